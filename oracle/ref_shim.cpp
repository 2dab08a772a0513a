// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference library (sslkit, built from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libsslref.so).  Every entry point here calls the reference's
// own public C++ API (namespace ssl) so that tests, the bench's
// `--impl reference` arm and the `cpu_baseline` leg can run the reference
// from Python through ctypes.  Nothing in this file re-implements numerics.
//
// Reference interfaces wrapped (paths relative to /root/reference/proj):
//   CorrelationWindow::push/normalized      include/ssl/correlation.hpp:29-51
//   NoiseModel / mat_inverse / PD gate       include/ssl/gsvd.hpp:31-50,71-72
//   gsvd / gsvd_reference / gsvd_matrix      include/ssl/gsvd.hpp:139-163
//   calc_average_power<T>                    include/ssl/music.hpp:76-79
//   DirectionTopology / peak_search          include/ssl/music.hpp:82-101
//   run_locate                               include/ssl/pipeline.hpp:71-75
//   synth + bench fixture generators         include/ssl/synth.hpp, bench.hpp

#include "ssl/bench.hpp"
#include "ssl/correlation.hpp"
#include "ssl/eig.hpp"
#include "ssl/gsvd.hpp"
#include "ssl/music.hpp"
#include "ssl/pipeline.hpp"
#include "ssl/rng.hpp"
#include "ssl/stft.hpp"
#include "ssl/synth.hpp"

#include <nlohmann/json.hpp>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#define SHIM_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

// 0 ok, 2 validation, 3 numerical, 4 io, 1 other — same mapping as the
// reference CLI (tools/sslkit.cpp:280-291).
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ssl::ValidationError& e) {
        return fail(2, e.what());
    } catch (const ssl::NumericalError& e) {
        return fail(3, e.what());
    } catch (const ssl::IoError& e) {
        return fail(4, e.what());
    } catch (const std::exception& e) {
        return fail(1, e.what());
    }
}

ssl::CMatrix<float> mat_from(const float* p, std::uint32_t m) {
    ssl::CMatrix<float> a(m, m);
    for (std::size_t i = 0; i < std::size_t(m) * m; ++i) a.data[i] = ssl::cfloat(p[2 * i], p[2 * i + 1]);
    return a;
}

ssl::CMatrix<double> matd_from(const double* p, std::uint32_t m) {
    ssl::CMatrix<double> a(m, m);
    for (std::size_t i = 0; i < std::size_t(m) * m; ++i) a.data[i] = ssl::cdouble(p[2 * i], p[2 * i + 1]);
    return a;
}

template <typename T>
void mat_to(const ssl::CMatrix<T>& a, double* p) {
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        p[2 * i] = double(a.data[i].real());
        p[2 * i + 1] = double(a.data[i].imag());
    }
}

ssl::CorrelationSet set_from(const float* p, std::uint32_t m, std::uint32_t bins) {
    ssl::CorrelationSet s;
    s.m = m;
    for (std::uint32_t b = 0; b < bins; ++b) s.bins.push_back(mat_from(p + std::size_t(b) * m * m * 2, m));
    return s;
}

ssl::SpectrumFrame frame_from(const float* x, std::uint32_t m, std::uint32_t bins, std::uint32_t index) {
    ssl::SpectrumFrame f;
    f.frame_index = index;
    f.spectra.resize(m);
    for (std::uint32_t c = 0; c < m; ++c) {
        f.spectra[c].resize(bins);
        for (std::uint32_t b = 0; b < bins; ++b) {
            const float* z = x + (std::size_t(c) * bins + b) * 2;
            f.spectra[c][b] = ssl::cfloat(z[0], z[1]);
        }
    }
    return f;
}

} // namespace

// ---------------------------------------------------------------------------
// POD configs
// ---------------------------------------------------------------------------

extern "C" {

typedef struct {
    std::uint32_t max_qr_sweeps;
    float tolerance_scale;
    int pivoting; // 0 none, 1 partial
    int compute_residual;
    int canonical_subspaces;
} sslref_solver;

typedef struct {
    std::uint32_t num_sources;
    float denominator_floor;
    int squared_denominator;
    float low_power_ratio;
} sslref_music;

enum { SSLREF_MAX_SOURCES = 16 };

typedef struct {
    int geometry_kind; // 0 circular, 1 spherical
    std::uint32_t mic_count;
    double radius;
    std::uint32_t frame_length, shift;
    int window; // 0 hann, 1 rectangular
    std::uint32_t bin_min, bin_max;
    std::uint32_t sample_rate;
    double duration_s;
    std::uint64_t seed;
    int has_diffuse;
    double diffuse_db;
    int n_sources;
    double src_az[SSLREF_MAX_SOURCES], src_el[SSLREF_MAX_SOURCES];
    double src_level_db[SSLREF_MAX_SOURCES], src_freq[SSLREF_MAX_SOURCES];
    int src_kind[SSLREF_MAX_SOURCES]; // 0 tone 1 white 2 multitone
    int src_noise_role[SSLREF_MAX_SOURCES];
    int grid_kind; // 0 azimuth ring, 1 fibonacci sphere, 2 az x el lattice
    double grid_step_deg;
    std::uint32_t sphere_count;
    double el_min_deg, el_max_deg, el_step_deg;
    int noise_kind; // 0 identity, 1 captured from the noise-role part, 2 random_noise_model
    std::uint64_t noise_seed;
    double noise_duration_s; // capture length for noise_kind 1 (<= 0: scene duration)
} sslref_scene;

} // extern "C"

namespace {

ssl::SolverConfig solver_from(const sslref_solver* s) {
    ssl::SolverConfig c;
    if (!s) return c;
    c.max_qr_sweeps = s->max_qr_sweeps;
    c.tolerance_scale = s->tolerance_scale;
    c.pivoting = s->pivoting ? ssl::Pivoting::partial : ssl::Pivoting::none;
    c.compute_residual = s->compute_residual != 0;
    c.canonical_subspaces = s->canonical_subspaces != 0;
    return c;
}

ssl::MusicConfig music_from(const sslref_music* m) {
    ssl::MusicConfig c;
    if (!m) return c;
    c.num_sources = m->num_sources;
    c.denominator_floor = m->denominator_floor;
    c.squared_denominator = m->squared_denominator != 0;
    c.low_power_ratio = m->low_power_ratio;
    return c;
}

ssl::StftConfig stft_from(const sslref_scene* s) {
    ssl::StftConfig c;
    c.frame_length = s->frame_length;
    c.shift = s->shift;
    c.window = s->window ? ssl::WindowKind::rectangular : ssl::WindowKind::hann;
    c.bin_min = s->bin_min;
    c.bin_max = s->bin_max;
    return c;
}

ssl::ArrayGeometry geometry_from(const sslref_scene* s) {
    return s->geometry_kind == 1 ? ssl::ArrayGeometry::spherical(s->mic_count, s->radius)
                                 : ssl::ArrayGeometry::circular(s->mic_count, s->radius);
}

ssl::SceneSpec scene_from(const sslref_scene* s) {
    ssl::SceneSpec sc;
    sc.duration_s = s->duration_s;
    sc.seed = s->seed;
    sc.has_diffuse = s->has_diffuse != 0;
    sc.diffuse_level_db = s->diffuse_db;
    for (int i = 0; i < s->n_sources && i < SSLREF_MAX_SOURCES; ++i) {
        ssl::SourceSpec src;
        src.direction = {s->src_az[i], s->src_el[i]};
        src.kind = s->src_kind[i] == 0   ? ssl::SourceKind::tone
                   : s->src_kind[i] == 1 ? ssl::SourceKind::white
                                         : ssl::SourceKind::multitone;
        src.frequency_hz = s->src_freq[i];
        src.level_db = s->src_level_db[i];
        src.noise_role = s->src_noise_role[i] != 0;
        sc.sources.push_back(src);
    }
    return sc;
}

std::vector<ssl::Direction> grid_from(const sslref_scene* s) {
    if (s->grid_kind == 1) return ssl::sphere_grid(s->sphere_count);
    if (s->grid_kind == 2) {
        // explicit azimuth x elevation lattice (no generator exists in the
        // reference; this is the SURVEY §8(d) C4 construction)
        std::vector<ssl::Direction> out;
        const auto ring = ssl::azimuth_grid(s->grid_step_deg);
        for (double el = s->el_min_deg; el <= s->el_max_deg + 1e-9; el += s->el_step_deg)
            for (const auto& d : ring) out.push_back({d.azimuth_deg, el});
        return out;
    }
    return ssl::azimuth_grid(s->grid_step_deg);
}

struct Workload {
    std::uint32_t m = 0, bins = 0;
    std::vector<ssl::SpectrumFrame> frames;
    ssl::SampleBlock audio;
    ssl::NoiseModel noise;
    ssl::SteeringField steering;
};

} // namespace

extern "C" {

SHIM_API const char* sslref_last_error() { return g_err.c_str(); }

SHIM_API int sslref_sizeof_scene() { return int(sizeof(sslref_scene)); }

// ---------------------------------------------------------------------------
// workload construction through the reference's own generators
// ---------------------------------------------------------------------------

SHIM_API int sslref_workload_new(const sslref_scene* s, void** out) {
    return guarded([&] {
        auto w = std::make_unique<Workload>();
        const auto geom = geometry_from(s);
        const auto stft = stft_from(s);
        const auto scene = scene_from(s);
        w->m = geom.channel_count();
        w->bins = stft.bin_count();
        w->audio = ssl::synthesize_scene(geom, scene, stft, s->sample_rate);
        ssl::stft_stream(w->audio, stft, [&](const ssl::SpectrumFrame& f) { w->frames.push_back(f); });
        if (s->noise_kind == 1) {
            ssl::SceneSpec ns = scene;
            if (s->noise_duration_s > 0) ns.duration_s = s->noise_duration_s;
            w->noise = ssl::capture_noise_model(geom, ns, stft, s->sample_rate);
        } else if (s->noise_kind == 2) {
            w->noise = ssl::random_noise_model(w->m, w->bins, s->noise_seed);
        } else {
            w->noise = ssl::NoiseModel::identity(w->m, w->bins);
        }
        w->steering = ssl::make_steering(geom, stft, s->sample_rate, grid_from(s));
        *out = w.release();
    });
}

SHIM_API void sslref_workload_free(void* h) { delete static_cast<Workload*>(h); }

SHIM_API void sslref_workload_dims(void* h, std::uint32_t* m, std::uint32_t* bins, std::uint32_t* dirs,
                                   std::uint32_t* frames, std::uint64_t* samples) {
    auto* w = static_cast<Workload*>(h);
    *m = w->m;
    *bins = w->bins;
    *dirs = std::uint32_t(w->steering.directions.size());
    *frames = std::uint32_t(w->frames.size());
    *samples = w->audio.frame_count();
}

// X: [frames][m][bins] cf32 (SpectrumFrame channel-major, types.hpp:56-61)
// K: [bins][m][m] cf32; H: [dirs][bins][m] cf32; dirs: [dirs][2] (az, el)
SHIM_API void sslref_workload_copy(void* h, float* x, float* k, float* hvec, double* dirs, float* audio) {
    auto* w = static_cast<Workload*>(h);
    if (x) {
        std::size_t o = 0;
        for (const auto& f : w->frames)
            for (const auto& ch : f.spectra)
                for (const auto& z : ch) {
                    x[o++] = z.real();
                    x[o++] = z.imag();
                }
    }
    if (k) {
        std::size_t o = 0;
        for (const auto& mat : w->noise.k.bins)
            for (const auto& z : mat.data) {
                k[o++] = z.real();
                k[o++] = z.imag();
            }
    }
    if (hvec) {
        std::size_t o = 0;
        for (const auto& z : w->steering.vectors) {
            hvec[o++] = z.real();
            hvec[o++] = z.imag();
        }
    }
    if (dirs) {
        for (std::size_t d = 0; d < w->steering.directions.size(); ++d) {
            dirs[2 * d] = w->steering.directions[d].azimuth_deg;
            dirs[2 * d + 1] = w->steering.directions[d].elevation_deg;
        }
    }
    if (audio) {
        const std::size_t n = w->audio.frame_count();
        for (std::size_t c = 0; c < w->audio.channel_count(); ++c)
            std::memcpy(audio + c * n, w->audio.channels[c].data(), n * sizeof(float));
    }
}

// bench.cpp:178-196 fixtures
SHIM_API int sslref_random_noise_model(std::uint32_t m, std::uint32_t bins, std::uint64_t seed, float* k) {
    return guarded([&] {
        const auto n = ssl::random_noise_model(m, bins, seed);
        std::size_t o = 0;
        for (const auto& mat : n.k.bins)
            for (const auto& z : mat.data) {
                k[o++] = z.real();
                k[o++] = z.imag();
            }
    });
}

SHIM_API int sslref_random_correlation(std::uint32_t m, std::uint32_t bins, std::uint64_t seed, float* r) {
    return guarded([&] {
        const auto s = ssl::random_correlation(m, bins, seed);
        std::size_t o = 0;
        for (const auto& mat : s.bins)
            for (const auto& z : mat.data) {
                r[o++] = z.real();
                r[o++] = z.imag();
            }
    });
}

// the acceptance sweep's pair (acceptance.cpp:130-132): one generator,
// K = random_psd(ridge 0.5) then R = random_psd(ridge 0)
SHIM_API void sslref_random_psd_pair(std::uint32_t m, std::uint64_t seed, std::uint64_t tag, float* k, float* r) {
    std::mt19937_64 rng(ssl::mix_seed(seed, tag));
    const auto kk = ssl::random_psd(m, rng, 0.5f);
    const auto rr = ssl::random_psd(m, rng, 0.0f);
    for (std::size_t i = 0; i < kk.data.size(); ++i) {
        k[2 * i] = kk.data[i].real();
        k[2 * i + 1] = kk.data[i].imag();
        r[2 * i] = rr.data[i].real();
        r[2 * i + 1] = rr.data[i].imag();
    }
}

// ---------------------------------------------------------------------------
// hot-path stages
// ---------------------------------------------------------------------------

// CorrelationWindow over F frames; writes normalized() for every filled push:
// r_out [F - T + 1][bins][m][m] cf32.  Returns the number of sets written.
SHIM_API int sslref_correlation(const float* x, std::uint32_t frames, std::uint32_t m, std::uint32_t bins,
                                std::uint32_t t, std::uint32_t rebuild_interval, float* r_out,
                                std::uint32_t* written) {
    return guarded([&] {
        ssl::CorrelationWindow win(t, rebuild_interval);
        std::size_t o = 0;
        std::uint32_t n = 0;
        for (std::uint32_t f = 0; f < frames; ++f) {
            win.push(frame_from(x + std::size_t(f) * m * bins * 2, m, bins, f));
            if (!win.filled()) continue;
            const auto r = win.normalized();
            for (const auto& mat : r.bins)
                for (const auto& z : mat.data) {
                    r_out[o++] = z.real();
                    r_out[o++] = z.imag();
                }
            ++n;
        }
        *written = n;
    });
}

SHIM_API int sslref_noise_check(const float* k, std::uint32_t m, std::uint32_t bins) {
    return guarded([&] {
        ssl::NoiseModel n;
        n.k = set_from(k, m, bins);
        n.check_positive_definite();
    });
}

// mat_inverse<T> (gsvd.cpp:21-62); precision 0 float, 1 double
SHIM_API int sslref_mat_inverse(const float* k, std::uint32_t m, int precision, int pivoting,
                                std::uint32_t bin_label, double* out) {
    return guarded([&] {
        const auto piv = pivoting ? ssl::Pivoting::partial : ssl::Pivoting::none;
        const auto kk = mat_from(k, m);
        if (precision == 0) mat_to(ssl::mat_inverse<float>(kk, piv, bin_label), out);
        else mat_to(ssl::mat_inverse<double>(ssl::convert<double>(kk), piv, bin_label), out);
    });
}

// Batched GSVD driver: path 0 = gsvd() (float batched), 1 = gsvd_reference().
// sigma [bins][m], e / er [bins][m][m] cf64 (float results widened exactly).
SHIM_API int sslref_gsvd(const float* k, const float* r, std::uint32_t m, std::uint32_t bins, int path,
                         unsigned threads, const sslref_solver* cfg, double* sigma, double* e, double* er,
                         std::uint32_t* iters, std::uint8_t* conv, double* resid) {
    return guarded([&] {
        ssl::NoiseModel noise;
        noise.k = set_from(k, m, bins);
        const auto rs = set_from(r, m, bins);
        const auto sc = solver_from(cfg);
        auto emit = [&](const auto& batch) {
            for (std::uint32_t b = 0; b < bins; ++b) {
                const auto& bin = batch.bins[b];
                for (std::uint32_t i = 0; i < m; ++i) sigma[std::size_t(b) * m + i] = double(bin.singular_values[i]);
                if (e) mat_to(bin.e, e + std::size_t(b) * m * m * 2);
                if (er) mat_to(bin.e_r, er + std::size_t(b) * m * m * 2);
                if (iters) iters[b] = bin.iterations;
                if (conv) conv[b] = bin.converged ? 1 : 0;
                if (resid) resid[b] = double(bin.recon_residual);
            }
        };
        if (path == 1) emit(ssl::gsvd_reference(noise, rs, sc, threads));
        else emit(ssl::gsvd(noise, rs, sc, threads));
    });
}

// Timing of the batched GSVD stage only (inverses prepared outside, as
// bench.cpp:209).  Returns median seconds per call over `repeats`.
SHIM_API int sslref_time_gsvd(const float* k, const float* r, std::uint32_t m, std::uint32_t bins, int path,
                              unsigned threads, int repeats, double* median_s) {
    return guarded([&] {
        ssl::NoiseModel noise;
        noise.k = set_from(k, m, bins);
        const auto rs = set_from(r, m, bins);
        ssl::SolverConfig sc;
        noise.prepare_inverses(sc.pivoting);
        std::vector<double> runs;
        for (int i = -1; i < repeats; ++i) { // i = -1: untimed warm-up call
            const auto t0 = std::chrono::steady_clock::now();
            if (path == 1) (void)ssl::gsvd_reference(noise, rs, sc, threads);
            else (void)ssl::gsvd(noise, rs, sc, threads);
            if (i >= 0) runs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(runs.begin(), runs.end());
        *median_s = runs[runs.size() / 2];
    });
}

// Timing of calc_average_power<float> alone (music.cpp:112-165) on the float
// path's own factors of `r` (gsvd(), computed outside the timer), as
// bench.cpp:198-231 times the spectrum stage.  Median seconds per call over
// `repeats` after one untimed warm-up call.
SHIM_API int sslref_time_spectrum(const float* k, const float* r, std::uint32_t m, std::uint32_t bins,
                                  const float* h, std::uint32_t dirs, const sslref_music* mcfg, unsigned threads,
                                  int repeats, double* median_s) {
    return guarded([&] {
        ssl::NoiseModel noise;
        noise.k = set_from(k, m, bins);
        const auto rs = set_from(r, m, bins);
        ssl::SolverConfig sc;
        const auto basis = ssl::gsvd(noise, rs, sc, threads);
        ssl::SteeringField sf;
        sf.m = m;
        sf.bin_min = 0;
        sf.bin_max = bins - 1;
        sf.directions.assign(dirs, ssl::Direction{});
        sf.vectors.resize(std::size_t(dirs) * bins * m);
        for (std::size_t i = 0; i < sf.vectors.size(); ++i) sf.vectors[i] = ssl::cfloat(h[2 * i], h[2 * i + 1]);
        const auto mc = music_from(mcfg);
        std::vector<double> runs;
        for (int i = -1; i < repeats; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            (void)ssl::calc_average_power<float>(basis, sf, mc, false, threads);
            if (i >= 0) runs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(runs.begin(), runs.end());
        *median_s = runs[runs.size() / 2];
    });
}

// Single-matrix composed solve gsvd_matrix<T> (gsvd.cpp:589-620) or the
// reference matrix solve (697-716) when precision == 2.
SHIM_API int sslref_gsvd_matrix(const double* kinv, const double* r, std::uint32_t m, int precision,
                                const sslref_solver* cfg, double* sigma, double* e, double* er,
                                std::uint32_t* iters, std::uint8_t* conv) {
    return guarded([&] {
        const auto sc = solver_from(cfg);
        const auto kd = matd_from(kinv, m);
        const auto rd = matd_from(r, m);
        auto emit = [&](const auto& bin) {
            for (std::uint32_t i = 0; i < m; ++i) sigma[i] = double(bin.singular_values[i]);
            if (e) mat_to(bin.e, e);
            if (er) mat_to(bin.e_r, er);
            if (iters) *iters = bin.iterations;
            if (conv) *conv = bin.converged ? 1 : 0;
        };
        if (precision == 0) emit(ssl::gsvd_matrix<float>(ssl::convert<float>(kd), ssl::convert<float>(rd), sc));
        else if (precision == 1) emit(ssl::gsvd_matrix<double>(kd, rd, sc));
        else emit(ssl::gsvd_reference_matrix(kd, rd, sc));
    });
}

SHIM_API int sslref_jacobi_svd(const double* a, std::uint32_t m, double* sigma, double* u, double* vh,
                               std::uint32_t* sweeps, std::uint8_t* conv) {
    return guarded([&] {
        const auto res = ssl::jacobi_svd(matd_from(a, m));
        for (std::uint32_t i = 0; i < m; ++i) sigma[i] = res.singular_values[i];
        if (u) mat_to(res.u, u);
        if (vh) mat_to(res.v_h, vh);
        if (sweeps) *sweeps = res.sweeps;
        if (conv) *conv = res.converged ? 1 : 0;
    });
}

SHIM_API int sslref_hermitian_eigenvalues(const double* a, std::uint32_t m, double* values) {
    return guarded([&] {
        const auto v = ssl::hermitian_eigenvalues(matd_from(a, m));
        for (std::uint32_t i = 0; i < m; ++i) values[i] = v[i];
    });
}

// calc_average_power<T> (music.cpp:112-165).  e: [bins][m][m] cf64 full
// left factors (narrowed to float when precision == 0); h: [dirs][bins][m].
SHIM_API int sslref_spectrum(const double* e, std::uint32_t m, std::uint32_t bins, const float* h,
                             std::uint32_t dirs, int precision, const sslref_music* mcfg, unsigned threads,
                             double* power, double* bin_power) {
    return guarded([&] {
        ssl::SteeringField sf;
        sf.m = m;
        sf.bin_min = 0;
        sf.bin_max = bins - 1;
        sf.directions.assign(dirs, ssl::Direction{});
        sf.vectors.resize(std::size_t(dirs) * bins * m);
        for (std::size_t i = 0; i < sf.vectors.size(); ++i) sf.vectors[i] = ssl::cfloat(h[2 * i], h[2 * i + 1]);
        const auto mc = music_from(mcfg);
        const bool keep = bin_power != nullptr;
        ssl::MusicSpectrum spec;
        if (precision == 0) {
            ssl::GsvdBatch<float> basis;
            basis.bins.resize(bins);
            for (std::uint32_t b = 0; b < bins; ++b)
                basis.bins[b].e = ssl::convert<float>(matd_from(e + std::size_t(b) * m * m * 2, m));
            spec = ssl::calc_average_power<float>(basis, sf, mc, keep, threads);
        } else {
            ssl::GsvdBatch<double> basis;
            basis.bins.resize(bins);
            for (std::uint32_t b = 0; b < bins; ++b) basis.bins[b].e = matd_from(e + std::size_t(b) * m * m * 2, m);
            spec = ssl::calc_average_power<double>(basis, sf, mc, keep, threads);
        }
        for (std::uint32_t d = 0; d < dirs; ++d) power[d] = spec.power[d];
        if (keep)
            for (std::uint32_t b = 0; b < bins; ++b)
                for (std::uint32_t d = 0; d < dirs; ++d) bin_power[std::size_t(b) * dirs + d] = spec.bin_power[b][d];
    });
}

// DirectionTopology::build (music.cpp:176-195) flattened to CSR.
// offsets [dirs + 1]; nbr capacity `cap`; returns 2 if cap is too small.
SHIM_API int sslref_topology(const double* dirs, std::uint32_t n, double radius_deg, std::uint32_t* offsets,
                             std::uint32_t* nbr, std::uint32_t cap) {
    return guarded([&] {
        std::vector<ssl::Direction> d(n);
        for (std::uint32_t i = 0; i < n; ++i) d[i] = {dirs[2 * i], dirs[2 * i + 1]};
        const auto topo = ssl::DirectionTopology::build(d, radius_deg);
        std::uint32_t o = 0;
        for (std::uint32_t i = 0; i < n; ++i) {
            offsets[i] = o;
            for (auto j : topo.neighbors[i]) {
                if (o >= cap) throw ssl::ValidationError("topology capacity exceeded");
                nbr[o++] = j;
            }
        }
        offsets[n] = o;
    });
}

// peak_search (music.cpp:197-236) on the reference topology with `radius`.
SHIM_API int sslref_peaks(const double* power, const double* dirs, std::uint32_t n, double radius_deg,
                          const sslref_music* mcfg, std::uint32_t* idx, double* pw, std::uint8_t* low,
                          std::uint32_t* count) {
    return guarded([&] {
        std::vector<ssl::Direction> d(n);
        for (std::uint32_t i = 0; i < n; ++i) d[i] = {dirs[2 * i], dirs[2 * i + 1]};
        const auto topo = ssl::DirectionTopology::build(d, radius_deg);
        const std::vector<double> p(power, power + n);
        const auto est = ssl::peak_search(p, d, topo, music_from(mcfg));
        *count = std::uint32_t(est.size());
        for (std::size_t i = 0; i < est.size(); ++i) {
            idx[i] = est[i].direction_index;
            pw[i] = est[i].power;
            low[i] = est[i].low_power ? 1 : 0;
        }
    });
}

// The per-frame loop of run_locate (pipeline.cpp:227-245) driven by
// precomputed STFT frames instead of audio, so both engines consume the same
// spectra.  path: 0 batched float, 1 naive (threads=1), 2 reference double.
// Outputs per emitted block: power [E][dirs], bin_power [E][bins][dirs]
// (nullable), estimates idx/pw/low [E][ns], counts [E].  Stage seconds in
// stage_s[4] = correlation, factorization, spectrum, peaks.
SHIM_API int sslref_locate_frames(const float* x, std::uint32_t frames, std::uint32_t m, std::uint32_t bins,
                                  std::uint32_t t, const float* k, const float* h, const double* dirs,
                                  std::uint32_t ndirs, int path, unsigned threads, const sslref_solver* scfg,
                                  const sslref_music* mcfg, double* power, double* bin_power,
                                  std::uint32_t* est_idx, double* est_pw, std::uint8_t* est_low,
                                  std::uint32_t* est_count, std::uint32_t* emitted, double* stage_s) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        ssl::NoiseModel noise;
        noise.k = set_from(k, m, bins);
        ssl::SteeringField sf;
        sf.m = m;
        sf.bin_min = 0;
        sf.bin_max = bins - 1;
        for (std::uint32_t d = 0; d < ndirs; ++d) sf.directions.push_back({dirs[2 * d], dirs[2 * d + 1]});
        sf.vectors.resize(std::size_t(ndirs) * bins * m);
        for (std::size_t i = 0; i < sf.vectors.size(); ++i) sf.vectors[i] = ssl::cfloat(h[2 * i], h[2 * i + 1]);
        const auto sc = solver_from(scfg);
        const auto mc = music_from(mcfg);
        const auto topo = ssl::DirectionTopology::build(sf.directions);
        noise.prepare_inverses(sc.pivoting);
        ssl::CorrelationWindow win(t);
        const bool keep = bin_power != nullptr;
        std::uint32_t e_out = 0;
        double st[4] = {0, 0, 0, 0};
        for (std::uint32_t f = 0; f < frames; ++f) {
            // stage clocks cover emitting frames only (steady-state per-block
            // cost; the T-1 window-filling pushes are excluded)
            auto mark = clk::now();
            win.push(frame_from(x + std::size_t(f) * m * bins * 2, m, bins, f));
            if (!win.filled()) continue;
            const auto r = win.normalized();
            st[0] += std::chrono::duration<double>(clk::now() - mark).count();
            ssl::MusicSpectrum spec;
            mark = clk::now();
            if (path == 2) {
                const auto basis = ssl::gsvd_reference(noise, r, sc, threads);
                st[1] += std::chrono::duration<double>(clk::now() - mark).count();
                mark = clk::now();
                spec = ssl::calc_average_power<double>(basis, sf, mc, keep, threads);
            } else {
                const unsigned tc = path == 1 ? 1 : threads;
                const auto basis = ssl::gsvd(noise, r, sc, tc);
                st[1] += std::chrono::duration<double>(clk::now() - mark).count();
                mark = clk::now();
                spec = ssl::calc_average_power<float>(basis, sf, mc, keep, tc);
            }
            st[2] += std::chrono::duration<double>(clk::now() - mark).count();
            mark = clk::now();
            const auto est = ssl::peak_search(spec.power, sf.directions, topo, mc);
            st[3] += std::chrono::duration<double>(clk::now() - mark).count();
            for (std::uint32_t d = 0; d < ndirs; ++d) power[std::size_t(e_out) * ndirs + d] = spec.power[d];
            if (keep)
                for (std::uint32_t b = 0; b < bins; ++b)
                    for (std::uint32_t d = 0; d < ndirs; ++d)
                        bin_power[(std::size_t(e_out) * bins + b) * ndirs + d] = spec.bin_power[b][d];
            est_count[e_out] = std::uint32_t(est.size());
            for (std::size_t i = 0; i < est.size(); ++i) {
                est_idx[std::size_t(e_out) * mc.num_sources + i] = est[i].direction_index;
                est_pw[std::size_t(e_out) * mc.num_sources + i] = est[i].power;
                est_low[std::size_t(e_out) * mc.num_sources + i] = est[i].low_power ? 1 : 0;
            }
            ++e_out;
        }
        *emitted = e_out;
        if (stage_s)
            for (int i = 0; i < 4; ++i) stage_s[i] = st[i];
    });
}

// run_locate (pipeline.cpp:210-247) on the workload's own audio, the full
// reference entry point including its STFT; estimates as above.
SHIM_API int sslref_run_locate(void* h, const sslref_scene* s, std::uint32_t t, int path, unsigned threads,
                               const sslref_solver* scfg, const sslref_music* mcfg, std::uint32_t* est_idx,
                               double* est_pw, std::uint8_t* est_low, std::uint32_t* est_count,
                               std::uint32_t* frame_index, std::uint32_t* emitted) {
    return guarded([&] {
        auto* w = static_cast<Workload*>(h);
        const auto mc = music_from(mcfg);
        const auto sp = path == 2 ? ssl::SolvePath::reference
                                  : (path == 1 ? ssl::SolvePath::naive : ssl::SolvePath::batched);
        std::uint32_t e = 0;
        ssl::run_locate(w->audio, stft_from(s), t, w->noise, w->steering, solver_from(scfg), mc, sp, threads,
                        [&](const ssl::FrameEstimates& fe) {
                            est_count[e] = std::uint32_t(fe.estimates.size());
                            frame_index[e] = std::uint32_t(fe.frame_index);
                            for (std::size_t i = 0; i < fe.estimates.size(); ++i) {
                                est_idx[std::size_t(e) * mc.num_sources + i] = fe.estimates[i].direction_index;
                                est_pw[std::size_t(e) * mc.num_sources + i] = fe.estimates[i].power;
                                est_low[std::size_t(e) * mc.num_sources + i] = fe.estimates[i].low_power ? 1 : 0;
                            }
                            ++e;
                        });
        *emitted = e;
    });
}


// ---------------------------------------------------------------------------
// on-disk formats through the reference's own readers and writers
// ---------------------------------------------------------------------------

SHIM_API int sslref_save_correlation(const char* path, std::uint32_t m, std::uint32_t bins, std::uint32_t t,
                                     const float* k) {
    return guarded([&] { ssl::save_correlation(path, set_from(k, m, bins), t); });
}

// load_correlation: header into m/bins/t, payload into k when non-null
SHIM_API int sslref_load_correlation(const char* path, std::uint32_t* m, std::uint32_t* bins, std::uint32_t* t,
                                     float* k) {
    return guarded([&] {
        std::uint32_t tt = 0;
        const auto set = ssl::load_correlation(path, &tt);
        *m = set.m;
        *bins = std::uint32_t(set.bins.size());
        *t = tt;
        if (k) {
            std::size_t o = 0;
            for (const auto& mat : set.bins)
                for (const auto& z : mat.data) {
                    k[o++] = z.real();
                    k[o++] = z.imag();
                }
        }
    });
}

SHIM_API int sslref_save_steering(const char* path, std::uint32_t m, std::uint32_t bin_min, std::uint32_t bin_max,
                                  std::uint32_t dirs, const double* dirs_deg, const float* h) {
    return guarded([&] {
        ssl::SteeringField f;
        f.m = m;
        f.bin_min = bin_min;
        f.bin_max = bin_max;
        for (std::uint32_t d = 0; d < dirs; ++d) f.directions.push_back({dirs_deg[2 * d], dirs_deg[2 * d + 1]});
        const std::size_t n = std::size_t(dirs) * (bin_max - bin_min + 1) * m;
        f.vectors.resize(n);
        for (std::size_t i = 0; i < n; ++i) f.vectors[i] = ssl::cfloat(h[2 * i], h[2 * i + 1]);
        ssl::save_steering(f, path);
    });
}

SHIM_API int sslref_load_steering(const char* path, std::uint32_t* m, std::uint32_t* bin_min, std::uint32_t* bin_max,
                                  std::uint32_t* dirs, double* dirs_deg, float* h) {
    return guarded([&] {
        const auto f = ssl::load_steering(path);
        *m = f.m;
        *bin_min = f.bin_min;
        *bin_max = f.bin_max;
        *dirs = std::uint32_t(f.directions.size());
        if (dirs_deg)
            for (std::size_t d = 0; d < f.directions.size(); ++d) {
                dirs_deg[2 * d] = f.directions[d].azimuth_deg;
                dirs_deg[2 * d + 1] = f.directions[d].elevation_deg;
            }
        if (h)
            for (std::size_t i = 0; i < f.vectors.size(); ++i) {
                h[2 * i] = f.vectors[i].real();
                h[2 * i + 1] = f.vectors[i].imag();
            }
    });
}

// The JSONL record run_locate_to_stream's sink writes (pipeline.cpp:268-283),
// built the same way with the same nlohmann::json.  Test infrastructure: the
// checker for the engine's record formatter.
SHIM_API int sslref_format_estimates(std::uint64_t frame, std::uint32_t count, const std::uint32_t* idx,
                                     const double* dirs_deg, const double* power, const std::uint8_t* low,
                                     char* buf, std::uint64_t cap) {
    return guarded([&] {
        nlohmann::json line;
        line["frame"] = frame;
        auto arr = nlohmann::json::array();
        for (std::uint32_t i = 0; i < count; ++i) {
            nlohmann::json e;
            e["azimuth_deg"] = dirs_deg[2 * std::size_t(idx[i])];
            e["elevation_deg"] = dirs_deg[2 * std::size_t(idx[i]) + 1];
            e["power"] = power[i];
            e["low_power"] = low[i] != 0;
            e["direction"] = idx[i];
            arr.push_back(std::move(e));
        }
        line["estimates"] = std::move(arr);
        const std::string s = line.dump();
        if (s.size() + 1 > cap) throw ssl::ValidationError("buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

} // extern "C"
