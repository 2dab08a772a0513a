// sslgpu/ssl.hpp — header-only C++ mirror of the reference's localization
// API (namespace ssl, /root/reference/proj/include/ssl/*.hpp) on top of the
// C ABI of libsslgpu.so (include/sslgpu.h).
//
// A C++ caller of the reference switches by including this header instead of
// <ssl/correlation.hpp>, <ssl/gsvd.hpp>, <ssl/music.hpp>, <ssl/pipeline.hpp>
// and linking libsslgpu.so.  Names, argument meaning and exceptions follow the
// reference (types.hpp:13-23); the `threads` arguments are accepted and
// ignored (results never depended on them, gsvd.hpp:157-159).  Everything
// lives in ssl::b200 and is re-exported into ssl by an inline namespace.
#pragma once

#include "../sslgpu.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace ssl {
inline namespace b200 {

// ---- errors (types.hpp:13-23) ---------------------------------------------
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc) {
    if (rc == SSLG_OK) return;
    const std::string msg = sslg_last_error();
    switch (rc) {
        case SSLG_VALIDATION: throw ValidationError(msg);
        case SSLG_NUMERICAL: throw NumericalError(msg);
        case SSLG_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

using cfloat = std::complex<float>;
using cdouble = std::complex<double>;

// ---- containers (mat.hpp:12-29, types.hpp, correlation.hpp, music.hpp) --------
template <typename T>
struct CMatrix {
    std::size_t rows = 0, cols = 0;
    std::vector<std::complex<T>> data;
    CMatrix() = default;
    CMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c) {}
    std::complex<T>& operator()(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    const std::complex<T>& operator()(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    static CMatrix identity(std::size_t n) {
        CMatrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = 1;
        return m;
    }
};

struct SpectrumFrame {
    std::uint32_t frame_index = 0;
    std::vector<std::vector<cfloat>> spectra;  // [m][bins]
};

struct CorrelationSet {
    std::uint32_t m = 0;
    std::uint32_t frame_index = 0;
    std::vector<CMatrix<float>> bins;
    std::size_t bin_count() const { return bins.size(); }
};

enum class Pivoting { none, partial };

struct SolverConfig {
    // SolverConfig (gsvd.hpp:14-26).  max_qr_sweeps > 0: a bin whose solve takes
    // more sweeps reports converged = false with the budget as its iteration
    // count (gsvd() only, like the reference's QR budget); tolerance_scale
    // scales the Jacobi no-rotation threshold.
    std::uint32_t max_qr_sweeps = 0;
    float tolerance_scale = 1.0f;
    Pivoting pivoting = Pivoting::partial;
    bool compute_residual = false;
    bool canonical_subspaces = true;
    void validate() const {
        if (!(tolerance_scale > 0)) throw ValidationError("tolerance_scale must be positive");
    }
};

struct MusicConfig {
    std::uint32_t num_sources = 1;
    float denominator_floor = 1e-12f;
    bool squared_denominator = false;
    float low_power_ratio = 1.25f;
};

struct Direction {
    double azimuth_deg = 0, elevation_deg = 0;
};

struct SteeringField {
    std::uint32_t m = 0, bin_min = 0, bin_max = 0;
    std::vector<Direction> directions;
    std::vector<cfloat> vectors;  // [dir][bin][mic]
    std::size_t bin_count() const { return std::size_t(bin_max) - bin_min + 1; }
    const cfloat* at(std::size_t dir, std::size_t bin) const { return &vectors[(dir * bin_count() + bin) * m]; }
    void validate() const {
        if (m == 0) throw ValidationError("steering field has no channels");
        if (bin_max < bin_min) throw ValidationError("steering field bin range is inverted");
        if (directions.empty()) throw ValidationError("steering field has no directions");
        if (vectors.size() != directions.size() * bin_count() * m)
            throw ValidationError("steering field payload size mismatch");
    }
};

template <typename T>
struct GsvdBinResult {
    std::vector<T> singular_values;  // non-increasing
    CMatrix<T> e;                    // left singular vectors as columns
    CMatrix<T> e_r;                  // right factor; row i pairs with value i (sslg_gsvd_ex)
    std::uint32_t iterations = 0;
    bool converged = true;
    T recon_residual = T(-1);  // relative Frobenius residual; < 0 if not computed
};

template <typename T>
struct GsvdBatch {
    std::vector<GsvdBinResult<T>> bins;
};

struct MusicSpectrum {
    std::uint64_t frame_index = 0;
    std::vector<double> power;
    std::vector<std::vector<double>> bin_power;
};

struct DirectionTopology {
    std::vector<std::vector<std::uint32_t>> neighbors;
    static DirectionTopology build(const std::vector<Direction>& dirs, double radius_deg = 10.0) {
        std::vector<double> d(dirs.size() * 2);
        for (std::size_t i = 0; i < dirs.size(); ++i) {
            d[2 * i] = dirs[i].azimuth_deg;
            d[2 * i + 1] = dirs[i].elevation_deg;
        }
        const auto n = std::uint32_t(dirs.size());
        std::vector<std::uint32_t> off(n + 1);
        std::uint32_t need = 0;
        sslg_build_topology(d.data(), n, radius_deg, off.data(), nullptr, 0, &need);
        std::vector<std::uint32_t> nbr(need ? need : 1);
        check(sslg_build_topology(d.data(), n, radius_deg, off.data(), nbr.data(), need, &need));
        DirectionTopology t;
        t.neighbors.resize(n);
        for (std::uint32_t i = 0; i < n; ++i) t.neighbors[i].assign(nbr.begin() + off[i], nbr.begin() + off[i + 1]);
        return t;
    }
};

struct SourceEstimate {
    std::uint32_t direction_index = 0;
    Direction direction;
    double power = 0;
    bool low_power = false;
};

struct FrameEstimates {
    std::uint64_t frame_index = 0;
    std::vector<SourceEstimate> estimates;
};

// ---- audio side (types.hpp:30-52) -----------------------------------------------
struct SampleBlock {
    std::uint32_t sample_rate = 16000;
    std::vector<std::vector<float>> channels;
    std::size_t channel_count() const { return channels.size(); }
    std::size_t frame_count() const { return channels.empty() ? 0 : channels[0].size(); }
    void validate() const {
        if (channels.empty()) throw ValidationError("sample block has no channels");
        for (const auto& c : channels)
            if (c.size() != channels[0].size()) throw ValidationError("channels differ in length");
    }
};

enum class WindowKind { hann, rectangular };

struct StftConfig {
    std::uint32_t frame_length = 512;
    std::uint32_t shift = 160;
    WindowKind window = WindowKind::hann;
    std::uint32_t bin_min = 16;
    std::uint32_t bin_max = 88;
    std::uint32_t bin_count() const { return bin_max - bin_min + 1; }
};

// pipeline.hpp:56: which solver the reference runs; the device engine always
// runs its FP64 path, so every value selects it.
enum class SolvePath { naive, batched, reference };

// ---- device contexts ---------------------------------------------------------
class Engine {
  public:
    Engine(std::uint32_t m, std::uint32_t bins, std::uint32_t window_frames, const MusicConfig& mc,
           const SolverConfig& sc, std::uint32_t max_batch = 16, int device = 0, std::uint32_t rebuild_interval = 1000) {
        sc.validate();
        sslg_config cfg;
        sslg_config_default(&cfg);
        cfg.m = m;
        cfg.bins = bins;
        cfg.window_frames = window_frames;
        cfg.rebuild_interval = rebuild_interval;
        cfg.num_sources = mc.num_sources;
        cfg.denominator_floor = mc.denominator_floor;
        cfg.squared_denominator = mc.squared_denominator ? 1 : 0;
        cfg.low_power_ratio = mc.low_power_ratio;
        cfg.pivoting = sc.pivoting == Pivoting::partial ? 1 : 0;
        cfg.canonical_subspaces = sc.canonical_subspaces ? 1 : 0;
        cfg.max_qr_sweeps = sc.max_qr_sweeps;
        cfg.tolerance_scale = sc.tolerance_scale;
        cfg.compute_residual = sc.compute_residual ? 1 : 0;
        cfg.max_batch = max_batch;
        cfg.device = device;
        sslg_ctx* c = nullptr;
        check(sslg_create(&c, &cfg));
        ctx_.reset(c);
        m_ = m;
        bins_ = bins;
        ns_ = mc.num_sources;
    }
    sslg_ctx* get() const { return ctx_.get(); }
    std::uint32_t m() const { return m_; }
    std::uint32_t bins() const { return bins_; }
    std::uint32_t num_sources() const { return ns_; }

  private:
    struct Del {
        void operator()(sslg_ctx* c) const { sslg_destroy(c); }
    };
    std::unique_ptr<sslg_ctx, Del> ctx_;
    std::uint32_t m_ = 0, bins_ = 0, ns_ = 1;
};

namespace detail {
inline std::vector<float> flatten(const std::vector<CMatrix<float>>& mats) {
    std::vector<float> out;
    for (const auto& a : mats)
        for (const auto& z : a.data) {
            out.push_back(z.real());
            out.push_back(z.imag());
        }
    return out;
}
inline std::vector<double> flat_dirs(const std::vector<Direction>& dirs) {
    std::vector<double> d;
    for (const auto& x : dirs) {
        d.push_back(x.azimuth_deg);
        d.push_back(x.elevation_deg);
    }
    return d;
}
inline std::uint64_t fnv1a(const void* p, std::size_t n, std::uint64_t h = 1469598103934665603ull) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
inline void validate_set(const CorrelationSet& s) {
    if (s.m < 1) throw ValidationError("correlation set has no channels");
    if (s.bins.empty()) throw ValidationError("correlation set has no bins");
    for (const auto& b : s.bins) {
        if (b.rows != s.m || b.cols != s.m) throw ValidationError("correlation matrix dimension mismatch");
        for (const auto& z : b.data)
            if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
                throw ValidationError("non-finite correlation entry");
    }
}
}  // namespace detail

// ---- CorrelationWindow (correlation.hpp:29-51) ------------------------------------
// The running FP64 sum, the ring and the periodic rebuild live on the device
// (correlation_kernel); normalized() reads the newest R back, bit-identical
// to the reference's (correlation.cpp:53-130).
class CorrelationWindow {
  public:
    explicit CorrelationWindow(std::uint32_t t, std::uint32_t rebuild_interval = 1000)
        : t_(t), rebuild_interval_(rebuild_interval < 1 ? 1 : rebuild_interval) {
        if (t_ < 1) throw ValidationError("correlation window length must be >= 1");
    }
    void push(const SpectrumFrame& frame) {
        const std::size_t m = frame.spectra.size();
        if (m == 0) throw ValidationError("empty spectrum frame");
        const std::size_t bins = frame.spectra[0].size();
        std::vector<float> x;
        x.reserve(m * bins * 2);
        for (const auto& ch : frame.spectra) {
            if (ch.size() != bins) throw ValidationError("ragged spectrum frame");
            for (const auto& z : ch) {
                if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
                    throw ValidationError("non-finite spectrum value");
                x.push_back(z.real());
                x.push_back(z.imag());
            }
        }
        if (!eng_) {
            eng_ = std::make_shared<Engine>(std::uint32_t(m), std::uint32_t(bins), t_, MusicConfig{}, SolverConfig{}, 1,
                                            0, rebuild_interval_);
        } else if (eng_->m() != m || eng_->bins() != bins) {
            throw ValidationError("spectrum frame shape changed mid-stream");
        }
        std::uint32_t emitted = 0;
        check(sslg_correlation(eng_->get(), x.data(), 1, nullptr, &emitted));
        last_frame_index_ = frame.frame_index;
        ++pushed_;
    }
    bool filled() const { return pushed_ >= t_; }
    std::uint32_t capacity() const { return t_; }
    CorrelationSet normalized() const {
        if (!filled())
            throw ValidationError("correlation window underfilled: " + std::to_string(pushed_) + " of " +
                                  std::to_string(t_) + " frames");
        const auto m = eng_->m(), nb = eng_->bins();
        std::vector<float> r(std::size_t(nb) * m * m * 2);
        check(sslg_last_correlation(eng_->get(), r.data()));
        CorrelationSet out;
        out.m = m;
        out.frame_index = last_frame_index_;
        out.bins.assign(nb, CMatrix<float>(m, m));
        for (std::uint32_t b = 0; b < nb; ++b)
            for (std::size_t i = 0; i < std::size_t(m) * m; ++i) {
                const std::size_t o = (std::size_t(b) * m * m + i) * 2;
                out.bins[b].data[i] = cfloat(r[o], r[o + 1]);
            }
        return out;
    }

  private:
    std::uint32_t t_, rebuild_interval_;
    std::uint64_t pushed_ = 0;
    std::uint32_t last_frame_index_ = 0;
    std::shared_ptr<Engine> eng_;
};

// ---- on-disk formats (correlation.hpp:53-58, music.hpp:103-104) --------------------
inline void save_correlation(const std::string& path, const CorrelationSet& set, std::uint32_t t) {
    detail::validate_set(set);
    const auto f = detail::flatten(set.bins);
    check(sslg_write_correlation_file(path.c_str(), set.m, std::uint32_t(set.bins.size()), t, f.data()));
}
inline CorrelationSet load_correlation(const std::string& path, std::uint32_t* t_out = nullptr) {
    std::uint32_t m = 0, nb = 0, t = 0;
    check(sslg_read_correlation_file(path.c_str(), &m, &nb, &t, nullptr, 0));
    std::vector<float> f(std::size_t(nb) * m * m * 2);
    check(sslg_read_correlation_file(path.c_str(), nullptr, nullptr, nullptr, f.data(), f.size()));
    if (t_out) *t_out = t;
    CorrelationSet s;
    s.m = m;
    s.bins.assign(nb, CMatrix<float>(m, m));
    for (std::uint32_t b = 0; b < nb; ++b)
        for (std::size_t i = 0; i < std::size_t(m) * m; ++i) {
            const std::size_t o = (std::size_t(b) * m * m + i) * 2;
            s.bins[b].data[i] = cfloat(f[o], f[o + 1]);
        }
    return s;
}
inline void save_steering(const SteeringField& field, const std::string& path) {
    field.validate();
    const auto d = detail::flat_dirs(field.directions);
    check(sslg_write_steering_file(path.c_str(), field.m, field.bin_min, field.bin_max,
                                   std::uint32_t(field.directions.size()), d.data(),
                                   reinterpret_cast<const float*>(field.vectors.data())));
}
inline SteeringField load_steering(const std::string& path) {
    std::uint32_t m = 0, lo = 0, hi = 0, nd = 0;
    check(sslg_read_steering_file(path.c_str(), &m, &lo, &hi, &nd, nullptr, nullptr, 0));
    SteeringField f;
    f.m = m;
    f.bin_min = lo;
    f.bin_max = hi;
    std::vector<double> d(std::size_t(nd) * 2);
    f.vectors.resize(std::size_t(nd) * (hi - lo + 1) * m);
    check(sslg_read_steering_file(path.c_str(), nullptr, nullptr, nullptr, nullptr, d.data(),
                                  reinterpret_cast<float*>(f.vectors.data()), nd));
    for (std::uint32_t i = 0; i < nd; ++i) f.directions.push_back({d[2 * i], d[2 * i + 1]});
    f.validate();
    return f;
}

// NoiseModel (gsvd.hpp:31-50): K on the host, the inverses built and cached
// on the device in a context the batched solves reuse (the reference caches
// them on the NoiseModel, gsvd.hpp:46-49; like it, changing k after
// prepare_inverses is not noticed).
struct NoiseModel {
    CorrelationSet k;

    static NoiseModel identity(std::uint32_t m, std::size_t bins) {
        NoiseModel n;
        n.k.m = m;
        n.k.bins.assign(bins, CMatrix<float>::identity(m));
        return n;
    }
    static NoiseModel from_file(const std::string& path) {
        NoiseModel n;
        n.k = load_correlation(path);
        n.check_positive_definite();
        return n;
    }
    // capture_noise_model (synth.cpp:329-373) from noise-only audio: the
    // device STFT and FP64 frame sums, bit-identical K, PD-gated.  (The
    // reference synthesizes that audio from a SceneSpec; synthesis is out of
    // scope here.)
    static NoiseModel capture(const SampleBlock& noise_audio, const StftConfig& stft) {
        noise_audio.validate();
        const auto m = std::uint32_t(noise_audio.channel_count());
        Engine e(m, stft.bin_count(), 1, MusicConfig{}, SolverConfig{}, 16);
        sslg_stft_config sc{stft.frame_length, stft.shift, stft.window == WindowKind::hann ? 0 : 1, stft.bin_min,
                            stft.bin_max};
        check(sslg_set_stft(e.get(), &sc));
        std::vector<float> pcm;
        for (const auto& c : noise_audio.channels) pcm.insert(pcm.end(), c.begin(), c.end());
        std::vector<float> kf(std::size_t(stft.bin_count()) * m * m * 2);
        std::uint32_t nf = 0;
        check(sslg_capture_noise_model(e.get(), pcm.data(), noise_audio.frame_count(), 0, kf.data(), &nf, nullptr));
        NoiseModel n;
        n.k.m = m;
        n.k.bins.assign(stft.bin_count(), CMatrix<float>(m, m));
        for (std::size_t b = 0; b < n.k.bins.size(); ++b)
            for (std::size_t i = 0; i < std::size_t(m) * m; ++i) {
                const std::size_t o = (b * m * m + i) * 2;
                n.k.bins[b].data[i] = cfloat(kf[o], kf[o + 1]);
            }
        return n;
    }
    void check_positive_definite() const {
        detail::validate_set(k);
        Engine e(k.m, std::uint32_t(k.bins.size()), 1, MusicConfig{}, SolverConfig{}, 1);
        const auto flat = detail::flatten(k.bins);
        check(sslg_set_noise_model(e.get(), flat.data(), 1, nullptr));
    }
    void prepare_inverses(Pivoting pivoting) const {
        SolverConfig sc;
        sc.pivoting = pivoting;
        context(sc);
    }
    CMatrix<float> inverse(std::size_t bin) const { return fetch_inverse<float>(bin, 0); }
    CMatrix<double> inverse_double(std::size_t bin) const { return fetch_inverse<double>(bin, 1); }

    // the cached device context for a solver configuration (internal)
    sslg_ctx* context(const SolverConfig& sc) const {
        const auto key = std::make_tuple(int(sc.pivoting), sc.canonical_subspaces, sc.max_qr_sweeps, sc.tolerance_scale,
                                         sc.compute_residual);
        if (!cache_ || cache_->key != key) {
            detail::validate_set(k);
            auto c = std::make_shared<Cache>();
            c->eng = std::make_shared<Engine>(k.m, std::uint32_t(k.bins.size()), 1, MusicConfig{}, sc, 1);
            const auto flat = detail::flatten(k.bins);
            check(sslg_set_noise_model(c->eng->get(), flat.data(), 0, nullptr));
            c->key = key;
            cache_ = c;
        }
        return cache_->eng->get();
    }

  private:
    struct Cache {
        std::shared_ptr<Engine> eng;
        std::tuple<int, bool, std::uint32_t, float, bool> key;
    };
    mutable std::shared_ptr<Cache> cache_;
    template <typename T>
    CMatrix<T> fetch_inverse(std::size_t bin, int precision) const {
        if (!cache_) throw ValidationError("noise model inverses not prepared");
        if (bin >= k.bins.size()) throw ValidationError("noise model inverses not prepared");
        const std::size_t m = k.m;
        std::vector<double> all(k.bins.size() * m * m * 2);
        check(sslg_noise_inverse(cache_->eng->get(), precision, all.data()));
        CMatrix<T> out(m, m);
        for (std::size_t i = 0; i < m * m; ++i)
            out.data[i] = std::complex<T>(T(all[(bin * m * m + i) * 2]), T(all[(bin * m * m + i) * 2 + 1]));
        return out;
    }
};

// ---- batched GSVD (gsvd.hpp:160-163) ------------------------------------------
namespace detail {
inline GsvdBatch<double> gsvd_device(const NoiseModel& noise, const CorrelationSet& r, SolverConfig cfg,
                                     bool budget) {
    cfg.validate();
    validate_set(r);
    validate_set(noise.k);
    if (noise.k.m != r.m) throw ValidationError("noise model channel count does not match correlation set");
    if (noise.k.bins.size() != r.bins.size())
        throw ValidationError("noise model bin count does not match correlation set");
    if (!budget) cfg.max_qr_sweeps = 0;  // gsvd_reference has no QR budget (gsvd.cpp:832-844)
    sslg_ctx* ctx = noise.context(cfg);
    const auto m = r.m;
    const auto nb = std::uint32_t(r.bins.size());
    const auto rf = flatten(r.bins);
    const std::size_t mm = std::size_t(m) * m;
    std::vector<double> sigma(std::size_t(nb) * m), ev(nb * mm * 2), er(nb * mm * 2), res(nb);
    std::vector<std::uint32_t> sweeps(nb);
    std::vector<std::uint8_t> conv(nb);
    check(sslg_gsvd_ex(ctx, rf.data(), 1, sigma.data(), ev.data(), er.data(), sweeps.data(), conv.data(), res.data()));
    GsvdBatch<double> out;
    out.bins.resize(nb);
    for (std::uint32_t b = 0; b < nb; ++b) {
        auto& o = out.bins[b];
        o.singular_values.assign(sigma.begin() + std::size_t(b) * m, sigma.begin() + std::size_t(b + 1) * m);
        o.e = CMatrix<double>(m, m);
        o.e_r = CMatrix<double>(m, m);
        for (std::size_t i = 0; i < mm; ++i) {
            o.e.data[i] = cdouble(ev[(b * mm + i) * 2], ev[(b * mm + i) * 2 + 1]);
            o.e_r.data[i] = cdouble(er[(b * mm + i) * 2], er[(b * mm + i) * 2 + 1]);
        }
        o.iterations = sweeps[b];
        o.converged = conv[b] != 0;
        o.recon_residual = res[b];
    }
    return out;
}
}  // namespace detail

inline GsvdBatch<double> gsvd_reference(const NoiseModel& noise, const CorrelationSet& r,
                                        const SolverConfig& cfg = {}, unsigned /*threads*/ = 0) {
    return detail::gsvd_device(noise, r, cfg, false);
}

inline GsvdBatch<float> gsvd(const NoiseModel& noise, const CorrelationSet& r, const SolverConfig& cfg = {},
                             unsigned /*threads*/ = 0) {
    const auto d = detail::gsvd_device(noise, r, cfg, true);
    GsvdBatch<float> out;
    out.bins.resize(d.bins.size());
    auto narrow = [](const CMatrix<double>& a) {
        CMatrix<float> o(a.rows, a.cols);
        for (std::size_t i = 0; i < o.data.size(); ++i) o.data[i] = cfloat(float(a.data[i].real()), float(a.data[i].imag()));
        return o;
    };
    for (std::size_t b = 0; b < d.bins.size(); ++b) {
        auto& o = out.bins[b];
        o.singular_values.assign(d.bins[b].singular_values.begin(), d.bins[b].singular_values.end());
        o.e = narrow(d.bins[b].e);
        o.e_r = narrow(d.bins[b].e_r);
        o.iterations = d.bins[b].iterations;
        o.converged = d.bins[b].converged;
        o.recon_residual = float(d.bins[b].recon_residual);
    }
    return out;
}

// ---- MUSIC spectrum + peaks (music.hpp:76-101) ----------------------------------
namespace detail {
// Device contexts of the stateless stage calls, reused across calls with the
// same configuration and inputs (a context holds the transposed steering
// table and the topology): one per thread, keyed by a content fingerprint.
struct StageCache {
    std::uint64_t key = 0;
    std::shared_ptr<Engine> eng;
};
inline StageCache& spectrum_cache() {
    thread_local StageCache c;
    return c;
}
inline StageCache& peaks_cache() {
    thread_local StageCache c;
    return c;
}
inline std::uint64_t music_key(const MusicConfig& cfg, std::uint64_t h) {
    h = fnv1a(&cfg.num_sources, sizeof cfg.num_sources, h);
    h = fnv1a(&cfg.denominator_floor, sizeof cfg.denominator_floor, h);
    const int sq = cfg.squared_denominator ? 1 : 0;
    h = fnv1a(&sq, sizeof sq, h);
    return fnv1a(&cfg.low_power_ratio, sizeof cfg.low_power_ratio, h);
}
}  // namespace detail

template <typename T>
MusicSpectrum calc_average_power(const GsvdBatch<T>& basis, const SteeringField& steering, const MusicConfig& cfg,
                                 bool keep_bins = false, unsigned /*threads*/ = 0) {
    steering.validate();
    const auto nb = std::uint32_t(basis.bins.size());
    if (nb != steering.bin_count()) throw ValidationError("steering field bin count does not match factorization");
    if (cfg.num_sources >= steering.m) throw ValidationError("num_sources must be smaller than the channel count");
    const auto m = steering.m;
    const auto nd = std::uint32_t(steering.directions.size());
    const auto dirs = detail::flat_dirs(steering.directions);
    std::uint64_t key = detail::fnv1a(steering.vectors.data(), steering.vectors.size() * sizeof(cfloat));
    key = detail::fnv1a(dirs.data(), dirs.size() * sizeof(double), key);
    key = detail::fnv1a(&m, sizeof m, detail::fnv1a(&nb, sizeof nb, detail::music_key(cfg, key)));
    auto& cache = detail::spectrum_cache();
    if (!cache.eng || cache.key != key) {
        cache.eng.reset();
        auto e = std::make_shared<Engine>(m, nb, 1, cfg, SolverConfig{}, 1);
        check(sslg_set_steering(e->get(), nd, reinterpret_cast<const float*>(steering.vectors.data()), dirs.data(),
                                nullptr, nullptr));
        cache.eng = e;
        cache.key = key;
    }
    std::vector<double> ev(std::size_t(nb) * m * m * 2);
    for (std::uint32_t b = 0; b < nb; ++b) {
        if (basis.bins[b].e.rows != m || basis.bins[b].e.cols != m)
            throw ValidationError("factorization channel count does not match steering field");
        for (std::size_t i = 0; i < std::size_t(m) * m; ++i) {
            ev[(std::size_t(b) * m * m + i) * 2] = double(basis.bins[b].e.data[i].real());
            ev[(std::size_t(b) * m * m + i) * 2 + 1] = double(basis.bins[b].e.data[i].imag());
        }
    }
    MusicSpectrum s;
    s.power.resize(nd);
    std::vector<double> bp(std::size_t(nb) * nd);
    check(sslg_spectrum(cache.eng->get(), ev.data(), 1, s.power.data(), bp.data()));
    if (keep_bins) {
        s.bin_power.assign(nb, std::vector<double>(nd));
        for (std::uint32_t b = 0; b < nb; ++b)
            for (std::uint32_t d = 0; d < nd; ++d) s.bin_power[b][d] = bp[std::size_t(b) * nd + d];
    }
    return s;
}

inline std::vector<SourceEstimate> peak_search(const std::vector<double>& power, const std::vector<Direction>& dirs,
                                               const DirectionTopology& topo, const MusicConfig& cfg) {
    if (power.size() != dirs.size() || topo.neighbors.size() != power.size())
        throw ValidationError("peak_search input sizes do not match");
    const auto nd = std::uint32_t(dirs.size());
    std::vector<std::uint32_t> off(nd + 1), nbr;
    for (std::uint32_t i = 0; i < nd; ++i) {
        off[i] = std::uint32_t(nbr.size());
        nbr.insert(nbr.end(), topo.neighbors[i].begin(), topo.neighbors[i].end());
    }
    off[nd] = std::uint32_t(nbr.size());
    if (nbr.empty()) nbr.push_back(0);
    const auto d = detail::flat_dirs(dirs);
    std::uint64_t key = detail::fnv1a(off.data(), off.size() * 4);
    key = detail::fnv1a(nbr.data(), nbr.size() * 4, key);
    key = detail::music_key(cfg, detail::fnv1a(d.data(), d.size() * sizeof(double), key));
    auto& cache = detail::peaks_cache();
    if (!cache.eng || cache.key != key) {
        cache.eng.reset();
        // a one-bin context whose steering vectors are placeholders: only the
        // topology and the grid size matter to the peak kernel
        auto e = std::make_shared<Engine>(cfg.num_sources + 1, 1, 1, cfg, SolverConfig{}, 1);
        std::vector<float> h(std::size_t(nd) * (cfg.num_sources + 1) * 2, 0.0f);
        check(sslg_set_steering(e->get(), nd, h.data(), d.data(), off.data(), nbr.data()));
        cache.eng = e;
        cache.key = key;
    }
    std::vector<std::uint32_t> idx(cfg.num_sources), cnt(1);
    std::vector<double> pw(cfg.num_sources);
    std::vector<std::uint8_t> low(cfg.num_sources);
    check(sslg_peaks(cache.eng->get(), power.data(), 1, idx.data(), pw.data(), low.data(), cnt.data()));
    std::vector<SourceEstimate> out;
    for (std::uint32_t i = 0; i < cnt[0]; ++i) out.push_back({idx[i], dirs[idx[i]], pw[i], low[i] != 0});
    return out;
}

// The JSONL record run_locate_to_stream writes per emitted block
// (pipeline.cpp:268-283), laid out as nlohmann::json::dump() does.
inline std::string format_estimates_json(const FrameEstimates& fe) {
    const auto n = std::uint32_t(fe.estimates.size());
    std::uint32_t top = 0;
    for (const auto& e : fe.estimates) top = std::max(top, e.direction_index + 1);
    // a grid just large enough to hold each estimate's direction at its index
    std::vector<double> dirs(2 * std::size_t(top ? top : 1));
    std::vector<std::uint32_t> idx(n ? n : 1);
    std::vector<double> pw(n ? n : 1);
    std::vector<std::uint8_t> low(n ? n : 1);
    for (std::uint32_t i = 0; i < n; ++i) {
        const auto& e = fe.estimates[i];
        idx[i] = e.direction_index;
        dirs[2 * std::size_t(e.direction_index)] = e.direction.azimuth_deg;
        dirs[2 * std::size_t(e.direction_index) + 1] = e.direction.elevation_deg;
        pw[i] = e.power;
        low[i] = e.low_power ? 1 : 0;
    }
    std::uint64_t len = 0;
    check(sslg_format_estimates_json(fe.frame_index, n, idx.data(), dirs.data(), pw.data(), low.data(), nullptr, 0,
                                     &len));
    std::string s(len + 1, '\0');
    check(sslg_format_estimates_json(fe.frame_index, n, idx.data(), dirs.data(), pw.data(), low.data(), &s[0],
                                     len + 1, &len));
    s.resize(len);
    return s;
}

// ---- streaming driver (run_locate's loop, pipeline.cpp:227-245) -------------------
// On STFT frames (SpectrumFrame); the SampleBlock overload below runs the STFT
// on the device.
inline std::size_t run_locate(const std::vector<SpectrumFrame>& frames, std::uint32_t window_frames,
                              const NoiseModel& noise, const SteeringField& steering, const SolverConfig& solver,
                              const MusicConfig& music, unsigned /*threads*/,
                              const std::function<void(const FrameEstimates&)>& sink,
                              std::uint32_t max_batch = 16) {
    if (window_frames == 0) throw ValidationError("window_frames must be at least 1");
    if (noise.k.m != steering.m) throw ValidationError("noise model channel count does not match steering field");
    const auto m = steering.m;
    const auto nb = std::uint32_t(steering.bin_count());
    if (noise.k.bins.size() != nb) throw ValidationError("noise model bin count does not match the analysis band");
    Engine e(m, nb, window_frames, music, solver, max_batch);
    const auto kf = detail::flatten(noise.k.bins);
    check(sslg_set_noise_model(e.get(), kf.data(), 0, nullptr));
    const auto nd = std::uint32_t(steering.directions.size());
    const auto d = detail::flat_dirs(steering.directions);
    check(sslg_set_steering(e.get(), nd, reinterpret_cast<const float*>(steering.vectors.data()), d.data(), nullptr,
                            nullptr));
    std::vector<float> x;
    x.reserve(frames.size() * m * nb * 2);
    for (const auto& f : frames) {
        if (f.spectra.size() != m) throw ValidationError("spectrum frame shape changed mid-stream");
        for (const auto& ch : f.spectra) {
            if (ch.size() != nb) throw ValidationError("ragged spectrum frame");
            for (const auto& z : ch) {
                x.push_back(z.real());
                x.push_back(z.imag());
            }
        }
    }
    const auto nf = std::uint32_t(frames.size());
    const auto ns = music.num_sources;
    std::vector<sslg_block_out> blocks(nf ? nf : 1);
    std::vector<std::uint32_t> idx(std::size_t(nf) * ns + 1);
    std::vector<double> pw(std::size_t(nf) * ns + 1);
    std::vector<std::uint8_t> low(std::size_t(nf) * ns + 1);
    std::uint32_t emitted = 0;
    // blocks before a non-finite frame reach the sink before the error (the
    // reference's per-frame loop has sunk them when the bad frame throws)
    const int rc =
        sslg_push_frames(e.get(), x.data(), nf, blocks.data(), idx.data(), pw.data(), low.data(), nullptr, &emitted);
    for (std::uint32_t b = 0; b < emitted; ++b) {
        FrameEstimates fe;
        fe.frame_index = frames[blocks[b].frame_index].frame_index;
        for (std::uint32_t i = 0; i < blocks[b].count; ++i) {
            const auto j = idx[std::size_t(b) * ns + i];
            fe.estimates.push_back({j, steering.directions[j], pw[std::size_t(b) * ns + i], low[std::size_t(b) * ns + i] != 0});
        }
        sink(fe);
    }
    check(rc);
    return emitted;
}

// run_locate with the reference's exact signature (pipeline.hpp:71-75): the
// SampleBlock goes through the device STFT (bit-identical frames, stft.cpp:38-68)
// straight into the correlation window.
inline std::size_t run_locate(const SampleBlock& audio, const StftConfig& stft, std::uint32_t window_frames,
                              const NoiseModel& noise, const SteeringField& steering, const SolverConfig& solver,
                              const MusicConfig& music, SolvePath /*path*/, unsigned /*threads*/,
                              const std::function<void(const FrameEstimates&)>& sink, std::uint32_t max_batch = 16) {
    audio.validate();
    if (window_frames == 0) throw ValidationError("window_frames must be at least 1");
    if (noise.k.m != steering.m) throw ValidationError("noise model channel count does not match steering field");
    if (audio.channel_count() != steering.m) throw ValidationError("sample block channel count does not match");
    const auto m = steering.m;
    const auto nb = std::uint32_t(steering.bin_count());
    if (noise.k.bins.size() != stft.bin_count() || nb != stft.bin_count())
        throw ValidationError("noise model bin count does not match the analysis band");
    Engine e(m, nb, window_frames, music, solver, max_batch);
    const auto kf = detail::flatten(noise.k.bins);
    check(sslg_set_noise_model(e.get(), kf.data(), 0, nullptr));
    const auto nd = std::uint32_t(steering.directions.size());
    const auto d = detail::flat_dirs(steering.directions);
    check(sslg_set_steering(e.get(), nd, reinterpret_cast<const float*>(steering.vectors.data()), d.data(), nullptr,
                            nullptr));
    sslg_stft_config sc{stft.frame_length, stft.shift, stft.window == WindowKind::hann ? 0 : 1, stft.bin_min,
                        stft.bin_max};
    check(sslg_set_stft(e.get(), &sc));
    const std::size_t n = audio.frame_count();
    std::vector<float> pcm;
    pcm.reserve(m * n);
    for (const auto& c : audio.channels) pcm.insert(pcm.end(), c.begin(), c.end());
    std::uint32_t frames = 0;
    check(sslg_stft(e.get(), pcm.data(), n, nullptr, 0, &frames));
    const std::uint32_t cap = frames >= window_frames ? frames - window_frames + 1 : 0;
    const auto ns = music.num_sources;
    std::vector<sslg_block_out> blocks(cap ? cap : 1);
    std::vector<std::uint32_t> idx(std::size_t(cap) * ns + 1);
    std::vector<double> pw(std::size_t(cap) * ns + 1);
    std::vector<std::uint8_t> low(std::size_t(cap) * ns + 1);
    std::uint32_t emitted = 0;
    const int rc = sslg_locate_samples(e.get(), pcm.data(), n, cap, blocks.data(), idx.data(), pw.data(), low.data(),
                                       nullptr, &emitted);
    for (std::uint32_t b = 0; b < emitted; ++b) {
        FrameEstimates fe;
        fe.frame_index = blocks[b].frame_index;
        for (std::uint32_t i = 0; i < blocks[b].count; ++i) {
            const auto j = idx[std::size_t(b) * ns + i];
            fe.estimates.push_back({j, steering.directions[j], pw[std::size_t(b) * ns + i], low[std::size_t(b) * ns + i] != 0});
        }
        sink(fe);
    }
    check(rc);
    return emitted;
}

}  // namespace b200
}  // namespace ssl
