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
    std::uint32_t max_qr_sweeps = 0;  // QR-solver knob of the reference; accepted, unused
    float tolerance_scale = 1.0f;     // idem
    Pivoting pivoting = Pivoting::partial;
    bool compute_residual = false;
    bool canonical_subspaces = true;
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
};

template <typename T>
struct GsvdBinResult {
    std::vector<T> singular_values;
    CMatrix<T> e;
    CMatrix<T> e_r;  // not produced by the engine (left vectors only)
    std::uint32_t iterations = 0;
    bool converged = true;
    T recon_residual = T(-1);
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
           const SolverConfig& sc, std::uint32_t max_batch = 16, int device = 0) {
        sslg_config cfg;
        sslg_config_default(&cfg);
        cfg.m = m;
        cfg.bins = bins;
        cfg.window_frames = window_frames;
        cfg.num_sources = mc.num_sources;
        cfg.denominator_floor = mc.denominator_floor;
        cfg.squared_denominator = mc.squared_denominator ? 1 : 0;
        cfg.low_power_ratio = mc.low_power_ratio;
        cfg.pivoting = sc.pivoting == Pivoting::partial ? 1 : 0;
        cfg.canonical_subspaces = sc.canonical_subspaces ? 1 : 0;
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
}  // namespace detail

// NoiseModel (gsvd.hpp:31-50): K kept on the host, inverses built on the device
struct NoiseModel {
    CorrelationSet k;
    static NoiseModel identity(std::uint32_t m, std::size_t bins) {
        NoiseModel n;
        n.k.m = m;
        n.k.bins.assign(bins, CMatrix<float>::identity(m));
        return n;
    }
    void check_positive_definite() const {
        Engine e(k.m, std::uint32_t(k.bins.size()), 1, MusicConfig{}, SolverConfig{});
        const auto flat = detail::flatten(k.bins);
        check(sslg_set_noise_model(e.get(), flat.data(), 1, nullptr));
    }
};

// ---- batched GSVD (gsvd.hpp:160-163) ------------------------------------------
inline GsvdBatch<double> gsvd_reference(const NoiseModel& noise, const CorrelationSet& r,
                                        const SolverConfig& cfg = {}, unsigned /*threads*/ = 0) {
    if (noise.k.m != r.m) throw ValidationError("noise model channel count does not match correlation set");
    if (noise.k.bins.size() != r.bins.size())
        throw ValidationError("noise model bin count does not match correlation set");
    const auto m = r.m;
    const auto nb = std::uint32_t(r.bins.size());
    Engine e(m, nb, 1, MusicConfig{}, cfg, 1);
    const auto kf = detail::flatten(noise.k.bins);
    check(sslg_set_noise_model(e.get(), kf.data(), 0, nullptr));
    const auto rf = detail::flatten(r.bins);
    std::vector<double> sigma(std::size_t(nb) * m), ev(std::size_t(nb) * m * m * 2);
    std::vector<std::uint32_t> sweeps(nb);
    std::vector<std::uint8_t> conv(nb);
    check(sslg_gsvd(e.get(), rf.data(), 1, sigma.data(), ev.data(), sweeps.data(), conv.data()));
    GsvdBatch<double> out;
    out.bins.resize(nb);
    for (std::uint32_t b = 0; b < nb; ++b) {
        auto& o = out.bins[b];
        o.singular_values.assign(sigma.begin() + std::size_t(b) * m, sigma.begin() + std::size_t(b + 1) * m);
        o.e = CMatrix<double>(m, m);
        for (std::size_t i = 0; i < std::size_t(m) * m; ++i)
            o.e.data[i] = cdouble(ev[(std::size_t(b) * m * m + i) * 2], ev[(std::size_t(b) * m * m + i) * 2 + 1]);
        o.iterations = sweeps[b];
        o.converged = conv[b] != 0;
    }
    return out;
}

inline GsvdBatch<float> gsvd(const NoiseModel& noise, const CorrelationSet& r, const SolverConfig& cfg = {},
                             unsigned threads = 0) {
    const auto d = gsvd_reference(noise, r, cfg, threads);
    GsvdBatch<float> out;
    out.bins.resize(d.bins.size());
    for (std::size_t b = 0; b < d.bins.size(); ++b) {
        auto& o = out.bins[b];
        o.singular_values.assign(d.bins[b].singular_values.begin(), d.bins[b].singular_values.end());
        o.e = CMatrix<float>(d.bins[b].e.rows, d.bins[b].e.cols);
        for (std::size_t i = 0; i < o.e.data.size(); ++i)
            o.e.data[i] = cfloat(float(d.bins[b].e.data[i].real()), float(d.bins[b].e.data[i].imag()));
        o.iterations = d.bins[b].iterations;
        o.converged = d.bins[b].converged;
    }
    return out;
}

// ---- MUSIC spectrum + peaks (music.hpp:76-101) ----------------------------------
template <typename T>
MusicSpectrum calc_average_power(const GsvdBatch<T>& basis, const SteeringField& steering, const MusicConfig& cfg,
                                 bool keep_bins = false, unsigned /*threads*/ = 0) {
    const auto nb = std::uint32_t(basis.bins.size());
    if (nb != steering.bin_count()) throw ValidationError("steering field bin count does not match factorization");
    if (cfg.num_sources >= steering.m) throw ValidationError("num_sources must be smaller than the channel count");
    const auto m = steering.m;
    const auto nd = std::uint32_t(steering.directions.size());
    Engine e(m, nb, 1, cfg, SolverConfig{}, 1);
    const auto dirs = detail::flat_dirs(steering.directions);
    check(sslg_set_steering(e.get(), nd, reinterpret_cast<const float*>(steering.vectors.data()), dirs.data(),
                            nullptr, nullptr));
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
    check(sslg_spectrum(e.get(), ev.data(), 1, s.power.data(), bp.data()));
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
    Engine e(cfg.num_sources + 1, 1, 1, cfg, SolverConfig{}, 1);
    std::vector<std::uint32_t> off(nd + 1), nbr;
    for (std::uint32_t i = 0; i < nd; ++i) {
        off[i] = std::uint32_t(nbr.size());
        nbr.insert(nbr.end(), topo.neighbors[i].begin(), topo.neighbors[i].end());
    }
    off[nd] = std::uint32_t(nbr.size());
    if (nbr.empty()) nbr.push_back(0);
    std::vector<float> h(std::size_t(nd) * (cfg.num_sources + 1) * 2, 0.0f);
    const auto d = detail::flat_dirs(dirs);
    check(sslg_set_steering(e.get(), nd, h.data(), d.data(), off.data(), nbr.data()));
    std::vector<std::uint32_t> idx(cfg.num_sources), cnt(1);
    std::vector<double> pw(cfg.num_sources);
    std::vector<std::uint8_t> low(cfg.num_sources);
    check(sslg_peaks(e.get(), power.data(), 1, idx.data(), pw.data(), low.data(), cnt.data()));
    std::vector<SourceEstimate> out;
    for (std::uint32_t i = 0; i < cnt[0]; ++i) out.push_back({idx[i], dirs[idx[i]], pw[i], low[i] != 0});
    return out;
}

// ---- streaming driver (run_locate's loop, pipeline.cpp:227-245) -------------------
// Frames are STFT frames (SpectrumFrame); the audio-side STFT is out of scope.
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
    check(sslg_push_frames(e.get(), x.data(), nf, blocks.data(), idx.data(), pw.data(), low.data(), nullptr, &emitted));
    for (std::uint32_t b = 0; b < emitted; ++b) {
        FrameEstimates fe;
        fe.frame_index = frames[blocks[b].frame_index].frame_index;
        for (std::uint32_t i = 0; i < blocks[b].count; ++i) {
            const auto j = idx[std::size_t(b) * ns + i];
            fe.estimates.push_back({j, steering.directions[j], pw[std::size_t(b) * ns + i], low[std::size_t(b) * ns + i] != 0});
        }
        sink(fe);
    }
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
    check(sslg_locate_samples(e.get(), pcm.data(), n, cap, blocks.data(), idx.data(), pw.data(), low.data(), nullptr,
                              &emitted));
    for (std::uint32_t b = 0; b < emitted; ++b) {
        FrameEstimates fe;
        fe.frame_index = blocks[b].frame_index;
        for (std::uint32_t i = 0; i < blocks[b].count; ++i) {
            const auto j = idx[std::size_t(b) * ns + i];
            fe.estimates.push_back({j, steering.directions[j], pw[std::size_t(b) * ns + i], low[std::size_t(b) * ns + i] != 0});
        }
        sink(fe);
    }
    return emitted;
}

}  // namespace b200
}  // namespace ssl
