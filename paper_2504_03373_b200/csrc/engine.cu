// Host engine behind the C ABI of include/sslgpu.h.
//
// Owns the device-resident state of one localization stream: the noise model
// (K and the FP64 K^-1), the transposed steering table with |h|^2, the
// topology CSR, the spectrum-frame ring and FP64 running correlation sum, and
// the per-block work buffers (R, sigma, E, P, Pbar, estimates).  A push of F
// frames is one pass over the hot path:
//
//   ring <- frames (H2D or D2D)      non-finite gate
//   correlation_kernel   grid bins                      -> R  [F'][bins][m][m]
//   jacobi_kernel        grid F' x bins                 -> sigma, E (sorted)
//   canonical_kernel     grid F' x bins                 -> E canonicalized
//   spectrum_kernel      grid F' x bins x dir-chunks    -> P  [F'][bins][dirs]
//   integrate_peaks      grid F'                        -> Pbar, estimates
//
// where F' = frames that complete a full window.  Everything runs on one CUDA
// stream (the caller's, if given) with CUDA events between stages; nothing on
// the path falls back to the CPU.
#include "../../include/sslgpu.h"
#include "common.cuh"
#include "kernels.cuh"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a profiler attaches

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

namespace sslg {

// [n][m][m] transpose of the trailing square (row-major <-> vector-major)
__global__ void transpose_sq_kernel(const double2* __restrict__ in, double2* __restrict__ out, int m, size_t n) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t mm = (size_t)m * m;
    if (idx >= n * mm) return;
    const size_t b = idx / mm;
    const int e = (int)(idx % mm);
    const int i = e / m, j = e % m;
    out[b * mm + (size_t)j * m + i] = in[idx];
}

}  // namespace sslg

using namespace sslg;

namespace {
thread_local std::string g_err;
}  // namespace

namespace sslg {
// the message of the last failure on this thread (sslg_last_error); shared
// with the format loaders (formats.cu)
int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace sslg

namespace {

int set_err(int code, const std::string& msg) { return sslg::set_error(code, msg); }

// grids from this size up take the tcgen05 spectrum (C4: 1368 directions)
constexpr uint32_t kSpectrumTcMinDirs = 512;

// NVTX range per hot-path stage: the host-side launch spans of
// correlation, GSVD, MUSIC + peaks, STFT and the pushes that contain them
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(SSLG_DEVICE, std::string(#call ": ") + cudaGetErrorString(e_));         \
    } while (0)

template <typename T>
int dalloc(T** p, size_t n) {
    *p = nullptr;
    if (n == 0) return 0;
    CU(cudaMalloc((void**)p, n * sizeof(T)));
    return 0;
}

}  // namespace

struct sslg_ctx {
    sslg_config cfg{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // noise model
    float2* k = nullptr;
    double2* kinv = nullptr;
    bool have_noise = false;
    // steering
    uint32_t dirs = 0;
    float2* h_raw = nullptr;  // [dirs][bins][m] staging
    float2* h_t = nullptr;    // [bins][dirs][m]
    double* num = nullptr;    // [bins][dirs]
    uint32_t* nbr_off = nullptr;
    uint32_t* nbr = nullptr;
    uint32_t nnz = 0;
    bool have_steering = false;
    // window
    float2* ring = nullptr;
    int cap = 0;
    double2* state = nullptr;
    long long pushed = 0;
    long long since = 0;
    // work buffers (max_batch blocks)
    float2* r = nullptr;
    double* sigma = nullptr;
    double2* e = nullptr;
    double2* e_tmp = nullptr;
    uint32_t* sweeps = nullptr;
    uint8_t* conv = nullptr;
    uint32_t* work = nullptr;  // generic-canonicalization worklist
    double2* ascratch = nullptr;  // A copies for the preconditioned back-multiply
    double2* wscratch = nullptr;  // W between the split solver kernels (m = 60)
    uint32_t* done = nullptr;     // per-(block, bin) sweep-completion epochs of the split solver
    uint32_t epoch = 0;           // last epoch handed to the split solver
    int* pivs = nullptr;          // QR pivots between them
    long long* phase_clk = nullptr;  // solver phase clocks (SSLG_PHASE_CLOCKS=1)
    double* p = nullptr;
    double* power = nullptr;
    uint32_t* est_idx = nullptr;
    double* est_pw = nullptr;
    uint8_t* est_low = nullptr;
    uint32_t* est_count = nullptr;
    unsigned int* flags = nullptr;  // [0] nonfinite, [1] bad_f, [2] bad_d, [3] herm, [4] pd
    // last push bookkeeping
    uint32_t last_emitted = 0;
    long long last_first_frame = 0;
    uint32_t launches = 0;
    cudaEvent_t ev[6] = {};
    bool timed = false;
    // STFT front end (sslg_set_stft)
    sslg_stft_config stft{};
    bool have_stft = false;
    float* win = nullptr;          // [frame_length]
    double2* twiddle = nullptr;    // [frame_length - 1]
    double2* dft = nullptr;        // non-power-of-two frame length: [bins][frame_length] (cos, sin)
    float* samp[2] = {nullptr, nullptr};  // [m][samp_cap] sample history, ping-pong
    size_t samp_cap = 0;           // frame_length + max_batch * shift
    size_t samp_fill = 0;          // samples held in samp[samp_cur]
    int samp_cur = 0;
    float2* frame_scratch = nullptr;  // [max_batch][m][bins] for the stage entry point
    // asynchronous streaming (sslg_push_samples_async / sslg_wait_results)
    unsigned int* abort = nullptr;  // device word: 0, or 1 + id of the first sub-push whose gate failed
    struct Slot {
        cudaEvent_t done = nullptr;
        uint32_t* idx = nullptr;   // pinned [max_batch][ns]
        double* pw = nullptr;      // pinned [max_batch][ns]
        uint8_t* low = nullptr;    // pinned [max_batch][ns]
        uint32_t* cnt = nullptr;   // pinned [max_batch + 1]; cnt[max_batch]: the abort word after this sub-push
        double* power = nullptr;   // pinned [max_batch][dirs] (allocated with the steering)
        uint32_t n = 0;
        long long first_frame = 0;
        long long pushed0 = 0, since0 = 0;  // window counters before this sub-push
        uint64_t id = 0;
        bool pending = false;
    };
    static constexpr int kSlots = 16;
    Slot slots[kSlots];
    uint64_t next_id = 0;       // sub-pushes enqueued
    uint64_t collected = 0;     // sub-pushes handed back by sslg_wait_results
    bool poisoned = false;
    uint32_t poison_code = 0;
    bool async_power = false;   // async pushes also copy back power [e][dirs] (sslg_set_async_power)
    bool slots_ready = false;   // pinned result ring allocated (ensure_slots)
    int last_corr = -1;         // index in r of the newest set emitted by sslg_correlation (-1: none)
    int spectrum_tc = -1;       // -1 auto (grids >= kSpectrumTcMinDirs), 0 FP64 DMMA, 1 tcgen05 tf32x3
    float* tc_slabs = nullptr;  // steering operand slabs of the tcgen05 spectrum (built on first use)
    int small_cta = 0;          // SSLG_SMALL_CTA=1: m <= 16 on the CTA solver (A/B measurement)
    // device-frame pushes (sslg_push_frames_device) gate on the device through
    // the same abort word; their window counters are kept until the next
    // synchronizing call verifies the word (check_device_gate)
    struct DevPush {
        uint32_t seq;
        long long pushed0, since0;
    };
    std::deque<DevPush> dev_unverified;
    uint32_t dev_seq = 0;
};

namespace {

int sync_flags(sslg_ctx* c, unsigned int* host, int n) {
    CU(cudaMemcpyAsync(host, c->flags, n * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return 0;
}

int reset_flags(sslg_ctx* c) {
    // [0] non-finite count, [1..4] first bad bin (float/double inverse, Hermitian, PD), [5] first bad frame
    unsigned int init[8] = {0, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0, 0};
    CU(cudaMemcpyAsync(c->flags, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    return 0;
}

// SSLG_SYNC_DEBUG=1 synchronizes after every launch so a fault is reported
// against the kernel that caused it.
bool sync_debug() {
    static const bool on = [] {
        const char* v = std::getenv("SSLG_SYNC_DEBUG");
        return v && v[0] == '1';
    }();
    return on;
}

int check_last_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && sync_debug()) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return set_err(SSLG_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    return 0;
}

#define TRY(x)                 \
    do {                       \
        int rc_ = (x);         \
        if (rc_) return rc_;   \
    } while (0)

// Runs GSVD -> (canonical) on n correlation sets already in c->r.
int run_gsvd(sslg_ctx* c, int n) {
    Nvtx range("sslg:gsvd");
    const sslg_config& g = c->cfg;
    CU(cudaMemsetAsync(c->work, 0, 2 * sizeof(uint32_t), c->stream));
    GsvdArgs ga{c->r,   c->kinv, c->sigma, c->e, c->sweeps, c->conv, c->work, (int)g.m, (int)g.bins,
                g.max_sweeps ? (int)g.max_sweeps : 60, g.canonical_subspaces, g.refine_leading,
                g.precondition, c->ascratch, c->phase_clk};
    ga.abort = c->abort;
    ga.wscratch = c->wscratch;
    ga.pivs = c->pivs;
    ga.tol2 = 1e-28 * (double)g.tolerance_scale * (double)g.tolerance_scale;
    ga.force_cta = c->small_cta;
    ga.done = c->done;
    if (++c->epoch == 0) c->epoch = 1;  // flags start at 0: never a live epoch
    ga.epoch = c->epoch;
    c->launches += launch_jacobi(ga, n, c->stream);
    TRY(check_last_launch("jacobi_kernel"));
    CU(cudaEventRecord(c->ev[2], c->stream));
    // the lane-group solver (m <= 16) canonicalizes every bin itself unless
    // refine mode asks for the full-space A A^H refinement: no worklist pass
    if (g.canonical_subspaces && !(small_jacobi_selected(ga) && !g.refine_leading)) {
        CanonArgs ca{c->r, c->kinv, c->sigma, c->e, c->work, (int)g.m, (int)g.bins, g.refine_leading};
        ca.abort = c->abort;
        launch_canonical(ca, n, c->stream);
        ++c->launches;
        TRY(check_last_launch("canonical_kernel"));
    }
    CU(cudaEventRecord(c->ev[3], c->stream));
    return 0;
}

int run_music(sslg_ctx* c, int n) {
    Nvtx range("sslg:music+peaks");
    const sslg_config& g = c->cfg;
    SpecArgs sa{c->e, c->h_t, c->num, c->p, (int)g.m, (int)g.bins, (int)c->dirs, (int)g.num_sources, 0, 0,
                (double)g.denominator_floor, g.squared_denominator};
    sa.abort = c->abort;
    // large grids run on the tcgen05 tensor cores (kind::tf32, 3-pass split:
    // <= 5.6e-7 per bin, <= 2.8e-7 broadband vs FP64); SSLG_SPECTRUM_TC=0/1 or
    // sslg_set_spectrum_path force the FP64 DMMA / tcgen05 path
    const bool tc = spectrum_tc_supported(sa) &&
                    (c->spectrum_tc > 0 || (c->spectrum_tc < 0 && c->dirs >= kSpectrumTcMinDirs));
    if (tc && !c->tc_slabs) {  // the steering as tf32 hi/lo operand slabs, once per steering field
        TRY(dalloc(&c->tc_slabs, spectrum_tc_slab_floats((int)g.m, (int)g.bins, (int)c->dirs)));
        launch_spectrum_tc_prep(c->h_t, (int)g.m, (int)g.bins, (int)c->dirs, c->tc_slabs, c->stream);
        ++c->launches;
        TRY(check_last_launch("spectrum_tc_prep_kernel"));
    }
    if (tc) launch_spectrum_tc(sa, c->tc_slabs, n, c->stream);
    else launch_spectrum(sa, n, c->stream);
    ++c->launches;
    TRY(check_last_launch("spectrum_kernel"));
    CU(cudaEventRecord(c->ev[4], c->stream));
    PeakArgs pa{c->p, c->power, c->nbr_off, c->nbr, c->est_idx, c->est_pw, c->est_low, c->est_count,
                (int)g.bins, (int)c->dirs, (int)g.num_sources, (double)g.low_power_ratio};
    pa.abort = c->abort;
    launch_peaks(pa, n, c->stream);
    ++c->launches;
    TRY(check_last_launch("integrate_peaks_kernel"));
    CU(cudaEventRecord(c->ev[5], c->stream));
    return 0;
}

int gate_frames(sslg_ctx* c, uint32_t nframes, uint32_t* good);

// copies nframes frames (src: host or device) into the ring after the
// current push count, then gates on non-finite values: *good = the number of
// leading frames before the first non-finite one (nframes if none)
int stage_frames(sslg_ctx* c, const float* src, uint32_t nframes, cudaMemcpyKind kind, uint32_t* good) {
    const sslg_config& g = c->cfg;
    const size_t fsz = (size_t)g.m * g.bins;
    uint32_t done = 0;
    while (done < nframes) {
        const int slot = (int)((c->pushed + done) % c->cap);
        const uint32_t run = std::min<uint32_t>(nframes - done, (uint32_t)(c->cap - slot));
        CU(cudaMemcpyAsync(c->ring + (size_t)slot * fsz, src + (size_t)done * fsz * 2, run * fsz * sizeof(float2),
                           kind, c->stream));
        done += run;
    }
    return gate_frames(c, nframes, good);
}

// non-finite gate over the nframes ring slots after the push count
// (CorrelationWindow::push -> instantaneous_correlation check,
// correlation.cpp:16-17), frame by frame: the reference rejects the first
// non-finite frame and keeps every frame pushed before it
int gate_frames(sslg_ctx* c, uint32_t nframes, uint32_t* good) {
    const sslg_config& g = c->cfg;
    const size_t fsz = (size_t)g.m * g.bins;
    TRY(reset_flags(c));
    // gate every staged slot (a wrapped range is two spans)
    uint32_t done = 0;
    while (done < nframes) {
        const int slot = (int)((c->pushed + done) % c->cap);
        const uint32_t run = std::min<uint32_t>(nframes - done, (uint32_t)(c->cap - slot));
        launch_first_nonfinite(reinterpret_cast<const float*>(c->ring + (size_t)slot * fsz), fsz * 2, (int)run, done,
                               c->flags + 5, c->stream);
        ++c->launches;
        done += run;
    }
    unsigned int fl[6];
    TRY(sync_flags(c, fl, 6));
    *good = std::min<uint32_t>(fl[5], nframes);
    return 0;
}

// one chunk of at most max_batch frames already validated in the ring
int process_chunk(sslg_ctx* c, uint32_t nframes, uint32_t* emitted) {
    const sslg_config& g = c->cfg;
    *emitted = 0;
    if (nframes == 0) return 0;
    Nvtx range("sslg:push_chunk");
    const long long first_emit = std::max<long long>(0, (long long)g.window_frames - 1 - c->pushed);
    const int n = (int)std::max<long long>(0, (long long)nframes - first_emit);
    CU(cudaEventRecord(c->ev[0], c->stream));
    CorrArgs ca{c->ring, c->state, c->r, (int)g.m, (int)g.bins, (int)g.window_frames, c->cap, (int)nframes,
                c->pushed, c->since, (int)(g.rebuild_interval ? g.rebuild_interval : 1)};
    ca.abort = c->abort;
    {
        Nvtx range("sslg:correlation");
        launch_correlation(ca, c->stream);
    }
    ++c->launches;
    TRY(check_last_launch("correlation_kernel"));
    CU(cudaEventRecord(c->ev[1], c->stream));
    // host mirror of the push counters (correlation.cpp:103-109)
    for (uint32_t f = 0; f < nframes; ++f) {
        ++c->pushed;
        if (++c->since >= (long long)(g.rebuild_interval ? g.rebuild_interval : 1)) c->since = 0;
    }
    c->last_first_frame = c->pushed - n;
    c->last_emitted = (uint32_t)n;
    if (n > 0) c->last_corr = n - 1;
    if (n > 0) {
        TRY(run_gsvd(c, n));
        TRY(run_music(c, n));
    } else {
        for (int i = 2; i < 6; ++i) CU(cudaEventRecord(c->ev[i], c->stream));
    }
    c->timed = true;
    *emitted = (uint32_t)n;
    return 0;
}

// Asynchronous sub-pushes not yet handed back by sslg_wait_results own the
// device window, the work buffers and the abort word: every synchronous entry
// point is refused until they are collected (or the window is reset).
int require_no_async(sslg_ctx* c) {
    if (c->next_id != c->collected)
        return set_err(SSLG_VALIDATION,
                       "asynchronous pushes are pending; collect them with sslg_wait_results or reset the window");
    return 0;
}

// Verifies the device-side gate of the device-frame pushes since the last
// check: if one of them saw a non-finite value, every kernel from its gate on
// was skipped, so the window is rewound to just before that push (its ring
// slots lie outside the live window) and the error is reported here.
int check_device_gate(sslg_ctx* c) {
    if (c->dev_unverified.empty()) return 0;
    CU(cudaStreamSynchronize(c->stream));
    unsigned int ab = 0;
    CU(cudaMemcpy(&ab, c->abort, sizeof ab, cudaMemcpyDeviceToHost));
    if (ab) {
        const uint32_t seq = ab - 1u;
        for (const auto& d : c->dev_unverified)
            if (d.seq == seq) {
                c->pushed = d.pushed0;
                c->since = d.since0;
                break;
            }
        c->last_emitted = 0;
        c->dev_unverified.clear();
        CU(cudaMemset(c->abort, 0, sizeof(unsigned int)));
        return set_err(SSLG_VALIDATION, "non-finite spectrum value");
    }
    c->dev_unverified.clear();
    return 0;
}

int require_ready(sslg_ctx* c, bool verify_device_gate = true) {
    if (!c) return set_err(SSLG_VALIDATION, "null context");
    if (!c->have_noise) return set_err(SSLG_VALIDATION, "noise model not set");
    if (!c->have_steering) return set_err(SSLG_VALIDATION, "steering field not set");
    if (c->cfg.num_sources >= c->cfg.m)
        return set_err(SSLG_VALIDATION, "num_sources must be smaller than the channel count");
    if (c->poisoned) return set_err(SSLG_VALIDATION, "stream stopped by a non-finite spectrum value; reset the window");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    if (verify_device_gate || c->dev_unverified.size() >= 1024) TRY(check_device_gate(c));
    return 0;
}

// The pinned result ring of sslg_push_samples_async, allocated on first use.
int ensure_slots(sslg_ctx* c) {
    if (c->slots_ready) return 0;
    const size_t NB = c->cfg.max_batch, ns = c->cfg.num_sources;
    for (auto& sl : c->slots) {
        if (cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess ||
            cudaMallocHost(&sl.idx, NB * ns * sizeof(uint32_t)) != cudaSuccess ||
            cudaMallocHost(&sl.pw, NB * ns * sizeof(double)) != cudaSuccess ||
            cudaMallocHost(&sl.low, NB * ns) != cudaSuccess ||
            cudaMallocHost(&sl.cnt, (NB + 1) * sizeof(uint32_t)) != cudaSuccess ||
            (c->dirs && cudaMallocHost(&sl.power, NB * c->dirs * sizeof(double)) != cudaSuccess))
            return set_err(SSLG_DEVICE, "pinned result ring allocation failed");  // sslg_destroy frees the rest
    }
    c->slots_ready = true;
    return 0;
}

// SolverConfig::max_qr_sweeps (gsvd.cpp:597-605, 819-827): a bin whose solve
// took more sweeps than a nonzero budget is flagged non-converged with the
// budget as its iteration count; its factors stay the converged FP64 ones,
// which is what the reference's salvage through the exact path returns.
void apply_sweep_budget(uint32_t budget, uint32_t* sweeps, uint8_t* conv, size_t n) {
    if (!budget || !sweeps) return;
    for (size_t i = 0; i < n; ++i)
        if (sweeps[i] > budget) {
            sweeps[i] = budget;
            if (conv) conv[i] = 0;
        }
}

}  // namespace

extern "C" {

void sslg_config_default(sslg_config* cfg) {
    std::memset(cfg, 0, sizeof *cfg);
    cfg->window_frames = 50;
    cfg->rebuild_interval = 1000;
    cfg->num_sources = 1;
    cfg->denominator_floor = 1e-12f;
    cfg->squared_denominator = 0;
    cfg->low_power_ratio = 1.25f;
    cfg->pivoting = 1;
    cfg->canonical_subspaces = 1;
    cfg->refine_leading = 0;
    cfg->precondition = 1;
    cfg->max_sweeps = 0;
    cfg->max_batch = 16;
    cfg->device = 0;
    cfg->stream = nullptr;
    cfg->max_qr_sweeps = 0;
    cfg->tolerance_scale = 1.0f;
    cfg->compute_residual = 0;
}

const char* sslg_last_error(void) { return g_err.c_str(); }

int sslg_create(sslg_ctx** out, const sslg_config* cfg) {
    if (!out || !cfg) return set_err(SSLG_VALIDATION, "null argument");
    *out = nullptr;
    const sslg_config& g = *cfg;
    if (g.m < 1 || g.m > SSLG_MAX_M)
        return set_err(SSLG_VALIDATION, "channel count must be in [1, " + std::to_string(SSLG_MAX_M) + "]");
    if (g.bins < 1) return set_err(SSLG_VALIDATION, "correlation set has no bins");
    if (g.window_frames < 1) return set_err(SSLG_VALIDATION, "correlation window length must be >= 1");
    if (g.num_sources == 0) return set_err(SSLG_VALIDATION, "num_sources must be at least 1");
    if (!(g.denominator_floor > 0)) return set_err(SSLG_VALIDATION, "denominator_floor must be positive");
    if (!(g.low_power_ratio >= 0)) return set_err(SSLG_VALIDATION, "low_power_ratio must be non-negative");
    if (g.max_batch < 1) return set_err(SSLG_VALIDATION, "max_batch must be >= 1");
    if (!(g.tolerance_scale > 0)) return set_err(SSLG_VALIDATION, "tolerance_scale must be positive");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_err(SSLG_DEVICE, "no CUDA device available (the engine has no CPU fallback)");
    if (g.device < 0 || g.device >= ndev) return set_err(SSLG_DEVICE, "device ordinal out of range");
    CU(cudaSetDevice(g.device));
    auto* c = new sslg_ctx();
    c->cfg = g;
    if (c->cfg.rebuild_interval < 1) c->cfg.rebuild_interval = 1;
    if (g.stream) {
        c->stream = static_cast<cudaStream_t>(g.stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return set_err(SSLG_DEVICE, "cudaStreamCreate failed");
        }
        c->own_stream = true;
    }
    const size_t mm = (size_t)g.m * g.m;
    const size_t B = g.bins, NB = g.max_batch;
    c->cap = (int)(g.window_frames + g.max_batch);
    int rc = 0;
    rc |= dalloc(&c->k, B * mm);
    rc |= dalloc(&c->kinv, B * mm);
    rc |= dalloc(&c->ring, (size_t)c->cap * g.m * B);
    rc |= dalloc(&c->state, B * mm);
    rc |= dalloc(&c->r, NB * B * mm);
    rc |= dalloc(&c->sigma, NB * B * g.m);
    rc |= dalloc(&c->e, NB * B * mm);
    rc |= dalloc(&c->e_tmp, NB * B * mm);
    rc |= dalloc(&c->sweeps, NB * B);
    rc |= dalloc(&c->conv, NB * B);
    rc |= dalloc(&c->work, NB * B + 2);
    if (g.precondition) rc |= dalloc(&c->ascratch, NB * B * mm);
    if (g.precondition && g.m == 60 && !std::getenv("SSLG_FUSED_SOLVER")) {
        rc |= dalloc(&c->wscratch, NB * B * mm);
        rc |= dalloc(&c->done, NB * B);
        if (!rc) cudaMemset(c->done, 0, NB * B * sizeof(uint32_t));
        rc |= dalloc(&c->pivs, NB * B * 64);
    }
    if (const char* tc = std::getenv("SSLG_SPECTRUM_TC")) c->spectrum_tc = tc[0] == '1' ? 1 : 0;
    if (const char* sm = std::getenv("SSLG_SMALL_CTA")) c->small_cta = sm[0] == '1';
    if (const char* pc = std::getenv("SSLG_PHASE_CLOCKS"); pc && pc[0] == '1') {
        rc |= dalloc(&c->phase_clk, 8);
        if (!rc) cudaMemset(c->phase_clk, 0, 8 * sizeof(long long));
    }
    rc |= dalloc(&c->est_count, NB);
    rc |= dalloc(&c->flags, 8);
    rc |= dalloc(&c->abort, 1);
    if (!rc && cudaMemsetAsync(c->abort, 0, sizeof(unsigned int), c->stream) != cudaSuccess)
        rc = set_err(SSLG_DEVICE, "cudaMemset failed");
    // the pinned result ring of the asynchronous path is allocated on its
    // first use (ensure_slots): most contexts never need its 80 pinned buffers
    for (int i = 0; i < 6 && !rc; ++i)
        if (cudaEventCreate(&c->ev[i]) != cudaSuccess) rc = set_err(SSLG_DEVICE, "cudaEventCreate failed");
    if (!rc && cudaMemsetAsync(c->state, 0, B * mm * sizeof(double2), c->stream) != cudaSuccess)
        rc = set_err(SSLG_DEVICE, "cudaMemset failed");
    if (rc) {
        sslg_destroy(c);
        return rc;
    }
    *out = c;
    return SSLG_OK;
}

void sslg_destroy(sslg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->cfg.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    void* ptrs[] = {c->k,      c->kinv,  c->h_raw, c->h_t,   c->num,     c->nbr_off, c->nbr,
                    c->ring,   c->state, c->r,     c->sigma, c->e,       c->e_tmp,   c->sweeps,
                    c->conv,   c->work, c->ascratch, c->wscratch, c->done, c->pivs, c->phase_clk, c->p,     c->power, c->est_idx, c->est_pw, c->est_low, c->est_count,
                    c->flags};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (void* p : {(void*)c->win, (void*)c->twiddle, (void*)c->samp[0], (void*)c->samp[1], (void*)c->frame_scratch,
                    (void*)c->abort, (void*)c->tc_slabs, (void*)c->dft})
        if (p) cudaFree(p);
    for (auto& sl : c->slots) {
        for (void* p : {(void*)sl.idx, (void*)sl.pw, (void*)sl.low, (void*)sl.cnt, (void*)sl.power})
            if (p) cudaFreeHost(p);
        if (sl.done) cudaEventDestroy(sl.done);
    }
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int sslg_get_config(const sslg_ctx* c, sslg_config* cfg) {
    if (!c || !cfg) return set_err(SSLG_VALIDATION, "null argument");
    *cfg = c->cfg;
    cfg->dirs = c->dirs;
    return SSLG_OK;
}

}  // extern "C"

namespace {

// check_positive_definite (gsvd.cpp:736-754) of a device K [bins][m][m]
int pd_gate(sslg_ctx* c, const float2* kdev, uint32_t* bad_bin) {
    const sslg_config& g = c->cfg;
    TRY(reset_flags(c));
    unsigned int fl[5];
    double* min_eig = nullptr;
    TRY(dalloc(&min_eig, g.bins));
    launch_pd_check(kdev, (int)g.m, (int)g.bins, c->flags + 3, c->flags + 4, min_eig, c->stream);
    int rc = check_last_launch("pd_check_kernel");
    if (!rc) rc = sync_flags(c, fl, 5);
    if (!rc && (fl[3] != 0xffffffffu || fl[4] != 0xffffffffu)) {
        // the reference checks bin by bin, Hermitian test first (gsvd.cpp:737-752)
        const unsigned b = std::min(fl[3], fl[4]);
        const bool herm = fl[3] == b;
        if (bad_bin) *bad_bin = b;
        double ev = 0;
        if (!herm) cudaMemcpy(&ev, min_eig + b, sizeof ev, cudaMemcpyDeviceToHost);
        char buf[64];
        std::snprintf(buf, sizeof buf, "%f", ev);  // std::to_string(double)
        rc = set_err(SSLG_NUMERICAL, herm ? "noise model is not Hermitian at bin " + std::to_string(b)
                                          : "noise model is not positive definite at bin " + std::to_string(b) +
                                                " (min eigenvalue " + buf + ")");
    }
    cudaFree(min_eig);
    return rc;
}

// NoiseModel::prepare_inverses (gsvd.cpp:756-768) of the K already in c->k
int install_noise(sslg_ctx* c, uint32_t* bad_bin) {
    const sslg_config& g = c->cfg;
    TRY(reset_flags(c));
    unsigned int fl[5];
    launch_gauss_jordan(c->k, (int)g.m, (int)g.bins, c->kinv, c->flags + 1, c->flags + 2, c->stream, g.pivoting);
    TRY(check_last_launch("gauss_jordan_kernel"));
    TRY(sync_flags(c, fl, 3));
    const unsigned bad = std::min(fl[1], fl[2]);
    if (bad != 0xffffffffu) {
        if (bad_bin) *bad_bin = bad;
        return set_err(SSLG_NUMERICAL, "noise matrix is singular at bin " + std::to_string(bad));
    }
    c->have_noise = true;
    return 0;
}

}  // namespace

extern "C" {

int sslg_set_noise_model(sslg_ctx* c, const float* k, int check_pd, uint32_t* bad_bin) {
    if (!c || !k) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    const sslg_config& g = c->cfg;
    const size_t mm = (size_t)g.m * g.m;
    const size_t n = g.bins * mm * 2;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(k[i])) return set_err(SSLG_VALIDATION, "non-finite correlation entry");
    c->have_noise = false;
    CU(cudaMemcpyAsync(c->k, k, g.bins * mm * sizeof(float2), cudaMemcpyHostToDevice, c->stream));
    if (check_pd) TRY(pd_gate(c, c->k, bad_bin));
    return install_noise(c, bad_bin);
}

int sslg_noise_inverse(sslg_ctx* c, int precision, double* out) {
    if (!c || !out) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->have_noise) return set_err(SSLG_VALIDATION, "noise model inverses not prepared");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    const sslg_config& g = c->cfg;
    const size_t n = (size_t)g.bins * g.m * g.m;
    if (precision) {
        CU(cudaMemcpyAsync(out, c->kinv, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        return SSLG_OK;
    }
    // the float inverse is not kept by the engine (the solver is FP64): rebuild it
    double2 *f = nullptr, *d = nullptr;
    TRY(dalloc(&f, n));
    int rc = dalloc(&d, n);
    if (!rc) rc = reset_flags(c);
    if (!rc) {
        launch_gauss_jordan(c->k, (int)g.m, (int)g.bins, d, c->flags + 1, c->flags + 2, c->stream, g.pivoting, f);
        rc = check_last_launch("gauss_jordan_kernel");
    }
    if (!rc && cudaMemcpyAsync(out, f, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
        rc = set_err(SSLG_DEVICE, "cudaMemcpy failed");
    if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = set_err(SSLG_DEVICE, "sync failed");
    cudaFree(f);
    if (d) cudaFree(d);
    return rc;
}

int sslg_set_noise_identity(sslg_ctx* c) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    const size_t mm = (size_t)c->cfg.m * c->cfg.m;
    std::vector<float> k(c->cfg.bins * mm * 2, 0.0f);
    for (size_t b = 0; b < c->cfg.bins; ++b)
        for (size_t i = 0; i < c->cfg.m; ++i) k[(b * mm + i * c->cfg.m + i) * 2] = 1.0f;
    return sslg_set_noise_model(c, k.data(), 0, nullptr);
}

int sslg_build_topology(const double* dirs_deg, uint32_t n, double radius_deg, uint32_t* nbr_off, uint32_t* nbr,
                        uint32_t cap, uint32_t* nnz) {
    // DirectionTopology::build (music.cpp:176-195): unit vectors in FP64,
    // neighbors where the dot product reaches cos(radius)
    const double pi = 3.14159265358979323846;
    std::vector<double> u(3 * (size_t)n);
    for (uint32_t i = 0; i < n; ++i) {
        const double az = dirs_deg[2 * i] * pi / 180.0;
        const double el = dirs_deg[2 * i + 1] * pi / 180.0;
        u[3 * i] = std::cos(el) * std::cos(az);
        u[3 * i + 1] = std::cos(el) * std::sin(az);
        u[3 * i + 2] = std::sin(el);
    }
    const double cr = std::cos(radius_deg * pi / 180.0);
    std::vector<std::vector<uint32_t>> lists(n);
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = i + 1; j < n; ++j) {
            const double dot = u[3 * i] * u[3 * j] + u[3 * i + 1] * u[3 * j + 1] + u[3 * i + 2] * u[3 * j + 2];
            if (dot >= cr) {
                lists[i].push_back(j);
                lists[j].push_back(i);
            }
        }
    uint32_t total = 0;
    for (uint32_t i = 0; i < n; ++i) total += (uint32_t)lists[i].size();
    if (nnz) *nnz = total;
    if (total > cap || !nbr_off || (!nbr && total))
        return set_err(SSLG_VALIDATION, "topology capacity too small: need " + std::to_string(total));
    uint32_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
        nbr_off[i] = o;
        for (uint32_t j : lists[i]) nbr[o++] = j;
    }
    nbr_off[n] = o;
    return SSLG_OK;
}

int sslg_set_steering(sslg_ctx* c, uint32_t dirs, const float* h, const double* dirs_deg, const uint32_t* nbr_off,
                      const uint32_t* nbr) {
    if (!c || !h) return set_err(SSLG_VALIDATION, "null argument");
    if (dirs == 0) return set_err(SSLG_VALIDATION, "steering field has no directions");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    const sslg_config& g = c->cfg;
    std::vector<uint32_t> off_own, nbr_own;
    if (!nbr_off) {
        if (!dirs_deg) return set_err(SSLG_VALIDATION, "directions are needed to build the topology");
        uint32_t need = 0;
        off_own.resize(dirs + 1);
        sslg_build_topology(dirs_deg, dirs, 10.0, off_own.data(), nullptr, 0, &need);
        nbr_own.resize(std::max<uint32_t>(need, 1));
        TRY(sslg_build_topology(dirs_deg, dirs, 10.0, off_own.data(), nbr_own.data(), need, &need));
        nbr_off = off_own.data();
        nbr = nbr_own.data();
    }
    const uint32_t nnz = nbr_off[dirs];
    for (uint32_t d = 0; d < dirs; ++d)
        if (nbr_off[d] > nbr_off[d + 1]) return set_err(SSLG_VALIDATION, "neighbor offsets must be non-decreasing");
    for (uint32_t k = 0; k < nnz; ++k)
        if (nbr[k] >= dirs) return set_err(SSLG_VALIDATION, "neighbor index out of range");
    const size_t hn = (size_t)dirs * g.bins * g.m;
    for (size_t i = 0; i < 2 * hn; ++i)
        if (!std::isfinite(h[i])) return set_err(SSLG_VALIDATION, "non-finite steering value");
    if (dirs != c->dirs) {
        // the new buffers are allocated first: on failure the context keeps
        // its previous steering field intact
        const size_t NB = g.max_batch;
        float2 *h_raw = nullptr, *h_t = nullptr;
        double *num = nullptr, *p = nullptr, *power = nullptr, *est_pw = nullptr;
        uint32_t* est_idx = nullptr;
        uint8_t* est_low = nullptr;
        double* slot_power[sslg_ctx::kSlots] = {};
        int rc = 0;
        rc |= dalloc(&h_raw, hn);
        rc |= dalloc(&h_t, hn);
        rc |= dalloc(&num, (size_t)g.bins * dirs);
        rc |= dalloc(&p, NB * g.bins * dirs);
        rc |= dalloc(&power, NB * dirs);
        rc |= dalloc(&est_idx, NB * g.num_sources);
        rc |= dalloc(&est_pw, NB * g.num_sources);
        rc |= dalloc(&est_low, NB * g.num_sources);
        for (int i = 0; i < sslg_ctx::kSlots && !rc && c->slots_ready; ++i)
            if (cudaMallocHost(&slot_power[i], NB * dirs * sizeof(double)) != cudaSuccess)
                rc = set_err(SSLG_DEVICE, "pinned result ring allocation failed");
        if (rc) {
            for (void* q : {(void*)h_raw, (void*)h_t, (void*)num, (void*)p, (void*)power, (void*)est_idx,
                            (void*)est_pw, (void*)est_low})
                if (q) cudaFree(q);
            for (double* q : slot_power)
                if (q) cudaFreeHost(q);
            return rc;
        }
        CU(cudaStreamSynchronize(c->stream));  // nothing in flight may still use the old buffers
        for (void* q : {(void*)c->h_raw, (void*)c->h_t, (void*)c->num, (void*)c->p, (void*)c->power,
                        (void*)c->est_idx, (void*)c->est_pw, (void*)c->est_low})
            if (q) cudaFree(q);
        c->h_raw = h_raw;
        c->h_t = h_t;
        c->num = num;
        c->p = p;
        c->power = power;
        c->est_idx = est_idx;
        c->est_pw = est_pw;
        c->est_low = est_low;
        for (int i = 0; i < sslg_ctx::kSlots && c->slots_ready; ++i) {
            if (c->slots[i].power) cudaFreeHost(c->slots[i].power);
            c->slots[i].power = slot_power[i];
        }
        c->dirs = dirs;
        c->last_emitted = 0;
    }
    if (c->nbr_off) cudaFree(c->nbr_off);
    if (c->nbr) cudaFree(c->nbr);
    c->nbr_off = c->nbr = nullptr;
    TRY(dalloc(&c->nbr_off, dirs + 1));
    TRY(dalloc(&c->nbr, std::max<uint32_t>(nnz, 1)));
    c->nnz = nnz;
    CU(cudaMemcpyAsync(c->nbr_off, nbr_off, (dirs + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    if (nnz) CU(cudaMemcpyAsync(c->nbr, nbr, nnz * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->h_raw, h, hn * sizeof(float2), cudaMemcpyHostToDevice, c->stream));
    if (c->tc_slabs) {  // rebuilt from the new field on the next tcgen05 launch
        CU(cudaStreamSynchronize(c->stream));
        cudaFree(c->tc_slabs);
        c->tc_slabs = nullptr;
    }
    launch_steering_prep(c->h_raw, c->h_t, c->num, (int)g.m, (int)g.bins, (int)dirs, c->stream);
    TRY(check_last_launch("steering_prep_kernel"));
    CU(cudaStreamSynchronize(c->stream));
    c->have_steering = true;
    return SSLG_OK;
}

int sslg_reset_window(sslg_ctx* c) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    CU(cudaSetDevice(c->cfg.device));
    CU(cudaMemsetAsync(c->state, 0, (size_t)c->cfg.bins * c->cfg.m * c->cfg.m * sizeof(double2), c->stream));
    c->pushed = 0;
    c->since = 0;
    c->last_emitted = 0;
    c->last_corr = -1;
    c->samp_fill = 0;
    // asynchronous pushes in flight are discarded
    CU(cudaMemsetAsync(c->abort, 0, sizeof(unsigned int), c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (auto& sl : c->slots) sl.pending = false;
    c->collected = c->next_id;
    c->poisoned = false;
    c->dev_unverified.clear();
    return SSLG_OK;
}

int sslg_synchronize(sslg_ctx* c) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    CU(cudaSetDevice(c->cfg.device));
    CU(cudaStreamSynchronize(c->stream));
    TRY(check_device_gate(c));
    return SSLG_OK;
}

int sslg_push_frames_device(sslg_ctx* c, const void* x_dev, uint32_t nframes, uint32_t* emitted) {
    if (emitted) *emitted = 0;
    TRY(require_ready(c, false));
    c->launches = 0;
    uint32_t total = 0;
    if (nframes > c->cfg.max_batch)
        return set_err(SSLG_VALIDATION, "push larger than max_batch; split it or raise max_batch");
    const sslg_config& g = c->cfg;
    const size_t fsz = (size_t)g.m * g.bins;
    const float* src = static_cast<const float*>(x_dev);
    // stream-ordered: frames into the ring, the device-side non-finite gate
    // (a failure makes every later kernel on the stream return early), the
    // hot path -- no host synchronization; check_device_gate reports a failure
    // at the next synchronizing call and rewinds the window to this push
    const uint32_t seq = c->dev_seq++ & 0x7fffffffu;
    c->dev_unverified.push_back({seq, c->pushed, c->since});
    for (uint32_t done = 0; done < nframes;) {
        const int slot = (int)((c->pushed + done) % c->cap);
        const uint32_t run = std::min<uint32_t>(nframes - done, (uint32_t)(c->cap - slot));
        CU(cudaMemcpyAsync(c->ring + (size_t)slot * fsz, src + (size_t)done * fsz * 2, run * fsz * sizeof(float2),
                           cudaMemcpyDeviceToDevice, c->stream));
        launch_gate_abort(reinterpret_cast<const float*>(c->ring + (size_t)slot * fsz), run * fsz * 2, c->abort, seq,
                          c->stream);
        ++c->launches;
        done += run;
    }
    TRY(process_chunk(c, nframes, &total));
    if (emitted) *emitted = total;
    return SSLG_OK;
}

int sslg_read_results(sslg_ctx* c, uint32_t n, sslg_block_out* blocks, uint32_t* est_idx, double* est_power,
                      uint8_t* est_low, double* power, double* bin_power, double* sigma, uint32_t* sweeps,
                      uint8_t* conv) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    if (n > c->last_emitted) return set_err(SSLG_VALIDATION, "fewer blocks available than requested");
    const sslg_config& g = c->cfg;
    const size_t ns = g.num_sources, D = c->dirs, B = g.bins;
    std::vector<uint32_t> cnt(n);
    if (n) CU(cudaMemcpyAsync(cnt.data(), c->est_count, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    if (est_idx && n) CU(cudaMemcpyAsync(est_idx, c->est_idx, n * ns * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    if (est_power && n) CU(cudaMemcpyAsync(est_power, c->est_pw, n * ns * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (est_low && n) CU(cudaMemcpyAsync(est_low, c->est_low, n * ns, cudaMemcpyDeviceToHost, c->stream));
    if (power && n) CU(cudaMemcpyAsync(power, c->power, n * D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (bin_power && n) CU(cudaMemcpyAsync(bin_power, c->p, n * B * D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (sigma && n) CU(cudaMemcpyAsync(sigma, c->sigma, n * B * g.m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (sweeps && n) CU(cudaMemcpyAsync(sweeps, c->sweeps, n * B * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    if (conv && n) CU(cudaMemcpyAsync(conv, c->conv, n * B, cudaMemcpyDeviceToHost, c->stream));
    std::vector<uint32_t> sw_tmp;
    if (conv && !sweeps && g.max_qr_sweeps && n) {
        sw_tmp.resize(n * B);
        CU(cudaMemcpyAsync(sw_tmp.data(), c->sweeps, n * B * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    CU(cudaStreamSynchronize(c->stream));
    apply_sweep_budget(g.max_qr_sweeps, sweeps ? sweeps : sw_tmp.data(), conv, sweeps || conv ? n * B : 0);
    if (blocks)
        for (uint32_t i = 0; i < n; ++i) {
            blocks[i].frame_index = (uint32_t)(c->last_first_frame + i);
            blocks[i].count = cnt[i];
        }
    return SSLG_OK;
}

int sslg_push_frames(sslg_ctx* c, const float* x, uint32_t nframes, sslg_block_out* blocks, uint32_t* est_idx,
                     double* est_power, uint8_t* est_low, double* power, uint32_t* emitted) {
    if (emitted) *emitted = 0;
    TRY(require_ready(c));
    const sslg_config& g = c->cfg;
    const size_t fsz = (size_t)g.m * g.bins * 2;
    const size_t ns = g.num_sources;
    uint32_t out = 0, done = 0, launches = 0;
    while (done < nframes) {
        const uint32_t chunk = std::min<uint32_t>(nframes - done, g.max_batch);
        c->launches = 0;
        uint32_t good = 0;
        TRY(stage_frames(c, x + done * fsz, chunk, cudaMemcpyHostToDevice, &good));
        // frames before the first non-finite one go through, as the
        // reference's per-frame loop has pushed and sunk them before it throws
        uint32_t e = 0;
        TRY(process_chunk(c, good, &e));
        launches += c->launches;
        TRY(sslg_read_results(c, e, blocks ? blocks + out : nullptr, est_idx ? est_idx + out * ns : nullptr,
                              est_power ? est_power + out * ns : nullptr, est_low ? est_low + out * ns : nullptr,
                              power ? power + (size_t)out * c->dirs : nullptr, nullptr, nullptr, nullptr, nullptr));
        out += e;
        if (emitted) *emitted = out;
        if (good < chunk) {
            c->launches = launches;
            return set_err(SSLG_VALIDATION, "non-finite spectrum value (frame " + std::to_string(done + good) + ")");
        }
        done += chunk;
    }
    c->launches = launches;
    return SSLG_OK;
}

int sslg_correlation(sslg_ctx* c, const float* x, uint32_t nframes, float* r_out, uint32_t* emitted) {
    if (emitted) *emitted = 0;
    if (!c || !x) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    const sslg_config& g = c->cfg;
    const size_t fsz = (size_t)g.m * g.bins * 2;
    const size_t rsz = (size_t)g.bins * g.m * g.m;
    uint32_t out = 0, done = 0;
    c->launches = 0;
    while (done < nframes) {
        uint32_t chunk = std::min<uint32_t>(nframes - done, g.max_batch);
        uint32_t good = 0;
        TRY(stage_frames(c, x + done * fsz, chunk, cudaMemcpyHostToDevice, &good));
        const bool bad = good < chunk;
        chunk = good;
        if (chunk == 0) {
            if (emitted) *emitted = out;
            return set_err(SSLG_VALIDATION, "non-finite spectrum value (frame " + std::to_string(done) + ")");
        }
        const long long first_emit = std::max<long long>(0, (long long)g.window_frames - 1 - c->pushed);
        const int n = (int)std::max<long long>(0, (long long)chunk - first_emit);
        CorrArgs ca{c->ring, c->state, c->r, (int)g.m, (int)g.bins, (int)g.window_frames, c->cap, (int)chunk,
                    c->pushed, c->since, (int)g.rebuild_interval};
        launch_correlation(ca, c->stream);
        ++c->launches;
        TRY(check_last_launch("correlation_kernel"));
        for (uint32_t f = 0; f < chunk; ++f) {
            ++c->pushed;
            if (++c->since >= (long long)g.rebuild_interval) c->since = 0;
        }
        if (n > 0) c->last_corr = n - 1;
        if (n > 0 && r_out)
            CU(cudaMemcpyAsync(r_out + out * rsz * 2, c->r, n * rsz * sizeof(float2), cudaMemcpyDeviceToHost,
                               c->stream));
        CU(cudaStreamSynchronize(c->stream));
        out += (uint32_t)n;
        done += chunk;
        if (emitted) *emitted = out;
        if (bad) return set_err(SSLG_VALIDATION, "non-finite spectrum value (frame " + std::to_string(done) + ")");
    }
    return SSLG_OK;
}

int sslg_last_correlation(sslg_ctx* c, float* r_out) {
    if (!c || !r_out) return set_err(SSLG_VALIDATION, "null argument");
    if (c->last_corr < 0) return set_err(SSLG_VALIDATION, "correlation window underfilled");
    CU(cudaSetDevice(c->cfg.device));
    const size_t rsz = (size_t)c->cfg.bins * c->cfg.m * c->cfg.m;
    CU(cudaMemcpyAsync(r_out, c->r + (size_t)c->last_corr * rsz, rsz * sizeof(float2), cudaMemcpyDeviceToHost,
                       c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return SSLG_OK;
}

int sslg_gsvd(sslg_ctx* c, const float* r, uint32_t nsets, double* sigma, double* e, uint32_t* sweeps,
              uint8_t* conv) {
    return sslg_gsvd_ex(c, r, nsets, sigma, e, nullptr, sweeps, conv, nullptr);
}

int sslg_gsvd_ex(sslg_ctx* c, const float* r, uint32_t nsets, double* sigma, double* e, double* er,
                 uint32_t* sweeps, uint8_t* conv, double* resid) {
    if (!c || !r) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    if (!c->have_noise) return set_err(SSLG_VALIDATION, "noise model not set");
    const sslg_config& g = c->cfg;
    const size_t mm = (size_t)g.m * g.m, B = g.bins;
    for (size_t i = 0; i < (size_t)nsets * B * mm * 2; ++i)
        if (!std::isfinite(r[i])) return set_err(SSLG_VALIDATION, "non-finite correlation entry");
    c->launches = 0;
    c->last_corr = -1;  // c->r now holds the caller's sets
    const bool want_resid = resid && g.compute_residual;
    std::vector<uint32_t> sw_tmp;
    for (uint32_t done = 0; done < nsets;) {
        const uint32_t n = std::min<uint32_t>(nsets - done, g.max_batch);
        CU(cudaMemcpyAsync(c->r, r + (size_t)done * B * mm * 2, n * B * mm * sizeof(float2), cudaMemcpyHostToDevice,
                           c->stream));
        CU(cudaEventRecord(c->ev[1], c->stream));
        TRY(run_gsvd(c, (int)n));
        double* resid_dev = nullptr;
        if (er || want_resid) {
            // E_r (into e_tmp) and the residual, from the final E
            if (want_resid) TRY(dalloc(&resid_dev, n * B));
            ErArgs ea{c->r, c->kinv, c->sigma, c->e, er ? c->e_tmp : nullptr, resid_dev, (int)g.m, (int)g.bins};
            launch_er(ea, (int)n, c->stream);
            ++c->launches;
            int rc = check_last_launch("er_kernel");
            if (!rc && er &&
                cudaMemcpyAsync(er + (size_t)done * B * mm * 2, c->e_tmp, n * B * mm * sizeof(double2),
                                cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
                rc = set_err(SSLG_DEVICE, "cudaMemcpy failed");
            if (!rc && want_resid &&
                cudaMemcpyAsync(resid + (size_t)done * B, resid_dev, n * B * sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream) != cudaSuccess)
                rc = set_err(SSLG_DEVICE, "cudaMemcpy failed");
            if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = set_err(SSLG_DEVICE, "sync failed");
            if (resid_dev) cudaFree(resid_dev);
            TRY(rc);
        }
        if (resid && !want_resid)
            for (size_t i = 0; i < n * B; ++i) resid[done * B + i] = -1.0;  // recon_residual < 0: not computed
        if (e) {
            const size_t tot = n * B * mm;
            transpose_sq_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(c->e, c->e_tmp, (int)g.m, n * B);
            ++c->launches;
            TRY(check_last_launch("transpose_sq_kernel"));
            CU(cudaMemcpyAsync(e + (size_t)done * B * mm * 2, c->e_tmp, tot * sizeof(double2), cudaMemcpyDeviceToHost,
                               c->stream));
        }
        if (sigma)
            CU(cudaMemcpyAsync(sigma + (size_t)done * B * g.m, c->sigma, n * B * g.m * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
        uint32_t* swp = sweeps ? sweeps + (size_t)done * B : nullptr;
        if (!swp && conv && g.max_qr_sweeps) {
            sw_tmp.resize(n * B);
            swp = sw_tmp.data();
        }
        if (swp) CU(cudaMemcpyAsync(swp, c->sweeps, n * B * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        if (conv) CU(cudaMemcpyAsync(conv + (size_t)done * B, c->conv, n * B, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        apply_sweep_budget(g.max_qr_sweeps, swp, conv ? conv + (size_t)done * B : nullptr, n * B);
        done += n;
    }
    return SSLG_OK;
}

int sslg_spectrum(sslg_ctx* c, const double* e, uint32_t nsets, double* power, double* bin_power) {
    if (!c || !e) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    TRY(check_device_gate(c));
    if (!c->have_steering) return set_err(SSLG_VALIDATION, "steering field not set");
    if (c->cfg.num_sources >= c->cfg.m)
        return set_err(SSLG_VALIDATION, "num_sources must be smaller than the channel count");
    CU(cudaSetDevice(c->cfg.device));
    const sslg_config& g = c->cfg;
    const size_t mm = (size_t)g.m * g.m, B = g.bins, D = c->dirs;
    c->launches = 0;
    for (uint32_t done = 0; done < nsets;) {
        const uint32_t n = std::min<uint32_t>(nsets - done, g.max_batch);
        const size_t tot = n * B * mm;
        CU(cudaMemcpyAsync(c->e_tmp, e + (size_t)done * B * mm * 2, tot * sizeof(double2), cudaMemcpyHostToDevice,
                           c->stream));
        transpose_sq_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(c->e_tmp, c->e, (int)g.m, n * B);
        ++c->launches;
        TRY(check_last_launch("transpose_sq_kernel"));
        TRY(run_music(c, (int)n));
        if (power)
            CU(cudaMemcpyAsync(power + (size_t)done * D, c->power, n * D * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
        if (bin_power)
            CU(cudaMemcpyAsync(bin_power + (size_t)done * B * D, c->p, n * B * D * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        done += n;
    }
    return SSLG_OK;
}

int sslg_peaks(sslg_ctx* c, const double* power, uint32_t nsets, uint32_t* est_idx, double* est_power,
               uint8_t* est_low, uint32_t* count) {
    if (!c || !power) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    TRY(check_device_gate(c));
    if (!c->have_steering) return set_err(SSLG_VALIDATION, "steering field not set");
    CU(cudaSetDevice(c->cfg.device));
    const sslg_config& g = c->cfg;
    const size_t D = c->dirs, ns = g.num_sources;
    c->launches = 0;
    for (uint32_t done = 0; done < nsets;) {
        const uint32_t n = std::min<uint32_t>(nsets - done, g.max_batch);
        // integrate over a single "bin" holding the given broadband power
        CU(cudaMemcpyAsync(c->p, power + (size_t)done * D, n * D * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        PeakArgs pa{c->p, c->power, c->nbr_off, c->nbr, c->est_idx, c->est_pw, c->est_low, c->est_count,
                    1, (int)D, (int)ns, (double)g.low_power_ratio};
        launch_peaks(pa, (int)n, c->stream);
        ++c->launches;
        TRY(check_last_launch("integrate_peaks_kernel"));
        if (est_idx) CU(cudaMemcpyAsync(est_idx + done * ns, c->est_idx, n * ns * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        if (est_power) CU(cudaMemcpyAsync(est_power + done * ns, c->est_pw, n * ns * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (est_low) CU(cudaMemcpyAsync(est_low + done * ns, c->est_low, n * ns, cudaMemcpyDeviceToHost, c->stream));
        if (count) CU(cudaMemcpyAsync(count + done, c->est_count, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        done += n;
    }
    return SSLG_OK;
}

int sslg_last_stage_ms(const sslg_ctx* c, float* ms5) {
    if (!c || !ms5) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->timed) return set_err(SSLG_VALIDATION, "nothing timed yet");
    for (int i = 0; i < 5; ++i) {
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
        ms5[i] = ms;
    }
    return SSLG_OK;
}

uint32_t sslg_last_launch_count(const sslg_ctx* c) { return c ? c->launches : 0; }

int sslg_copy_bin_power_device(sslg_ctx* c, void* dst, uint32_t n) {
    if (!c || !dst) return set_err(SSLG_VALIDATION, "null argument");
    if (n > c->last_emitted) return set_err(SSLG_VALIDATION, "fewer blocks available than requested");
    CU(cudaSetDevice(c->cfg.device));
    const size_t bytes = (size_t)n * c->cfg.bins * c->dirs * sizeof(double);
    if (bytes) CU(cudaMemcpyAsync(dst, c->p, bytes, cudaMemcpyDeviceToDevice, c->stream));
    return SSLG_OK;
}

int sslg_integrate_peaks_device(sslg_ctx* c, const void* p_dev, uint32_t n, uint32_t bins_total) {
    if (!c || !p_dev) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->have_steering) return set_err(SSLG_VALIDATION, "steering field not set");
    if (n > c->cfg.max_batch) return set_err(SSLG_VALIDATION, "more blocks than max_batch");
    CU(cudaSetDevice(c->cfg.device));
    const sslg_config& g = c->cfg;
    c->launches = 0;
    CU(cudaEventRecord(c->ev[4], c->stream));
    PeakArgs pa{static_cast<const double*>(p_dev), c->power, c->nbr_off, c->nbr, c->est_idx, c->est_pw, c->est_low,
                c->est_count, (int)bins_total, (int)c->dirs, (int)g.num_sources, (double)g.low_power_ratio};
    launch_peaks(pa, (int)n, c->stream);
    ++c->launches;
    TRY(check_last_launch("integrate_peaks_kernel"));
    CU(cudaEventRecord(c->ev[5], c->stream));
    c->last_emitted = n;
    return SSLG_OK;
}

int sslg_debug_phase_clocks(sslg_ctx* c, double* out8, int reset) {
    if (!c || !out8) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->phase_clk) return set_err(SSLG_VALIDATION, "phase clocks disabled (set SSLG_PHASE_CLOCKS=1)");
    long long h[8];
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpy(h, c->phase_clk, sizeof h, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 8; ++i) out8[i] = (double)h[i];
    if (reset) CU(cudaMemset(c->phase_clk, 0, sizeof h));
    return SSLG_OK;
}

// ---- STFT front end ----------------------------------------------------------

void sslg_stft_config_default(sslg_stft_config* s) {
    s->frame_length = 512;  // StftConfig defaults (types.hpp:43-52)
    s->shift = 160;
    s->window = 0;
    s->bin_min = 16;
    s->bin_max = 88;
}

int sslg_set_stft(sslg_ctx* c, const sslg_stft_config* s) {
    if (!c || !s) return set_err(SSLG_VALIDATION, "null argument");
    // StftConfig::validate (stft.cpp:9-16)
    if (s->frame_length == 0) return set_err(SSLG_VALIDATION, "frame_length must be positive");
    if (s->shift == 0) return set_err(SSLG_VALIDATION, "shift must be positive");
    if (s->shift > s->frame_length) return set_err(SSLG_VALIDATION, "shift must not exceed frame_length");
    if (s->bin_min > s->bin_max) return set_err(SSLG_VALIDATION, "bin_min must not exceed bin_max");
    if (s->bin_max > s->frame_length / 2)
        return set_err(SSLG_VALIDATION, "bin_max exceeds the half spectrum of frame_length");
    if (s->window != 0 && s->window != 1) return set_err(SSLG_VALIDATION, "unknown window");
    const bool pow2 = (s->frame_length & (s->frame_length - 1)) == 0;
    if (pow2 ? s->frame_length > 8192 : s->frame_length > 4096)
        return set_err(SSLG_VALIDATION,
                       "the device STFT takes frame lengths up to 8192 (power of two) or 4096 (direct sum)");
    if (s->bin_max - s->bin_min + 1 != c->cfg.bins)
        return set_err(SSLG_VALIDATION, "STFT band does not match the engine's bin count");
    CU(cudaSetDevice(c->cfg.device));
    const uint32_t n = s->frame_length;
    // make_window (stft.cpp:28-36) and the per-stage twiddle recurrence of
    // fft_pow2 (fft.hpp:29-38), both on the host exactly as the reference
    // evaluates them (libm cos/sin, textbook complex product, no contraction)
    std::vector<float> w(n, 1.0f);
    if (s->window == 0)
        for (uint32_t i = 0; i < n; ++i) w[i] = float(0.5 - 0.5 * std::cos(2.0 * M_PI * double(i) / double(n)));
    std::vector<double2> tw(n > 1 ? n - 1 : 1);
    for (uint32_t len = 2; len <= n; len <<= 1) {
        const double ang = -2.0 * M_PI / double(len);
        const double wlr = std::cos(ang), wli = std::sin(ang);
        double wr = 1.0, wi = 0.0;
        for (uint32_t k = 0; k < len / 2; ++k) {
            tw[len / 2 - 1 + k] = make_double2(wr, wi);
            const volatile double a = wr * wlr, b = wi * wli, e = wr * wli, f = wi * wlr;
            wr = a - b;
            wi = e + f;
        }
    }
    for (void* p : {(void*)c->win, (void*)c->twiddle, (void*)c->samp[0], (void*)c->samp[1], (void*)c->frame_scratch,
                    (void*)c->dft})
        if (p) cudaFree(p);
    c->win = nullptr;
    c->twiddle = nullptr;
    c->dft = nullptr;
    c->samp[0] = c->samp[1] = nullptr;
    c->frame_scratch = nullptr;
    c->have_stft = false;
    c->samp_cap = (size_t)n + (size_t)c->cfg.max_batch * s->shift;
    TRY(dalloc(&c->win, n));
    TRY(dalloc(&c->twiddle, tw.size()));
    TRY(dalloc(&c->samp[0], c->samp_cap * c->cfg.m));
    TRY(dalloc(&c->samp[1], c->samp_cap * c->cfg.m));
    TRY(dalloc(&c->frame_scratch, (size_t)c->cfg.max_batch * c->cfg.m * c->cfg.bins));
    CU(cudaMemcpy(c->win, w.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->twiddle, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    if (!pow2) {
        // real_dft_half's direct sum (fft.hpp:55-65): the angle evaluated as
        // the reference writes it, -2.0 * M_PI * double(k) * double(i) / double(n)
        std::vector<double2> cs((size_t)c->cfg.bins * n);
        for (uint32_t b = 0; b < c->cfg.bins; ++b)
            for (uint32_t i = 0; i < n; ++i) {
                const volatile double ang = -2.0 * M_PI * double(s->bin_min + b) * double(i) / double(n);
                cs[(size_t)b * n + i] = make_double2(std::cos(ang), std::sin(ang));
            }
        TRY(dalloc(&c->dft, cs.size()));
        CU(cudaMemcpy(c->dft, cs.data(), cs.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    c->stft = *s;
    c->samp_fill = 0;
    c->samp_cur = 0;
    c->have_stft = true;
    return SSLG_OK;
}

namespace {

int launch_stft_frames(sslg_ctx* c, const float* pcm_dev, size_t pitch, int nframes, float2* out, int cap,
                       long long slot0) {
    Nvtx range("sslg:stft");
    StftArgs sa{pcm_dev, c->win, c->twiddle, out, pitch, (int)c->cfg.m, (int)c->stft.frame_length,
                (int)c->stft.shift, (int)c->stft.bin_min, (int)c->cfg.bins, cap, slot0};
    sa.dft = c->dft;
    launch_stft(sa, nframes, c->stream);
    ++c->launches;
    return check_last_launch("stft_kernel");
}

// appends up to `n` samples per channel (host, row pitch `ld`) to the
// sample history; returns the count taken
int append_samples(sslg_ctx* c, const float* pcm, size_t ld, size_t n, size_t* took) {
    const size_t take = std::min(n, c->samp_cap - c->samp_fill);
    if (take)
        CU(cudaMemcpy2DAsync(c->samp[c->samp_cur] + c->samp_fill, c->samp_cap * sizeof(float), pcm, ld * sizeof(float),
                             take * sizeof(float), c->cfg.m, cudaMemcpyHostToDevice, c->stream));
    c->samp_fill += take;
    *took = take;
    return 0;
}

// drops the first `consumed` samples of the history (ping-pong copy of the tail)
int consume_samples(sslg_ctx* c, size_t consumed) {
    const size_t tail = c->samp_fill - consumed;
    if (tail)
        CU(cudaMemcpy2DAsync(c->samp[c->samp_cur ^ 1], c->samp_cap * sizeof(float), c->samp[c->samp_cur] + consumed,
                             c->samp_cap * sizeof(float), tail * sizeof(float), c->cfg.m, cudaMemcpyDeviceToDevice,
                             c->stream));
    c->samp_cur ^= 1;
    c->samp_fill = tail;
    return 0;
}

uint32_t frames_ready(const sslg_ctx* c) {
    const size_t L = c->stft.frame_length;
    if (c->samp_fill < L) return 0;
    return (uint32_t)std::min<size_t>((c->samp_fill - L) / c->stft.shift + 1, c->cfg.max_batch);
}

}  // namespace

int sslg_stft(sslg_ctx* c, const float* pcm, uint64_t nsamples, float* frames, uint32_t cap_frames, uint32_t* nframes) {
    if (!c || !pcm) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->have_stft) return set_err(SSLG_VALIDATION, "STFT not configured (sslg_set_stft)");
    CU(cudaSetDevice(c->cfg.device));
    const size_t L = c->stft.frame_length, S = c->stft.shift;
    const uint64_t total = nsamples < L ? 0 : (nsamples - L) / S + 1;  // stft_frame_count (stft.cpp:38-42)
    if (nframes) *nframes = (uint32_t)total;
    if (!frames) return SSLG_OK;
    if (total > cap_frames) return set_err(SSLG_VALIDATION, "frame buffer too small for this block");
    const size_t fsz = (size_t)c->cfg.m * c->cfg.bins;
    c->launches = 0;
    // stage the block through the second history buffer, one max_batch chunk at a time
    float* stage = c->samp[c->samp_cur ^ 1];
    for (uint64_t f0 = 0; f0 < total; f0 += c->cfg.max_batch) {
        const int nf = (int)std::min<uint64_t>(total - f0, c->cfg.max_batch);
        const size_t span = (size_t)(nf - 1) * S + L;
        CU(cudaMemcpy2DAsync(stage, c->samp_cap * sizeof(float), pcm + f0 * S, nsamples * sizeof(float),
                             span * sizeof(float), c->cfg.m, cudaMemcpyHostToDevice, c->stream));
        TRY(launch_stft_frames(c, stage, c->samp_cap, nf, c->frame_scratch, nf, 0));
        CU(cudaMemcpyAsync(frames + f0 * fsz * 2, c->frame_scratch, nf * fsz * sizeof(float2), cudaMemcpyDeviceToHost,
                           c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    return SSLG_OK;
}

int sslg_capture_noise_model(sslg_ctx* c, const float* pcm, uint64_t nsamples, int install, float* k_out,
                             uint32_t* nframes, uint32_t* bad_bin) {
    if (!c || (!pcm && nsamples)) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->have_stft) return set_err(SSLG_VALIDATION, "STFT not configured (sslg_set_stft)");
    TRY(require_no_async(c));
    CU(cudaSetDevice(c->cfg.device));
    TRY(check_device_gate(c));
    const sslg_config& g = c->cfg;
    const size_t L = c->stft.frame_length, S = c->stft.shift;
    const uint64_t total = nsamples < L ? 0 : (nsamples - L) / S + 1;  // stft_frame_count (stft.cpp:38-42)
    if (nframes) *nframes = (uint32_t)total;
    if (total == 0) return set_err(SSLG_VALIDATION, "noise capture scene is shorter than one frame");
    const size_t mm = (size_t)g.m * g.m, n = g.bins * mm;
    // acc: FP64 sums [bins][m][m] (e_tmp); K: cf32 (the first set of R)
    double2* acc = c->e_tmp;
    float2* kdev = c->r;
    c->last_corr = -1;
    c->launches = 0;
    CU(cudaMemsetAsync(acc, 0, n * sizeof(double2), c->stream));
    float* stage = c->samp[c->samp_cur ^ 1];
    for (uint64_t f0 = 0; f0 < total; f0 += g.max_batch) {
        const int nf = (int)std::min<uint64_t>(total - f0, g.max_batch);
        const size_t span = (size_t)(nf - 1) * S + L;
        CU(cudaMemcpy2DAsync(stage, c->samp_cap * sizeof(float), pcm + f0 * S, nsamples * sizeof(float),
                             span * sizeof(float), g.m, cudaMemcpyHostToDevice, c->stream));
        TRY(launch_stft_frames(c, stage, c->samp_cap, nf, c->frame_scratch, nf, 0));
        launch_capture_accum(c->frame_scratch, nf, (int)g.m, (int)g.bins, acc, c->stream);
        ++c->launches;
        TRY(check_last_launch("capture_accum_kernel"));
    }
    launch_capture_narrow(acc, n, 1.0 / double(total), kdev, c->stream);
    ++c->launches;
    TRY(check_last_launch("capture_narrow_kernel"));
    if (k_out) CU(cudaMemcpyAsync(k_out, kdev, n * sizeof(float2), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    // capture_noise_model ends with check_positive_definite (synth.cpp:370)
    TRY(pd_gate(c, kdev, bad_bin));
    if (!install) return SSLG_OK;
    c->have_noise = false;
    CU(cudaMemcpyAsync(c->k, kdev, n * sizeof(float2), cudaMemcpyDeviceToDevice, c->stream));
    return install_noise(c, bad_bin);
}

int sslg_samples_pending(const sslg_ctx* c, uint64_t nsamples, uint32_t* frames, uint32_t* blocks) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    if (!c->have_stft) return set_err(SSLG_VALIDATION, "STFT not configured (sslg_set_stft)");
    const uint64_t have = c->samp_fill + nsamples, L = c->stft.frame_length;
    const uint64_t f = have < L ? 0 : (have - L) / c->stft.shift + 1;
    const long long need = (long long)c->cfg.window_frames - 1 - c->pushed;  // frames still filling the window
    const long long b = (long long)f - std::max<long long>(0, need);
    if (frames) *frames = (uint32_t)f;
    if (blocks) *blocks = (uint32_t)std::max<long long>(0, b);
    return SSLG_OK;
}

int sslg_push_samples(sslg_ctx* c, const float* pcm, uint64_t nsamples, uint32_t cap_blocks, sslg_block_out* blocks,
                      uint32_t* est_idx, double* est_power, uint8_t* est_low, double* power, uint32_t* emitted) {
    if (emitted) *emitted = 0;
    TRY(require_ready(c));
    if (!c->have_stft) return set_err(SSLG_VALIDATION, "STFT not configured (sslg_set_stft)");
    if (!pcm && nsamples) return set_err(SSLG_VALIDATION, "null argument");
    uint32_t need = 0;
    TRY(sslg_samples_pending(c, nsamples, nullptr, &need));
    if (need > cap_blocks) return set_err(SSLG_VALIDATION, "result arrays too small for the emitted blocks");
    const size_t ns = c->cfg.num_sources;
    uint32_t out = 0, launches = 0;
    uint64_t off = 0;
    for (;;) {
        size_t took = 0;
        c->launches = 0;
        TRY(append_samples(c, pcm + off, nsamples, nsamples - off, &took));
        off += took;
        const uint32_t nf = frames_ready(c);
        if (nf == 0) {
            if (off >= nsamples) break;
            continue;
        }
        TRY(launch_stft_frames(c, c->samp[c->samp_cur], c->samp_cap, (int)nf, c->ring, c->cap, c->pushed));
        uint32_t good = 0;
        TRY(gate_frames(c, nf, &good));
        // frames before the first non-finite one go through (run_locate has
        // pushed and sunk them when the bad frame throws, pipeline.cpp:227-245)
        uint32_t e = 0;
        TRY(process_chunk(c, good, &e));
        TRY(consume_samples(c, (size_t)good * c->stft.shift));
        launches += c->launches;
        TRY(sslg_read_results(c, e, blocks ? blocks + out : nullptr, est_idx ? est_idx + out * ns : nullptr,
                              est_power ? est_power + out * ns : nullptr, est_low ? est_low + out * ns : nullptr,
                              power ? power + (size_t)out * c->dirs : nullptr, nullptr, nullptr, nullptr, nullptr));
        out += e;
        if (emitted) *emitted = out;
        if (good < nf) {
            c->launches = launches;
            return set_err(SSLG_VALIDATION, "non-finite spectrum value (frame " + std::to_string(c->pushed) + ")");
        }
    }
    c->launches = launches;
    return SSLG_OK;
}

int sslg_locate_samples(sslg_ctx* c, const float* pcm, uint64_t nsamples, uint32_t cap_blocks, sslg_block_out* blocks,
                        uint32_t* est_idx, double* est_power, uint8_t* est_low, double* power, uint32_t* emitted) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    TRY(sslg_reset_window(c));
    c->samp_fill = 0;
    return sslg_push_samples(c, pcm, nsamples, cap_blocks, blocks, est_idx, est_power, est_low, power, emitted);
}

// ---- asynchronous streaming --------------------------------

int sslg_set_spectrum_path(sslg_ctx* c, int mode) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    if (mode < -1 || mode > 1) return set_err(SSLG_VALIDATION, "spectrum path must be -1 (auto), 0 or 1");
    c->spectrum_tc = mode;
    return SSLG_OK;
}

int sslg_set_async_power(sslg_ctx* c, int on) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    TRY(require_no_async(c));
    c->async_power = on != 0;
    return SSLG_OK;
}

int sslg_push_samples_async(sslg_ctx* c, const float* pcm, uint64_t nsamples, uint64_t* ticket) {
    if (!c) return set_err(SSLG_VALIDATION, "null context");
    {
        // asynchronous pushes may queue behind each other: only the
        // collected-vs-enqueued check of require_ready is skipped here
        const uint64_t nid = c->next_id, col = c->collected;
        c->collected = nid;
        const int rc = require_ready(c);
        c->collected = col;
        TRY(rc);
    }
    if (!c->have_stft) return set_err(SSLG_VALIDATION, "STFT not configured (sslg_set_stft)");
    if (!pcm && nsamples) return set_err(SSLG_VALIDATION, "null argument");
    if (c->poisoned) return set_err(SSLG_VALIDATION, "stream stopped by a non-finite spectrum value; reset the window");
    TRY(check_device_gate(c));
    TRY(ensure_slots(c));
    uint32_t frames = 0;
    TRY(sslg_samples_pending(c, nsamples, &frames, nullptr));
    const uint32_t subs = (frames + c->cfg.max_batch - 1) / c->cfg.max_batch;
    if (c->next_id - c->collected + subs > (uint64_t)sslg_ctx::kSlots)
        return set_err(SSLG_VALIDATION, "asynchronous result ring full; collect results with sslg_wait_results");
    const sslg_config& g = c->cfg;
    const size_t ns = g.num_sources;
    uint64_t off = 0;
    for (;;) {
        size_t took = 0;
        TRY(append_samples(c, pcm + off, nsamples, nsamples - off, &took));
        off += took;
        const uint32_t nf = frames_ready(c);
        if (nf == 0) {
            if (off >= nsamples) break;
            continue;
        }
        auto& sl = c->slots[c->next_id % sslg_ctx::kSlots];
        sl.id = c->next_id;
        sl.pushed0 = c->pushed;
        sl.since0 = c->since;
        c->launches = 0;
        TRY(launch_stft_frames(c, c->samp[c->samp_cur], c->samp_cap, (int)nf, c->ring, c->cap, c->pushed));
        // device-side gate: the first failing sub-push stops everything after it
        const size_t fsz = (size_t)g.m * g.bins;
        for (uint32_t done = 0; done < nf;) {
            const int slot = (int)((c->pushed + done) % c->cap);
            const uint32_t run = std::min<uint32_t>(nf - done, (uint32_t)(c->cap - slot));
            launch_gate_abort(reinterpret_cast<const float*>(c->ring + (size_t)slot * fsz), run * fsz * 2, c->abort,
                              (unsigned)sl.id, c->stream);
            done += run;
        }
        uint32_t e = 0;
        TRY(process_chunk(c, nf, &e));
        TRY(consume_samples(c, (size_t)nf * c->stft.shift));
        sl.n = e;
        sl.first_frame = c->last_first_frame;
        if (e) {
            CU(cudaMemcpyAsync(sl.idx, c->est_idx, e * ns * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(sl.pw, c->est_pw, e * ns * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(sl.low, c->est_low, e * ns, cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(sl.cnt, c->est_count, e * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
            if (c->async_power)
                CU(cudaMemcpyAsync(sl.power, c->power, (size_t)e * c->dirs * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream));
        }
        // the abort word as of this sub-push, read by sslg_wait_results from
        // pinned memory after the event (no synchronous copy on that path)
        CU(cudaMemcpyAsync(sl.cnt + c->cfg.max_batch, c->abort, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaEventRecord(sl.done, c->stream));
        sl.pending = true;
        ++c->next_id;
    }
    if (ticket) *ticket = c->next_id;  // every sub-push before this id belongs to the call
    return SSLG_OK;
}

int sslg_wait_results(sslg_ctx* c, uint64_t ticket, uint32_t cap_blocks, sslg_block_out* blocks, uint32_t* est_idx,
                      double* est_power, uint8_t* est_low, double* power, uint32_t* emitted) {
    if (!c) return set_err(SSLG_VALIDATION, "null argument");
    CU(cudaSetDevice(c->cfg.device));
    if (emitted) *emitted = 0;
    if (c->poisoned) return set_err(SSLG_VALIDATION, "non-finite spectrum value");
    if (ticket > c->next_id) return set_err(SSLG_VALIDATION, "unknown ticket");
    const size_t ns = c->cfg.num_sources, D = c->dirs;
    // wait for the last requested sub-push, then check the abort word once
    // (its copy taken on the stream right after that sub-push)
    unsigned int ab = 0;
    if (ticket > c->collected) {
        const auto& last = c->slots[(ticket - 1) % sslg_ctx::kSlots];
        CU(cudaEventSynchronize(last.done));
        ab = last.cnt[c->cfg.max_batch];
    }
    // the whole requested range must fit before any slot is consumed
    {
        uint64_t total = 0;
        for (uint64_t id = c->collected; id < ticket; ++id) {
            const auto& sl = c->slots[id % sslg_ctx::kSlots];
            if (ab && sl.id + 1 >= ab) break;
            total += sl.n;
        }
        if (total > cap_blocks) return set_err(SSLG_VALIDATION, "result arrays too small for the emitted blocks");
    }
    if (power && !c->async_power)
        return set_err(SSLG_VALIDATION, "power was not requested for asynchronous pushes (sslg_set_async_power)");
    uint32_t out = 0;
    while (c->collected < ticket) {
        auto& sl = c->slots[c->collected % sslg_ctx::kSlots];
        if (ab && sl.id + 1 >= ab) {
            // this sub-push's gate (or an earlier one of this stream) failed:
            // nothing from here on touched the window; rewind to it
            c->pushed = sl.pushed0;
            c->since = sl.since0;
            c->samp_fill = 0;
            c->poisoned = true;
            for (auto& s2 : c->slots) s2.pending = false;
            c->collected = c->next_id;
            CU(cudaMemsetAsync(c->abort, 0, sizeof(unsigned int), c->stream));
            if (emitted) *emitted = out;
            return set_err(SSLG_VALIDATION, "non-finite spectrum value");
        }
        for (uint32_t b = 0; b < sl.n; ++b) {
            if (blocks) {
                blocks[out + b].frame_index = (uint32_t)(sl.first_frame + b);
                blocks[out + b].count = sl.cnt[b];
            }
        }
        if (est_idx) std::memcpy(est_idx + out * ns, sl.idx, sl.n * ns * sizeof(uint32_t));
        if (est_power) std::memcpy(est_power + out * ns, sl.pw, sl.n * ns * sizeof(double));
        if (est_low) std::memcpy(est_low + out * ns, sl.low, sl.n * ns);
        if (power) std::memcpy(power + (size_t)out * D, sl.power, (size_t)sl.n * D * sizeof(double));
        out += sl.n;
        sl.pending = false;
        ++c->collected;
    }
    if (emitted) *emitted = out;
    return SSLG_OK;
}

}  // extern "C"
