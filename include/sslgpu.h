/*
 * sslgpu.h — C ABI of the B200-native GSVD-MUSIC sound-source-localization
 * engine (libsslgpu.so).
 *
 * This is the drop-in boundary for the reference's localization hot path.
 * The reference (sslkit, /root/reference/proj) exposes that path only as a
 * C++ API over STL value types in namespace ssl; every entry point below
 * replaces one of those calls with plain pointers, sizes and an int status,
 * so any FFI (ctypes, cgo, JNI, N-API) or the C++ shim in
 * include/sslgpu/ssl.hpp can bind it.  Reference interfaces are cited as
 * include/ssl/<file>:<line> relative to /root/reference/proj.
 *
 * Tensor layouts are the reference's own (interleaved complex, row-major):
 *   spectrum frame  X  [m][bins]        cf32  (SpectrumFrame::spectra[m][b], types.hpp:56-61)
 *   correlation     R  [bins][m][m]     cf32  (CorrelationSet::bins[b], correlation.hpp:14-21)
 *   noise model     K  [bins][m][m]     cf32  (NoiseModel::k, gsvd.hpp:31-50)
 *   steering        H  [dirs][bins][m]  cf32  (SteeringField::vectors, music.hpp:32-47)
 *   left factors    E  [bins][m][m]     cf64  row-major, column j = vector j
 *                                             (GsvdBinResult::e, gsvd.hpp:52-60)
 *   power           P  [dirs] f64, bin power [bins][dirs] f64 (MusicSpectrum, music.hpp:66-71)
 *
 * Status codes mirror the reference's error taxonomy (types.hpp:13-23) and
 * its CLI exit codes (tools/sslkit.cpp:280-291).  There is no CPU fallback:
 * every compute entry point runs on the GPU and fails with SSLG_DEVICE if no
 * device is usable.
 *
 * Contexts are not thread-safe (one per stream, like CorrelationWindow,
 * SPEC.md:124); many contexts may share one device.
 */
#ifndef SSLGPU_H
#define SSLGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSLG_OK 0
#define SSLG_VALIDATION 2 /* ssl::ValidationError */
#define SSLG_NUMERICAL 3  /* ssl::NumericalError */
#define SSLG_IO 4         /* ssl::IoError */
#define SSLG_DEVICE 5     /* CUDA failure / no device */

#define SSLG_MAX_M 64 /* channels handled by the SMEM-resident solver */

typedef struct sslg_ctx sslg_ctx;

/* Engine configuration.  Solver / music fields mirror ssl::SolverConfig
 * (gsvd.hpp:14-26) and ssl::MusicConfig (music.hpp:49-62). */
typedef struct sslg_config {
    uint32_t m;                  /* channels (<= SSLG_MAX_M) */
    uint32_t bins;               /* retained STFT bins (StftConfig::bin_count) */
    uint32_t dirs;               /* direction-grid size; 0 until set_steering */
    uint32_t window_frames;      /* T of CorrelationWindow (correlation.hpp:29-31) */
    uint32_t rebuild_interval;   /* CorrelationWindow rebuild cadence, default 1000 */
    uint32_t num_sources;        /* MusicConfig::num_sources */
    float denominator_floor;     /* MusicConfig::denominator_floor, default 1e-12 */
    int squared_denominator;     /* MusicConfig::squared_denominator */
    float low_power_ratio;       /* MusicConfig::low_power_ratio, default 1.25 */
    int pivoting;                /* SolverConfig::pivoting: 0 none (pivot-free elimination, gsvd.cpp:27-40),
                                    1 partial */
    int canonical_subspaces;     /* SolverConfig::canonical_subspaces */
    int refine_leading;          /* A A^H sharpening of the kept span (gsvd.cpp:440-466); default 0 =
                                    canonicalize in the span of the FP64 Jacobi basis (fused), 1 =
                                    the reference's full-space procedure (canonical_kernel) */
    int precondition;            /* 1 (default): Householder QR with column pivoting, Jacobi on R^H
                                    (converges in ~8 instead of ~18 sweeps); 0: Jacobi on A as
                                    jacobi_svd (gsvd.cpp:622-695) */
    uint32_t max_sweeps;         /* Jacobi sweep cap, 0 = 60 (jacobi_svd, gsvd.cpp:631) */
    uint32_t max_batch;          /* blocks (frames) processed per launch; sizes device buffers */
    int device;                  /* CUDA device ordinal */
    void* stream;                /* cudaStream_t to launch on; NULL = the context's own stream */
    uint32_t max_qr_sweeps;      /* SolverConfig::max_qr_sweeps (gsvd.hpp:15): 0 = no budget.  A bin whose
                                    solve needs more Jacobi sweeps than a nonzero budget reports
                                    converged = 0 and iterations = the budget, with the converged FP64
                                    factors -- what gsvd()'s salvage returns (gsvd.cpp:819-827) */
    float tolerance_scale;       /* SolverConfig::tolerance_scale (gsvd.hpp:16, > 0): scales the Jacobi
                                    no-rotation threshold, |a_pq| <= 1e-14 * scale * |w_p| |w_q| */
    int compute_residual;        /* SolverConfig::compute_residual: sslg_gsvd fills `resid` */
} sslg_config;

/* Fills `cfg` with the reference defaults (gsvd.hpp:14-26, music.hpp:49-62,
 * pipeline.hpp:23, correlation.hpp:31). */
void sslg_config_default(sslg_config* cfg);

int sslg_create(sslg_ctx** out, const sslg_config* cfg);
void sslg_destroy(sslg_ctx* ctx);
/* Message of the last failure on this thread (any context). */
const char* sslg_last_error(void);
/* Reads back the effective configuration. */
int sslg_get_config(const sslg_ctx* ctx, sslg_config* cfg);

/* ---- setup ------------------------------------------------------------ */

/* NoiseModel: uploads K, builds K^-1 on the device with the float and double
 * Gauss-Jordan of mat_inverse<T> (gsvd.cpp:21-62, prepare_inverses 756-768;
 * cfg.pivoting selects partial or none); with check_pd also runs
 * check_positive_definite (gsvd.cpp:736-754: Hermitian test, then the
 * smallest eigenvalue of hermitian_eigenvalues, eig.cpp:11-84).
 * Failures return SSLG_NUMERICAL and set *bad_bin (nullable) to the first
 * offending bin, like the reference's "... at bin b" messages. */
int sslg_set_noise_model(sslg_ctx* ctx, const float* k, int check_pd, uint32_t* bad_bin);
/* NoiseModel::inverse / inverse_double (gsvd.hpp:43-44) of the current noise
 * model: out [bins][m][m] cf64 row-major; precision 0 = the float inverse
 * (widened exactly), 1 = the double inverse the solver uses.  Both are
 * bit-identical to mat_inverse<T> with the context's pivoting. */
int sslg_noise_inverse(sslg_ctx* ctx, int precision, double* out);
/* NoiseModel::identity (gsvd.cpp:722-727). */
int sslg_set_noise_identity(sslg_ctx* ctx);

/* SteeringField + DirectionTopology: h [dirs][bins][m] cf32, dirs_deg
 * [dirs][2] (azimuth, elevation), and the neighbor lists of
 * DirectionTopology::build (music.cpp:176-195) as CSR (nbr_off [dirs+1],
 * nbr [nbr_off[dirs]]).  Pass nbr_off == NULL to build the topology here
 * with sslg_build_topology(radius_deg = 10, pipeline.cpp:222). */
int sslg_set_steering(sslg_ctx* ctx, uint32_t dirs, const float* h, const double* dirs_deg,
                      const uint32_t* nbr_off, const uint32_t* nbr);

/* DirectionTopology::build (music.cpp:176-195) on the host, same FP64 test
 * dot >= cos(radius): writes nbr_off [n+1] and up to `cap` neighbors.
 * Returns SSLG_VALIDATION (and the needed size in *nnz) if cap is short. */
int sslg_build_topology(const double* dirs_deg, uint32_t n, double radius_deg, uint32_t* nbr_off, uint32_t* nbr,
                        uint32_t cap, uint32_t* nnz);

/* ---- streaming hot path (run_locate's per-frame loop, pipeline.cpp:227-245) */

/* Estimates of one emitted block.  Mirrors FrameEstimates + SourceEstimate
 * (pipeline.hpp:63-66, music.hpp:88-93); arrays hold num_sources slots, the
 * first `count` valid (unused slots: index 0xffffffff, power 0, low 0). */
typedef struct sslg_block_out {
    uint32_t frame_index; /* frame that completed the block */
    uint32_t count;       /* estimates written (<= num_sources) */
} sslg_block_out;

/* Pushes `nframes` spectrum frames x [nframes][m][bins] cf32 (host memory)
 * through the correlation window; for every frame that leaves the window
 * full runs GSVD -> MUSIC -> integration -> peak search on the device and
 * writes one block of results: blocks[e], est_idx / est_power / est_low
 * [e][num_sources], and (nullable) power [e][dirs].  *emitted receives the
 * block count (nframes minus the frames still filling the window). */
int sslg_push_frames(sslg_ctx* ctx, const float* x, uint32_t nframes, sslg_block_out* blocks, uint32_t* est_idx,
                     double* est_power, uint8_t* est_low, double* power, uint32_t* emitted);

/* Same on device-resident frames (x_dev: device pointer, same layout);
 * results stay on the device until sslg_read_results.  Asynchronous on the
 * context stream, with no host synchronization: the non-finite gate runs on
 * the device (a failure makes every later kernel return early), and the
 * next synchronizing call (sslg_read_results, sslg_synchronize, any
 * push or stage call) reports SSLG_VALIDATION and rewinds the window to just
 * before the failing push.
 *
 * Every synchronous entry point returns SSLG_VALIDATION while asynchronous
 * pushes (sslg_push_samples_async) are uncollected.  The host-buffer pushes
 * gate frame by frame like CorrelationWindow::push (correlation.cpp:16-17):
 * the frames before the first non-finite one are pushed and their blocks
 * written and counted in *emitted before the error is returned. */
int sslg_push_frames_device(sslg_ctx* ctx, const void* x_dev, uint32_t nframes, uint32_t* emitted);
/* Copies the results of the last push (blocks [0, n)) to host arrays
 * (any may be NULL). */
int sslg_read_results(sslg_ctx* ctx, uint32_t n, sslg_block_out* blocks, uint32_t* est_idx, double* est_power,
                      uint8_t* est_low, double* power, double* bin_power, double* sigma, uint32_t* sweeps,
                      uint8_t* conv);
/* Bin sharding across GPUs (one array's bins split over ranks): copies the
 * per-bin powers P [n][bins][dirs] f64 of the last push's first n blocks to
 * the device buffer `dst` (stream-ordered on the context stream). */
int sslg_copy_bin_power_device(sslg_ctx* ctx, void* dst, uint32_t n);
/* Integration + peak search (music.cpp:143-160, 197-236) of externally
 * assembled per-bin powers p_dev [n][bins_total][dirs] f64 (device), summed
 * in ascending bin order; results are read with sslg_read_results. */
int sslg_integrate_peaks_device(sslg_ctx* ctx, const void* p_dev, uint32_t n, uint32_t bins_total);
/* Clears the correlation window (a fresh CorrelationWindow). */
int sslg_reset_window(sslg_ctx* ctx);
/* Blocks until the context stream is idle. */
int sslg_synchronize(sslg_ctx* ctx);

/* ---- STFT front end: SampleBlock in (run_locate, pipeline.cpp:210-247) --- */

/* StftConfig (types.hpp:41-52). window: 0 hann (periodic), 1 rectangular. */
typedef struct sslg_stft_config {
    uint32_t frame_length; /* power of two, <= 8192 on the device */
    uint32_t shift;
    int window;
    uint32_t bin_min, bin_max; /* inclusive; bin_max - bin_min + 1 == sslg_config.bins */
} sslg_stft_config;

/* StftConfig defaults: 512 / 160 / hann / 16..88 (types.hpp:43-52). */
void sslg_stft_config_default(sslg_stft_config* s);
/* Validates like StftConfig::validate (stft.cpp:9-16), builds make_window
 * (stft.cpp:28-36) and the fft_pow2 twiddles (fft.hpp:29-38) and sizes the
 * device sample history.  Frames are bit-identical to stft_frame. */
int sslg_set_stft(sslg_ctx* ctx, const sslg_stft_config* s);
/* stft_stream over one SampleBlock (stft.cpp:61-68): pcm [m][nsamples] f32
 * channel-major (SampleBlock::channels); frames [nframes][m][bins] cf32 with
 * nframes = stft_frame_count (stft.cpp:38-42), at most cap_frames (pass
 * frames == NULL to query *nframes).  Does not touch the correlation window. */
int sslg_stft(sslg_ctx* ctx, const float* pcm, uint64_t nsamples, float* frames, uint32_t cap_frames,
              uint32_t* nframes);
/* Frames and result blocks the next sslg_push_samples of nsamples samples
 * per channel will produce (sizing aid for the result arrays). */
int sslg_samples_pending(const sslg_ctx* ctx, uint64_t nsamples, uint32_t* frames, uint32_t* blocks);
/* Streaming run_locate: appends pcm [m][nsamples] to the context's sample
 * history (frames continue across calls at multiples of shift), transforms
 * every complete frame on the device straight into the correlation window
 * and runs the hot path as sslg_push_frames.  Result arrays hold cap_blocks
 * blocks; SSLG_VALIDATION if the push would emit more. */
int sslg_push_samples(sslg_ctx* ctx, const float* pcm, uint64_t nsamples, uint32_t cap_blocks,
                      sslg_block_out* blocks, uint32_t* est_idx, double* est_power, uint8_t* est_low, double* power,
                      uint32_t* emitted);
/* run_locate (pipeline.cpp:210-247): a fresh correlation window and sample
 * history, then sslg_push_samples over the whole SampleBlock; frame indices
 * count from the block's first frame. */
int sslg_locate_samples(sslg_ctx* ctx, const float* pcm, uint64_t nsamples, uint32_t cap_blocks,
                        sslg_block_out* blocks, uint32_t* est_idx, double* est_power, uint8_t* est_low,
                        double* power, uint32_t* emitted);

/* ---- asynchronous streaming -------------------------------------------------
 * sslg_push_samples_async enqueues a push (H2D of the PCM, device STFT, a
 * device-side non-finite gate, the hot path, D2H of the estimates into a
 * pinned result ring) on the context stream and returns without waiting; any
 * number of pushes may be in flight (up to 16 max_batch chunks uncollected).
 * `pcm` must stay valid until the push is collected; pinned (cudaHostAlloc)
 * memory lets the copy overlap the previous push's kernels.  *ticket marks
 * the end of this call's results.  sslg_wait_results waits for every push up
 * to `ticket` and copies their blocks out in order.  A non-finite value stops
 * the stream on the device (later pushes skip their kernels), the window is
 * rewound to just before the failing push and SSLG_VALIDATION is returned;
 * sslg_reset_window restarts the stream. */
int sslg_push_samples_async(sslg_ctx* ctx, const float* pcm, uint64_t nsamples, uint64_t* ticket);
/* Which kernel evaluates the MUSIC contraction: -1 auto (the default: the
 * tcgen05 kind::tf32 3-pass-split kernel for grids of >= 512 directions, the
 * FP64 tensor-core DMMA kernel below), 0 always FP64 (DMMA / DFMA), 1 the
 * tcgen05 kernel whenever m <= 64.  The tf32x3 path is within 5.6e-7 relative
 * per bin and 2.8e-7 on the broadband power of the FP64 one on the C4 grid
 * (tests/test_gpu_spectrum_tc.py; the reference's own float path: ~1e-4). */
int sslg_set_spectrum_path(sslg_ctx* ctx, int mode);
/* Whether asynchronous pushes also copy the broadband power [e][dirs] back
 * (needed for sslg_wait_results' `power`; off by default: FrameEstimates,
 * pipeline.hpp:63-66, carries only the estimates).  Refused while pushes are
 * pending. */
int sslg_set_async_power(sslg_ctx* ctx, int on);
int sslg_wait_results(sslg_ctx* ctx, uint64_t ticket, uint32_t cap_blocks, sslg_block_out* blocks, uint32_t* est_idx,
                      double* est_power, uint8_t* est_low, double* power, uint32_t* emitted);

/* ---- stage entry points (host buffers, one call per reference function) */

/* CorrelationWindow push + normalized (correlation.cpp:86-130) for nframes
 * frames; r_out [emitted][bins][m][m] cf32 bit-identical to the reference. */
int sslg_correlation(sslg_ctx* ctx, const float* x, uint32_t nframes, float* r_out, uint32_t* emitted);

/* The newest correlation set the window produced (by sslg_correlation or a
 * push): r_out [bins][m][m] cf32 -- CorrelationWindow::normalized
 * (correlation.cpp:112-130).  SSLG_VALIDATION while the window is underfilled. */
int sslg_last_correlation(sslg_ctx* ctx, float* r_out);

/* gsvd / gsvd_reference batch drivers (gsvd.hpp:160-163) for nsets
 * correlation sets r [nsets][bins][m][m]: sigma [nsets][bins][m] descending,
 * e [nsets][bins][m][m] (row-major, column j = vector j), sweeps / conv
 * [nsets][bins] (nullable).  FP64 one-sided Jacobi + canonicalization. */
int sslg_gsvd(sslg_ctx* ctx, const float* r, uint32_t nsets, double* sigma, double* e, uint32_t* sweeps,
              uint8_t* conv);
/* The same with the right factor and the residual (GsvdBinResult::e_r and
 * recon_residual, gsvd.hpp:52-60): er [nsets][bins][m][m] row-major, row i
 * pairs with sigma_i so that A = E diag(sigma) E_r with A = K^-1 R; rows of
 * non-vanishing values are the reference's (the polar factor of E_g^H A per
 * tied group g -- for a single value, e_i^H A / sigma_i -- which is what the
 * reference's W^H rotation of V^H yields, gsvd.cpp:512-543), rows of the
 * vanishing block complete E_r to a unitary matrix (canonical completion, as
 * pick_orthonormal builds E's, gsvd.cpp:402-436).  resid [nsets][bins] =
 * ||A - E diag(sigma) E_r||_F / ||A||_F (reconstruction_residual,
 * gsvd.cpp:573-585), or -1 unless compute_residual is set.  Every output is
 * nullable. */
int sslg_gsvd_ex(sslg_ctx* ctx, const float* r, uint32_t nsets, double* sigma, double* e, double* er,
                 uint32_t* sweeps, uint8_t* conv, double* resid);

/* calc_average_power (music.cpp:112-165) on left factors e [nsets][bins][m][m]
 * (as returned by sslg_gsvd): power [nsets][dirs], bin_power
 * [nsets][bins][dirs] (nullable). */
int sslg_spectrum(sslg_ctx* ctx, const double* e, uint32_t nsets, double* power, double* bin_power);

/* peak_search (music.cpp:197-236) on power [nsets][dirs] with the context's
 * topology: est_* [nsets][num_sources], count [nsets]. */
int sslg_peaks(sslg_ctx* ctx, const double* power, uint32_t nsets, uint32_t* est_idx, double* est_power,
               uint8_t* est_low, uint32_t* count);

/* ---- on-disk formats and output records ----------------
 * File access is host I/O; what is loaded lands in the device context. */

/* load_correlation (correlation.cpp:169-193): SSLC tensor file ("SSLC",
 * u32le m, bins, T, then bins x m x m cf32 row-major).  Pass data == NULL to
 * read the header only.  SSLG_IO on a bad magic / implausible header /
 * truncated payload with the reference's messages. */
int sslg_read_correlation_file(const char* path, uint32_t* m, uint32_t* bins, uint32_t* t, float* data,
                               uint64_t cap_floats);
/* save_correlation (correlation.cpp:148-167). */
int sslg_write_correlation_file(const char* path, uint32_t m, uint32_t bins, uint32_t t, const float* data);
/* NoiseModel::from_file (gsvd.cpp:729-734) into the context: the SSLC file,
 * its positive-definiteness gate and the inverses.  *t (nullable) receives
 * the header's frame count. */
int sslg_load_noise_model(sslg_ctx* ctx, const char* path, uint32_t* bad_bin, uint32_t* t);
/* load_steering (music.cpp:72-106): JSON header line + [dirs][bins][m] cf32
 * payload.  Pass dirs_deg == h == NULL to read the header only; dirs_deg
 * [dirs][2], h [dirs][bins][m] cf32 (cap_dirs = capacity in directions). */
int sslg_read_steering_file(const char* path, uint32_t* m, uint32_t* bin_min, uint32_t* bin_max, uint32_t* dirs,
                            double* dirs_deg, float* h, uint64_t cap_dirs);
/* save_steering (music.cpp:47-70): the header as nlohmann::json dumps it. */
int sslg_write_steering_file(const char* path, uint32_t m, uint32_t bin_min, uint32_t bin_max, uint32_t dirs,
                             const double* dirs_deg, const float* h);
/* load_steering into the context (plus DirectionTopology::build at 10 degrees,
 * pipeline.cpp:222); *bin_min (nullable) receives the field's first bin. */
int sslg_load_steering(sslg_ctx* ctx, const char* path, uint32_t* bin_min);
/* capture_noise_model (synth.cpp:329-373) on the device from noise-only PCM
 * pcm [m][nsamples] f32: the device STFT (bit-identical frames), K = sum_f
 * x x^H / F accumulated in FP64 in frame order and narrowed to cf32
 * (bit-identical to the reference's), then check_positive_definite.
 * k_out (nullable) receives K [bins][m][m] cf32; install != 0 makes it the
 * context's noise model (inverses built).  Needs sslg_set_stft. */
int sslg_capture_noise_model(sslg_ctx* ctx, const float* pcm, uint64_t nsamples, int install, float* k_out,
                             uint32_t* nframes, uint32_t* bad_bin);
/* One JSONL record of run_locate_to_stream (pipeline.cpp:265-286) for a
 * block: {"estimates":[{"azimuth_deg","direction","elevation_deg",
 * "low_power","power"},...],"frame"} laid out as nlohmann::json::dump()
 * writes it (sorted keys, shortest round-trip doubles).  idx/power/low hold
 * `count` estimates, dirs_deg the grid [dirs][2]; buf == NULL queries *len. */
int sslg_format_estimates_json(uint64_t frame, uint32_t count, const uint32_t* idx, const double* dirs_deg,
                               const double* power, const uint8_t* low, char* buf, uint64_t cap, uint64_t* len);

/* ---- measurement ---------------------------------------------------------- */

/* Device time (ms) of each stage of the last push, measured with CUDA events
 * on the context stream: [0] correlation, [1] jacobi, [2] canonical,
 * [3] spectrum, [4] peaks. */
int sslg_last_stage_ms(const sslg_ctx* ctx, float* ms5);
/* Number of kernel launches issued by the last push / stage call. */
uint32_t sslg_last_launch_count(const sslg_ctx* ctx);
/* Measured FP64 FMA throughput of `device` (TFLOP/s): the roofline
 * denominator for the FP64 solver kernels. */
int sslg_probe_fp64_tflops(int device, double* tflops);
/* Measured FP32 FMA throughput of `device` (TFLOP/s): the ceiling a float
 * solver would have (reported beside the FP64 fraction). */
int sslg_probe_fp32_tflops(int device, double* tflops);
/* Diagnostics: SM clocks summed over all GSVD CTAs per solver phase
 * (whiten, QR, sweeps, sigma/back-multiply, basis completion, canonical
 * picker + phase, store) since the last reset; needs SSLG_PHASE_CLOCKS=1 in
 * the environment when the context is created. */
int sslg_debug_phase_clocks(sslg_ctx* ctx, double* out8, int reset);

#ifdef __cplusplus
}
#endif
#endif /* SSLGPU_H */
