// Launch interfaces of the sm_100a kernels, shared by the kernel translation
// units and the host engine (engine.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sslg {

struct StftArgs {
    const float* pcm;        // [m][pitch] samples, channel-major (SampleBlock::channels)
    const float* window;     // [n] make_window (host-evaluated, stft.cpp:28-36)
    const double2* twiddle;  // [n-1] per-stage recurrence twiddles, stage len at offset len/2-1
    float2* out;             // frame ring [cap][m][bins]
    size_t pitch;            // samples per channel row
    int m, n, shift, bin_min, bins;
    int cap;
    long long slot0;         // ring index of frame 0 of this launch
    const double2* dft = nullptr;  // non-power-of-two n: [bins][n] (cos, sin) of the retained bins
};
void launch_stft(const StftArgs& a, int nframes, cudaStream_t s);

struct CorrArgs {
    const float2* ring;  // [cap][m][bins] spectra, frame g at slot g % cap
    double2* state;      // [bins][m][m] FP64 running sum
    float2* r_out;       // [n_emit][bins][m][m]
    int m, bins, t, cap;
    int frames;          // frames ingested by this launch
    long long pushed0;   // pushes before this launch (== global index of first frame)
    long long since0;    // pushes since the last rebuild
    int rebuild_interval;
    const unsigned int* abort = nullptr;  // nonzero: a failed gate earlier on the stream, skip (async path)
};
void launch_correlation(const CorrArgs& a, cudaStream_t s);
void launch_count_nonfinite(const float* p, size_t n, unsigned int* bad, cudaStream_t s);
// synchronous per-frame gate: min(frame0 + f) over frames f holding a non-finite value -> *first
void launch_first_nonfinite(const float* p, size_t per_frame, int nframes, unsigned int frame0, unsigned int* first,
                            cudaStream_t s);
// async gate: the first failing push id + 1 lands in *abort (atomicCAS from 0)
void launch_gate_abort(const float* p, size_t n, unsigned int* abort, unsigned int id, cudaStream_t s);

// mat_inverse<float> and mat_inverse<double> (gsvd.cpp:21-62) of every bin:
// inv_out <- the double inverse, inv_f_out (nullable) <- the float inverse widened
void launch_gauss_jordan(const float2* k, int m, int bins, double2* inv_out, unsigned int* bad_f,
                         unsigned int* bad_d, cudaStream_t s, int pivoting = 1, double2* inv_f_out = nullptr);
// check_positive_definite (gsvd.cpp:736-754): Hermitian test + smallest eigenvalue
// of hermitian_eigenvalues (eig.cpp:11-84) per bin into min_eig (nullable)
void launch_pd_check(const float2* k, int m, int bins, unsigned int* bad_herm, unsigned int* bad_pd,
                     double* min_eig, cudaStream_t s);

struct GsvdArgs {
    const float2* r;      // [nblk][bins][m][m] row-major R
    const double2* kinv;  // [bins][m][m] row-major K^-1
    double* sigma;        // [nblk][bins][m]
    double2* e;           // [nblk][bins][m vec][m row]
    uint32_t* sweeps;     // [nblk][bins]
    uint8_t* conv;        // [nblk][bins]
    uint32_t* work;       // generic-canonicalization worklist: [0] count, [1] cursor, [2..] indices
    int m, bins, max_sweeps;
    int canonical, refine;
    int precondition;     // QR-preconditioned Jacobi (needs ascratch)
    double2* ascratch;    // [nblk][bins][m][m] column-major copy of A (precondition)
    long long* phase_clk; // optional [8] summed SM clocks per solver phase (diagnostics)
    const unsigned int* abort = nullptr;  // nonzero: a failed gate earlier on the stream, skip (async path)
    double2* wscratch = nullptr;  // [nblk][bins][m][m] W between the split solver kernels (m = 60)
    int* pivs = nullptr;          // [nblk][bins][64] QR column pivots between them
    int force_cta = 0;            // m <= 8: use the CTA solver instead of the warp solver (A/B, SSLG_SMALL_CTA=1)
    double tol2 = 1e-28;          // no-rotation test |a_pq|^2 <= tol2 |w_p|^2 |w_q|^2 (gsvd.cpp:648);
                                  // 1e-28 * SolverConfig::tolerance_scale^2
    uint32_t* done = nullptr;     // [nblk][bins] split solver: the launch epoch once a bin's sweeps are stored
    uint32_t epoch = 0;           // this launch's epoch (nonzero, new per launch)
};
// returns the number of kernels launched (1, or 3 when the solver is split
// around a 128-thread sweep kernel)
int launch_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s);
// m <= 8: one warp per (block, bin) (small.cu)
bool small_jacobi_supported(const GsvdArgs& a);
// the lane-group solver will run (launch_jacobi's choice for m <= 16); it
// canonicalizes every bin itself unless refine mode is on
bool small_jacobi_selected(const GsvdArgs& a);
void launch_small_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s);

struct CanonArgs {
    const float2* r;         // [nblk][bins][m][m]
    const double2* kinv;     // [bins][m][m]
    const double* sigma;     // [nblk][bins][m]
    double2* e;              // [nblk][bins][m vec][m row]  (in/out)
    uint32_t* work;          // worklist filled by jacobi_kernel (see GsvdArgs)
    int m, bins, refine;
    const unsigned int* abort = nullptr;  // nonzero: a failed gate earlier on the stream, skip (async path)
};
void launch_canonical(const CanonArgs& a, int nblk, cudaStream_t s);

// E_r rows and the reconstruction residual from the final E (er.cu)
struct ErArgs {
    const float2* r;      // [nblk][bins][m][m]
    const double2* kinv;  // [bins][m][m]
    const double* sigma;  // [nblk][bins][m]
    const double2* e;     // [nblk][bins][m vec][m row]
    double2* er;          // [nblk][bins][m][m] row-major (nullable)
    double* resid;        // [nblk][bins] (nullable)
    int m, bins;
    const unsigned int* abort = nullptr;
};
void launch_er(const ErArgs& a, int nblk, cudaStream_t s);

struct SpecArgs {
    const double2* e;    // [nblk][bins][m vec][m mic]
    const float2* h;     // [bins][dirs][m]
    const double* num;   // [bins][dirs]  |h|^2
    double* p;           // [nblk][bins][dirs]
    int m, bins, dirs, ns, dchunk, nsplit;
    double floor_;
    int squared;
    const unsigned int* abort = nullptr;  // nonzero: a failed gate earlier on the stream, skip (async path)
};
void launch_spectrum(SpecArgs a, int nblk, cudaStream_t s);
// the tcgen05 kind::tf32 (3-pass split) spectrum of large grids (music_tc.cu):
// the steering is prepared once into tf32 hi/lo slabs (spectrum_tc_slab_floats)
bool spectrum_tc_supported(const SpecArgs& a);
size_t spectrum_tc_slab_floats(int m, int bins, int dirs);
void launch_spectrum_tc_prep(const float2* h_t, int m, int bins, int dirs, float* slabs, cudaStream_t s);
void launch_spectrum_tc(const SpecArgs& a, const float* slabs, int nblk, cudaStream_t s);
// capture_noise_model (synth.cpp:329-373): FP64 sums of x x^H over frames, then K = float(sum / F)
void launch_capture_accum(const float2* frames, int nframes, int m, int bins, double2* acc, cudaStream_t s);
void launch_capture_narrow(const double2* acc, size_t n, double inv, float2* k, cudaStream_t s);
void launch_steering_prep(const float2* h_in, float2* h_t, double* num, int m, int bins, int dirs,
                          cudaStream_t s);

struct PeakArgs {
    const double* p;          // [nblk][bins][dirs]
    double* power;            // [nblk][dirs]
    const uint32_t* nbr_off;  // [dirs + 1]
    const uint32_t* nbr;      // [nnz]
    uint32_t* est_idx;        // [nblk][ns]
    double* est_pw;           // [nblk][ns]
    uint8_t* est_low;         // [nblk][ns]
    uint32_t* est_count;      // [nblk]
    int bins, dirs, ns;
    double low_ratio;         // double(float ratio)
    const unsigned int* abort = nullptr;  // nonzero: a failed gate earlier on the stream, skip (async path)
    int peak_chunk = 1;                   // bins staged per pass (set by launch_peaks)
};
void launch_peaks(PeakArgs a, int nblk, cudaStream_t s);

}  // namespace sslg
