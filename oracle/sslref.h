/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the checker.
 *
 * C restatement of the reference (sslkit) double-precision path for the
 * GSVD-MUSIC hot path.  Every function cites the reference file:line it
 * follows (paths relative to /root/reference/proj).  Complex matrices are
 * row-major interleaved (re, im) pairs, exactly as the reference stores
 * CMatrix<T> (include/ssl/mat.hpp:12-29).
 *
 * Status codes follow the reference error taxonomy (include/ssl/types.hpp:13-23,
 * tools/sslkit.cpp:280-291): 0 ok, 2 validation, 3 numerical.
 */
#ifndef SSLREF_ORACLE_H
#define SSLREF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* CorrelationWindow push/normalized (correlation.cpp:53-130). */
int orc_correlation(const float* x, uint32_t frames, uint32_t m, uint32_t bins, uint32_t t,
                    uint32_t rebuild_interval, float* r_out, uint32_t* written);

/* mat_inverse<double> on the widened float K (gsvd.cpp:21-62, 764). */
int orc_mat_inverse(const float* k, uint32_t m, int pivoting, uint32_t bin_label, double* out);

/* jacobi_svd (gsvd.cpp:622-695). vh may be NULL. */
int orc_jacobi_svd(const double* a, uint32_t m, double* sigma, double* u, double* vh,
                   uint32_t* sweeps, uint8_t* conv);

/* canonicalize_subspaces<double> (gsvd.cpp:470-565). er may be NULL. */
void orc_canonicalize(const double* a, uint32_t m, const double* sigma, double* e, double* er);

/* gsvd_reference over bins (gsvd.cpp:697-716, 832-844).  kinv: [bins][m][m] cf64
 * (NULL: invert k here), k/r: [bins][m][m] cf32.  er/iters/conv nullable. */
int orc_gsvd_reference(const float* k, const double* kinv, const float* r, uint32_t m, uint32_t bins,
                       int canonical, int threads, double* sigma, double* e, double* er,
                       uint32_t* sweeps, uint8_t* conv);

/* calc_average_power<double> (music.cpp:112-165).  e: [bins][m][m] cf64;
 * h: [dirs][bins][m] cf32.  bin_power nullable ([bins][dirs]). */
int orc_spectrum(const double* e, uint32_t m, uint32_t bins, const float* h, uint32_t dirs,
                 uint32_t num_sources, float floor, int squared, int threads, double* power,
                 double* bin_power);

/* DirectionTopology::build (music.cpp:176-195) as CSR. */
int orc_topology(const double* dirs, uint32_t n, double radius_deg, uint32_t* offsets, uint32_t* nbr,
                 uint32_t cap);

/* peak_search (music.cpp:197-236) on a CSR topology. */
int orc_peaks(const double* power, uint32_t n, const uint32_t* offsets, const uint32_t* nbr,
              uint32_t num_sources, float low_power_ratio, uint32_t* idx, double* pw, uint8_t* low,
              uint32_t* count);

/* make_window (stft.cpp:28-36): w [length] f32; kind 0 hann (periodic), 1 rectangular. */
void orc_window(int kind, uint32_t length, float* w);

/* stft_stream / stft_frame (stft.cpp:38-68) with real_dft_half / fft_pow2
 * (fft.hpp:15-68): pcm [m][nsamples] f32 channel-major (SampleBlock::channels);
 * frames [nframes][m][bin_max-bin_min+1] cf32, nframes = (nsamples-len)/shift+1
 * (0 if nsamples < len).  Power-of-two lengths only (the fast path). */
int orc_stft(const float* pcm, uint32_t m, uint64_t nsamples, uint32_t frame_length, uint32_t shift, int window,
             uint32_t bin_min, uint32_t bin_max, float* frames, uint32_t* nframes);

#ifdef __cplusplus
}
#endif
#endif
