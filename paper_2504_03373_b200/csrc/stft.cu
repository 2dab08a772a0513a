// Kernel (0): the STFT front end, SampleBlock -> SpectrumFrame
// (stft_frame / stft_stream, reference proj/src/stft.cpp:44-68, with
// real_dft_half / fft_pow2, proj/include/ssl/fft.hpp:15-68; other frame
// lengths through the direct sum, dft_kernel below).
//
// One warp per (frame, channel): the windowed frame (float product
// src[i] * window[i], stft.cpp:53) is stored bit-reversed in shared memory,
// then the log2(N) radix-2 stages run with the reference's arithmetic —
// butterflies in FP64 on the widened float data, v = b * w as the textbook
// complex product (the reference is built with -fcx-limited-range), u +- v
// rounded to float after every stage — so every output bin is bit-identical
// to the reference's.  The twiddles w_k of each stage are the reference's
// recurrence w *= wlen (fft.hpp:29-38) evaluated on the host (same libm,
// same order, no contraction) and read from a table.  The retained band
// [bin_min, bin_max] of every channel lands directly in the engine's frame
// ring ([m][bins] cf32 per slot), where the correlation kernel reads it.
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

__global__ void stft_kernel(StftArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int wpc = blockDim.x / kWarp;
    const int f = blockIdx.x;
    const int ch = blockIdx.y * wpc + warp;
    if (ch >= a.m) return;  // no block-wide barrier below
    const int n = a.n;
    float2* buf = reinterpret_cast<float2*>(smem_raw) + (size_t)warp * n;
    const float* src = a.pcm + (size_t)ch * a.pitch + (size_t)f * a.shift;
    const int lg = 31 - __clz(n);
    for (int i = lane; i < n; i += kWarp) {
        const int j = (int)(__brev((unsigned)i) >> (32 - lg));
        buf[j] = make_float2(__fmul_rn(src[i], a.window[i]), 0.0f);
    }
    __syncwarp();
    const double2* tw = a.twiddle;
    for (int half = 1; half < n; half <<= 1) {  // len = 2 * half
        for (int t = lane; t < n / 2; t += kWarp) {
            const int k = t & (half - 1);
            const int i0 = ((t - k) << 1) + k, i1 = i0 + half;
            const double2 w = tw[half - 1 + k];
            const float2 fa = buf[i0], fb = buf[i1];
            const double ur = fa.x, ui = fa.y, br = fb.x, bi = fb.y;
            const double vr = __dsub_rn(__dmul_rn(br, w.x), __dmul_rn(bi, w.y));
            const double vi = __dadd_rn(__dmul_rn(br, w.y), __dmul_rn(bi, w.x));
            buf[i0] = make_float2(__double2float_rn(__dadd_rn(ur, vr)), __double2float_rn(__dadd_rn(ui, vi)));
            buf[i1] = make_float2(__double2float_rn(__dsub_rn(ur, vr)), __double2float_rn(__dsub_rn(ui, vi)));
        }
        __syncwarp();
    }
    float2* dst = a.out + ((size_t)((a.slot0 + f) % a.cap) * a.m + ch) * a.bins;
    for (int b = lane; b < a.bins; b += kWarp) dst[b] = buf[a.bin_min + b];
}

// Non-power-of-two frame lengths: the reference's direct sum
// (real_dft_half, fft.hpp:55-65): out[k] = sum_i double(x_i) (cos, sin)(ang),
// ang = -2 pi k i / n, accumulated in i order in FP64 and rounded to float.
// The (cos, sin) table of the retained bins is evaluated on the host with
// the reference's libm calls and operation order (sslg_set_stft), so with
// unfused products and sums every bin is bit-identical.  One warp per
// (frame, channel), lanes over the retained bins.
__global__ void dft_kernel(StftArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int wpc = blockDim.x / kWarp;
    const int f = blockIdx.x;
    const int ch = blockIdx.y * wpc + warp;
    if (ch >= a.m) return;
    const int n = a.n;
    float* x = reinterpret_cast<float*>(smem_raw) + (size_t)warp * n;
    const float* src = a.pcm + (size_t)ch * a.pitch + (size_t)f * a.shift;
    for (int i = lane; i < n; i += kWarp) x[i] = __fmul_rn(src[i], a.window[i]);
    __syncwarp();
    float2* dst = a.out + ((size_t)((a.slot0 + f) % a.cap) * a.m + ch) * a.bins;
    for (int b = lane; b < a.bins; b += kWarp) {
        const double2* cs = a.dft + (size_t)b * n;
        double re = 0.0, im = 0.0;
        for (int i = 0; i < n; ++i) {
            const double xi = x[i];
            const double2 c = cs[i];
            re = __dadd_rn(re, __dmul_rn(xi, c.x));
            im = __dadd_rn(im, __dmul_rn(xi, c.y));
        }
        dst[b] = make_float2(__double2float_rn(re), __double2float_rn(im));
    }
}

// Warps (frame-channel transforms) per CTA: up to 8 within 32 KB of shared
// memory, fewer when the launch has fewer than 8 transforms per SM (C1: 32
// frames x 8 channels -- one warp per CTA spreads them over the SMs instead
// of 32 SMs running eight each: 16.9 -> 15.3 us per launch).
int stft_warps_per_cta(int n, int transforms) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 148;
    }
    int w = 16384 / n;
    if (w > 8) w = 8;
    const int spread = transforms / sms;
    if (w > spread) w = spread;
    if (w < 1) w = 1;
    return w;
}

void launch_stft(const StftArgs& a, int nframes, cudaStream_t s) {
    const int wpc = stft_warps_per_cta(a.n, nframes * a.m);
    const size_t smem = (size_t)wpc * a.n * sizeof(float2);
    if (smem > 48 * 1024) cudaFuncSetAttribute(stft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nframes, (a.m + wpc - 1) / wpc);
    if (a.dft) {  // non-power-of-two length: direct sum, one float per sample staged
        const size_t smem_d = (size_t)wpc * a.n * sizeof(float);
        if (smem_d > 48 * 1024) cudaFuncSetAttribute(dft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        dft_kernel<<<grid, wpc * kWarp, smem_d, s>>>(a);
        return;
    }
    stft_kernel<<<grid, wpc * kWarp, smem, s>>>(a);
}

}  // namespace sslg
