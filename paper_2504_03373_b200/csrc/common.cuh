// Shared device helpers for the sm_100a GSVD-MUSIC kernels.
//
// Complex values are interleaved (re, im) pairs: float2 for the FP32 tensors
// the reference stores (spectra, R, K, steering: include/ssl/types.hpp:25-26,
// correlation.hpp:14-21, music.hpp:32-47) and double2 for everything the
// solver computes (A, W, E, P), so every stored tensor keeps the reference's
// memory layout and only the arithmetic precision is chosen here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sslg {

constexpr int kMaxM = 64;       // channels handled by the SMEM-resident solver
constexpr int kWarp = 32;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// conj(a) * b
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cnorm(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 f2d(float2 a) { return make_double2((double)a.x, (double)a.y); }
__device__ __forceinline__ double2 f2d(double2 a) { return a; }

__device__ __forceinline__ double shfl_xor_d(double v, int m, unsigned mask = 0xffffffffu) {
    return __shfl_xor_sync(mask, v, m);
}

// 1/sqrt(x) and 1/x for positive normal FP64 arguments: the MUFU seed
// (rsqrt/rcp.approx.ftz.f64, ~2^-22 relative) refined by two Newton steps to
// full precision, without the special-case paths of the library versions.
// Used on the Jacobi rotation-parameter chain, which is latency-bound.
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
}
// gpu-scope release store / acquire load (cross-CTA hand-off flags)
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    return y;
}

// Lanes of the aligned W-lane group that contains this thread.  Reductions
// over a group name only that group, so groups may diverge independently.
template <int W>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (W >= 32) {
        return 0xffffffffu;
    } else {
        return ((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1));
    }
}

template <int W>
__device__ __forceinline__ double group_sum(double v) {
    const unsigned mask = group_mask<W>();
#pragma unroll
    for (int m = W / 2; m > 0; m >>= 1) v += __shfl_xor_sync(mask, v, m);
    return v;
}

template <int W>
__device__ __forceinline__ double2 group_sum2(double2 v) {
    const unsigned mask = group_mask<W>();
#pragma unroll
    for (int m = W / 2; m > 0; m >>= 1) {
        v.x += __shfl_xor_sync(mask, v.x, m);
        v.y += __shfl_xor_sync(mask, v.y, m);
    }
    return v;
}

// store(e, src[e]) for e = t, t + nt, ... < n with B loads in flight per
// thread: a plain load-store loop through generic pointers is compiled as one
// dependent global round trip per element (the store may alias the next load)
template <int B, class T, class F>
__device__ __forceinline__ void batched_copy(int t, int nt, int n, const T* __restrict__ src, F store) {
    for (int e0 = t; e0 < n; e0 += B * nt) {
        T v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int e = e0 + u * nt;
            if (e < n) v[u] = src[e];
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int e = e0 + u * nt;
            if (e < n) store(e, v[u]);
        }
    }
}

// block-wide helpers -------------------------------------------------------

// Round-robin (circle method) pairing for an even number of columns n:
// round r in [0, n-1), pair g in [0, n/2).  Every unordered pair appears
// exactly once per sweep and each column once per round.
__device__ __forceinline__ void rr_pair(int r, int g, int n, int& p, int& q) {
    int a, b;
    if (g == 0) {
        a = n - 1;
        b = r;
    } else {  // r < n - 1 and g < n / 2: one conditional subtraction replaces the modulo
        a = r + g;
        if (a >= n - 1) a -= n - 1;
        b = r - g + (n - 1);
        if (b >= n - 1) b -= n - 1;
    }
    p = a < b ? a : b;
    q = a < b ? b : a;
}

}  // namespace sslg
