// A = K^-1 R for one bin, formed in shared memory (shared by the Jacobi and
// canonicalization kernels).  The product follows gsvd.cpp:596/702 in FP64:
// K^-1 is the FP64 inverse of the FP32 noise model, R the FP32 correlation
// widened exactly.
#pragma once
#include "common.cuh"

namespace sslg {

// A = K^-1 R into W (column-major), staging R as float2 in the upper half of
// the W buffer (bytes [8 m^2, 16 m^2)).  Columns j < m/2 live entirely in the
// lower half and are written as soon as they are formed; the remaining
// columns overlap the staged R and are held in registers until R is dead.
__device__ __forceinline__ void form_whitened(const float2* __restrict__ rb, const double2* __restrict__ kb,
                                              int m, double2* W) {
    const int tid = threadIdx.x;
    const int mm = m * m;
    float2* rs = reinterpret_cast<float2*>(W) + mm;
    for (int e = tid; e < mm; e += blockDim.x) rs[e] = rb[e];
    __syncthreads();
    int parts = blockDim.x / m;
    if (parts > m) parts = m;
    const int jl = m / 2;  // columns [0, jl) do not overlap the staged R
    const bool active = tid < m * parts;
    const int i = active ? tid / parts : 0;
    const int part = active ? tid % parts : 0;
    // pass 1: columns 0..jl-1, written directly
    if (active) {
        for (int j0 = part; j0 < jl; j0 += 8 * parts) {
            double2 acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = make_double2(0, 0);
            for (int k = 0; k < m; ++k) {
                const double2 kv = __ldg(&kb[i * m + k]);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + u * parts;
                    if (j < jl) acc[u] = cadd(acc[u], cmul(kv, f2d(rs[k * m + j])));
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + u * parts;
                if (j < jl) W[j * m + i] = acc[u];
            }
        }
    }
    // pass 2: columns jl..m-1 overlap R; at most 8 per thread for m <= 64
    double2 hold[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) hold[u] = make_double2(0, 0);
    if (active) {
        for (int k = 0; k < m; ++k) {
            const double2 kv = __ldg(&kb[i * m + k]);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = jl + part + u * parts;
                if (j < m) hold[u] = cadd(hold[u], cmul(kv, f2d(rs[k * m + j])));
            }
        }
    }
    __syncthreads();
    if (active) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = jl + part + u * parts;
            if (j < m) W[j * m + i] = hold[u];
        }
    }
    __syncthreads();
}

}  // namespace sslg
