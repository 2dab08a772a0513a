// A = K^-1 R for one bin, formed in shared memory (shared by the Jacobi and
// canonicalization kernels).  The product follows gsvd.cpp:596/702 in FP64:
// K^-1 is the FP64 inverse of the FP32 noise model, R the FP32 correlation
// widened exactly.
#pragma once
#include "common.cuh"

namespace sslg {

constexpr int kWhitenBatch = 8;  // K^-1 loads in flight per thread

// acc[u] += sum_k K^-1[i][k] R[k][j_u], K^-1 row i streamed from global in
// batches of kWhitenBatch independent loads (the row is L2-resident; a
// dependent load per k would serialize ~m L2 round trips per thread).
template <typename RT, typename ColFn>
__device__ __forceinline__ void whiten_rows(const double2* __restrict__ krow, const RT* rs, int m, int ld, double2* acc,
                                            ColFn col) {
    for (int k0 = 0; k0 < m; k0 += kWhitenBatch) {
        double2 kv[kWhitenBatch];
#pragma unroll
        for (int b = 0; b < kWhitenBatch; ++b) kv[b] = (k0 + b < m) ? __ldg(&krow[k0 + b]) : make_double2(0, 0);
#pragma unroll
        for (int b = 0; b < kWhitenBatch; ++b) {
            const int k = k0 + b;
            if (k < m) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = col(u);
                    if (j >= 0) {
                        const double2 r = f2d(rs[k * ld + j]);
                        acc[u].x = fma(kv[b].x, r.x, fma(-kv[b].y, r.y, acc[u].x));
                        acc[u].y = fma(kv[b].x, r.y, fma(kv[b].y, r.x, acc[u].y));
                    }
                }
            }
        }
    }
}

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
    const double2* krow = kb + (size_t)i * m;
    // pass 1: columns 0..jl-1, written directly
    if (active) {
        for (int j0 = part; j0 < jl; j0 += 8 * parts) {
            double2 acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = make_double2(0, 0);
            whiten_rows(krow, rs, m, m, acc, [&](int u) {
                const int j = j0 + u * parts;
                return j < jl ? j : -1;
            });
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
    if (active)
        whiten_rows(krow, rs, m, m, hold, [&](int u) {
            const int j = jl + part + u * parts;
            return j < m ? j : -1;
        });
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

// A = K^-1 R into W with R widened to FP64 once, one column half at a time,
// in a separate buffer `stage` (>= m * ceil(m/2) entries): the inner loop is
// one 16-byte shared load per complex MAC instead of a load and two
// conversions, and W is written directly.  Bit-identical to form_whitened.
__device__ __forceinline__ void form_whitened_staged(const float2* __restrict__ rb, const double2* __restrict__ kb,
                                                     int m, double2* W, double2* stage) {
    const int tid = threadIdx.x;
    const int nt = blockDim.x;
    int parts = nt / m;
    if (parts > m) parts = m;
    const bool active = tid < m * parts;
    const int i = active ? tid / parts : 0;
    const int part = active ? tid % parts : 0;
    const double2* krow = kb + (size_t)i * m;
    const int jh = (m + 1) / 2;
    for (int h = 0; h < 2; ++h) {
        const int j0 = h ? jh : 0, nj = h ? m - jh : jh;
        for (int e = tid; e < m * nj; e += nt) {
            const int k = e / nj, jj = e - k * nj;
            stage[e] = f2d(rb[k * m + j0 + jj]);
        }
        __syncthreads();
        // 8 columns per thread and pass (one pass at 256 threads, m <= 64)
        for (int jb = 0; active && jb < nj; jb += 8 * parts) {
            double2 acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = make_double2(0, 0);
            whiten_rows(krow, stage, m, nj, acc, [&](int u) {
                const int jj = jb + part + u * parts;
                return jj < nj ? jj : -1;
            });
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int jj = jb + part + u * parts;
                if (jj < nj) W[(j0 + jj) * m + i] = acc[u];
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// A = K^-1 R on the FP64 tensor cores (DMMA m8n8k4), for the split solver's
// prologue: K^-1 is staged in W (row-major, the A operand), R in `stage` as
// float2 (the B operand, widened exactly at the fragment load); warp w
// computes the 8-row strip 8w..8w+7 of A (8 complex 8x8 tiles, four real
// MMAs per 4-wide k-step: Re += Kr Rr - Ki Ri, Im += Kr Ri + Ki Rr) in
// registers, then writes it column-major over W and to `ag` (the saved copy
// the back-multiplication reads).  NT threads, NT / 32 >= ceil(m / 8) warps.
// Same products as form_whitened, summed in the tensor core's order.
template <int NT>
__device__ __forceinline__ void form_whitened_mma(const float2* __restrict__ rb, const double2* __restrict__ kb,
                                                  int m, double2* W, float2* stage, double2* ag) {
    const int t = threadIdx.x;
    batched_copy<4>(t, NT, m * m, kb, [&](int e, double2 v) { W[e] = v; });
    batched_copy<4>(t, NT, m * m, rb, [&](int e, float2 v) { stage[e] = v; });
    __syncthreads();
    const int warp = t >> 5, lane = t & 31, r = lane >> 2, c = lane & 3;
    const int nt8 = (m + 7) >> 3;
    double re[8][2], im[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) re[j][0] = re[j][1] = im[j][0] = im[j][1] = 0.0;
    const int i = warp * 8 + r;
    if (warp < nt8) {
        for (int k0 = 0; k0 < m; k0 += 4) {
            const int k = k0 + c;
            const double2 av = (i < m && k < m) ? W[i * m + k] : make_double2(0, 0);
            const double nai = -av.y;
            double2 bv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int col = j * 8 + r;
                bv[j] = (j < nt8 && k < m && col < m) ? f2d(stage[k * m + col]) : make_double2(0, 0);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nt8) {
                    dmma_8x8x4(re[j][0], re[j][1], av.x, bv[j].x);
                    dmma_8x8x4(im[j][0], im[j][1], av.x, bv[j].y);
                }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nt8) {
                    dmma_8x8x4(re[j][0], re[j][1], nai, bv[j].y);
                    dmma_8x8x4(im[j][0], im[j][1], av.y, bv[j].x);
                }
        }
    }
    __syncthreads();  // K^-1 in W is consumed
    if (warp < nt8) {
        const int row = warp * 8 + r;
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = j * 8 + 2 * c + e;
                if (row < m && col < m) {
                    const double2 v = make_double2(re[j][e], im[j][e]);
                    W[col * m + row] = v;
                    if (ag) ag[col * m + row] = v;
                }
            }
    }
    __syncthreads();
}

}  // namespace sslg
