// Throughput harness for the Jacobi sweep loop (development aid): many CTAs
// (2 per SM), random 60x60 complex W in shared memory, a fixed number of
// round-robin sweeps with the production rotate_pair / neighbor hand-off.
// Variants: -DSB_NOSTORE (no write-back), -DSB_NOROT (dot products only).
// Measured on B200 (SM-cycles per round per bin, all pairs rotating): base
// 1607, no stores 816, dot products only 702 -- the round's shared-memory
// stores cost as much as everything else together.
#include "../../paper_2504_03373_b200/csrc/gsvd.cu"
#include <cstdio>
using namespace sslg;
__global__ void __launch_bounds__(256, 2) sweep_bench(double2* out, int m, int sweeps, long long* clk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    __shared__ double cn[kMaxM];
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) {
        unsigned h = (unsigned)(e * 2654435761u) ^ (unsigned)(blockIdx.x * 40503u);
        W[e] = make_double2((h & 0xffff) / 65536.0 - 0.5, ((h >> 16) & 0xffff) / 65536.0 - 0.5);
    }
    if (tid < m) cn[tid] = 0;
    __syncthreads();
    const int g = tid / kLPP, s = tid % kLPP;
    const int n_even = (m + 1) & ~1, npairs = n_even / 2;
    for (int j = g * 2; j < g * 2 + 2 && j < m; ++j) {
        double v = 0;
        for (int u = 0; u < kRows; ++u) { const int row = s + u * kLPP; if (row < m) v += cnorm(W[j * m + row]); }
        v = group_sum<kLPP>(v);
        if (s == 0) cn[j] = v;
    }
    __syncthreads();
    long long t0 = clock64();
    double mymax = 0;
    int rots = 0;
#ifdef SB_HALVE
    int n2 = 2;
    while (n2 < m) n2 <<= 1;
    const bool gact = g < n2 / 2;
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int S = n2; S >= 2; S >>= 1) {
            const int h = S >> 1;
            const int kset = g / h, gi = g % h;
            const int ia = kset * S + gi;
            int ib = kset * S + h + gi;
            double2 Aa[kRows], Bb[kRows];
            double ca = 0.0, cb = 0.0;
            bool adirty = false;
            if (gact) {
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    Aa[u] = (row < m && ia < m) ? W[ia * m + row] : make_double2(0, 0);
                    Bb[u] = (row < m && ib < m) ? W[ib * m + row] : make_double2(0, 0);
                }
                ca = ia < m ? cn[ia] : 0.0;
                cb = ib < m ? cn[ib] : 0.0;
            }
            for (int rnd = 0; rnd < h; ++rnd) {
                if (gact && ia < m && ib < m) {
                    if (rotate_pair<kRows, kLPP>(Aa, Bb, ca, cb, 0.0, s, m, mymax)) {
                        adirty = true;
                        ++rots;
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            if (row < m) W[ib * m + row] = Bb[u];
                        }
                        if (s == 0) cn[ib] = cb;
                    }
                }
                if (rnd + 1 < h) {
                    __syncthreads();
                    ib = kset * S + h + ((gi + rnd + 1) & (h - 1));
                    if (gact) {
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            Bb[u] = (row < m && ib < m) ? W[ib * m + row] : make_double2(0, 0);
                        }
                        cb = ib < m ? cn[ib] : 0.0;
                    }
                }
            }
            if (gact && adirty) {
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    if (row < m) W[ia * m + row] = Aa[u];
                }
                if (s == 0) cn[ia] = ca;
            }
            __syncthreads();
        }
    }
#else
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                double2 P[kRows], Q[kRows];
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    P[u] = row < m ? W[p * m + row] : make_double2(0, 0);
                    Q[u] = row < m ? W[q * m + row] : make_double2(0, 0);
                }
                double cp = cn[p], cq = cn[q];
#ifdef SB_NOROT
                double d0 = 0;
                for (int u = 0; u < kRows; ++u) d0 = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d0));
                d0 = group_sum<kLPP>(d0);
                rots += d0 > 1e300;
#else
                if (rotate_pair<kRows, kLPP>(P, Q, cp, cq, 0.0, s, m, mymax)) {
                    ++rots;
#ifndef SB_NOSTORE
#pragma unroll
                    for (int u = 0; u < kRows; ++u) {
                        const int row = s + u * kLPP;
                        if (row < m) {
                            W[p * m + row] = P[u];
                            W[q * m + row] = Q[u];
                        }
                    }
                    if (s == 0) { cn[p] = cp; cn[q] = cq; }
#endif
                }
#endif
            }
            __syncthreads();
        }
    }
#endif
    long long t1 = clock64();
    if (tid == 0) atomicAdd((unsigned long long*)clk, (unsigned long long)(t1 - t0));
    if (tid == 0) out[blockIdx.x] = make_double2(W[0].x + rots, mymax);
}
int main() {
    const int m = 60, sweeps = 4, ctas = 148 * 2 * 4;
    double2* out; long long* clk;
    cudaMalloc(&out, ctas * sizeof(double2)); cudaMalloc(&clk, 8);
    const int smem = m * m * 16;
    cudaFuncSetAttribute(sweep_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(clk, 0, 8);
        cudaEventRecord(a);
        sweep_bench<<<ctas, 256, smem>>>(out, m, sweeps, clk);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double rounds = (double)sweeps * (m - 1);
        printf("%-12s %.3f ms  per-CTA cycles/round %.0f  SM-cycles/round-of-one-bin %.0f (%s)\n", VARIANT, ms,
               (double)c / ctas / rounds, ms * 1e-3 * 1.965e9 * 148 / (ctas * rounds), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
