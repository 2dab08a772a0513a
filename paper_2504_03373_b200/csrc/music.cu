// Kernels (3) and (4): MUSIC pseudo-spectrum, broadband integration, peaks.
//
// (3) P(theta, w) = |h|^2 / max(floor, sum_{i >= Ns} |h^H e_i|)
//     (calc_average_power, reference proj/src/music.cpp:112-165; squared
//     denominator optional, music.hpp:55-57), FP64 arithmetic on the FP32
//     steering table.  One CTA per (block, bin, direction chunk): the bin's
//     noise vectors E_n (FP64) and the chunk's steering vectors (transposed to
//     [mic][dir] so consecutive threads read consecutive directions) are staged
//     in SMEM; thread (direction, part) accumulates |h^H e_i| over its share of
//     the noise vectors four at a time (one steering load feeds four complex
//     FMAs).  Every direction runs the identical instruction sequence, so
//     bit-identical steering vectors give bit-identical powers (exact ties
//     survive to the peak search, music.cpp:215-223).
// (4) Pbar(theta) = sum_w P(theta, w) in ascending-bin FP64 order
//     (music.cpp:160), then the local-maximum test on the host-built neighbor
//     topology, stable (power desc, index asc) top-Ns and the low-power flag
//     against the sequential FP64 mean (peak_search, music.cpp:197-236).
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

constexpr int kSpecThreads = 256;

// |z| as sqrt(x^2 + y^2): the projections are far from the overflow and
// underflow ranges hypot guards against, and its guarded sequence was a large
// share of the spectrum's FP64 work; every direction still runs the identical
// instruction sequence (exact ties survive)
__device__ __forceinline__ double cabs_fast(double2 z) { return sqrt(fma(z.x, z.x, z.y * z.y)); }
constexpr int kSpecVec = 4;  // noise vectors per steering load

__global__ void __launch_bounds__(kSpecThreads) spectrum_kernel(SpecArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    const int nn = m - a.ns;
    double2* En = reinterpret_cast<double2*>(smem_raw);             // [nn][m]
    float2* Hs = reinterpret_cast<float2*>(En + (size_t)nn * m);   // [m][dchunk]
    double* part_den = reinterpret_cast<double*>(Hs + (size_t)m * a.dchunk);  // [nsplit][dchunk]

    const int blkbin = blockIdx.x;  // block * bins + bin
    const int bin = blkbin % a.bins;
    const int d0 = blockIdx.y * a.dchunk;
    const int nd = min(a.dchunk, a.dirs - d0);
    const int t = threadIdx.x;

    const double2* eb = a.e + ((size_t)blkbin * m + a.ns) * m;
    for (int x = t; x < nn * m; x += blockDim.x) En[x] = eb[x];
    const float2* hb = a.h + ((size_t)bin * a.dirs + d0) * m;
    for (int x = t; x < nd * m; x += blockDim.x) {
        const int d = x / m, mic = x % m;
        Hs[mic * a.dchunk + d] = hb[x];
    }
    __syncthreads();

    const int d = t % a.dchunk;
    const int part = t / a.dchunk;
    if (part < a.nsplit && d < nd) {
        double den = 0;
        // vector chunks of kSpecVec assigned round-robin to parts
        for (int v0 = part * kSpecVec; v0 < nn; v0 += a.nsplit * kSpecVec) {
            double2 acc[kSpecVec];
#pragma unroll
            for (int u = 0; u < kSpecVec; ++u) acc[u] = make_double2(0, 0);
            for (int mic = 0; mic < m; ++mic) {
                const double2 hv = f2d(Hs[mic * a.dchunk + d]);
#pragma unroll
                for (int u = 0; u < kSpecVec; ++u)
                    if (v0 + u < nn) acc[u] = cadd(acc[u], cmulc(hv, En[(v0 + u) * m + mic]));
            }
#pragma unroll
            for (int u = 0; u < kSpecVec; ++u) {
                if (v0 + u < nn) {
                    const double mag = cabs_fast(acc[u]);
                    den += a.squared ? mag * mag : mag;
                }
            }
        }
        part_den[part * a.dchunk + d] = den;
    }
    __syncthreads();
    if (t < nd) {
        double den = part_den[t];
        for (int pp = 1; pp < a.nsplit; ++pp) den += part_den[pp * a.dchunk + t];
        if (den < a.floor_) den = a.floor_;
        const double num = a.num[(size_t)bin * a.dirs + d0 + t];
        a.p[(size_t)blkbin * a.dirs + d0 + t] = num / den;
    }
}


// Small arrays (m <= 8: C1): one WARP per
// (block, bin), eight per CTA.  The bin's noise vectors sit in the warp's
// slice of shared memory (broadcast reads); each lane takes directions
// lane, lane + 32, ... with its steering vector in registers and runs the
// noise vectors in order, so every direction runs the identical instruction
// sequence (exact ties survive) and the denominator sums in the reference's
// vector order (music.cpp:140-152).  One CTA-wide load of the direction chunk
// per (block, bin) in spectrum_kernel cost more than the arithmetic at these
// sizes (C1: 68 us per 32 blocks).
constexpr int kSpecWarps = 8;

template <int MCAP>
__global__ void __launch_bounds__(32 * kSpecWarps) spectrum_warp_kernel(SpecArgs a, int nbb) {
    if (a.abort && *a.abort) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m, nn = m - a.ns;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* En = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * nn * m;
    const int bb = blockIdx.x * kSpecWarps + warp;  // block * bins + bin
    if (bb >= nbb) return;                          // a whole warp
    const int bin = bb % a.bins;
    const double2* eb = a.e + ((size_t)bb * m + a.ns) * m;
    for (int x = lane; x < nn * m; x += 32) En[x] = eb[x];
    __syncwarp();
    for (int d = lane; d < a.dirs; d += 32) {
        const float2* hb = a.h + ((size_t)bin * a.dirs + d) * m;
        double2 h[MCAP];
#pragma unroll
        for (int i = 0; i < MCAP; ++i) h[i] = i < m ? f2d(hb[i]) : make_double2(0, 0);
        double den = 0;
        for (int v = 0; v < nn; ++v) {
            const double2* ev = En + v * m;
            double2 acc = make_double2(0, 0);
#pragma unroll
            for (int i = 0; i < MCAP; ++i)
                if (i < m) acc = cadd(acc, cmulc(h[i], ev[i]));
            const double mag = cabs_fast(acc);
            den += a.squared ? mag * mag : mag;
        }
        if (den < a.floor_) den = a.floor_;
        a.p[(size_t)bb * a.dirs + d] = a.num[(size_t)bin * a.dirs + d] / den;
    }
}

// FP64 tensor-core variant (DMMA, mma.sync m8n8k4 .f64), used whenever the
// noise subspace has 16..64 vectors (C3, C4; C1/C2 keep the kernel above):
// the contraction
// h^H e for a warp's 8 directions x 64 noise-vector slots is 8 complex 8x8
// tiles, each k-step of 4 mics four real MMAs (Re += Hr Er + Hi Ei,
// Im += Hr Ei - Hi Er).  One instruction carries 256 FMAs, so the issue
// overhead of an FFMA-tiled kernel (loads, conversions, index math per
// 4 FMAs) disappears; B200 runs DMMA at 37 TFLOP/s vs 33 for DFMA
// (tools/ubench/dmma.cu).  Fragment layouts (PTX m8n8k4 .f64): A[r][c] at
// lane 4r + c, B[k][n] at lane 4n + k, C[r][2c + i] at lane 4r + c.  Every
// direction's denominator is reduced in the same order (its lane's two
// columns per tile over the tiles, then the 4 lanes of its row), so exact
// steering ties stay exact.
constexpr int kMmaN = 64;  // noise-vector slots (8 tiles of 8)

__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__host__ __device__ inline int mma_kpad(int m) { return (m + 3) & ~3; }
// noise-vector row stride (double2): = 4 mod 8, so the two vectors a quarter
// warp reads land in opposite bank halves
__host__ __device__ inline int mma_estride(int m) { return ((mma_kpad(m) + 3) & ~7) + 4; }
// steering row stride (float2): = 4 or 12 mod 16 (two rows per quarter warp
// in different banks); m itself when m = 4 mod 8 (bulk-copied rows)
__host__ __device__ inline int mma_hstride(int m) { return (m & 7) == 4 ? m : ((mma_kpad(m) + 11) & ~15) + 4; }

// 1-D bulk copies (TMA engine, cp.async.bulk) global -> shared, completed on
// an mbarrier with a transaction byte count
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
}

template <int WPC>
__global__ void __launch_bounds__(32 * WPC, 2) spectrum_mma_kernel(SpecArgs a, int nblk) {
    constexpr int kChunk = 8 * WPC;
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    const int nn = m - a.ns;
    const int kp = mma_kpad(m), es = mma_estride(m), hs = mma_hstride(m);
    double2* Es = reinterpret_cast<double2*>(smem_raw);                 // [kMmaN][es]
    float2* Hs = reinterpret_cast<float2*>(Es + (size_t)kMmaN * es);  // [kChunk][hs]
    // one CTA per (bin, block), blocks of a bin adjacent (its steering stays
    // in L2); the noise vectors are staged once and every direction chunk of
    // the grid streams past them
    const int bin = blockIdx.x / nblk, blk = blockIdx.x % nblk;
    const int blkbin = blk * a.bins + bin;
    const int t = threadIdx.x;

    const double2* eb = a.e + ((size_t)blkbin * m + a.ns) * m;  // [nn][m]
    const int nchunk = (a.dirs + kChunk - 1) / kChunk;
    // m = 4 mod 8: the staged layouts equal the global ones (row strides m),
    // so the noise vectors — and the steering rows when one chunk covers the
    // grid — arrive by bulk copy (one TMA request each) while the threads
    // zero the padding rows
    const bool bulk = (m & 7) == 4;
    const bool hbulk = bulk && nchunk == 1;
    __shared__ unsigned long long bar;
    if (bulk) {
        if (t == 0) mbar_init(&bar, 1);
        __syncthreads();
        const int nd0 = min(kChunk, a.dirs);
        if (t == 0) {
            const unsigned eb_bytes = (unsigned)(nn * m * sizeof(double2));
            const unsigned hb_bytes = hbulk ? (unsigned)(nd0 * m * sizeof(float2)) : 0u;
            mbar_expect_tx(&bar, eb_bytes + hb_bytes);
            bulk_g2s(Es, eb, eb_bytes, &bar);
            if (hbulk) bulk_g2s(Hs, a.h + (size_t)bin * a.dirs * m, hb_bytes, &bar);
        }
        for (int x = t; x < (kMmaN - nn) * m; x += blockDim.x) Es[nn * m + x] = make_double2(0, 0);
        if (hbulk)
            for (int x = t; x < (kChunk - nd0) * m; x += blockDim.x) Hs[nd0 * m + x] = make_float2(0.f, 0.f);
        mbar_wait(&bar, 0);
    } else {
        for (int x = t; x < kMmaN * kp; x += blockDim.x) {
            const int v = x / kp, mic = x - v * kp;
            Es[v * es + mic] = (v < nn && mic < m) ? eb[(size_t)v * m + mic] : make_double2(0, 0);
        }
    }
    const int warp = t >> 5, lane = t & 31;
    const int r = lane >> 2, c = lane & 3;
    float2* Hw = Hs + warp * 8 * hs;  // this warp's 8 steering rows (warp-private)
    __syncthreads();                  // the noise vectors (and padding) are staged
    for (int chunk = 0; chunk < nchunk; ++chunk) {
        const int d0 = chunk * kChunk;
        const int nd = min(kChunk, a.dirs - d0);
        if (hbulk) goto compute;  // the steering rows came with the bulk copy
        // each warp stages its own 8 directions: no block barrier per chunk
        __syncwarp();  // the previous chunk's rows are consumed
        {
        const int dw = d0 + warp * 8;
        const float2* hb = a.h + ((size_t)bin * a.dirs + dw) * m;
        for (int x = lane; x < 8 * kp; x += 32) {
            const int d = x / kp, mic = x - d * kp;
            Hw[d * hs + mic] = (dw + d < a.dirs && warp * 8 + d < nd && mic < m) ? hb[(size_t)d * m + mic]
                                                                               : make_float2(0.f, 0.f);
        }
        __syncwarp();
        }
    compute:
        const float2* hrow = Hs + (warp * 8 + r) * hs + c;  // A[r][c] = h(dir r, mic k0 + c)
        double den = 0.0;
        // two passes of 4 vector tiles (32 accumulator registers each); the
        // second holds only zero padding when nn <= 32 (it would add 0.0)
        const int halves = nn > 32 ? 2 : 1;
#pragma unroll 1
        for (int half = 0; half < halves; ++half) {
            const double2* ecol = Es + (half * 32 + r) * es + c;  // B[c][r] = e(vector 8j + r, mic k0 + c)
            double re[4][2], im[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) re[j][0] = re[j][1] = im[j][0] = im[j][1] = 0.0;
            for (int k0 = 0; k0 < kp; k0 += 4) {
                const float2 hv = hrow[k0];
                const double hr = hv.x, hi = hv.y, nhi = -hi;
                double2 ev[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) ev[j] = ecol[j * 8 * es + k0];
                // 8 independent accumulators between two updates of the same one
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    dmma8x8x4(re[j][0], re[j][1], hr, ev[j].x);
                    dmma8x8x4(im[j][0], im[j][1], hr, ev[j].y);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    dmma8x8x4(re[j][0], re[j][1], hi, ev[j].y);
                    dmma8x8x4(im[j][0], im[j][1], nhi, ev[j].x);
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double mag = hypot(re[j][i], im[j][i]);  // 0 on padded vectors
                    den += a.squared ? mag * mag : mag;
                }
        }
        den += __shfl_xor_sync(0xffffffffu, den, 1);
        den += __shfl_xor_sync(0xffffffffu, den, 2);
        const int d = warp * 8 + r;
        if (c == 0 && d < nd) {
            if (den < a.floor_) den = a.floor_;
            const double num = a.num[(size_t)bin * a.dirs + d0 + d];
            a.p[(size_t)blkbin * a.dirs + d0 + d] = num / den;
        }
    }
}

// |h|^2 per (bin, dir) in the reference's order: sequential over mics,
// (re^2 + im^2) rounded once (both squares exact in double).
__global__ void steering_prep_kernel(const float2* __restrict__ h_in,  // [dirs][bins][m]
                                     float2* __restrict__ h_t,         // [bins][dirs][m]
                                     double* __restrict__ num, int m, int bins, int dirs) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)bins * dirs) return;
    const int b = (int)(idx / dirs), d = (int)(idx % dirs);
    const float2* src = h_in + ((size_t)d * bins + b) * m;
    float2* dst = h_t + ((size_t)b * dirs + d) * m;
    double acc = 0;
    for (int mic = 0; mic < m; ++mic) {
        const float2 v = src[mic];
        dst[mic] = v;
        const double re = v.x, im = v.y;
        acc = __dadd_rn(acc, __fma_rn(re, re, __dmul_rn(im, im)));
    }
    num[idx] = acc;
}

constexpr int kPeakThreads = 512;

__global__ void __launch_bounds__(kPeakThreads) integrate_peaks_kernel(PeakArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* pw = reinterpret_cast<double*>(smem_raw);              // [dirs]
    int* is_peak = reinterpret_cast<int*>(pw + a.dirs);            // [dirs]
    __shared__ double s_mean;
    const int blk = blockIdx.x;
    const int t = threadIdx.x;
    const double* pb = a.p + (size_t)blk * a.bins * a.dirs;
    // ascending-bin FP64 sum per direction (music.cpp:160)
    if (a.peak_chunk > 1) {
        // small grids: chunks of cb bins ([cb][dirs], contiguous in P) are
        // staged by the whole CTA with coalesced loads, then every
        // direction's running sum walks its column
        double* stage = reinterpret_cast<double*>(is_peak + a.dirs + (a.dirs & 1));  // [cb][dirs]
        const int cb = a.peak_chunk;
        for (int d = t; d < a.dirs; d += blockDim.x) pw[d] = 0.0;
        for (int b0 = 0; b0 < a.bins; b0 += cb) {
            const int nb = min(cb, a.bins - b0);
            __syncthreads();
            const double* src = pb + (size_t)b0 * a.dirs;
            // sixteen loads in flight per thread (a load-store loop through
            // generic pointers is serialized: one L2 round trip per element)
            const int n = nb * a.dirs;
            for (int x0 = t; x0 < n; x0 += 16 * blockDim.x) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int x = x0 + u * blockDim.x;
                    v[u] = x < n ? __ldg(src + x) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int x = x0 + u * blockDim.x;
                    if (x < n) stage[x] = v[u];
                }
            }
            __syncthreads();
            for (int d = t; d < a.dirs; d += blockDim.x) {
                double acc = pw[d];
                for (int u = 0; u < nb; ++u) acc = __dadd_rn(acc, stage[u * a.dirs + d]);
                pw[d] = acc;
            }
        }
    } else {
        // large grids: a thread per direction, 32 bins' loads in flight
        for (int d = t; d < a.dirs; d += blockDim.x) {
            double acc = 0.0;
            int b = 0;
            for (; b + 32 <= a.bins; b += 32) {
                double v[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) v[u] = __ldg(pb + (size_t)(b + u) * a.dirs + d);
#pragma unroll
                for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, v[u]);
            }
            for (; b < a.bins; ++b) acc = __dadd_rn(acc, pb[(size_t)b * a.dirs + d]);
            pw[d] = acc;
        }
    }
    for (int d = t; d < a.dirs; d += blockDim.x) a.power[(size_t)blk * a.dirs + d] = pw[d];
    __syncthreads();
    if (t == 0) {
        double mean = 0;
        for (int d = 0; d < a.dirs; ++d) mean = __dadd_rn(mean, pw[d]);
        if (a.dirs) mean = __ddiv_rn(mean, (double)a.dirs);
        s_mean = mean;
    }
    for (int d = t; d < a.dirs; d += blockDim.x) {
        // local-maximum test over the CSR neighbor list, 8 neighbor indices
        // loaded together per step (the list lives in global memory)
        const double v = pw[d];
        const uint32_t k1 = a.nbr_off[d + 1];
        int ok = 1;
        for (uint32_t k = a.nbr_off[d]; k < k1 && ok; k += 8) {
            uint32_t nb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) nb[u] = k + u < k1 ? a.nbr[k + u] : (uint32_t)d;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v < pw[nb[u]]) ok = 0;
        }
        is_peak[d] = ok;
    }
    __syncthreads();
    if (t < 32) {
        // insertion into a bounded list ordered by (power desc, index asc);
        // peaks are visited in index order, so equal powers keep index order.
        // Warp 0 finds the peak directions 32 at a time by ballot; lane 0
        // inserts them.
        uint32_t best[64];
        int nb = 0;
        const int cap = a.ns < 64 ? a.ns : 64;
        for (int d0 = 0; d0 < a.dirs; d0 += 32) {
            unsigned bal = __ballot_sync(0xffffffffu, d0 + t < a.dirs && is_peak[d0 + t]);
            if (t != 0) continue;
            for (; bal; bal &= bal - 1) {
            const int d = d0 + __ffs(bal) - 1;
            const double v = pw[d];
            int pos = nb;
            while (pos > 0 && v > pw[best[pos - 1]]) --pos;
            if (pos >= cap) continue;
            const int last = nb < cap ? nb : cap - 1;
            for (int k = last; k > pos; --k) best[k] = best[k - 1];
            best[pos] = (uint32_t)d;
            if (nb < cap) ++nb;
            }
        }
        if (t != 0) return;
        const double thr = a.low_ratio * s_mean;
        for (int k = 0; k < nb; ++k) {
            a.est_idx[(size_t)blk * a.ns + k] = best[k];
            a.est_pw[(size_t)blk * a.ns + k] = pw[best[k]];
            a.est_low[(size_t)blk * a.ns + k] = pw[best[k]] < thr ? 1 : 0;
        }
        for (int k = nb; k < a.ns; ++k) {  // unused slots: no estimate
            a.est_idx[(size_t)blk * a.ns + k] = 0xffffffffu;
            a.est_pw[(size_t)blk * a.ns + k] = 0.0;
            a.est_low[(size_t)blk * a.ns + k] = 0;
        }
        a.est_count[blk] = (uint32_t)nb;
    }
}

void spectrum_shape(int m, int ns, int dirs, int& dchunk, int& nsplit, size_t& smem) {
    dchunk = dirs < 128 ? dirs : 128;
    nsplit = kSpecThreads / dchunk;
    const int nn = m - ns;
    const int max_split = (nn + kSpecVec - 1) / kSpecVec;
    if (nsplit > max_split) nsplit = max_split;
    if (nsplit < 1) nsplit = 1;
    smem = (size_t)nn * m * sizeof(double2) + (size_t)m * dchunk * sizeof(float2) +
           (size_t)nsplit * dchunk * sizeof(double);
}

void launch_spectrum(SpecArgs a, int nblk, cudaStream_t s) {
    if (a.m - a.ns <= kMmaN && a.m - a.ns >= 16) {  // FP64 tensor cores (m = 16, Ns = 2 on them: 181 vs 130 us per C2 launch)
        auto mma = [&](auto kern, int wpc) {
            const int chunk = 8 * wpc;
            const size_t smem2 = (size_t)kMmaN * mma_estride(a.m) * sizeof(double2) +
                                 (size_t)chunk * mma_hstride(a.m) * sizeof(float2);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
            kern<<<nblk * a.bins, 32 * wpc, smem2, s>>>(a, nblk);
        };
        if (a.dirs % 72 == 0) mma(spectrum_mma_kernel<9>, 9);
        else mma(spectrum_mma_kernel<8>, 8);
        return;
    }
    if (a.m <= 8) {  // the smallest arrays: a warp per (block, bin) (C2's m = 16 measured slower: 170 vs 133 us)
        const int nbb = nblk * a.bins;
        const size_t smemw = (size_t)kSpecWarps * (a.m - a.ns) * a.m * sizeof(double2);
        cudaFuncSetAttribute(spectrum_warp_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemw);
        spectrum_warp_kernel<8><<<(nbb + kSpecWarps - 1) / kSpecWarps, 32 * kSpecWarps, smemw, s>>>(a, nbb);
        return;
    }
    size_t smem;
    spectrum_shape(a.m, a.ns, a.dirs, a.dchunk, a.nsplit, smem);
    cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nblk * a.bins, (a.dirs + a.dchunk - 1) / a.dchunk);
    spectrum_kernel<<<grid, kSpecThreads, smem, s>>>(a);
}

void launch_steering_prep(const float2* h_in, float2* h_t, double* num, int m, int bins, int dirs,
                          cudaStream_t s) {
    const size_t n = (size_t)bins * dirs;
    steering_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h_in, h_t, num, m, bins, dirs);
}

void launch_peaks(PeakArgs a, int nblk, cudaStream_t s) {
    // small grids stage up to 160 KB of P per pass (the whole block at D = 72:
    // one memory latency instead of four), in chunks of >= 16 bins; large
    // grids read directly
    a.peak_chunk = (int)(163840 / ((size_t)a.dirs * sizeof(double)));
    if (a.peak_chunk < 16) a.peak_chunk = 1;
    if (a.peak_chunk > a.bins) a.peak_chunk = a.bins;
    const size_t smem = (size_t)a.dirs * sizeof(double) + (size_t)(a.dirs + (a.dirs & 1)) * sizeof(int) +
                        (size_t)a.peak_chunk * a.dirs * sizeof(double);
    cudaFuncSetAttribute(integrate_peaks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    integrate_peaks_kernel<<<nblk, kPeakThreads, smem, s>>>(a);
}

}  // namespace sslg
