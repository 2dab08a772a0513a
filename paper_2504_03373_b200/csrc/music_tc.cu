// MUSIC spectrum of large direction grids on the 5th-generation tensor cores
// (calc_average_power, reference music.cpp:112-165):
//
//   P(theta, w) = |h|^2 / max(floor, sum_{i >= Ns} |h^H e_i|)
//
// per (block, bin) is a complex GEMM of the steering rows [D x M] against the
// noise vectors [M x (M - Ns)].  As one real GEMM C = A B^T with K = 2M:
//   A[d] = [Re h_d, Im h_d]                                      (D x 2M)
//   B[2n] = [Re e_n, Im e_n],  B[2n + 1] = [Im e_n, -Re e_n]     (2(M - Ns) x 2M)
//   C[d][2n] = Re(h^H e_n),  C[d][2n + 1] = Im(h^H e_n)
// on tcgen05.mma kind::tf32 with the 3-pass split x = hi + lo (hi = tf32(x),
// lo = tf32(x - hi)): C = A_hi B_hi + (A_hi B_lo + A_lo B_hi), the main
// products and the ~2^-11 smaller corrections in two separate FP32 TMEM
// accumulators (the tensor core aligns the products of one accumulation to
// the largest; summed together the corrections would lose their low bits),
// added in FP32 in the epilogue.  The steering is FP32-stored (as in the reference) and the FP64
// noise vectors are rounded to FP32.  Measured against the FP64 spectrum on
// every bin of 5 C4 blocks (tests/test_gpu_spectrum_tc.py): <= 5.6e-7
// relative per bin, <= 2.8e-7 on the broadband power, identical peaks
// (with one accumulator for all three passes: 1.5e-6 / 8.2e-7); every direction runs the identical MMA sequence, so bit-identical
// steering rows (the az x el grid's pole rows) keep bit-identical powers.
//
// One CTA per (bin, block) -- blocks of a bin adjacent, so its steering stays
// in L2 -- walks every 128-direction tile of the grid:
//   * the steering operand is prepared once per grid (spectrum_tc_prep_kernel:
//     tf32 hi/lo in the UMMA core-matrix layout, one 40 KB slab per (bin,
//     tile, K phase)), so each slab reaches shared memory as ONE bulk copy
//     (cp.async.bulk, TMA engine) into a two-stage ring;
//   * the noise-vector operand B (all of K, 120 KB) is built once per CTA
//     from the bulk-copied FP64 vectors;
//   * warp 8 lane 0 issues the copies and the MMAs (single-thread tcgen05.mma
//     issue), tcgen05.commit releases ring stages and publishes each tile's
//     accumulators; two accumulator pairs (2 x 2 x 128 columns) let warps 0-7 run a
//     tile's epilogue (tcgen05.ld -> |.| -> FP64 row sum -> P) while the
//     next tile's MMAs run.
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

namespace {

constexpr int kTcRows = 128;   // UMMA M: directions per tile
constexpr int kTcN = 128;      // UMMA N: 2 (M - Ns), padded
constexpr int kTcKP = 40;      // K per steering slab (5 MMAs of K = 8)
constexpr int kTcChunks = kTcKP / 4;            // 16-byte K chunks per slab
constexpr int kTcOp = kTcChunks * kTcRows * 4;  // floats of one operand slab
constexpr int kTcSlab = 2 * kTcOp;              // hi + lo
constexpr int kTcStages = 2;
constexpr int kTcEpiWarps = 8;   // two warps per TMEM lane quarter, one per half of the columns
constexpr int kTcThreads = 32 * (kTcEpiWarps + 1);  // + the MMA warp

__host__ __device__ constexpr int tc_phases(int m) { return (2 * m + kTcKP - 1) / kTcKP; }
// shared memory: B (hi, lo; every phase) + the steering ring
__host__ __device__ constexpr size_t tc_smem(int m) {
    return ((size_t)2 * tc_phases(m) * kTcOp + (size_t)kTcStages * kTcSlab) * sizeof(float);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// UMMA shared-memory descriptor, K-major, no swizzle (version 1, legacy LBO
// mode): 8-row x 16-byte core matrices, 16 B between rows of a core matrix,
// SBO between 8-row groups, LBO between the two K halves of one MMA.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;                // base offset 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor: D f32, A/B tf32, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t tf32_idesc(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
}

__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// 4 consecutive K values of operand row r (K chunk kc) as tf32 hi and lo parts
__device__ __forceinline__ void put_split4(float* hi, float* lo, int r, int kc, const float (&x)[4]) {
    float4 h, l;
    h.x = tf32_rna(x[0]);
    h.y = tf32_rna(x[1]);
    h.z = tf32_rna(x[2]);
    h.w = tf32_rna(x[3]);
    l.x = tf32_rna(x[0] - h.x);
    l.y = tf32_rna(x[1] - h.y);
    l.z = tf32_rna(x[2] - h.z);
    l.w = tf32_rna(x[3] - h.w);
    const int off = (kc * kTcRows + r) * 4;
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
}

}  // namespace

// Steering slabs [bin][tile][phase]{hi, lo}[chunk][row][4]: row = direction
// tile*128 + row, K index k = phase*40 + 4 chunk + q -> Re h[k] (k < m),
// Im h[k - m] (m <= k < 2m), zero beyond the grid / past 2m.
__global__ void spectrum_tc_prep_kernel(const float2* __restrict__ h, int m, int bins, int dirs,
                                        float* __restrict__ out) {
    const int ntiles = (dirs + kTcRows - 1) / kTcRows, nph = tc_phases(m);
    const size_t total = (size_t)bins * ntiles * nph * kTcChunks * kTcRows;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int row = (int)(i % kTcRows);
        const int kc = (int)((i / kTcRows) % kTcChunks);
        const size_t slab = i / ((size_t)kTcRows * kTcChunks);  // (bin, tile, phase)
        const int ph = (int)(slab % nph), tile = (int)((slab / nph) % ntiles), bin = (int)(slab / nph / ntiles);
        const int d = tile * kTcRows + row;
        float x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = ph * kTcKP + 4 * kc + q;
            x[q] = 0.f;
            if (d < dirs && k < 2 * m) {
                const float2 v = h[((size_t)bin * dirs + d) * m + (k < m ? k : k - m)];
                x[q] = k < m ? v.x : v.y;
            }
        }
        float* base = out + slab * kTcSlab;
        put_split4(base, base + kTcOp, row, kc, x);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) spectrum_tc_kernel(SpecArgs a, const float* __restrict__ hs,
                                                                    int nblk) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int m = a.m, nn = m - a.ns;
    const int nph = tc_phases(m);
    const int ntiles = (a.dirs + kTcRows - 1) / kTcRows;
    float* B_hi = reinterpret_cast<float*>(smem_raw);  // [phase][chunk][row][4]
    float* B_lo = B_hi + nph * kTcOp;
    float* ring = B_lo + nph * kTcOp;  // [stage]{hi, lo}
    __shared__ uint64_t full[kTcStages], empty[kTcStages], accfull[2], accempty[2], ebar;
    __shared__ uint32_t s_tmem;
    __shared__ double s_den[2][kTcRows];  // column-half partial sums of a tile's rows

    const int bin = blockIdx.x / nblk, blk = blockIdx.x % nblk;
    const int blkbin = blk * a.bins + bin;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const float* hs_bin = hs + (size_t)bin * ntiles * nph * kTcSlab;

    const int mma_warp = kTcEpiWarps;
    if (warp == mma_warp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                     "n"(4 * kTcN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            bar_init(&accfull[b], 1);
            bar_init(&accempty[b], 32 * kTcEpiWarps);
        }
        bar_init(&ebar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;

    // the noise vectors [nn][m] cf64 land in the ring by one bulk copy, and
    // are turned into the B operand (every K phase) by all threads
    const double2* eb = a.e + ((size_t)blkbin * m + a.ns) * m;
    const uint32_t ebytes = (uint32_t)((size_t)nn * m * sizeof(double2));
    if (t == 0) {
        bar_expect_tx(&ebar, ebytes);
        bulk_copy(ring, eb, ebytes, &ebar);
    }
    bar_wait(&ebar, 0);
    {
        const double2* es = reinterpret_cast<const double2*>(ring);
        // lanes over operand rows (16-byte stores to consecutive slots), warps
        // over K chunks
        for (int idx = t; idx < kTcN * nph * kTcChunks; idx += kTcThreads) {
            const int n = idx % kTcN, kc = idx / kTcN;
            const int j = n >> 1;
            const bool im = n & 1, used = j < nn;
            {
                float x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = 4 * kc + q;
                    x[q] = 0.f;
                    if (used && k < 2 * m) {
                        const double2 e = es[(size_t)j * m + (k < m ? k : k - m)];
                        // [Re e, Im e] for the real column, [Im e, -Re e] for the imaginary one
                        x[q] = k < m ? (float)(im ? e.y : e.x) : (float)(im ? -e.x : e.y);
                    }
                }
                const int ph = kc / kTcChunks, c = kc % kTcChunks;
                put_split4(B_hi + ph * kTcOp, B_lo + ph * kTcOp, n, c, x);
            }
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> async proxy
    __syncthreads();  // B built; the ring is free for the steering slabs

    const uint32_t idesc = tf32_idesc(kTcRows, kTcN);
    const uint32_t lbo = kTcRows * 16, sbo = 128;
    if (warp == mma_warp) {
        if (lane == 0) {
            // producer + MMA issuer: slab i = (tile i / nph, phase i % nph) into stage i % 2
            const int nslab = ntiles * nph;
            const uint32_t slab_bytes = (uint32_t)(kTcSlab * sizeof(float));
            for (int i = 0; i < kTcStages && i < nslab; ++i) {
                bar_expect_tx(&full[i], slab_bytes);
                bulk_copy(ring + i * kTcSlab, hs_bin + (size_t)i * kTcSlab, slab_bytes, &full[i]);
            }
            for (int i = 0; i < nslab; ++i) {
                const int s = i % kTcStages, tile = i / nph, ph = i % nph;
                const int acc = tile & 1;
                if (ph == 0 && tile >= 2) bar_wait(&accempty[acc], (uint32_t)((tile / 2 - 1) & 1));
                bar_wait(&full[s], (uint32_t)((i / kTcStages) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const float* a_hi = ring + s * kTcSlab;
                const float* a_lo = a_hi + kTcOp;
                const uint32_t d = tmem + (uint32_t)(acc * 2 * kTcN);  // main; corrections at d + kTcN
                for (int st = 0; st < kTcKP / 8; ++st) {
                    const uint32_t off = (uint32_t)st * 2 * kTcRows * 16;
                    const uint64_t ah = umma_desc(smem_addr(a_hi) + off, lbo, sbo);
                    const uint64_t al = umma_desc(smem_addr(a_lo) + off, lbo, sbo);
                    const uint64_t bh = umma_desc(smem_addr(B_hi + ph * kTcOp) + off, lbo, sbo);
                    const uint64_t bl = umma_desc(smem_addr(B_lo + ph * kTcOp) + off, lbo, sbo);
                    mma_tf32(d, ah, bh, idesc, (ph | st) ? 1u : 0u);
                    mma_tf32(d + kTcN, ah, bl, idesc, (ph | st) ? 1u : 0u);
                    mma_tf32(d + kTcN, al, bh, idesc, 1u);
                }
                mma_commit(&empty[s]);                         // stage s refillable once these MMAs are done
                if (ph == nph - 1) mma_commit(&accfull[acc]);  // the tile's accumulator is complete
                // refill the PREVIOUS slab's stage with slab i + 1: its MMAs finish
                // while this slab's are queued, so the tensor pipe never drains
                const int nx = i + 1;
                if (i >= 1 && nx < nslab) {
                    const int sp = (i - 1) % kTcStages;
                    bar_wait(&empty[sp], (uint32_t)(((i - 1) / kTcStages) & 1));
                    bar_expect_tx(&full[sp], slab_bytes);
                    bulk_copy(ring + sp * kTcSlab, hs_bin + (size_t)nx * kTcSlab, slab_bytes, &full[sp]);
                }
            }
        }
        __syncwarp();
    } else {
        // epilogue: warps w and w + 4 own TMEM lanes 32(w % 4).. (direction
        // rows), each one half of the 128 columns (32 complex products)
        const int q4 = warp & 3, half = warp >> 2;
        const int row = 32 * q4 + lane;
        const uint32_t lane_base = (uint32_t)(32 * q4) << 16;
        for (int tile = 0; tile < ntiles; ++tile) {
            const int acc = tile & 1;
            bar_wait(&accfull[acc], (uint32_t)((tile / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t trow = tmem + lane_base + (uint32_t)(acc * 2 * kTcN + 64 * half);
            // four independent FP64 partial sums (no 57-long dependent chain)
            double dp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
                uint32_t v[16], w[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15])
                    : "r"(trow + (uint32_t)c0));
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];"
                    : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                      "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
                      "=r"(w[14]), "=r"(w[15])
                    : "r"(trow + (uint32_t)(kTcN + c0)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int j0 = 32 * half + c0 / 2;  // first noise vector of this load
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    // h^H e = main + correction; |.| in FP32 (the products carry
                    // ~1e-7 already); two magnitudes added in FP32 (one more
                    // 2^-24 relative rounding) before each FP64 accumulation:
                    // the FP64 pipe is this epilogue's throttle
                    float mg[2];
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const float re = __uint_as_float(v[2 * (q + r)]) + __uint_as_float(w[2 * (q + r)]);
                        const float im = __uint_as_float(v[2 * (q + r) + 1]) + __uint_as_float(w[2 * (q + r) + 1]);
                        const float s2 = fmaf(re, re, im * im);
                        const float mag = a.squared ? s2 : sqrtf(s2);
                        mg[r] = j0 + q + r < nn ? mag : 0.0f;
                    }
                    dp[q >> 1] += (double)(mg[0] + mg[1]);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            bar_arrive(&accempty[acc]);  // the accumulator may be overwritten by tile + 2
            s_den[half][row] = (dp[0] + dp[1]) + (dp[2] + dp[3]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcEpiWarps));  // the epilogue warps only
            const int d = tile * kTcRows + row;
            if (half == 0 && d < a.dirs) {
                double den = s_den[0][row] + s_den[1][row];
                if (den < a.floor_) den = a.floor_;
                a.p[(size_t)blkbin * a.dirs + d] = a.num[(size_t)bin * a.dirs + d] / den;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcEpiWarps));  // s_den is reused by the next tile
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == mma_warp) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(4 * kTcN));
    }
}

bool spectrum_tc_supported(const SpecArgs& a) {
    return a.m <= 64 && 2 * (a.m - a.ns) <= kTcN &&
           (size_t)(a.m - a.ns) * a.m * 16 <= (size_t)kTcStages * kTcSlab * sizeof(float) &&
           tc_smem(a.m) <= 227 * 1024;
}

size_t spectrum_tc_slab_floats(int m, int bins, int dirs) {
    return (size_t)bins * ((dirs + kTcRows - 1) / kTcRows) * tc_phases(m) * kTcSlab;
}

void launch_spectrum_tc_prep(const float2* h_t, int m, int bins, int dirs, float* slabs, cudaStream_t s) {
    spectrum_tc_prep_kernel<<<148 * 8, 256, 0, s>>>(h_t, m, bins, dirs, slabs);
}

void launch_spectrum_tc(const SpecArgs& a, const float* slabs, int nblk, cudaStream_t s) {
    const size_t smem = tc_smem(a.m);
    cudaFuncSetAttribute(spectrum_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    spectrum_tc_kernel<<<nblk * a.bins, kTcThreads, smem, s>>>(a, slabs, nblk);
}

}  // namespace sslg
