// Kernel (2): batched complex GSVD, one CTA per (block, frequency bin).
//
//   A = K^-1 R                    (gsvd.cpp:596 / 702, FP64)
//   one-sided Jacobi on A         (jacobi_svd, gsvd.cpp:622-695)
//   sigma_j = |w_j|, u_j = w_j / sigma_j, stable descending order
//   canonical bases for vanishing / tied groups + phase rule
//                                 (canonicalize_subspaces, gsvd.cpp:470-565)
//
// The solver is the reference's FP64 oracle algorithm (gsvd_reference),
// organized for the GPU:
//  * the Jacobi pairs of a sweep follow the round-robin (circle) ordering, so
//    the M/2 disjoint pairs of a round rotate concurrently, one 8-lane group
//    per pair, inner products reduced with group-masked shuffles;
//  * W = A V lives in shared memory (M x M complex double, column-major);
//  * rotation angle, skip tests (drop 1e-20 max|w|^2, |a_pq|^2 <= 1e-28
//    |w_p|^2 |w_q|^2), convergence (a sweep without rotations) and the
//    60-sweep cap are the reference's;
//  * canonicalization runs fused in the epilogue whenever the converged W is
//    an orthonormal basis (every column survived the drop rule, so the final
//    sweep certified all pairs orthogonal): the canonical vectors of a group
//    with span N are N z, and the reference's picker (candidates P e_j in
//    index order, thresholds {0.05, 1e-8, 0}) runs on the coordinates
//    z_j = N^H e_j — the same vectors the reference builds in the full
//    space, at O(M d^2) cost for a d-dimensional group.  Other bins (and
//    refine_leading mode) are flagged for the generic kernel (canonical.cu).
//
// Outputs per (block, bin): sigma [M] descending, E [M vectors][M rows]
// (vector-major: the [bin][vector][mic] gather of music.cpp:127-135), sweeps,
// convergence flag, and the generic-canonicalization flag.
#include "common.cuh"
#include "kernels.cuh"
#include "whiten.cuh"
#include "jacobi_rot.cuh"

namespace sslg {

#ifndef SSLG_JAC_LPP
#define SSLG_JAC_LPP 8
#endif
constexpr int kLPP = SSLG_JAC_LPP;   // lanes per column pair
constexpr int kJacThreads = 32 * kLPP;  // 32 column-pair groups
// small arrays (m <= 16: at most 8 pairs) run 64-thread CTAs with a scratch
// sized for them, so several bins share an SM instead of one CTA idling 3/4
template <int MC>
constexpr int jac_threads() { return (MC > 0 && MC <= 16) ? 64 : kJacThreads; }
constexpr int kRows = kMaxM / kLPP;  // rows per lane (8)
constexpr double kReorth = 1e-5;  // re-orthonormalization line (relative to sigma_max)
constexpr int kZMax = 28;            // largest group handled by the fused picker
constexpr int kYld = kZMax + 1;      // padded row stride of the coordinate buffer
// scratch after W: picker coordinates, C^H D products and the packed D^H D
constexpr int kScratch = kMaxM * (kMaxM + 1) / 2 > kMaxM * kYld ? kMaxM * (kMaxM + 1) / 2 : kMaxM * kYld;
// scratch entries for a compile-time channel count (0: any m <= 64): the
// packed Cholesky (m(m+1)/2), the sequential picker's rows (m kYld) and the
// concurrent pickers' G and Z slices (<= 2 m^2 for m <= 16)
constexpr int cmax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
__host__ __device__ constexpr int scratch_entries(int mc) {
    return (mc > 0 && mc <= 16) ? cmax3(mc * (mc + 1) / 2, mc * kYld, 2 * mc * mc) : kScratch;
}

// Per-CTA canonicalization state, sized for the channel count (MM) and the
// largest group the coordinate-space picker takes (ZM): small arrays keep
// their static shared memory small so more bins share an SM.
template <int MM, int ZM>
struct CanonScratchT {
    double nrm[MM];
    double norm0[MM];
    double2 q[ZM];
    double2 z[ZM][ZM];  // accepted coordinate vectors, column t = vector t
    int cols[MM];       // W columns of the current group
    int groups[MM][2];  // rank ranges of tied groups
    double2 up[MM];     // phase factor per rank
    unsigned ball[2];
    int dropped[MM];    // columns below the final sweep's drop line
    int certcols[MM];   // certified columns
    double invd[MM];    // 1 / L_jj of the CholeskyQR (column norms before it)
    double dn2[MM];     // column norms after the first projection
    int ngroups, nvanish, eligible, ndropped, ncert, collapsed, again;
};
template <int MC>
using CanonScratchFor = CanonScratchT<(MC > 0 ? MC : kMaxM), (MC > 0 && MC < kZMax ? MC : kZMax)>;

// C = op(A) B on the FP64 tensor cores (DMMA m8n8k4) over 8x8 complex tiles,
// warps round-robin over the tiles; fa(i, k) and fb(k, j) return the operand
// entries (zero outside M x K / K x N), conj(A) when CONJ; fc(i, j, v) takes
// each result.  Used for the basis-completion projections of the split
// solver's epilogue.
template <bool CONJ, class FA, class FB, class FC>
__device__ __forceinline__ void cgemm_tiles_mma(int M, int N, int K, FA fa, FB fb, FC fc) {
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, r = lane >> 2, c = lane & 3;
    const int tm = (M + 7) >> 3, tn = (N + 7) >> 3;
    for (int tile = warp; tile < tm * tn; tile += blockDim.x >> 5) {
        const int i0 = (tile / tn) * 8, j0 = (tile % tn) * 8;
        double re0 = 0, re1 = 0, im0 = 0, im1 = 0;
        for (int k0 = 0; k0 < K; k0 += 4) {
            const double2 av = fa(i0 + r, k0 + c);
            const double2 bv = fb(k0 + c, j0 + r);
            const double ai = CONJ ? -av.y : av.y;
            dmma_8x8x4(re0, re1, av.x, bv.x);
            dmma_8x8x4(im0, im1, av.x, bv.y);
            dmma_8x8x4(re0, re1, -ai, bv.y);
            dmma_8x8x4(im0, im1, ai, bv.x);
        }
        fc(i0 + r, j0 + 2 * c, make_double2(re0, im0));
        fc(i0 + r, j0 + 2 * c + 1, make_double2(re1, im1));
    }
}

// Completes the basis: the columns below the drop line (list D, rank order)
// are orthonormalized against the certified columns C and then among
// themselves.  Block form: D -= C (C^H D) (Gram product in the scratch G,
// |C||D| <= m^2/4 entries), repeated only where the first pass removed more
// than half of a column's energy, then CholeskyQR2 of D (the rank-order
// Gram-Schmidt result).  Clears cs.eligible if a column collapses.
template <int MC, bool MMA = false>
__device__ void complete_basis(double2* W, double2* G, int m_rt, CanonScratchFor<MC>& cs) {
    const int m = MC > 0 ? MC : m_rt;
    const int t = threadIdx.x, nt = blockDim.x;
    const int nc = cs.ncert, nd = cs.ndropped;
    if (t == 0) cs.collapsed = 0;  // published by the first barrier below
    // squared norms of the D columns (four lanes per column, nd <= 64)
    auto dnorms = [&](double* out) {
        const int part = t & 3;
        for (int b0 = 0; b0 < nd; b0 += nt / 4) {
            const int b = b0 + (t >> 2);
            double v = 0;
            if (b < nd) {
                const double2* wd = W + cs.dropped[b] * m;
                for (int i = part; i < m; i += 4) v = fma(wd[i].x, wd[i].x, fma(wd[i].y, wd[i].y, v));
            }
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (b < nd && part == 0) out[b] = v;
        }
    };
    dnorms(cs.invd);
    for (int pass = 0; pass < 2; ++pass) {
      if constexpr (MMA) {
        // G = C^H D and D -= C G on the tensor cores
        cgemm_tiles_mma<true>(
            nc, nd, m,
            [&](int a, int k) { return (a < nc && k < m) ? W[cs.certcols[a] * m + k] : make_double2(0, 0); },
            [&](int k, int b) { return (k < m && b < nd) ? W[cs.dropped[b] * m + k] : make_double2(0, 0); },
            [&](int a, int b, double2 v) {
                if (a < nc && b < nd) G[a * nd + b] = v;
            });
        __syncthreads();
        cgemm_tiles_mma<false>(
            m, nd, nc,
            [&](int i, int a) { return (i < m && a < nc) ? W[cs.certcols[a] * m + i] : make_double2(0, 0); },
            [&](int a, int b) { return (a < nc && b < nd) ? G[a * nd + b] : make_double2(0, 0); },
            [&](int i, int b, double2 v) {
                if (i < m && b < nd) {
                    double2* w = W + cs.dropped[b] * m + i;
                    *w = csub(*w, v);
                }
            });
        __syncthreads();
      } else {
        // G[a][b] = e_C[a]^H w_D[b], four lanes per product
        for (int e0 = 0; e0 < nc * nd; e0 += nt / 4) {
            const int e = e0 + (t >> 2), part = t & 3;
            double2 d = make_double2(0, 0);
            if (e < nc * nd) {
                const double2* ec = W + cs.certcols[e / nd] * m;
                const double2* wd = W + cs.dropped[e % nd] * m;
                for (int i = part; i < m; i += 4) {
                    const double2 a = ec[i], b = wd[i];
                    d.x = fma(a.x, b.x, fma(a.y, b.y, d.x));
                    d.y = fma(a.x, b.y, fma(-a.y, b.x, d.y));
                }
            }
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 1);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 1);
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 2);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 2);
            if (e < nc * nd && (t & 3) == 0) G[e] = d;
        }
        __syncthreads();
        // w_D[b][i] -= sum_a G[a][b] e_C[a][i]  (four independent partial sums)
        for (int o = t; o < nd * m; o += nt) {
            const int b = o / m, i = o % m;
            double2 acc[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
            int a = 0;
            for (; a + 4 <= nc; a += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double2 g = G[(a + u) * nd + b], ev = W[cs.certcols[a + u] * m + i];
                    acc[u].x = fma(g.x, ev.x, fma(-g.y, ev.y, acc[u].x));
                    acc[u].y = fma(g.x, ev.y, fma(g.y, ev.x, acc[u].y));
                }
            }
            for (; a < nc; ++a) {
                const double2 g = G[a * nd + b], ev = W[cs.certcols[a] * m + i];
                acc[0].x = fma(g.x, ev.x, fma(-g.y, ev.y, acc[0].x));
                acc[0].y = fma(g.x, ev.y, fma(g.y, ev.x, acc[0].y));
            }
            double2* w = W + cs.dropped[b] * m + i;
            *w = csub(*w, cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])));
        }
        __syncthreads();
      }
        if (pass == 0) {
            // "twice is enough" (Kahan): a second projection is needed only
            // where the first removed more than half of a column's energy
            dnorms(cs.dn2);
            __syncthreads();
            bool again = false;
            for (int b = t; b < nd; b += nt) again |= cs.dn2[b] < 0.5 * cs.invd[b];
            if (!__syncthreads_or(again)) break;
        }
    }
    // D <- D L^-H with D^H D = L L^H (CholeskyQR, twice): the Q factor of D
    // in rank order, i.e. the Gram-Schmidt result; L_jj is the norm of column
    // j after projection against the earlier ones (collapse test).
    double* invd = cs.invd;
    for (int pass = 0; pass < 2; ++pass) {
        // packed lower Gram G[i(i+1)/2 + k] = d_i^H d_k, k <= i
        const int np = nd * (nd + 1) / 2;
        if constexpr (MMA) {
            cgemm_tiles_mma<true>(
                nd, nd, m,
                [&](int i, int r) { return (i < nd && r < m) ? W[cs.dropped[i] * m + r] : make_double2(0, 0); },
                [&](int r, int k) { return (r < m && k < nd) ? W[cs.dropped[k] * m + r] : make_double2(0, 0); },
                [&](int i, int k, double2 v) {
                    if (i < nd && k <= i) G[i * (i + 1) / 2 + k] = v;
                });
        } else
        for (int e0 = 0; e0 < np; e0 += nt / 4) {
            const int e = e0 + (t >> 2), part = t & 3;
            double2 d = make_double2(0, 0);
            if (e < np) {
                int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
                while (i * (i + 1) / 2 > e) --i;
                while ((i + 1) * (i + 2) / 2 <= e) ++i;
                const int k = e - i * (i + 1) / 2;
                const double2* di = W + cs.dropped[i] * m;
                const double2* dk = W + cs.dropped[k] * m;
                for (int r = part; r < m; r += 4) {
                    const double2 a = di[r], b = dk[r];
                    d.x = fma(a.x, b.x, fma(a.y, b.y, d.x));
                    d.y = fma(a.x, b.y, fma(-a.y, b.x, d.y));
                }
            }
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 1);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 1);
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 2);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 2);
            if (e < np && (t & 3) == 0) G[e] = d;
        }
        __syncthreads();
        if constexpr (MMA) {
            // right-looking Cholesky over the whole CTA (the split solver's
            // epilogue has no co-resident sweeps to hide a one-warp chain):
            // two barriers per column, the trailing triangle flattened over
            // every thread; per entry the same operations as the warp form
            __syncthreads();
            for (int j = 0; j < nd; ++j) {
                const double gjj = G[j * (j + 1) / 2 + j].x;
                if (!(gjj > 1e-12)) {  // projected norm <= 1e-6: collapsed (uniform)
                    if (t == 0) {
                        cs.eligible = 0;
                        cs.collapsed = 1;
                    }
                    break;
                }
                const double inv = fast_rsqrt(gjj);
                for (int i = j + 1 + t; i < nd; i += nt) {
                    double2& gij = G[i * (i + 1) / 2 + j];
                    gij = cscale(inv, gij);
                }
                if (t == 0) invd[j] = inv;
                __syncthreads();
                const int n = nd - j - 1;
                for (int e = t; e < n * (n + 1) / 2; e += nt) {
                    int ii = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
                    while (ii * (ii + 1) / 2 > e) --ii;
                    while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
                    const int i = j + 1 + ii, k = j + 1 + (e - ii * (ii + 1) / 2);
                    const double2 lij = G[i * (i + 1) / 2 + j], lkj = G[k * (k + 1) / 2 + j];
                    double2& gik = G[i * (i + 1) / 2 + k];
                    gik.x -= fma(lij.x, lkj.x, lij.y * lkj.y);
                    gik.y -= fma(lij.y, lkj.x, -lij.x * lkj.y);
                }
                __syncthreads();
            }
            if (t == 0 && !cs.collapsed) {
                double lo = invd[0], hi = invd[0];
                for (int j = 1; j < nd; ++j) {
                    lo = fmin(lo, invd[j]);
                    hi = fmax(hi, invd[j]);
                }
                cs.again = hi <= 100.0 * lo ? 0 : 1;
            }
        } else if (t < kWarp) {  // right-looking Cholesky, one warp
            for (int j = 0; j < nd; ++j) {
                const double gjj = G[j * (j + 1) / 2 + j].x;
                if (!(gjj > 1e-12)) {  // projected norm <= 1e-6: collapsed
                    if (t == 0) {
                        cs.eligible = 0;
                        cs.collapsed = 1;
                    }
                    break;
                }
                const double inv = fast_rsqrt(gjj);
                for (int i = j + 1 + t; i < nd; i += kWarp) {
                    double2& gij = G[i * (i + 1) / 2 + j];
                    gij = cscale(inv, gij);
                }
                __syncwarp();
                // trailing lower triangle, one (i, k) entry per lane at a time
                const int n = nd - j - 1;
                for (int e = t; e < n * n; e += kWarp) {
                    const int i = j + 1 + e / n, k = j + 1 + e % n;
                    if (k > i) continue;
                    const double2 lij = G[i * (i + 1) / 2 + j], lkj = G[k * (k + 1) / 2 + j];
                    double2& gik = G[i * (i + 1) / 2 + k];
                    gik.x -= fma(lij.x, lkj.x, lij.y * lkj.y);
                    gik.y -= fma(lij.y, lkj.x, -lij.x * lkj.y);
                }
                if (t == 0) invd[j] = inv;
                __syncwarp();
            }
            if (t == 0 && !cs.collapsed) {
                // CholeskyQR loses orthogonality like eps kappa(D)^2; with the
                // Cholesky diagonal spread (a lower bound on kappa) below 100 the
                // first pass is already orthonormal to ~1e-12 and the second is
                // skipped
                double lo = invd[0], hi = invd[0];
                for (int j = 1; j < nd; ++j) {
                    lo = fmin(lo, invd[j]);
                    hi = fmax(hi, invd[j]);
                }
                cs.again = hi <= 100.0 * lo ? 0 : 1;
            }
        }
        __syncthreads();
        if (cs.collapsed) return;  // uniform: written before the barrier above
        // row solve q_rb = (d_rb - sum_{a<b} q_ra conj(L_ba)) / L_bb
        if constexpr (MMA) {  // one thread per row, two partial sums
            for (int r = t; r < m; r += nt) {
                for (int b = 0; b < nd; ++b) {
                    double2 acc0 = make_double2(0, 0), acc1 = make_double2(0, 0);
                    const double2* lb = G + b * (b + 1) / 2;
                    int a = 0;
                    for (; a + 2 <= b; a += 2) {
                        const double2 q0 = W[cs.dropped[a] * m + r], l0 = lb[a];
                        const double2 q1 = W[cs.dropped[a + 1] * m + r], l1 = lb[a + 1];
                        acc0.x = fma(q0.x, l0.x, fma(q0.y, l0.y, acc0.x));
                        acc0.y = fma(q0.y, l0.x, fma(-q0.x, l0.y, acc0.y));
                        acc1.x = fma(q1.x, l1.x, fma(q1.y, l1.y, acc1.x));
                        acc1.y = fma(q1.y, l1.x, fma(-q1.x, l1.y, acc1.y));
                    }
                    if (a < b) {
                        const double2 q0 = W[cs.dropped[a] * m + r], l0 = lb[a];
                        acc0.x = fma(q0.x, l0.x, fma(q0.y, l0.y, acc0.x));
                        acc0.y = fma(q0.y, l0.x, fma(-q0.x, l0.y, acc0.y));
                    }
                    double2* w = W + cs.dropped[b] * m + r;
                    *w = cscale(invd[b], csub(*w, cadd(acc0, acc1)));
                }
            }
        } else {  // four lanes per row
            const int part = t & 3;
            const unsigned gm = 0xfu << ((t & 31) & ~3);
            for (int r = t >> 2; r < m; r += nt / 4) {
                for (int b = 0; b < nd; ++b) {
                    double2 acc = make_double2(0, 0);
                    const double2* lb = G + b * (b + 1) / 2;
                    for (int a = part; a < b; a += 4) {
                        const double2 q = W[cs.dropped[a] * m + r], l = lb[a];
                        acc.x = fma(q.x, l.x, fma(q.y, l.y, acc.x));
                        acc.y = fma(q.y, l.x, fma(-q.x, l.y, acc.y));
                    }
                    acc.x += __shfl_xor_sync(gm, acc.x, 1);
                    acc.y += __shfl_xor_sync(gm, acc.y, 1);
                    acc.x += __shfl_xor_sync(gm, acc.x, 2);
                    acc.y += __shfl_xor_sync(gm, acc.y, 2);
                    if (part == 0) {
                        double2* w = W + cs.dropped[b] * m + r;
                        *w = cscale(invd[b], csub(*w, acc));
                    }
                    __syncwarp(gm);
                }
            }
        }
        __syncthreads();
        if (pass == 0 && !cs.again) break;  // uniform: written before the barrier above
    }
}

// Fast path of the picker.  The reference's sequential two-pass Gram-Schmidt
// over the candidates in index order (pick_orthonormal, gsvd.cpp:404-436,
// first threshold pass) is a Cholesky factorization of the candidates' Gram
// matrix G = Y^H Y in which a candidate is accepted when its residual norm
// R_jj exceeds 0.05 n0_j and a rejected candidate is simply skipped (its row
// never enters the trailing updates).  One warp forms G for the first
// K = min(m, d + 8) candidates (rows of conj(N)), factors it with skipping
// until d are accepted, and forms the accepted vectors' coordinates
// Z = Y_sel R^-1.  Returns false (nothing written) when fewer than d of the K
// candidates pass; the caller then runs the sequential picker over all m.
// No block barrier inside: warp 0 only.
template <class CS>
__device__ bool pick_fast(const double2* W, double2* G, int m, int d, bool unit_norm0, CS& cs) {
    __shared__ int s_ok;
    __shared__ int s_sel[kZMax];
    const int t = threadIdx.x;
    if (t < kWarp) {
        const int lane = t;
        const int K = min(m, d + 8);
        // G[a][b] = y_a^H y_b (a <= b < K),  y_j[k] = conj(W[cols[k]][j])
        for (int e = lane; e < K * K; e += kWarp) {
            const int a = e / K, b = e % K;
            if (b < a) continue;
            double gx = 0, gy = 0;
            for (int k = 0; k < d; ++k) {
                const double2 wa = W[cs.cols[k] * m + a], wb = W[cs.cols[k] * m + b];
                gx = fma(wa.x, wb.x, fma(wa.y, wb.y, gx));
                gy = fma(wa.y, wb.x, fma(-wa.x, wb.y, gy));
            }
            G[a * K + b] = make_double2(gx, gy);
        }
        __syncwarp();
        // candidate norms before projection: lanes own j = lane, lane + 32
        const double n0a = unit_norm0 ? 1.0 : (lane < K ? sqrt(G[lane * K + lane].x) : 0.0);
        const double n0b = unit_norm0 ? 1.0 : (lane + kWarp < K ? sqrt(G[(lane + kWarp) * K + lane + kWarp].x) : 0.0);
        int taken = 0;
        for (int j = 0; j < K && taken < d; ++j) {
            const double n0j = __shfl_sync(0xffffffffu, j < kWarp ? n0a : n0b, j & 31);
            const double gjj = G[j * K + j].x;
            const double inv = gjj > 1e-300 ? fast_rsqrt(gjj) : 0.0;
            const double rjj = gjj * inv;
            if (!(n0j > 1e-140) || !(rjj > 0.05 * n0j) || !(rjj > 0)) continue;  // rejected: skipped (warp-uniform)
            for (int b = j + 1 + lane; b < K; b += kWarp) G[j * K + b] = cscale(inv, G[j * K + b]);
            __syncwarp();
            // trailing upper triangle, column b per lane: G[a][b] -= conj(R[j][a]) R[j][b];
            // four rows per batch, loads first (row j is read-only here)
            for (int b = j + 1 + lane; b < K; b += kWarp) {
                const double2 rb = G[j * K + b];
                int a = j + 1;
                for (; a + 4 <= b + 1; a += 4) {
                    double2 ra[4], g[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        ra[u] = G[j * K + a + u];
                        g[u] = G[(a + u) * K + b];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        g[u].x -= fma(ra[u].x, rb.x, ra[u].y * rb.y);
                        g[u].y -= fma(ra[u].x, rb.y, -ra[u].y * rb.x);
                        G[(a + u) * K + b] = g[u];
                    }
                }
                for (; a <= b; ++a) {
                    const double2 ra = G[j * K + a];
                    double2& g = G[a * K + b];
                    g.x -= fma(ra.x, rb.x, ra.y * rb.y);
                    g.y -= fma(ra.x, rb.y, -ra.y * rb.x);
                }
            }
            if (lane == 0) {
                G[j * K + j] = make_double2(rjj, 0.0);
                cs.nrm[taken] = inv;
                s_sel[taken] = j;
            }
            ++taken;
            __syncwarp();
        }
        const bool ok = taken == d;
        if (ok && lane < d) {  // Z = Y_sel R_sel^-1 column by column, lane = coordinate
            const int k = lane;
            for (int tt = 0; tt < d; ++tt) {
                const int jt = s_sel[tt];
                const double2 w = W[cs.cols[k] * m + jt];
                double2 acc0 = make_double2(w.x, -w.y), acc1 = make_double2(0, 0);  // y_jt[k]
                int s2 = 0;
                for (; s2 + 2 <= tt; s2 += 2) {
                    acc0 = csub(acc0, cmul(cs.z[k][s2], G[s_sel[s2] * K + jt]));
                    acc1 = csub(acc1, cmul(cs.z[k][s2 + 1], G[s_sel[s2 + 1] * K + jt]));
                }
                if (s2 < tt) acc0 = csub(acc0, cmul(cs.z[k][s2], G[s_sel[s2] * K + jt]));
                cs.z[k][tt] = cscale(cs.nrm[tt], cadd(acc0, acc1));
            }
        }
        if (lane == 0) s_ok = ok ? 1 : 0;
    }
    __syncthreads();
    return s_ok != 0;
}

// Upper-triangle packed index of (a, b), a <= b, of a d x d matrix.
__device__ __forceinline__ int tri(int a, int b, int d) { return a * d - a * (a - 1) / 2 + (b - a); }
__device__ __forceinline__ void tri_ab(int e, int d, int& a, int& b) {
    a = (int)((2.0f * d + 1.0f - sqrtf((2.0f * d + 1.0f) * (2.0f * d + 1.0f) - 8.0f * e)) * 0.5f);
    if (a < 0) a = 0;
    while (a > 0 && a * d - a * (a - 1) / 2 > e) --a;
    while ((a + 1) * d - (a + 1) * a / 2 <= e) ++a;
    b = a + (e - (a * d - a * (a - 1) / 2));
}

// Concurrent form of pick_fast for the fused canonicalization, in three
// stages over all groups at once (group columns s_perm[i0+k], scratch slice
// G [d][d] then Z [d][d], coordinate k of vector t at k*d+t):
//   gram_group   G = Y^H Y, y_j[k] = conj(W[cols[k]][j]), by the whole CTA;
//   chol_group   one warp per group: the Cholesky G = R^H R with the
//                acceptance test R_jj > 0.05 n0_j of pick_orthonormal
//                (gsvd.cpp:404-436) at every step; false when a candidate
//                would be rejected (the caller then runs the sequential picker);
//   z_rows       Z = Y R^-1, kZL threads per coordinate row, by the whole CTA.
template <int MC>
__device__ __forceinline__ void gram_group(const double2* W, const int* cols, double2* G, int m_rt, int d) {
    const int m = MC > 0 ? MC : m_rt;
    constexpr int nt = jac_threads<MC>();
    const int np = d * (d + 1) / 2;
    for (int e = threadIdx.x; e < np; e += nt) {
        int a, b;
        tri_ab(e, d, a, b);  // row-major over the upper triangle
        double gx = 0, gy = 0;
        for (int k = 0; k < d; ++k) {
            const double2 wa = W[cols[k] * m + a], wb = W[cols[k] * m + b];
            gx = fma(wa.x, wb.x, fma(wa.y, wb.y, gx));
            gy = fma(wa.y, wb.x, fma(-wa.x, wb.y, gy));
        }
        G[a * d + b] = make_double2(gx, gy);
    }
}

__device__ __forceinline__ bool chol_group(double2* G, double* n0b, double* ivb, int d, bool unit_norm0) {
    const int lane = threadIdx.x & 31;
    if (lane < d) n0b[lane] = unit_norm0 ? 1.0 : sqrt(G[lane * d + lane].x);
    __syncwarp();
    for (int j = 0; j < d; ++j) {
        const double gjj = G[j * d + j].x;
        const double n0 = n0b[j];
        // 1 / R_jj and R_jj from one refined rsqrt (the step's serial chain)
        const double inv = gjj > 1e-300 ? fast_rsqrt(gjj) : 0.0;
        const double rjj = gjj * inv;
        if (!(n0 > 1e-140) || !(rjj > 0.05 * n0) || !(rjj > 0)) return false;  // warp-uniform
        for (int b = j + 1 + lane; b < d; b += kWarp) G[j * d + b] = cscale(inv, G[j * d + b]);
        __syncwarp();
        // trailing upper triangle, column b per lane: G[a][b] -= conj(R[j][a]) R[j][b];
        // four rows per batch, loads first (row j is read-only here)
        for (int b = j + 1 + lane; b < d; b += kWarp) {
            const double2 rb = G[j * d + b];
            int a = j + 1;
            for (; a + 4 <= b + 1; a += 4) {
                double2 ra[4], g[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    ra[u] = G[j * d + a + u];
                    g[u] = G[(a + u) * d + b];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    g[u].x -= fma(ra[u].x, rb.x, ra[u].y * rb.y);
                    g[u].y -= fma(ra[u].x, rb.y, -ra[u].y * rb.x);
                    G[(a + u) * d + b] = g[u];
                }
            }
            for (; a <= b; ++a) {
                const double2 ra = G[j * d + a];
                double2& g = G[a * d + b];
                g.x -= fma(ra.x, rb.x, ra.y * rb.y);
                g.y -= fma(ra.x, rb.y, -ra.y * rb.x);
            }
        }
        if (lane == 0) {
            G[j * d + j] = make_double2(rjj, 0.0);
            ivb[j] = inv;
        }
        __syncwarp();
    }
    return true;
}

// Z[k][tt] = (y_tt[k] - sum_{s<tt} Z[k][s] R[s][tt]) / R[tt][tt] for row k of
// one group; the kZL lanes split the sum (lane part keeps, and alone reads
// back, the entries s = part mod kZL).
template <int kZL>
__device__ __forceinline__ void z_row(const double2* W, const int* cols, const double2* G, double2* Z,
                                      const double* ivb, int m, int d, int k, int part) {
    for (int tt = 0; tt < d; ++tt) {
        double2 acc = make_double2(0, 0);
        for (int s2 = part; s2 < tt; s2 += kZL) {
            const double2 zv = Z[k * d + s2], r = G[s2 * d + tt];
            acc.x = fma(zv.x, r.x, fma(-zv.y, r.y, acc.x));
            acc.y = fma(zv.x, r.y, fma(zv.y, r.x, acc.y));
        }
        acc = group_sum2<kZL>(acc);
        if (part == tt % kZL) {
            const double2 w = W[cols[k] * m + tt];
            Z[k * d + tt] = cscale(ivb[tt], make_double2(w.x - acc.x, -w.y - acc.y));
        }
    }
}

// The vanishing block when it exceeds kZMax (short windows, T < m / 2): its
// projector is written through the lead vectors B (ranks 0..m-z-1),
// P = I - B B^H — the form the reference itself builds (gsvd.cpp:466-503) —
// so no z x z buffer is needed.  G = P[0:z, 0:z] (the candidates e_0..e_z-1)
// goes packed into the scratch, its Cholesky runs with the acceptance test
// (candidate norms 1), and row i of the new block, P[i, 0:z] R^-1, is formed
// and back-substituted in place in row i of the vanishing columns.  False
// (nothing written) when a candidate would be rejected: seq_vanish then
// runs the reference's sequential picker.
template <int MC>
__device__ bool big_vanish(double2* W, const int* perm, int m_rt, int z, double2* Rp, double* ivb) {
    const int m = MC > 0 ? MC : m_rt;
    constexpr int nt = jac_threads<MC>();
    constexpr int kZL = 4;
    const int tid = threadIdx.x;
    const int lead = m - z;
    const int* vcols = perm + lead;
    __shared__ int s_ok;
    for (int e = tid; e < z * (z + 1) / 2; e += nt) {
        int a, b;
        tri_ab(e, z, a, b);
        double gx = 0, gy = 0;
        for (int l = 0; l < lead; ++l) {
            const double2 wa = W[perm[l] * m + a], wb = W[perm[l] * m + b];
            gx = fma(wa.x, wb.x, fma(wa.y, wb.y, gx));
            gy = fma(wa.y, wb.x, fma(-wa.x, wb.y, gy));
        }
        Rp[e] = make_double2((a == b ? 1.0 : 0.0) - gx, -gy);
    }
    __syncthreads();
    if (tid < kWarp) {
        const int lane = tid;
        bool ok = true;
        for (int j = 0; j < z; ++j) {
            const double gjj = Rp[tri(j, j, z)].x;
            const double rjj = gjj > 0 ? sqrt(gjj) : 0.0;
            if (!(rjj > 0.05)) {  // acceptance test, n0 = 1 (gsvd.cpp:404-436)
                ok = false;
                break;
            }
            const double inv = 1.0 / rjj;
            const int rj = tri(j, j, z);
            for (int b = j + 1 + lane; b < z; b += kWarp) Rp[rj + b - j] = cscale(inv, Rp[rj + b - j]);
            __syncwarp();
            for (int b = j + 1 + lane; b < z; b += kWarp) {
                const double2 rb = Rp[rj + b - j];
                for (int a2 = j + 1; a2 <= b; ++a2) {
                    const double2 ra = Rp[rj + a2 - j];
                    double2& g = Rp[tri(a2, b, z)];
                    g.x -= fma(ra.x, rb.x, ra.y * rb.y);
                    g.y -= fma(ra.x, rb.y, -ra.y * rb.x);
                }
            }
            if (lane == 0) {
                Rp[rj] = make_double2(rjj, 0.0);
                ivb[j] = inv;
            }
            __syncwarp();
        }
        if (lane == 0) s_ok = ok ? 1 : 0;
    }
    __syncthreads();
    if (!s_ok) return false;
    // row i: x_t = P[i][t] into W[vcols[t]][i] (lane part owns t = part mod
    // kZL), then w R = x by forward substitution, in place
    const int part = tid % kZL;
    for (int i = tid / kZL; i < m; i += nt / kZL) {
        for (int t = part; t < z; t += kZL) {
            double gx = 0, gy = 0;
            for (int l = 0; l < lead; ++l) {
                const double2 wa = W[perm[l] * m + i], wb = W[perm[l] * m + t];
                gx = fma(wa.x, wb.x, fma(wa.y, wb.y, gx));
                gy = fma(wa.y, wb.x, fma(-wa.x, wb.y, gy));
            }
            W[vcols[t] * m + i] = make_double2((i == t ? 1.0 : 0.0) - gx, -gy);
        }
        for (int t = 0; t < z; ++t) {
            double2 acc = make_double2(0, 0);
            for (int s2 = part; s2 < t; s2 += kZL) {
                const double2 wv = W[vcols[s2] * m + i], r = Rp[tri(s2, t, z)];
                acc.x = fma(wv.x, r.x, fma(-wv.y, r.y, acc.x));
                acc.y = fma(wv.x, r.y, fma(wv.y, r.x, acc.y));
            }
            acc = group_sum2<kZL>(acc);
            if (part == t % kZL) {
                const double2 x = W[vcols[t] * m + i];
                W[vcols[t] * m + i] = cscale(ivb[t], make_double2(x.x - acc.x, x.y - acc.y));
            }
        }
    }
    __syncthreads();
    return true;
}

// The reference's sequential picker (pick_orthonormal, gsvd.cpp:404-436) for
// a vanishing block big_vanish could not take in one pass (a candidate
// rejected): candidates e_j in index order over the three threshold passes,
// each projected twice against the lead vectors B and the vectors already
// taken; accepted vectors go straight into the vanishing columns (the old
// basis of the block is not needed in this representation).  Thread i < m
// holds c[i]; cbuf / dots are m-entry scratch.
template <int MC>
__device__ void seq_vanish(double2* W, const int* perm, int m_rt, int z, double2* cbuf, double2* dots) {
    const int m = MC > 0 ? MC : m_rt;
    constexpr int nt = jac_threads<MC>();
    constexpr int nw = nt / kWarp;
    const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
    const int lead = m - z;
    const int* vcols = perm + lead;
    __shared__ double s_red[nw];
    auto project = [&](double2& c, const int* cols, int n) {
        if (n == 0) return;
        if (tid < m) cbuf[tid] = c;
        __syncthreads();
        for (int l = warp; l < n; l += nw) {
            double2 d = make_double2(0, 0);
            for (int i = lane; i < m; i += kWarp) {
                const double2 b = W[cols[l] * m + i], v = cbuf[i];
                d.x = fma(b.x, v.x, fma(b.y, v.y, d.x));
                d.y = fma(b.x, v.y, fma(-b.y, v.x, d.y));
            }
            d = group_sum2<kWarp>(d);
            if (lane == 0) dots[l] = d;
        }
        __syncthreads();
        if (tid < m)
            for (int l = 0; l < n; ++l) {
                const double2 b = W[cols[l] * m + tid], d = dots[l];
                c.x -= fma(d.x, b.x, -d.y * b.y);
                c.y -= fma(d.x, b.y, d.y * b.x);
            }
    };
    unsigned long long used = 0;
    int taken = 0;
    const double thresholds[3] = {0.05, 1e-8, 0.0};
    for (int tp = 0; tp < 3 && taken < z; ++tp) {
        for (int j = 0; j < m && taken < z; ++j) {
            if ((used >> j) & 1ull) continue;
            double2 c = make_double2(tid == j ? 1.0 : 0.0, 0.0);
            for (int pass = 0; pass < 2; ++pass) {
                project(c, perm, lead);
                project(c, vcols, taken);
            }
            double v = tid < m ? fma(c.x, c.x, c.y * c.y) : 0.0;
            v = group_sum<kWarp>(v);
            if (lane == 0) s_red[warp] = v;
            __syncthreads();
            double n2 = 0;
#pragma unroll
            for (int w = 0; w < nw; ++w) n2 += s_red[w];
            const double nrm = sqrt(n2);
            __syncthreads();  // s_red and cbuf reused by the next candidate
            if (!(nrm > thresholds[tp]) || !(nrm > 0)) continue;
            if (tid < m) W[vcols[taken] * m + tid] = cscale(1.0 / nrm, c);
            used |= 1ull << j;
            ++taken;
        }
    }
    // unfilled slots stay zero, as the reference's zero-initialized output
    for (int e = tid; e < (z - taken) * m; e += nt) W[vcols[taken + e / m] * m + e % m] = make_double2(0, 0);
    __syncthreads();
}

// New columns of one group from a Z slice: W[:, cols[s]] <- sum_k W[:, cols[k]] Z[k][s]
template <int MC>
__device__ void apply_span_z(double2* W, int m_rt, int d, const int* cols, const double2* Z, int zld = 0) {
    const int m = MC > 0 ? MC : m_rt;
    constexpr int nt = jac_threads<MC>();
    constexpr int kOut = ((MC > 0 ? MC : kMaxM) * kZMax + nt - 1) / nt;
    const int t = threadIdx.x;
    double2 out[kOut];
#pragma unroll
    for (int c = 0; c < kOut; ++c) {
        const int e = t + c * nt;
        if (e < m * d) {
            const int i = e % m, sv = e / m;
            double2 acc = make_double2(0, 0);
            for (int k = 0; k < d; ++k) {
                const double2 a = W[cols[k] * m + i], b = Z[k * (zld ? zld : d) + sv];
                acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
                acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
            }
            out[c] = acc;
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kOut; ++c) {
        const int e = t + c * nt;
        if (e < m * d) W[cols[e / m] * m + (e % m)] = out[c];
    }
    __syncthreads();
}

// Reference picker (pick_orthonormal, gsvd.cpp:404-436) on the coordinates of
// one group: candidate j is row j of conj(N), N = W[cols[0..d)].  Threads
// j < m own candidate j; the accepted coordinate vectors land in cs.z.
template <class CS>
__device__ void pick_in_span(const double2* W, double2* Y, int m, int d, bool unit_norm0, CS& cs) {
    if (d <= kZMax && pick_fast(W, Y, m, d, unit_norm0, cs)) return;
    const int t = threadIdx.x;
    double2* yr = Y + t * kYld;
    bool used = false;
    if (t < m) {
        double n2 = 0;
        for (int k = 0; k < d; ++k) {
            const double2 v = W[cs.cols[k] * m + t];
            yr[k] = make_double2(v.x, -v.y);
            n2 = fma(v.x, v.x, fma(v.y, v.y, n2));
        }
        cs.nrm[t] = sqrt(n2);
        cs.norm0[t] = unit_norm0 ? 1.0 : sqrt(n2);
    }
    __syncthreads();
    int taken = 0;
    const double thresholds[3] = {0.05, 1e-8, 0.0};
    for (int tp = 0; tp < 3 && taken < d; ++tp) {
        const double thr = thresholds[tp];
        int start = 0;
        while (taken < d) {
            if (t < 64) {
                bool ok = false;
                if (t < m && t >= start && !used) {
                    const double n0 = cs.norm0[t], nr = cs.nrm[t];
                    ok = (n0 > 1e-140) && (nr > thr * n0) && (nr > 0);
                }
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                if ((t & 31) == 0) cs.ball[t >> 5] = b;
            }
            __syncthreads();
            int sel = -1;
            if (cs.ball[0]) sel = __ffs(cs.ball[0]) - 1;
            else if (cs.ball[1]) sel = 32 + __ffs(cs.ball[1]) - 1;
            if (sel < 0) break;
            if (t < d) {
                const double inv = 1.0 / cs.nrm[sel];
                const double2 qv = cscale(inv, Y[sel * kYld + t]);
                cs.q[t] = qv;
                cs.z[t][taken] = qv;
            }
            __syncthreads();
            if (t == sel) used = true;
            start = sel + 1;
            ++taken;
            // two projection passes of the remaining candidates against q
            if (t < m && !used) {
                for (int rep = 0; rep < 2; ++rep) {
                    double2 dt = make_double2(0, 0);
                    for (int k = 0; k < d; ++k) {
                        const double2 qk = cs.q[k], yk = yr[k];
                        dt.x = fma(qk.x, yk.x, fma(qk.y, yk.y, dt.x));
                        dt.y = fma(qk.x, yk.y, fma(-qk.y, yk.x, dt.y));
                    }
                    double n2 = 0;
                    for (int k = 0; k < d; ++k) {
                        const double2 qk = cs.q[k];
                        double2 yk = yr[k];
                        yk.x = fma(-dt.x, qk.x, fma(dt.y, qk.y, yk.x));
                        yk.y = fma(-dt.x, qk.y, fma(-dt.y, qk.x, yk.y));
                        yr[k] = yk;
                        n2 = fma(yk.x, yk.x, fma(yk.y, yk.y, n2));
                    }
                    if (rep == 1) cs.nrm[t] = sqrt(n2);
                }
            }
            __syncthreads();
        }
    }
    // unfilled slots (fewer acceptable candidates than d) stay zero, as the
    // reference's zero-initialized output
    for (int e = t; e < d * d; e += blockDim.x) {
        const int k = e / d, s = e % d;
        if (s >= taken) cs.z[k][s] = make_double2(0, 0);
    }
    __syncthreads();
}

// W[:, cols[s]] <- sum_k W[:, cols[k]] z[k][s]  (new vectors of one group)
template <int MC, class CS>
__device__ void apply_span(double2* W, int m, int d, CS& cs) {
    apply_span_z<MC>(W, m, d, cs.cols, &cs.z[0][0], (int)(sizeof(cs.z[0]) / sizeof(double2)));
}

// ---------------------------------------------------------------------------
// QR preconditioning (Drmac-Veselic): A P = Q R by Householder with column
// pivoting, then the one-sided Jacobi runs on X = R^H, whose graded columns
// converge in ~8 round-robin sweeps instead of ~18 on A itself (measured on
// the C3 scenes).  Q is never formed: with X V_X = U_X S, the left singular
// vectors of A are U_A = A P U_X S^-1 (A P = U_A S V_R^H, U_X = V_R), one
// GEMM against the saved A.
// ---------------------------------------------------------------------------

struct QrScratch {
    double2 u[kMaxM];       // Householder vector of the current step (zero above k)
    unsigned key[kMaxM];    // pivot key per physical column (0: already pivoted)
    int piv[kMaxM];         // column k of A P is column piv[k] of A
    double tau;
};

// Pivot key: the remaining squared norm as float bits (monotonic for x >= 0)
// with the low 6 bits replaced by 63 - column, so one unsigned max picks the
// largest norm (to 2^-17 relative) and the lowest column among equals.
__device__ __forceinline__ unsigned pivot_key(double n2, int c) {
    const float f = __double2float_rz(fmin(n2, 1e38));
    return ((__float_as_uint(f) & ~63u) | (unsigned)(63 - c)) + 1u;
}

// sqrt for positive normal FP64 values (x * rsqrt(x), Newton-refined)
__device__ __forceinline__ double fast_sqrt(double x) { return x > 0 ? x * fast_rsqrt(x) : 0.0; }


// Column-resident QRCP: 4 lanes own one physical column of A in registers
// (rows l, l+4, ...), so a step moves only the Householder vector through
// shared memory.  Per step: every warp reduces the pivot keys with one
// redux.max; the pivot's group forms the reflector H = I - tau u u^H
// (H x = beta e_k) from the exact norm of its rows >= k that it computed in
// the previous step; one barrier; every other unpivoted group applies H to
// its column and accumulates the exact norm of its rows > k in the same pass;
// one barrier.  The pivot section is kept to a few dozen instructions: it is
// the serial part of every step.
template <int MC>
__device__ void qrcp_to_rh(double2* W, int m, QrScratch& qs) {
    constexpr int QL = jac_threads<MC>() / kMaxM > 0 ? jac_threads<MC>() / kMaxM : 1;  // lanes per column
    constexpr int RP = MC > 0 ? (MC + QL - 1) / QL : kMaxM / QL;
    const int t = threadIdx.x, c = t / QL, l = t % QL, lane = t & 31;
    const bool own = c < m;
    const unsigned gmask = ((1u << QL) - 1u) << (lane & ~(QL - 1));
    double2 y[RP];
#pragma unroll
    for (int v = 0; v < RP; ++v) {
        const int i = l + QL * v;
        y[v] = (own && i < m) ? W[c * m + i] : make_double2(0, 0);
    }
    double nrm;  // exact squared norm of rows >= k (rows > k - 1 after the previous update)
    {
        double a0 = 0, a1 = 0;
#pragma unroll
        for (int v = 0; v < RP; v += 2) a0 = fma(y[v].x, y[v].x, fma(y[v].y, y[v].y, a0));
#pragma unroll
        for (int v = 1; v < RP; v += 2) a1 = fma(y[v].x, y[v].x, fma(y[v].y, y[v].y, a1));
        nrm = a0 + a1;
#pragma unroll
        for (int o = 1; o < QL; o <<= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        if (own && l == 0) qs.key[c] = pivot_key(nrm, c);
        if (t < kMaxM) {
            qs.u[t] = make_double2(0, 0);
            if (t >= m) qs.key[t] = 0u;
        }
    }
    int mypos = -1;
    double2 mybeta = make_double2(0, 0);
    __syncthreads();
    for (int k = 0; k < m; ++k) {
        const unsigned kk = __reduce_max_sync(0xffffffffu, max(qs.key[lane], qs.key[lane + 32]));
        const int p = 63 - (int)((kk - 1u) & 63u);
        if (c == p) {
            double2 x0 = make_double2(0, 0);
#pragma unroll
            for (int v = 0; v < RP; ++v) {
                const int i = l + QL * v;
                if (i == k) x0 = y[v];
                if (i >= k && i < m) qs.u[i] = y[v];
            }
            if (l == k % QL) {  // the lane that owns row k finishes the reflector
                const double ax2 = fma(x0.x, x0.x, x0.y * x0.y);
                const double alpha = fast_sqrt(nrm);
                double2 ph = make_double2(1.0, 0.0);
                double ax0 = 0.0;
                if (ax2 > 0) {
                    const double ri = fast_rsqrt(ax2);
                    ax0 = ax2 * ri;
                    ph = make_double2(x0.x * ri, x0.y * ri);
                }
                mybeta = make_double2(-ph.x * alpha, -ph.y * alpha);
                qs.u[k] = make_double2(x0.x + ph.x * alpha, x0.y + ph.y * alpha);
                qs.tau = alpha > 0 ? fast_rcp(alpha * (alpha + ax0)) : 0.0;
                qs.piv[k] = p;
            }
            mypos = k;
        }
        __syncthreads();
        {  // every group runs the update (no divergence around the group
           // shuffles); pivoted and padding groups apply a zero multiple
            const bool act = own && mypos < 0;
            const double tau = act ? qs.tau : 0.0;
            // rows above k have u = 0, so whole segments of 3 row chunks below
            // the first active chunk are skipped (warp-uniform) and the rest
            // run unpredicated; a segment issues its 3 Householder loads
            // before its FMAs, keeping them in flight together
            const int v0 = k / QL;
            constexpr int SEG = 3;
            double sx0 = 0, sy0 = 0, sx1 = 0, sy1 = 0;
#pragma unroll
            for (int s0 = 0; s0 < RP; s0 += SEG) {
                if (v0 <= s0 + SEG - 1) {
                    double2 uu[SEG];
#pragma unroll
                    for (int j = 0; j < SEG; ++j) uu[j] = s0 + j < RP ? qs.u[l + QL * (s0 + j)] : make_double2(0, 0);
#pragma unroll
                    for (int j = 0; j < SEG; ++j) {
                        const int v = s0 + j;
                        if (v < RP) {
                            if (v & 1) {
                                sx1 = fma(uu[j].x, y[v].x, fma(uu[j].y, y[v].y, sx1));
                                sy1 = fma(uu[j].x, y[v].y, fma(-uu[j].y, y[v].x, sy1));
                            } else {
                                sx0 = fma(uu[j].x, y[v].x, fma(uu[j].y, y[v].y, sx0));
                                sy0 = fma(uu[j].x, y[v].y, fma(-uu[j].y, y[v].x, sy0));
                            }
                        }
                    }
                }
            }
            double sx = sx0 + sx1, sy = sy0 + sy1;
#pragma unroll
            for (int o = 1; o < QL; o <<= 1) {
                sx += __shfl_xor_sync(gmask, sx, o);
                sy += __shfl_xor_sync(gmask, sy, o);
            }
            const double fx = tau * sx, fy = tau * sy;
            double a0 = 0, a1 = 0;
#pragma unroll
            for (int s0 = 0; s0 < RP; s0 += SEG) {
                if (v0 <= s0 + SEG - 1) {
                    double2 uu[SEG];
#pragma unroll
                    for (int j = 0; j < SEG; ++j) uu[j] = s0 + j < RP ? qs.u[l + QL * (s0 + j)] : make_double2(0, 0);
#pragma unroll
                    for (int j = 0; j < SEG; ++j) {
                        const int v = s0 + j;
                        if (v < RP) {
                            y[v].x = fma(-fx, uu[j].x, fma(fy, uu[j].y, y[v].x));
                            y[v].y = fma(-fx, uu[j].y, fma(-fy, uu[j].x, y[v].y));
                            const double e = (l + QL * v > k) ? fma(y[v].x, y[v].x, y[v].y * y[v].y) : 0.0;
                            if (v & 1) a1 += e;
                            else a0 += e;
                        }
                    }
                }
            }
            nrm = a0 + a1;
#pragma unroll
            for (int o = 1; o < QL; o <<= 1) nrm += __shfl_xor_sync(gmask, nrm, o);
            if (act && l == 0) qs.key[c] = pivot_key(nrm, c);
            // the pivot leaves the key set only now: every warp read this
            // step's keys before the barrier above
            if (c == p && l == 0) qs.key[c] = 0u;
        }
        __syncthreads();
        if (c == p && l == k % QL) qs.u[k] = make_double2(0, 0);  // keep u zero above the next step
    }
    // X = R^H: the group at pivot position j holds row j of X (conjugated
    // column j of R: rows < j in registers, beta on the diagonal); X is
    // lower triangular
    const int bsrc = (lane & ~(QL - 1)) | (mypos & (QL - 1));
    const double2 bj = make_double2(__shfl_sync(0xffffffffu, mybeta.x, bsrc), __shfl_sync(0xffffffffu, mybeta.y, bsrc));
    if (own) {
#pragma unroll
        for (int v = 0; v < RP; ++v) {
            const int r = l + QL * v;
            if (r < m) W[r * m + mypos] = r < mypos ? cconj(y[v]) : (r == mypos ? cconj(bj) : make_double2(0, 0));
        }
    }
    __syncthreads();
}

// U_A[:, j] = A[:, piv] U_X[:, j] / sigma_j, A from the global copy (column
// major), U_X in W; processed in column chunks so each chunk only reads the
// U_X columns it overwrites.
__device__ void back_multiply(double2* W, const double2* __restrict__ ag, int m, const QrScratch& qs,
                              const double* sig) {
    const int t = threadIdx.x;
    int parts = blockDim.x / m;
    if (parts > m) parts = m;
    const bool active = t < m * parts;
    // part-major: a warp covers consecutive rows i of one column set, so its
    // W reads are broadcasts and its A loads coalesce
    const int i = active ? t % m : 0;
    const int part = active ? t / m : 0;
    const int per = (m + parts - 1) / parts;  // columns per thread
    for (int u0 = 0; u0 < per; u0 += 8) {
        double2 acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = make_double2(0, 0);
        if (active)
            for (int k0 = 0; k0 < m; k0 += 8) {
                double2 av[8];  // independent loads in flight (A written earlier by this CTA)
#pragma unroll
                for (int b = 0; b < 8; ++b) av[b] = k0 + b < m ? ag[qs.piv[k0 + b] * m + i] : make_double2(0, 0);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const int k = k0 + b;
                    if (k < m) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = part + parts * (u0 + u);
                            if (u0 + u < per && j < m) {
                                const double2 w = W[j * m + k];
                                acc[u].x = fma(av[b].x, w.x, fma(-av[b].y, w.y, acc[u].x));
                                acc[u].y = fma(av[b].x, w.y, fma(av[b].y, w.x, acc[u].y));
                            }
                        }
                    }
                }
            }
        __syncthreads();
        if (active)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = part + parts * (u0 + u);
                if (u0 + u < per && j < m) W[j * m + i] = sig[j] > 0 ? cscale(1.0 / sig[j], acc[u]) : make_double2(0, 0);
            }
        __syncthreads();
    }
}

// rotate_pair<R, L>'s no-rotation test (jacobi_rot.cuh) for columns a and b
// in its exact operation order, for both orientations (which column the sweep
// loads as P is a property of its ordering): lane s of the pair's group sums
// rows s + L u into two accumulators by the parity of u, and group_sum2 adds
// the lanes' partials by the xor butterfly.  True iff either orientation
// would rotate.
template <int L>
__device__ bool pair_rotates_exact(const double2* W, int m, int a, int b, double ca, double cb, double tol2) {
    for (int o = 0; o < 2; ++o) {
        const double2* P = W + (o ? b : a) * m;
        const double2* Q = W + (o ? a : b) * m;
        const double cp = o ? cb : ca, cq = o ? ca : cb;
        double2 v[L];
#pragma unroll
        for (int s = 0; s < L; ++s) {
            double d0x = 0, d0y = 0, d1x = 0, d1y = 0;
            for (int u = 0; s + u * L < m; ++u) {
                const double2 x = P[s + u * L], y = Q[s + u * L];
                if (u & 1) {
                    d1x = fma(x.x, y.x, fma(x.y, y.y, d1x));
                    d1y = fma(x.x, y.y, fma(-x.y, y.x, d1y));
                } else {
                    d0x = fma(x.x, y.x, fma(x.y, y.y, d0x));
                    d0y = fma(x.x, y.y, fma(-x.y, y.x, d0y));
                }
            }
            v[s] = make_double2(d0x + d1x, d0y + d1y);
        }
#pragma unroll
        for (int h = L / 2; h > 0; h >>= 1) {
            double2 nv[L];
#pragma unroll
            for (int s = 0; s < L; ++s) nv[s] = make_double2(v[s].x + v[s ^ h].x, v[s].y + v[s ^ h].y);
#pragma unroll
            for (int s = 0; s < L; ++s) v[s] = nv[s];
        }
        const double mag2 = fma(v[0].x, v[0].x, v[0].y * v[0].y);
        if (!(mag2 <= tol2 * cp * cq)) return true;
    }
    return false;
}

// True iff every pair of columns above the drop line satisfies the
// reference's no-rotation test |x_p^H x_q|^2 <= 1e-28 |x_p|^2 |x_q|^2, i.e.
// iff the next sweep would rotate nothing (gsvd.cpp:642-649).  Evaluated as
// one 4x4-register-tiled Gram product over the upper triangle instead of a
// full verification sweep of round-synchronized pair visits; a pair the Gram
// product's summation order puts above the line is re-tested in the order of
// the sweep it stands in for (L lanes per pair), so a coupling at the 1e-14
// line does not cost a sweep that would rotate nothing (C3: 7.18 -> 7.14
// sweeps per bin; most certificates that fail do so for a pair the sweep
// then rotates).
template <int MC, int TS = 2, int L = 4>  // 2x2 tiles keep the fused kernel's register budget
__device__ bool gram_converged(const double2* W, int m_rt, const double* cn, double drop, double tol2) {
    const int m = MC > 0 ? MC : m_rt;
    const int nt = (m + TS - 1) / TS;
    const int ntiles = nt * (nt + 1) / 2;
    bool bad = false;
    for (int idx0 = threadIdx.x; idx0 < ntiles; idx0 += blockDim.x) {
        int idx = idx0, ti = 0;
        while (idx >= nt - ti) {  // upper-triangle tile enumeration
            idx -= nt - ti;
            ++ti;
        }
        const int p0 = TS * ti, q0 = TS * (ti + idx);
        double2 acc[TS][TS];
#pragma unroll
        for (int u = 0; u < TS; ++u)
#pragma unroll
            for (int v = 0; v < TS; ++v) acc[u][v] = make_double2(0, 0);
        // rows visited from a lane-dependent start: the lanes of a quarter-warp
        // read 8 different rows of their (different) columns, not one bank
        const int k0 = threadIdx.x & 7;
        for (int kk = 0; kk < m; ++kk) {
            int k = kk + k0;
            if (k >= m) k -= m;
            double2 xp[TS], xq[TS];
#pragma unroll
            for (int u = 0; u < TS; ++u) {
                xp[u] = p0 + u < m ? W[(p0 + u) * m + k] : make_double2(0, 0);
                xq[u] = q0 + u < m ? W[(q0 + u) * m + k] : make_double2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < TS; ++u)
#pragma unroll
                for (int v = 0; v < TS; ++v) {
                    acc[u][v].x = fma(xp[u].x, xq[v].x, fma(xp[u].y, xq[v].y, acc[u][v].x));
                    acc[u][v].y = fma(xp[u].x, xq[v].y, fma(-xp[u].y, xq[v].x, acc[u][v].y));
                }
        }
        unsigned flagged = 0u;
#pragma unroll
        for (int u = 0; u < TS; ++u)
#pragma unroll
            for (int v = 0; v < TS; ++v) {
                const int p = p0 + u, q = q0 + v;
                if (p < q && q < m && cn[p] > drop && cn[q] > drop) {
                    const double mag2 = fma(acc[u][v].x, acc[u][v].x, acc[u][v].y * acc[u][v].y);
                    if (mag2 > tol2 * cn[p] * cn[q]) flagged |= 1u << (u * TS + v);
                }
            }
#pragma unroll 1
        for (; flagged && !bad; flagged &= flagged - 1) {
            const int f = __ffs(flagged) - 1, p = p0 + f / TS, q = q0 + f % TS;
            bad = pair_rotates_exact<L>(W, m, p, q, cn[p], cn[q], tol2);
        }
    }
    return !__syncthreads_or(bad);
}

// U_A = A P U_X S^-1 on the FP64 tensor cores (DMMA m8n8k4) for the split
// solver's epilogue: warp w owns output rows 8w..8w+7 (8 complex 8x8 tiles),
// the A operand (rows of A P, column piv[k] of the saved A) comes straight
// from global memory (L2), the B operand (U_X = normalized W) from shared
// memory; the strip is held in registers until every warp has read W.
template <int NT>
__device__ void back_multiply_mma(double2* W, const double2* __restrict__ ag, int m, const QrScratch& qs,
                                  const double* sig) {
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31, r = lane >> 2, c = lane & 3;
    const int nt8 = (m + 7) >> 3;
    double re[8][2], im[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) re[j][0] = re[j][1] = im[j][0] = im[j][1] = 0.0;
    const int i = warp * 8 + r;
    if (warp < nt8) {
        double2 an = (i < m && c < m) ? ag[qs.piv[c] * m + i] : make_double2(0, 0);
        for (int k0 = 0; k0 < m; k0 += 4) {
            const int k = k0 + c;
            const double2 av = an;  // A_P[i][k]
            const int kn = k + 4;
            an = (i < m && kn < m) ? ag[qs.piv[kn] * m + i] : make_double2(0, 0);  // next step's fragment
            const double nai = -av.y;
            double2 bv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int col = j * 8 + r;
                bv[j] = (j < nt8 && k < m && col < m) ? W[col * m + k] : make_double2(0, 0);
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
    __syncthreads();  // every warp has read U_X
    if (warp < nt8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = j * 8 + 2 * c + e;
                if (i < m && col < m)
                    W[col * m + i] = sig[col] > 0 ? cscale(1.0 / sig[col], make_double2(re[j][e], im[j][e]))
                                                  : make_double2(0, 0);
            }
    }
    __syncthreads();
}

// The one-sided Jacobi sweeps (gsvd.cpp:622-695) on W in shared memory with
// LPP-lane pair groups (RW = 64 / LPP rows per lane); shared by the fused
// solver (LPP = 8) and the split sweep kernel (LPP = 4, 128 threads).
// Returns the sweep count and convergence; drop_out is the last sweep's
// drop line (the non-preconditioned path marks columns below it).
template <int MC, int LPP>
__device__ void run_sweeps(double2* W, int m, double* cn, bool precond, const GsvdArgs& a, int& sweep_out,
                           bool& conv_out, double& drop_out) {
    constexpr int RW = kMaxM / LPP;
    const int tid = threadIdx.x;
    __shared__ double s_drop;
    const int g = tid / LPP;
    const int s = tid % LPP;
    const int n_even = (m + 1) & ~1;
    const int npairs = n_even / 2;

    __shared__ int s_rots;
    __shared__ unsigned long long s_maxrel;  // 1: a pair coupled above 1e-8 relative was rotated this sweep
    if (tid == 0) {
        s_rots = 0;
        s_maxrel = 0ull;
    }
    int prev_rots = 1 << 30;
    double prev_maxrel = 1.0;
    const int total_pairs = m * (m - 1) / 2;
    int sweep = 0;
    bool converged = false;
    while (sweep < a.max_sweeps) {
        // fresh squared column norms (gsvd.cpp:633-637)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int j = 2 * g + cc;
            if (j < m) {
                double v = 0;
#pragma unroll
                for (int u = 0; u < RW; ++u) {
                    const int row = s + u * LPP;
                    if (row < m) {
                        const double2 w = W[j * m + row];
                        v = fma(w.x, w.x, fma(w.y, w.y, v));
                    }
                }
                v = group_sum<LPP>(v);
                if (s == 0) cn[j] = v;
            }
        }
        __syncthreads();
        if (tid < kWarp) {
            double mx = 0;
            for (int j = tid; j < m; j += kWarp) mx = fmax(mx, cn[j]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            // Preconditioned path: no column is skipped (only exact zeros) —
            // the back-multiplication A P U_X / sigma_j would amplify the
            // un-rotated coupling to a dropped column by sigma_max / sigma_j.
            if (tid == 0) s_drop = precond ? 0.0 : 1e-20 * mx;
        }
        __syncthreads();
        const double drop = s_drop;
        // A sweep after one that rotated fewer than half of the pairs (the
        // quadratic tail: at C3 the 8th sweep after a 30%-rotating 7th is
        // rotation-free in 98% of bins), or only pairs coupled by <= 1e-8
        // relative, is usually rotation-free: certify that with one Gram
        // product instead of running it (7.44 -> 7.06 sweeps at C3).
        if (sweep > 0 && (2 * prev_rots < total_pairs || prev_maxrel == 0.0) && gram_converged<MC, LPP == 4 ? 4 : 2, LPP>(W, m, cn, drop, a.tol2)) {
            converged = true;
            break;
        }
        if (tid == 0) {
            s_rots = 0;
            s_maxrel = 0ull;
        }
        int myrots = 0;
        double mymax = 0.0;
        bool rot = false;
        // round-robin (circle) ordering: the m/2 disjoint pairs of a round
        // rotate concurrently, one LPP-lane group per pair
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                if (q < m) {
                    double2 P[RW], Q[RW];
#pragma unroll
                    for (int u = 0; u < RW; ++u) {
                        const int row = s + u * LPP;
                        P[u] = row < m ? W[p * m + row] : make_double2(0, 0);
                        Q[u] = row < m ? W[q * m + row] : make_double2(0, 0);
                    }
                    double cp = cn[p], cq = cn[q];
                    if (rotate_pair<RW, LPP>(P, Q, cp, cq, drop, s, m, mymax, a.tol2)) {
#pragma unroll
                        for (int u = 0; u < RW; ++u) {
                            const int row = s + u * LPP;
                            if (row < m) {
                                W[p * m + row] = P[u];
                                W[q * m + row] = Q[u];
                            }
                        }
                        // lane 0 writes the norms the whole group loaded; the
                        // group barrier orders those loads before the write
                        // under the CUDA memory model (the group's shuffles
                        // already did in practice)
                        __syncwarp(group_mask<LPP>());
                        if (s == 0) {
                            cn[p] = cp;
                            cn[q] = cq;
                            ++myrots;
                        }
                        rot = true;
                    }
                }
            }
            __syncthreads();
        }
        ++sweep;
        if (myrots) {
            atomicAdd(&s_rots, myrots);
            if (mymax > 0) atomicMax(&s_maxrel, 1ull);
        }
        if (!__syncthreads_or(rot)) {
            converged = true;
            break;
        }
        prev_rots = s_rots;
        prev_maxrel = s_maxrel ? 1.0 : 0.0;
    }

    sweep_out = sweep;
    conv_out = converged;
    drop_out = s_drop;
}

// resident CTAs per SM: 2 for the 60/64-channel solver (shared memory), 12 at
// m = 8 and 8 at m = 16 (registers; measured best: C1 0.44 -> 0.36 ms,
// C2 1.03 -> 0.93 ms per 32 blocks against 6)
template <int MC>
constexpr int jac_ctas() { return MC > 0 && MC <= 8 ? 12 : (MC > 0 && MC <= 16 ? 8 : 2); }

// MC > 0: channel count fixed at compile time (loop bounds, predicates and
// addressing fold away); MC == 0: any m <= 64 at run time.
// PART 0: the whole solve; 1: whitening + QR, W and the pivots to global;
// 3: the rest, after sweep_kernel ran the sweeps on the stored W.
template <int MC, int PART = 0>
__global__ void __launch_bounds__(jac_threads<MC>(), jac_ctas<MC>()) jacobi_kernel(GsvdArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    if constexpr (PART == 3) {
        // launched while the sweep kernel's last CTAs still run (programmatic
        // dependent launch): wait for this CTA's own bin only
        if (a.done) {
            if (threadIdx.x == 0)
                while (ld_acquire_gpu(a.done + blockIdx.x) != a.epoch) __nanosleep(200);
            __syncthreads();
        }
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = MC > 0 ? MC : a.m;
    double2* W = reinterpret_cast<double2*>(smem_raw);  // [m cols][m rows]
    double2* Y = W + m * m;                             // [kMaxM][kYld] picker coordinates
    __shared__ double cn[kMaxM];
    __shared__ int s_perm[kMaxM];  // rank -> column
    __shared__ double s_sig[kMaxM];
    __shared__ CanonScratchFor<MC> cs;
    __shared__ QrScratch qs;

    const int blk = blockIdx.x;
    const int bin = blk % a.bins;
    const int tid = threadIdx.x;

    // optional phase clocks (SSLG_PHASE_CLOCKS): whiten, QR, sweeps, sigma /
    // back-multiply, canonicalization, store
    long long clk0 = 0;
    auto mark = [&](int ph) {
        if (a.phase_clk && tid == 0) {
            const long long now = clock64();
            atomicAdd(reinterpret_cast<unsigned long long*>(a.phase_clk + ph), (unsigned long long)(now - clk0));
            clk0 = now;
        }
    };
    if (tid == 0) clk0 = clock64();
    const bool precond = a.precondition && a.ascratch;
    double2* ag = precond ? a.ascratch + (size_t)blk * m * m : nullptr;
    int sweep = 0;
    bool converged = false;
    double drop_last = 0.0;
    if constexpr (PART == 1) {
        // prologue of the split solver: the whitening on the FP64 tensor
        // cores (no sweeps share this kernel's SM time), A saved on the way
        form_whitened_mma<jac_threads<MC>()>(a.r + (size_t)blk * m * m, a.kinv + (size_t)bin * m * m, m, W,
                                            reinterpret_cast<float2*>(Y), ag);
        mark(0);
        qrcp_to_rh<MC>(W, m, qs);
        mark(1);
    } else if constexpr (PART == 0) {
        form_whitened_staged(a.r + (size_t)blk * m * m, a.kinv + (size_t)bin * m * m, m, W, Y);
        mark(0);
        if (precond) {
            for (int e = tid; e < m * m; e += blockDim.x) ag[e] = W[e];
            qrcp_to_rh<MC>(W, m, qs);
        }
        mark(1);
    }
    if constexpr (PART == 1) {
        double2* wg = a.wscratch + (size_t)blk * m * m;
        for (int e = tid; e < m * m; e += blockDim.x) wg[e] = W[e];
        if (tid < m) a.pivs[(size_t)blk * kMaxM + tid] = qs.piv[tid];
        return;
    }
    if constexpr (PART == 3) {
        const double2* wg = a.wscratch + (size_t)blk * m * m;
        batched_copy<4>(tid, (int)blockDim.x, m * m, wg, [&](int e, double2 v) { W[e] = v; });
        if (tid < m) qs.piv[tid] = a.pivs[(size_t)blk * kMaxM + tid];
        sweep = (int)a.sweeps[blk];
        converged = a.conv[blk] != 0;
        __syncthreads();
    }

    if constexpr (PART == 0) run_sweeps<MC, kLPP>(W, m, cn, precond, a, sweep, converged, drop_last);
    const int g = tid / kLPP;
    const int s = tid % kLPP;
    mark(2);
    // sigma_j = |w_j| (gsvd.cpp:677-686), normalize in place
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        const int j = 2 * g + cc;
        if (j < m) {
            double v = 0;
#pragma unroll
            for (int u = 0; u < kRows; ++u) {
                const int row = s + u * kLPP;
                if (row < m) {
                    const double2 w = W[j * m + row];
                    v = fma(w.x, w.x, fma(w.y, w.y, v));
                }
            }
            v = group_sum<kLPP>(v);
            if (s == 0) s_sig[j] = sqrt(v);
        }
    }
    __syncthreads();
    // stable descending rank (gsvd.cpp:331-338)
    if (tid < m) {
        const double v = s_sig[tid];
        int rank = 0;
        for (int k = 0; k < m; ++k) {
            const double o = s_sig[k];
            rank += (o > v) || (o == v && k < tid);
        }
        s_perm[rank] = tid;
    }
    __shared__ double s_inv[kMaxM];  // 1 / sigma_j, one division per column
    if (tid < m) s_inv[tid] = s_sig[tid] > 0 ? 1.0 / s_sig[tid] : 0.0;
    __syncthreads();
    for (int e = tid; e < m * m; e += blockDim.x) W[e] = cscale(s_inv[e / m], W[e]);
    __syncthreads();
    if (precond) {  // left vectors of X -> of A
        if constexpr (PART == 3) back_multiply_mma<jac_threads<MC>()>(W, ag, m, qs, s_sig);
        else back_multiply(W, ag, m, qs, s_sig);
    }
    mark(3);

    // ---- canonicalization (gsvd.cpp:470-565) ---------------------------
    // Structure of the sorted values, by warp 0 with ballots over the ranks
    // (two 32-rank halves): the vanishing suffix, the tied runs above it,
    // the re-orthonormalization line and the dropped / certified lists.
    //
    // Fused path: the final (rotation-free) sweep certified every pair of
    // columns above that sweep's drop line orthogonal (its cn[] are the final
    // squared norms).  Columns at or below the line (sigma <= 1e-10
    // sigma_max, always in the vanishing block) are completed to an
    // orthonormal basis below.  In the preconditioned path u_j = A P x_j /
    // sigma_j carries the Jacobi's residual coupling to larger-sigma vectors
    // amplified by sigma_k / sigma_j; every vector below kReorth sigma_max
    // (and the whole vanishing block) is therefore re-orthonormalized, in rank
    // order, against all larger ones -- which removes exactly those components
    // (the ones above keep an error <= 1/kReorth x the Jacobi's 1e-14
    // relative orthogonality, i.e. <= 1e-9).
    if (tid < kWarp) {
        const int lane = tid;
        const double smax = s_sig[s_perm[0]] > 0 ? s_sig[s_perm[0]] : 0.0;
        const double gap = 1e-5 * smax;  // kDegenerateGap (gsvd.cpp:381)
        double v[2], vn[2];
        int jj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rk = lane + 32 * h;
            jj[h] = rk < m ? s_perm[rk] : 0;
            v[h] = rk < m ? s_sig[jj[h]] : -1.0;
            vn[h] = rk + 1 < m ? s_sig[s_perm[rk + 1]] : -1.0;
        }
        // vanishing values form a suffix of the ranks
        const unsigned van0 = __ballot_sync(0xffffffffu, lane < m && v[0] <= gap);
        const unsigned van1 = __ballot_sync(0xffffffffu, lane + 32 < m && v[1] <= gap);
        const int z = __popc(van0) + __popc(van1);
        const int lead_end = m - z;
        // rank rk ties with rk + 1 (both above the vanishing line)
        const unsigned long long tie =
            (unsigned long long)__ballot_sync(0xffffffffu, lane + 1 < lead_end && v[0] - vn[0] <= gap) |
            ((unsigned long long)__ballot_sync(0xffffffffu, lane + 33 < lead_end && v[1] - vn[1] <= gap) << 32);
        const unsigned long long starts = tie & ~(tie << 1);  // first rank of each tied run
        const unsigned long long ends = tie & ~(tie >> 1);    // last tied rank of each run (its group ends one later)
        int dmax = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rk = lane + 32 * h;
            if (rk < 64 && ((starts >> rk) & 1ull)) {
                const int gi = __popcll(starts & ((1ull << rk) - 1ull));
                const int e = __ffsll((long long)(ends >> rk)) - 1 + rk + 1;  // group's last rank
                cs.groups[gi][0] = rk;
                cs.groups[gi][1] = e;
                dmax = max(dmax, e - rk + 1);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        // the re-orthonormalization line: the first lead rank below kReorth sigma_max
        int r0 = lead_end;
        if (precond) {
            const unsigned b0 = __ballot_sync(0xffffffffu, lane < lead_end && v[0] < kReorth * smax);
            const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < lead_end && v[1] < kReorth * smax);
            if (b0) r0 = __ffs(b0) - 1;
            else if (b1) r0 = 32 + __ffs(b1) - 1;
        }
        // dropped (rank order) and certified lists, by stable compaction
        unsigned dropm[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rk = lane + 32 * h;
            const bool dr = rk < m && (precond ? (rk >= r0) : !(cn[jj[h]] > drop_last));
            dropm[h] = __ballot_sync(0xffffffffu, dr);
        }
        const int nd0 = __popc(dropm[0]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rk = lane + 32 * h;
            if (rk < m) {
                const unsigned below = lane ? (dropm[h] & ((1u << lane) - 1u)) : 0u;
                const int dpos = (h ? nd0 : 0) + __popc(below);
                if ((dropm[h] >> lane) & 1u) cs.dropped[dpos] = jj[h];
                else cs.certcols[rk - dpos] = jj[h];
            }
        }
        if (lane == 0) {
            cs.ndropped = nd0 + __popc(dropm[1]);
            cs.ncert = m - cs.ndropped;
            cs.ngroups = __popcll(starts);
            cs.nvanish = z;
            cs.eligible = a.canonical && !a.refine && converged && dmax <= kZMax && m <= 64;
        }
    }
    __syncthreads();
    // the preconditioned vectors are re-orthonormalized whichever kernel
    // canonicalizes them (the generic one reads the lead vectors too)
    if ((cs.eligible || precond) && cs.ndropped > 0) complete_basis<MC, PART == 3>(W, Y, m, cs);
    mark(4);
    bool fused = cs.eligible;
    int zf = cs.nvanish;  // the vanishing block, when the group machinery below takes it
    if (a.canonical && fused && zf > kZMax) {
        if (!big_vanish<MC>(W, s_perm, m, zf, Y, cs.nrm)) seq_vanish<MC>(W, s_perm, m, zf, Y, Y + kMaxM);
        zf = 0;
    }
    if (a.canonical && fused) {
        const int z = zf;
        // the groups (the vanishing block first, then the tied groups) are
        // disjoint column sets; each runs the QR-form picker
        const int ngt = cs.ngroups + (z > 0 ? 1 : 0);
        auto grp = [&](int gi, int& i0, int& d) {
            if (z > 0 && gi == 0) {
                i0 = m - z;
                d = z;
            } else {
                const int q = gi - (z > 0 ? 1 : 0);
                i0 = cs.groups[q][0];
                d = cs.groups[q][1] - i0 + 1;
            }
        };
        __shared__ int s_fast[kMaxM];
        __shared__ int s_off[kMaxM + 1];
        __shared__ int s_row[kMaxM + 1];
        if (tid == 0) {
            int off = 0, rows = 0;
            for (int gi = 0; gi < ngt; ++gi) {
                int i0, d;
                grp(gi, i0, d);
                s_off[gi] = off;
                s_row[gi] = rows;
                off += 2 * d * d;
                rows += d;
            }
            s_off[ngt] = off;
            s_row[ngt] = rows;
        }
        __syncthreads();
        // groups that do not fit the scratch together, or exceed kZMax, take
        // the sequential picker afterwards
        const bool concurrent = s_off[ngt] <= scratch_entries(MC);
        if (concurrent) {
            for (int gi = 0; gi < ngt; ++gi) {
                int i0, d;
                grp(gi, i0, d);
                if (d <= kZMax) gram_group<MC>(W, s_perm + i0, Y + s_off[gi], m, d);
            }
            __syncthreads();
            const int warp = tid / kWarp;
            for (int gi = warp; gi < ngt; gi += jac_threads<MC>() / kWarp) {
                int i0, d;
                grp(gi, i0, d);
                const bool ok =
                    d <= kZMax && chol_group(Y + s_off[gi], cs.norm0 + i0, cs.nrm + i0, d, z > 0 && gi == 0);
                if ((tid & 31) == 0) s_fast[gi] = ok ? 1 : 0;
            }
            __syncthreads();
            constexpr int kZL = 4;
            for (int r = tid / kZL; r < s_row[ngt]; r += jac_threads<MC>() / kZL) {
                int gi = 0;
                while (s_row[gi + 1] <= r) ++gi;
                if (!s_fast[gi]) continue;  // uniform over the kZL lanes of the row
                int i0, d;
                grp(gi, i0, d);
                const double2* G = Y + s_off[gi];
                z_row<kZL>(W, s_perm + i0, G, Y + s_off[gi] + d * d, cs.nrm + i0, m, d, r - s_row[gi], tid % kZL);
            }
            __syncthreads();
            for (int gi = 0; gi < ngt; ++gi) {
                int i0, d;
                grp(gi, i0, d);
                if (s_fast[gi]) apply_span_z<MC>(W, m, d, s_perm + i0, Y + s_off[gi] + d * d);
            }
        } else {
            for (int gi = tid; gi < ngt; gi += jac_threads<MC>()) s_fast[gi] = 0;
            __syncthreads();
        }
        mark(7);
        for (int gi = 0; gi < ngt; ++gi) {  // after every Z slice is consumed: the scratch is free
            int i0, d;
            grp(gi, i0, d);
            if (s_fast[gi]) continue;
            if (tid < d) cs.cols[tid] = s_perm[i0 + tid];
            __syncthreads();
            pick_in_span(W, Y, m, d, z > 0 && gi == 0, cs);
            apply_span<MC>(W, m, d, cs);
        }
        // phase rule (gsvd.cpp:545-564): eight lanes per vector, four vectors
        // per warp; the first entry of largest magnitude sets the phase
        const int warp = tid / kWarp, lane = tid % kWarp, sl = lane & 7;
        for (int rk0 = 4 * warp; rk0 < m; rk0 += 4 * (jac_threads<MC>() / kWarp)) {
            const int rk = rk0 + (lane >> 3);
            const bool on = rk < m;
            const int j = on ? s_perm[rk] : 0;
            double best = -1;
            int bi = 0;
            if (on) {
                for (int i = sl; i < m; i += 8) {
                    const double2 v = W[j * m + i];
                    const double mg = hypot(v.x, v.y);
                    if (mg > best) {
                        best = mg;
                        bi = i;
                    }
                }
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (on && sl == 0) {
                double2 up = make_double2(1.0, 0.0);
                if (best > 0) {
                    const double2 val = W[j * m + bi];
                    const double av = hypot(val.x, val.y);
                    up = make_double2(val.x / av, -(val.y / av));
                }
                cs.up[rk] = up;
            }
        }
    } else if (tid < m) {
        cs.up[tid] = make_double2(1.0, 0.0);
    }
    __syncthreads();

    mark(5);
    const size_t base = (size_t)blk * m;
    if (tid < m) a.sigma[base + tid] = s_sig[s_perm[tid]];
    double2* eb = a.e + (size_t)blk * m * m;
    for (int e = tid; e < m * m; e += blockDim.x) {
        const int rank = e / m, row = e % m;
        eb[e] = cmul(W[s_perm[rank] * m + row], cs.up[rank]);
    }
    if (tid == 0) {
        a.sweeps[blk] = (uint32_t)sweep;
        a.conv[blk] = converged ? 1 : 0;
    }
    mark(6);
    if (tid == 0) {
        if (a.canonical && !fused) a.work[2 + atomicAdd(a.work, 1u)] = (uint32_t)blk;
    }
}

// The sweeps of the split solver in a recursive bipartite ordering (m = 60
// padded to 64 columns, 32 processors of four lanes, 15 rows per lane):
//   level S = 32, 16, 8, 4, 2, 1 (groups of S processors, 2S columns):
//     every processor keeps a resident BOTTOM column in registers for the
//     whole level, and the group's S TOP columns sit in S slots; each round
//     pairs every bottom with a different top, so that over the level's S
//     rounds every top meets every bottom of the group once: for S >= 8 in
//     blocks of eight warp-local rounds (warp wi of the group visits the
//     tops of warp wi + k/8's slots, processor pw slot (pw + k) mod 8), so a
//     CTA barrier is needed only between blocks, not between rounds;
//     then the group splits: its tops form one group of S/2 processors (the
//     lower half takes the tops of the upper slots as its new bottoms) and
//     its bottoms the other (the lower half's old bottoms become the upper
//     group's tops, in those slots).
// 32 + 16 + 8 + 4 + 2 + 1 = 63 rounds visit each of the 64*63/2 pairs once.
// Slots hold column ids; W stays in shared memory by column id, so a round
// loads and stores ONE column per processor (the top) where the circle
// ordering (run_sweeps) loads and stores both, and 8 CTA barriers per sweep
// replace 59.  Every sweep starts from the same arrangement: carrying the
// end-of-sweep arrangement into the next sweep changes the cyclic order and
// costs a sweep (numpy on the C3 matrices: 8.27 against 7.18 counted sweeps;
// this ordering 7.12 in numpy, 7.18 on the GPU; the circle ordering 7.09 /
// 7.06).  Measured against the circle-ordered kernel it replaced (128
// threads, run_sweeps<60, 4> on W in shared memory) on C3: 206k vs 214k SM cycles per
// CTA-sweep (three CTAs per SM), 20.70 vs 21.04 ms of solver per 32 blocks:
// halving the shared-memory traffic and removing 51 barriers per sweep
// gains only 4% per sweep -- the round is bound by its own dependent chain
// (dot product, shuffle reduction, rotation parameters) at three warps per
// scheduler with the FP64 pipe 52% busy.
// The rotation, skip and convergence rules are the reference's
// (gsvd.cpp:642-674); the Gram certificate is run_sweeps'.
constexpr int kBipRows = 15;  // 60 rows over 4 lanes

// Shared-memory position of column c: columns 4k+2 and 4k+3 trade places.
// The two processors of a quarter-warp load the tops of adjacent slots, and
// the tops start as the even columns: at a column stride of 60 x 16 bytes a
// column's bank half is its parity, so every such pair hit the same 16 banks
// (2-way conflicts on every top load and store, 400M conflicts per 8-block
// launch); with the swap adjacent even columns alternate (1.5% of the pairs
// conflict over a sweep).  W, cn and the Gram certificate all live in
// position space; the ordering works on column ids.
__device__ __forceinline__ int bip_pos(int c) { return c ^ ((c >> 1) & 1); }

// the warps of this thread's S-processor group (eight processors per warp)
__device__ __forceinline__ void bip_group_sync(int S, int warp) {
    if (S >= 32) {
        __syncthreads();
    } else {  // S = 16: a warp pair
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
    }
}

template <int MC>
__global__ void __launch_bounds__(32 * 4, 3) sweep_bip_kernel(GsvdArgs a) {
    static_assert(MC == 4 * kBipRows, "bipartite-ordered sweeps: m = 60");
    if (a.abort && *a.abort) return;
    // the epilogue kernel may be scheduled once every sweep CTA is resident:
    // it fills the SMs this launch's tail leaves idle, bin by bin (a.done)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int m = MC, R = kBipRows;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);  // [column id][row]
    __shared__ double cn[64];
    __shared__ int slot_id[32];
    __shared__ int s_rots;
    __shared__ unsigned s_maxrel;
    const int tid = threadIdx.x;
    const int g = tid >> 2, s = tid & 3;  // processor, lane in it
    const long long clk0 = clock64();
    double2* wg = a.wscratch + (size_t)blockIdx.x * m * m;
    batched_copy<4>(tid, (int)blockDim.x, m * m, wg, [&](int e, double2 v) { W[bip_pos(e / m) * m + e % m] = v; });
    if (tid == 0) {
        s_rots = 0;
        s_maxrel = 0u;
    }
    __syncthreads();
    const int total_pairs = m * (m - 1) / 2;
    int prev_rots = 1 << 30;
    bool prev_maxrel = true;
    int sweep = 0;
    bool converged = false;
    while (sweep < a.max_sweeps) {
        // fresh squared column norms (gsvd.cpp:633-637): four lanes per column
        {
            const int j = tid >> 1, part = tid & 1;
            double v = 0.0;
            if (j < m)
                for (int i = part; i < m; i += 2) v = fma(W[j * m + i].x, W[j * m + i].x, fma(W[j * m + i].y, W[j * m + i].y, v));
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            if (part == 0) cn[j] = j < m ? v : 0.0;
        }
        if (s == 0) slot_id[g] = 2 * g;  // the sweep's starting arrangement: tops 2g
        __syncthreads();
        // the Gram certificate of a probably rotation-free sweep (see run_sweeps)
        if (sweep > 0 && (2 * prev_rots < total_pairs || !prev_maxrel) &&
            gram_converged<MC, 4, 4>(W, m, cn, 0.0, a.tol2)) {
            converged = true;
            break;
        }
        int qid = 2 * g + 1;  // resident bottom
        double2 Q[R];
#pragma unroll
        for (int u = 0; u < R; ++u) Q[u] = qid < m ? W[bip_pos(qid) * m + s + 4 * u] : make_double2(0, 0);
        double cq = cn[bip_pos(qid)];
        bool qdirty = false;
        __syncthreads();  // every thread has read s_rots / s_maxrel
        if (tid == 0) {
            s_rots = 0;
            s_maxrel = 0u;
        }
        int myrots = 0;
        double mymax = 0.0;
        bool rot = false;
#pragma unroll 1
        for (int S = 32; S >= 1; S >>= 1) {
            const int b = g & ~(S - 1), pos = g - b;
            const int wi = pos >> 3, pw = pos & 7, nw = S >> 3;  // S >= 8: warp in the group, processor in the warp
#pragma unroll 1
            for (int k = 0; k < S; ++k) {
                // S >= 8: blocks of eight warp-local rounds over one slot
                // region (the tops of warp wi + k/8 of the group)
                const int sl = S >= 8 ? b + (((wi + (k >> 3)) & (nw - 1)) << 3) + ((pw + k) & 7)
                                      : b + ((pos + k) & (S - 1));
                const int pid = slot_id[sl];
                if (pid < m && qid < m) {
                    double2 P[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) P[u] = W[bip_pos(pid) * m + s + 4 * u];
                    double cp = cn[bip_pos(pid)];
                    if (rotate_pair<R, 4>(P, Q, cp, cq, 0.0, s, m, mymax, a.tol2)) {
#pragma unroll
                        for (int u = 0; u < R; ++u) W[bip_pos(pid) * m + s + 4 * u] = P[u];
                        __syncwarp(group_mask<4>());  // the group's loads of cn[bip_pos(pid)] precede the write
                        if (s == 0) {
                            cn[bip_pos(pid)] = cp;
                            ++myrots;
                        }
                        qdirty = true;
                        rot = true;
                    }
                }
                if (S >= 16 && (k & 7) == 7) {
                    bip_group_sync(S, tid >> 5);  // the next block reads another warp's slots
                } else {
                    __syncwarp();
                }
            }
            if (S == 1) break;
            // split: the lower half swaps its bottom with the top in slot
            // b + S/2 + pos (that top becomes its bottom, its bottom a top of
            // the upper half's group)
            const int h = S >> 1;
            if (pos < h) {
                const int sl = b + h + pos;
                const int nid = slot_id[sl];
                if (qid < m) {
                    if (qdirty) {
#pragma unroll
                        for (int u = 0; u < R; ++u) W[bip_pos(qid) * m + s + 4 * u] = Q[u];
                    }
                    __syncwarp(group_mask<4>());
                    if (s == 0) cn[bip_pos(qid)] = cq;
                }
                qdirty = false;
#pragma unroll
                for (int u = 0; u < R; ++u) Q[u] = nid < m ? W[bip_pos(nid) * m + s + 4 * u] : make_double2(0, 0);
                cq = cn[bip_pos(nid)];
                __syncwarp(group_mask<4>());
                if (s == 0) slot_id[sl] = qid;
                qid = nid;
            }
            if (S >= 16) {
                bip_group_sync(S, tid >> 5);
            } else {
                __syncwarp();
            }
        }
        // the resident bottoms go home
        if (qid < m && qdirty) {
#pragma unroll
            for (int u = 0; u < R; ++u) W[bip_pos(qid) * m + s + 4 * u] = Q[u];
        }
        ++sweep;
        if (s == 0 && myrots) {
            atomicAdd(&s_rots, myrots);
            if (mymax > 0) atomicMax(&s_maxrel, 1u);
        }
        if (!__syncthreads_or(rot)) {
            converged = true;
            break;
        }
        prev_rots = s_rots;
        prev_maxrel = s_maxrel != 0u;
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += blockDim.x) wg[e] = W[bip_pos(e / m) * m + e % m];
    if (tid == 0) {
        a.sweeps[blockIdx.x] = (uint32_t)sweep;
        a.conv[blockIdx.x] = converged ? 1 : 0;
    }
    if (a.done) {  // release this bin to the epilogue: every thread's stores, then the epoch
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release_gpu(a.done + blockIdx.x, a.epoch);
        }
    }
    if (tid == 0) {
        if (a.phase_clk)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.phase_clk + 2), (unsigned long long)(clock64() - clk0));
    }
}

int launch_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    auto launch = [&](auto kern, int threads, int mc) {
        const size_t smem = (size_t)a.m * a.m * sizeof(double2) + (size_t)scratch_entries(mc) * sizeof(double2);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nblk * a.bins, threads, smem, s>>>(a);
    };
    if (a.m == 60 && a.precondition && a.ascratch && a.wscratch && a.pivs) {
        // split around the 128-thread sweep kernel
        launch(jacobi_kernel<60, 1>, jac_threads<60>(), 60);
        const size_t smem = (size_t)60 * 60 * sizeof(double2);
        cudaFuncSetAttribute(sweep_bip_kernel<60>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sweep_bip_kernel<60><<<nblk * a.bins, 128, smem, s>>>(a);
        if (a.done && a.epoch) {
            // programmatic dependent launch: the epilogue's CTAs start as the
            // sweep kernel's tail frees SMs, each waiting only for its own
            // bin (a.done holds the epoch once its sweeps are stored).  The
            // launch waits until every sweep CTA has started, so a waiting
            // epilogue CTA never holds an SM a sweep CTA still needs.  (The
            // same hand-off from the prologue to the sweep kernel measured
            // slower: 1640 vs 1659 blocks/s at C3.)
            auto pdl = [&](auto kern, int threads, size_t dsmem) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(nblk * a.bins);
                cfg.blockDim = dim3(threads);
                cfg.dynamicSmemBytes = dsmem;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, kern, a);
            };
            pdl(jacobi_kernel<60, 3>, jac_threads<60>(), smem + (size_t)scratch_entries(60) * sizeof(double2));
        } else {
            launch(jacobi_kernel<60, 3>, jac_threads<60>(), 60);
        }
        return 3;
    }
    if (small_jacobi_selected(a)) {  // C1 / C2 sizes: a lane group per bin
        launch_small_jacobi(a, nblk, s);
        return 1;
    }
    switch (a.m) {  // the BASELINE configs' channel counts get specialized code
        case 8: launch(jacobi_kernel<8>, jac_threads<8>(), 8); break;
        case 16: launch(jacobi_kernel<16>, jac_threads<16>(), 16); break;
        case 60: launch(jacobi_kernel<60>, jac_threads<60>(), 60); break;
        case 64: launch(jacobi_kernel<64>, jac_threads<64>(), 64); break;
        default: launch(jacobi_kernel<0>, jac_threads<0>(), 0); break;
    }
    return 1;
}

}  // namespace sslg
