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

namespace sslg {

#ifndef SSLG_JAC_LPP
#define SSLG_JAC_LPP 8
#endif
constexpr int kLPP = SSLG_JAC_LPP;   // lanes per column pair
constexpr int kJacThreads = 32 * kLPP;  // 32 column-pair groups
constexpr int kRows = kMaxM / kLPP;  // rows per lane (8)
constexpr int kZMax = 24;            // largest group handled by the fused picker
constexpr int kYld = kZMax + 1;      // padded row stride of the coordinate buffer

struct CanonScratch {
    double nrm[kMaxM];
    double norm0[kMaxM];
    double2 q[kZMax];
    double2 z[kZMax][kZMax];  // accepted coordinate vectors, column t = vector t
    int cols[kMaxM];          // W columns of the current group
    int groups[kMaxM][2];     // rank ranges of tied groups
    double2 up[kMaxM];        // phase factor per rank
    unsigned ball[2];
    int cert[kMaxM];          // column certified orthonormal to the others
    int dropped[kMaxM];       // columns below the final sweep's drop line
    double2 dots[kMaxM];
    double nrm1;
    int ngroups, nvanish, eligible, ndropped;
};

// Completes the basis: every column below the drop line is orthonormalized
// (two classical Gram-Schmidt passes) against all certified columns, then
// certified itself.  Clears cs.eligible if a column collapses.
__device__ void complete_basis(double2* W, int m, CanonScratch& cs) {
    const int t = threadIdx.x;
    const int k = t >> 2, part = t & 3;  // 4 lanes per column / row
    for (int qd = 0; qd < cs.ndropped; ++qd) {
        const int jd = cs.dropped[qd];
        for (int pass = 0; pass < 2; ++pass) {
            double2 d = make_double2(0, 0);
            if (k < m && k != jd && cs.cert[k])
                for (int i = part; i < m; i += 4) {
                    const double2 a = W[k * m + i], b = W[jd * m + i];
                    d.x = fma(a.x, b.x, fma(a.y, b.y, d.x));
                    d.y = fma(a.x, b.y, fma(-a.y, b.x, d.y));
                }
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 1);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 1);
            d.x += __shfl_xor_sync(0xffffffffu, d.x, 2);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, 2);
            if (k < m && part == 0) cs.dots[k] = (k != jd && cs.cert[k]) ? d : make_double2(0, 0);
            __syncthreads();
            // row i = k: w_jd[i] -= sum_kk dots[kk] e_kk[i]
            double2 acc = make_double2(0, 0);
            if (k < m)
                for (int kk = part; kk < m; kk += 4) {
                    const double2 dk = cs.dots[kk], e = W[kk * m + k];
                    acc.x = fma(dk.x, e.x, fma(-dk.y, e.y, acc.x));
                    acc.y = fma(dk.x, e.y, fma(dk.y, e.x, acc.y));
                }
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
            __syncthreads();
            if (k < m && part == 0) W[jd * m + k] = csub(W[jd * m + k], acc);
            __syncthreads();
        }
        if (t < kWarp) {
            double v = 0;
            for (int i = t; i < m; i += kWarp) v += cnorm(W[jd * m + i]);
            v = group_sum<kWarp>(v);
            if (t == 0) cs.nrm1 = sqrt(v);
        }
        __syncthreads();
        const double nrm = cs.nrm1;
        if (!(nrm > 1e-6)) {  // collapsed: leave this bin to the generic kernel
            if (t == 0) cs.eligible = 0;
            __syncthreads();
            return;
        }
        if (t < m) W[jd * m + t] = cscale(1.0 / nrm, W[jd * m + t]);
        if (t == 0) cs.cert[jd] = 1;
        __syncthreads();
    }
}

// Reference picker (pick_orthonormal, gsvd.cpp:404-436) on the coordinates of
// one group: candidate j is row j of conj(N), N = W[cols[0..d)].  Threads
// j < m own candidate j; the accepted coordinate vectors land in cs.z.
__device__ void pick_in_span(const double2* W, double2* Y, int m, int d, bool unit_norm0, CanonScratch& cs) {
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
__device__ void apply_span(double2* W, int m, int d, CanonScratch& cs) {
    const int t = threadIdx.x;
    double2 out[6];
    int cnt = 0;
    for (int e = t; e < m * d && cnt < 6; e += blockDim.x, ++cnt) {
        const int i = e % m, s = e / m;
        double2 acc = make_double2(0, 0);
        for (int k = 0; k < d; ++k) {
            const double2 a = W[cs.cols[k] * m + i], b = cs.z[k][s];
            acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
            acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
        }
        out[cnt] = acc;
    }
    __syncthreads();
    cnt = 0;
    for (int e = t; e < m * d && cnt < 6; e += blockDim.x, ++cnt) W[cs.cols[e / m] * m + (e % m)] = out[cnt];
    __syncthreads();
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
    double nrm2[kMaxM];
    int piv[kMaxM];  // column k of A P is column piv[k] of A
    double2 u0, beta;
    double tau;
    int p;
};

__device__ void qrcp_to_rh(double2* W, int m, QrScratch& qs) {
    const int t = threadIdx.x, warp = t / kWarp, lane = t % kWarp;
    constexpr int kWarps = kJacThreads / kWarp;
    for (int j = warp; j < m; j += kWarps) {
        double v = 0;
        for (int i = lane; i < m; i += kWarp) v += cnorm(W[j * m + i]);
        v = group_sum<kWarp>(v);
        if (lane == 0) qs.nrm2[j] = v;
    }
    if (t < m) qs.piv[t] = t;
    __syncthreads();
    for (int k = 0; k < m; ++k) {
        // warp 0 alone: pivot (first column of largest remaining norm), column
        // swap, and the reflector H = I - tau u u^H with H x = beta e_k
        if (warp == 0) {
            double best = -1;
            int bi = k;
            for (int j = k + lane; j < m; j += kWarp)
                if (qs.nrm2[j] > best) {
                    best = qs.nrm2[j];
                    bi = j;
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            const int p = bi;
            double a2 = 0;
            for (int i = lane; i < m; i += kWarp) {
                double2 xk = W[k * m + i];
                if (p != k) {
                    const double2 xp = W[p * m + i];
                    W[p * m + i] = xk;
                    W[k * m + i] = xp;
                    xk = xp;
                }
                if (i >= k) a2 = fma(xk.x, xk.x, fma(xk.y, xk.y, a2));
            }
            a2 = group_sum<kWarp>(a2);
            __syncwarp();
            if (lane == 0) {
                if (p != k) {
                    const double x = qs.nrm2[k];
                    qs.nrm2[k] = qs.nrm2[p];
                    qs.nrm2[p] = x;
                    const int i = qs.piv[k];
                    qs.piv[k] = qs.piv[p];
                    qs.piv[p] = i;
                }
                const double2 x0 = W[k * m + k];
                const double alpha = sqrt(a2);
                const double ax2 = fma(x0.x, x0.x, x0.y * x0.y);
                double2 ph = make_double2(1.0, 0.0);
                double ax0 = 0.0;
                if (ax2 > 0) {
                    const double ri = fast_rsqrt(ax2);
                    ax0 = ax2 * ri;
                    ph = make_double2(x0.x * ri, x0.y * ri);
                }
                qs.beta = make_double2(-ph.x * alpha, -ph.y * alpha);
                qs.u0 = make_double2(x0.x + ph.x * alpha, x0.y + ph.y * alpha);
                qs.tau = alpha > 0 ? fast_rcp(alpha * (alpha + ax0)) : 0.0;
            }
        }
        __syncthreads();
        const double tau = qs.tau;
        const double2 u0 = qs.u0;
        if (tau != 0.0) {  // trailing columns, 4 lanes per column, all in parallel
            const int j = k + 1 + (t >> 2), part = t & 3;
            double2 sdot = make_double2(0, 0);
            if (j < m)
                for (int i = k + 1 + part; i < m; i += 4) {
                    const double2 u = W[k * m + i], y = W[j * m + i];
                    sdot.x = fma(u.x, y.x, fma(u.y, y.y, sdot.x));
                    sdot.y = fma(u.x, y.y, fma(-u.y, y.x, sdot.y));
                }
            sdot.x += __shfl_xor_sync(0xffffffffu, sdot.x, 1);
            sdot.y += __shfl_xor_sync(0xffffffffu, sdot.y, 1);
            sdot.x += __shfl_xor_sync(0xffffffffu, sdot.x, 2);
            sdot.y += __shfl_xor_sync(0xffffffffu, sdot.y, 2);
            if (j < m) {
                const double2 yk = W[j * m + k];
                sdot.x = fma(u0.x, yk.x, fma(u0.y, yk.y, sdot.x));
                sdot.y = fma(u0.x, yk.y, fma(-u0.y, yk.x, sdot.y));
                const double2 f = cscale(tau, sdot);
                for (int i = k + 1 + part; i < m; i += 4) W[j * m + i] = csub(W[j * m + i], cmul(f, W[k * m + i]));
            }
            __syncwarp();  // every lane of the group has read y_k
            if (j < m) {
                const double2 yk = W[j * m + k];
                const double2 f = cscale(tau, sdot);
                if (part == 0) {
                    const double2 nk = csub(yk, cmul(f, u0));
                    W[j * m + k] = nk;
                    qs.nrm2[j] = fmax(0.0, qs.nrm2[j] - cnorm(nk));
                }
            }
        }
        __syncthreads();
        if (t == 0) W[k * m + k] = qs.beta;
    }
    __syncthreads();
    // X = R^H: column j of X is the conjugated row j of R (lower triangular)
    for (int e = t; e < m * m; e += blockDim.x) {
        const int j = e / m, i = e % m;  // X column j, row i
        if (i > j) {
            const double2 rji = W[i * m + j];
            W[j * m + i] = cconj(rji);
            W[i * m + j] = make_double2(0, 0);
        } else if (i == j) {
            W[e] = cconj(W[e]);
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
    const int i = active ? t / parts : 0;
    const int part = active ? t % parts : 0;
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

// One Jacobi pair in registers (gsvd.cpp:642-672): P is the lower-index
// column.  Returns whether a rotation was applied.
template <int R, int L>
__device__ __forceinline__ bool rotate_pair(double2 (&P)[R], double2 (&Q)[R], double& cp, double& cq, double drop,
                                            int s, int m) {
    double d0x = 0, d0y = 0, d1x = 0, d1y = 0;
#pragma unroll
    for (int u = 0; u < R; ++u) {
        if (s + u * L < m) {  // conj(p) * q, two independent accumulators
            if (u & 1) {
                d1x = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d1x));
                d1y = fma(P[u].x, Q[u].y, fma(-P[u].y, Q[u].x, d1y));
            } else {
                d0x = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d0x));
                d0y = fma(P[u].x, Q[u].y, fma(-P[u].y, Q[u].x, d0y));
            }
        }
    }
    const double2 dot = group_sum2<L>(make_double2(d0x + d1x, d0y + d1y));
    const double mag2 = fma(dot.x, dot.x, dot.y * dot.y);
    if (cp <= drop || cq <= drop || mag2 <= 1e-28 * cp * cq) return false;
    // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = (cq - cp) / (2 |apq|)
    const double inv_mag = fast_rsqrt(mag2);
    const double mag = mag2 * inv_mag;
    const double phx = dot.x * inv_mag, phy = dot.y * inv_mag;
    const double tau = (cq - cp) * (0.5 * inv_mag);
    const double atau = fabs(tau);
    double t;
    if (atau < 1e150) {
        const double tt = fma(tau, tau, 1.0);
        t = copysign(fast_rcp(atau + tt * fast_rsqrt(tt)), tau);
    } else {  // tau^2 would overflow: t = 1 / (2 |tau|)
        t = copysign(0.5 / atau, tau);
    }
    const double c = fast_rsqrt(fma(t, t, 1.0));
    const double sn = t * c;
    const double alx = sn * phx, aly = -sn * phy;  // s * conj(ph)
    const double bex = c * phx, bey = -c * phy;    // c * conj(ph)
#pragma unroll
    for (int u = 0; u < R; ++u) {
        const double2 x = P[u], y = Q[u];
        P[u].x = fma(c, x.x, fma(-alx, y.x, aly * y.y));
        P[u].y = fma(c, x.y, fma(-alx, y.y, -aly * y.x));
        Q[u].x = fma(sn, x.x, fma(bex, y.x, -bey * y.y));
        Q[u].y = fma(sn, x.y, fma(bex, y.y, bey * y.x));
    }
    const double cs2 = 2.0 * c * sn * mag;
    const double np = c * c * cp - cs2 + sn * sn * cq;
    cq = sn * sn * cp + cs2 + c * c * cq;
    cp = np;
    return true;
}

// True iff every pair of columns above the drop line satisfies the
// reference's no-rotation test |x_p^H x_q|^2 <= 1e-28 |x_p|^2 |x_q|^2, i.e.
// iff the next sweep would rotate nothing (gsvd.cpp:642-649).  Evaluated as
// one 4x4-register-tiled Gram product over the upper triangle instead of a
// full verification sweep of round-synchronized pair visits.
__device__ bool gram_converged(const double2* W, int m, const double* cn, double drop) {
    constexpr int TS = 2;  // 2x2 tiles keep the kernel's register budget
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
        for (int k = 0; k < m; ++k) {
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
#pragma unroll
        for (int u = 0; u < TS; ++u)
#pragma unroll
            for (int v = 0; v < TS; ++v) {
                const int p = p0 + u, q = q0 + v;
                if (p < q && q < m && cn[p] > drop && cn[q] > drop) {
                    const double mag2 = fma(acc[u][v].x, acc[u][v].x, acc[u][v].y * acc[u][v].y);
                    if (mag2 > 1e-28 * cn[p] * cn[q]) bad = true;
                }
            }
    }
    return !__syncthreads_or(bad);
}

// MC > 0: channel count fixed at compile time (loop bounds, predicates and
// addressing fold away); MC == 0: any m <= 64 at run time.
template <int MC>
__global__ void __launch_bounds__(kJacThreads, 2) jacobi_kernel(GsvdArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = MC > 0 ? MC : a.m;
    double2* W = reinterpret_cast<double2*>(smem_raw);  // [m cols][m rows]
    double2* Y = W + m * m;                             // [kMaxM][kYld] picker coordinates
    __shared__ double cn[kMaxM];
    __shared__ double s_drop;
    __shared__ int s_perm[kMaxM];  // rank -> column
    __shared__ double s_sig[kMaxM];
    __shared__ CanonScratch cs;
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
    form_whitened(a.r + (size_t)blk * m * m, a.kinv + (size_t)bin * m * m, m, W);
    mark(0);
    const bool precond = a.precondition && a.ascratch;
    double2* ag = precond ? a.ascratch + (size_t)blk * m * m : nullptr;
    if (precond) {
        for (int e = tid; e < m * m; e += blockDim.x) ag[e] = W[e];
        qrcp_to_rh(W, m, qs);
    }
    mark(1);

    const int g = tid / kLPP;
    const int s = tid % kLPP;
    const int n_even = (m + 1) & ~1;
    const int npairs = n_even / 2;

    __shared__ int s_rots;
    if (tid == 0) s_rots = 0;
    int prev_rots = 1 << 30;
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
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    if (row < m) {
                        const double2 w = W[j * m + row];
                        v = fma(w.x, w.x, fma(w.y, w.y, v));
                    }
                }
                v = group_sum<kLPP>(v);
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
        // A sweep after one that rotated few pairs is usually rotation-free:
        // certify that with one Gram product instead of running it.
        if (sweep > 0 && 16 * prev_rots < total_pairs && gram_converged(W, m, cn, drop)) {
            converged = true;
            break;
        }
        if (tid == 0) s_rots = 0;
        int myrots = 0;
        bool rot = false;
        // round-robin (circle) ordering: the m/2 disjoint pairs of a round
        // rotate concurrently, one kLPP-lane group per pair
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                if (q < m) {
                    double2 P[kRows], Q[kRows];
#pragma unroll
                    for (int u = 0; u < kRows; ++u) {
                        const int row = s + u * kLPP;
                        P[u] = row < m ? W[p * m + row] : make_double2(0, 0);
                        Q[u] = row < m ? W[q * m + row] : make_double2(0, 0);
                    }
                    double cp = cn[p], cq = cn[q];
                    if (rotate_pair<kRows, kLPP>(P, Q, cp, cq, drop, s, m)) {
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            if (row < m) {
                                W[p * m + row] = P[u];
                                W[q * m + row] = Q[u];
                            }
                        }
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
        if (myrots) atomicAdd(&s_rots, myrots);
        if (!__syncthreads_or(rot)) {
            converged = true;
            break;
        }
        prev_rots = s_rots;
    }

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
    for (int e = tid; e < m * m; e += blockDim.x) {
        const int j = e / m;
        const double nrm = s_sig[j];
        W[e] = nrm > 0 ? cscale(1.0 / nrm, W[e]) : make_double2(0, 0);
    }
    __syncthreads();
    if (precond) back_multiply(W, ag, m, qs, s_sig);  // left vectors of X -> of A
    mark(3);

    // ---- canonicalization (gsvd.cpp:470-565) ---------------------------
    if (tid == 0) {
        const double smax = s_sig[s_perm[0]] > 0 ? s_sig[s_perm[0]] : 0.0;
        const double gap = 1e-5 * smax;  // kDegenerateGap (gsvd.cpp:381)
        int z = 0;
        while (z < m && s_sig[s_perm[m - 1 - z]] <= gap) ++z;
        const int lead_end = m - z;
        int ng = 0, dmax = z;
        for (int i = 0; i < lead_end;) {
            int end = i;
            while (end + 1 < lead_end && s_sig[s_perm[end]] - s_sig[s_perm[end + 1]] <= gap) ++end;
            if (end > i) {
                cs.groups[ng][0] = i;
                cs.groups[ng][1] = end;
                ++ng;
                dmax = max(dmax, end - i + 1);
            }
            i = end + 1;
        }
        // fused path: the final (rotation-free) sweep certified every pair of
        // columns above that sweep's drop line orthogonal (its cn[] are the
        // final squared norms).  Columns at or below the line (sigma <=
        // 1e-10 sigma_max, always in the vanishing block) are completed to an
        // orthonormal basis below.
        // In the preconditioned path u_j = A P x_j / sigma_j carries the
        // Jacobi's residual coupling to larger-sigma vectors amplified by
        // sigma_k / sigma_j; every vector below 1e-4 sigma_max (and the whole
        // vanishing block) is therefore re-orthonormalized, in rank order,
        // against all larger ones — which removes exactly those components
        // (the ones above keep an error <= 1e4 x the Jacobi tolerance).
        int r0 = lead_end;
        if (precond)
            for (int rk = 0; rk < lead_end; ++rk)
                if (s_sig[s_perm[rk]] < 1e-4 * smax) {
                    r0 = rk;
                    break;
                }
        int nd = 0;
        for (int rk = 0; rk < m; ++rk) {
            const int j = s_perm[rk];
            const bool dropped = precond ? (rk >= r0) : !(cn[j] > s_drop);
            cs.cert[j] = dropped ? 0 : 1;
            if (dropped) cs.dropped[nd++] = j;
        }
        cs.ndropped = nd;
        const bool clean = converged;
        cs.ngroups = ng;
        cs.nvanish = z;
        cs.eligible = a.canonical && !a.refine && clean && dmax <= kZMax && m <= 64;
    }
    __syncthreads();
    // the preconditioned vectors are re-orthonormalized whichever kernel
    // canonicalizes them (the generic one reads the lead vectors too)
    if ((cs.eligible || precond) && cs.ndropped > 0) complete_basis(W, m, cs);
    mark(4);
    const bool fused = cs.eligible;
    if (a.canonical && fused) {
        const int z = cs.nvanish;
        if (z > 0) {
            if (tid < z) cs.cols[tid] = s_perm[m - z + tid];
            __syncthreads();
            pick_in_span(W, Y, m, z, true, cs);
            apply_span(W, m, z, cs);
        }
        for (int gi = 0; gi < cs.ngroups; ++gi) {
            const int i0 = cs.groups[gi][0];
            const int d = cs.groups[gi][1] - i0 + 1;
            if (tid < d) cs.cols[tid] = s_perm[i0 + tid];
            __syncthreads();
            pick_in_span(W, Y, m, d, false, cs);
            apply_span(W, m, d, cs);
        }
        // phase rule (gsvd.cpp:545-564): warp per vector
        const int warp = tid / kWarp, lane = tid % kWarp;
        for (int rk = warp; rk < m; rk += kJacThreads / kWarp) {
            const int j = s_perm[rk];
            double best = -1;
            int bi = 0;
            for (int i = lane; i < m; i += kWarp) {
                const double2 v = W[j * m + i];
                const double mg = hypot(v.x, v.y);
                if (mg > best) {
                    best = mg;
                    bi = i;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (lane == 0) {
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

size_t jacobi_smem_bytes(int m) { return (size_t)m * m * sizeof(double2) + (size_t)kMaxM * kYld * sizeof(double2); }

void launch_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = jacobi_smem_bytes(a.m);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nblk * a.bins, kJacThreads, smem, s>>>(a);
    };
    switch (a.m) {  // the BASELINE configs' channel counts get specialized code
        case 8: launch(jacobi_kernel<8>); break;
        case 16: launch(jacobi_kernel<16>); break;
        case 60: launch(jacobi_kernel<60>); break;
        case 64: launch(jacobi_kernel<64>); break;
        default: launch(jacobi_kernel<0>); break;
    }
}

}  // namespace sslg
