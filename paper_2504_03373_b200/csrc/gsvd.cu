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

constexpr int kJacThreads = 256;
constexpr int kLPP = 8;              // lanes per column pair
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

__global__ void __launch_bounds__(kJacThreads, 2) jacobi_kernel(GsvdArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    double2* W = reinterpret_cast<double2*>(smem_raw);  // [m cols][m rows]
    double2* Y = W + m * m;                             // [kMaxM][kYld] picker coordinates
    __shared__ double cn[kMaxM];
    __shared__ double s_drop;
    __shared__ int s_perm[kMaxM];  // rank -> column
    __shared__ double s_sig[kMaxM];
    __shared__ CanonScratch cs;

    const int blk = blockIdx.x;
    const int bin = blk % a.bins;
    const int tid = threadIdx.x;

    form_whitened(a.r + (size_t)blk * m * m, a.kinv + (size_t)bin * m * m, m, W);

    const int n_even = (m + 1) & ~1;
    const int npairs = n_even / 2;
    const int g = tid / kLPP;
    const int s = tid % kLPP;

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
            if (tid == 0) s_drop = 1e-20 * mx;
        }
        __syncthreads();
        const double drop = s_drop;
        bool rot = false;
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                if (q < m) {
                    double2 wp[kRows], wq[kRows];
                    double d0x = 0, d0y = 0, d1x = 0, d1y = 0;
#pragma unroll
                    for (int u = 0; u < kRows; ++u) {
                        const int row = s + u * kLPP;
                        if (row < m) {
                            wp[u] = W[p * m + row];
                            wq[u] = W[q * m + row];
                            // conj(wp) * wq, two independent accumulators
                            if (u & 1) {
                                d1x = fma(wp[u].x, wq[u].x, fma(wp[u].y, wq[u].y, d1x));
                                d1y = fma(wp[u].x, wq[u].y, fma(-wp[u].y, wq[u].x, d1y));
                            } else {
                                d0x = fma(wp[u].x, wq[u].x, fma(wp[u].y, wq[u].y, d0x));
                                d0y = fma(wp[u].x, wq[u].y, fma(-wp[u].y, wq[u].x, d0y));
                            }
                        }
                    }
                    const double2 dot = group_sum2<kLPP>(make_double2(d0x + d1x, d0y + d1y));
                    const double cp = cn[p], cq = cn[q];
                    const double mag2 = fma(dot.x, dot.x, dot.y * dot.y);
                    if (!(cp <= drop || cq <= drop) && !(mag2 <= 1e-28 * cp * cq)) {
                        // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = (cq - cp) / (2 |apq|)
                        const double inv_mag = rsqrt(mag2);
                        const double mag = mag2 * inv_mag;
                        const double phx = dot.x * inv_mag, phy = dot.y * inv_mag;
                        const double tau = (cq - cp) * (0.5 * inv_mag);
                        const double tt = fma(tau, tau, 1.0);
                        const double t = copysign(1.0, tau) / (fabs(tau) + tt * rsqrt(tt));
                        const double c = rsqrt(fma(t, t, 1.0));
                        const double sn = t * c;
                        const double alx = sn * phx, aly = -sn * phy;  // s * conj(ph)
                        const double bex = c * phx, bey = -c * phy;    // c * conj(ph)
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            if (row < m) {
                                const double2 x = wp[u], y = wq[u];
                                double2 np, nq;
                                np.x = fma(c, x.x, fma(-alx, y.x, aly * y.y));
                                np.y = fma(c, x.y, fma(-alx, y.y, -aly * y.x));
                                nq.x = fma(sn, x.x, fma(bex, y.x, -bey * y.y));
                                nq.y = fma(sn, x.y, fma(bex, y.y, bey * y.x));
                                W[p * m + row] = np;
                                W[q * m + row] = nq;
                            }
                        }
                        if (s == 0) {
                            const double cs2 = 2.0 * c * sn * mag;
                            cn[p] = c * c * cp - cs2 + sn * sn * cq;
                            cn[q] = sn * sn * cp + cs2 + c * c * cq;
                        }
                        rot = true;
                    }
                }
            }
            __syncthreads();
        }
        ++sweep;
        if (!__syncthreads_or(rot)) {
            converged = true;
            break;
        }
    }

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
        int nd = 0;
        for (int j = 0; j < m; ++j) {
            const bool dropped = !(cn[j] > s_drop);
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
    if (cs.eligible && cs.ndropped > 0) complete_basis(W, m, cs);
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
        if (a.canonical && !fused) a.work[2 + atomicAdd(a.work, 1u)] = (uint32_t)blk;
    }
}

size_t jacobi_smem_bytes(int m) { return (size_t)m * m * sizeof(double2) + (size_t)kMaxM * kYld * sizeof(double2); }

void launch_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = jacobi_smem_bytes(a.m);
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    jacobi_kernel<<<nblk * a.bins, kJacThreads, smem, s>>>(a);
}

}  // namespace sslg
