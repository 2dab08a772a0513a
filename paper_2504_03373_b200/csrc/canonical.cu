// Kernel (2b): canonical bases for degenerate singular groups, FP64.
//
// Restates canonicalize_subspaces (reference proj/src/gsvd.cpp:470-565) for
// one (block, bin) per CTA, on the sorted left vectors written by the Jacobi
// kernel:
//   (a) trailing values <= 1e-5 * sigma_max ("vanishing", gsvd.cpp:479-500):
//       lead vectors sharpened by one A A^H subspace step + two-pass
//       Gram-Schmidt (refine_leading, 440-466), then the canonical complement
//       picked from e_0 .. e_{n-1} in index order with accept thresholds
//       {0.05, 1e-8, 0} (pick_orthonormal, 404-436);
//   (b) runs of tied values (adjacent gap <= 1e-5 * sigma_max, 505-543):
//       basis rebuilt from the group projector applied to e_j, same picker;
//   (c) phase: largest-magnitude entry of every vector made real positive
//       (545-564).
// The picker's "visit candidates in index order, project out what was taken
// so far" is run right-looking: when a vector is accepted every remaining
// candidate is orthogonalized against it (twice), so the next candidate's
// residual is ready without a sequential sweep over the taken set.  The
// A A^H step and the projector products are 4x4-register-tiled complex GEMMs
// over SMEM-resident operands.
#include "common.cuh"
#include "kernels.cuh"
#include "whiten.cuh"

namespace sslg {

constexpr int kCanThreads = 256;

// C(i,j) = sum_k fa(i,k) fb(k,j) for i < M, j < N; one 4x4 tile per thread
// (M, N <= 64 with 256 threads).  Results are held in registers across a
// barrier so `fo` may overwrite an operand.
template <class FA, class FB, class FO>
__device__ __forceinline__ void cgemm(int M, int N, int K, FA fa, FB fb, FO fo) {
    const int tn = (N + 3) / 4;
    const int tiles = ((M + 3) / 4) * tn;
    const int t = threadIdx.x;
    double2 acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = make_double2(0, 0);
    const int i0 = (t / tn) * 4, j0 = (t % tn) * 4;
    if (t < tiles) {
        for (int k = 0; k < K; ++k) {
            double2 av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) av[u] = (i0 + u < M) ? fa(i0 + u, k) : make_double2(0, 0);
#pragma unroll
            for (int v = 0; v < 4; ++v) bv[v] = (j0 + v < N) ? fb(k, j0 + v) : make_double2(0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = cadd(acc[u][v], cmul(av[u], bv[v]));
        }
    }
    __syncthreads();
    if (t < tiles) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (i0 + u < M && j0 + v < N) fo(i0 + u, j0 + v, acc[u][v]);
    }
    __syncthreads();
}

struct PickScratch {
    double norm0[kMaxM];
    double nrm[kMaxM];
    double2 dot[kMaxM];
    double2 q[kMaxM];
    int used[kMaxM];
    int sel;
    int taken;
};

// squared norms of candidate columns k (not used) of cand, 4 threads per column
__device__ __forceinline__ void cand_norms(const double2* cand, int m, PickScratch& ps, bool into_norm0) {
    const int t = threadIdx.x;
    const int k = t >> 2, part = t & 3;
    double v = 0;
    if (k < m)
        for (int i = part; i < m; i += 4) v += cnorm(cand[k * m + i]);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (k < m && part == 0) {
        if (into_norm0) ps.norm0[k] = sqrt(v);
        ps.nrm[k] = sqrt(v);
    }
}

// pick_orthonormal (gsvd.cpp:404-436), right-looking over the candidate
// columns of `cand` (already projected against the exclude set).  Accepted
// vectors go to out[(off + t) * m + i].
__device__ void pick_right_looking(double2* cand, int m, int need, double2* out, int off, PickScratch& ps,
                                   bool unit_norm0) {
    const int t = threadIdx.x;
    if (t < m) ps.used[t] = 0;
    if (t == 0) ps.taken = 0;
    cand_norms(cand, m, ps, true);
    __syncthreads();
    if (unit_norm0 && t < m) ps.norm0[t] = 1.0;  // candidates were e_j
    __syncthreads();
    const double thresholds[3] = {0.05, 1e-8, 0.0};
    for (int tp = 0; tp < 3; ++tp) {
        const double thr = thresholds[tp];
        int start = 0;
        while (true) {
            if (ps.taken >= need) break;
            if (t < kWarp) {
                int found = -1;
                for (int base = start; base < m && found < 0; base += kWarp) {
                    const int j = base + t;
                    bool ok = false;
                    if (j < m && !ps.used[j]) {
                        const double n0 = ps.norm0[j], nr = ps.nrm[j];
                        ok = (n0 > 1e-140) && (nr > thr * n0) && (nr > 0);
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, ok);
                    if (bal) found = base + __ffs(bal) - 1;
                }
                if (t == 0) ps.sel = found;
            }
            __syncthreads();
            const int sel = ps.sel;
            if (sel < 0) break;
            const double inv = 1.0 / ps.nrm[sel];
            const int slot = ps.taken;
            if (t < m) {
                const double2 qv = cscale(inv, cand[sel * m + t]);
                ps.q[t] = qv;
                out[(off + slot) * m + t] = qv;
            }
            __syncthreads();
            if (t == 0) {
                ps.used[sel] = 1;
                ps.taken = slot + 1;
            }
            start = sel + 1;
            __syncthreads();
            // two projection passes of every remaining candidate against q
            for (int rep = 0; rep < 2; ++rep) {
                {
                    const int k = t >> 2, part = t & 3;
                    double2 d = make_double2(0, 0);
                    if (k < m && !ps.used[k])
                        for (int i = part; i < m; i += 4) d = cadd(d, cmulc(ps.q[i], cand[k * m + i]));
                    d.x += __shfl_xor_sync(0xffffffffu, d.x, 1);
                    d.y += __shfl_xor_sync(0xffffffffu, d.y, 1);
                    d.x += __shfl_xor_sync(0xffffffffu, d.x, 2);
                    d.y += __shfl_xor_sync(0xffffffffu, d.y, 2);
                    if (k < m && part == 0) ps.dot[k] = d;
                }
                __syncthreads();
                for (int e = t; e < m * m; e += blockDim.x) {
                    const int k = e / m, i = e % m;
                    if (!ps.used[k]) cand[e] = csub(cand[e], cmul(ps.dot[k], ps.q[i]));
                }
                __syncthreads();
            }
            cand_norms(cand, m, ps, false);
            __syncthreads();
        }
        if (ps.taken >= need) break;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCanThreads, 1) canonical_kernel(CanonArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    const int mm = m * m;
    double2* Es = reinterpret_cast<double2*>(smem_raw);  // [vec][row]
    double2* Ab = Es + mm;                               // A / S / candidates
    double2* X = Ab + mm;                                // T1 / P
    __shared__ double s_sig[kMaxM];
    __shared__ int s_z;
    __shared__ int s_groups[kMaxM][2];
    __shared__ int s_ngroups;
    __shared__ double2 s_dots[kMaxM];
    __shared__ double s_nrm;
    __shared__ PickScratch ps;

    // persistent CTAs drain the worklist of bins the Jacobi epilogue could not
    // canonicalize (work[0] = count, work[1] = cursor, work[2..] = indices)
    __shared__ int s_blk;
    for (;;) {
    if (threadIdx.x == 0) {
        const unsigned i = atomicAdd(a.work + 1, 1u);
        s_blk = i < a.work[0] ? (int)a.work[2 + i] : -1;
    }
    __syncthreads();
    const int blk = s_blk;
    if (blk < 0) break;
    const int bin = blk % a.bins;
    const int t = threadIdx.x;
    const double* sg = a.sigma + (size_t)blk * m;
    double2* eg = a.e + (size_t)blk * mm;

    if (t < m) s_sig[t] = sg[t];
    for (int e = t; e < mm; e += blockDim.x) Es[e] = eg[e];
    __syncthreads();
    const double smax = s_sig[0] > 0 ? s_sig[0] : 0.0;
    const double gap = 1e-5 * smax;  // kDegenerateGap (gsvd.cpp:381)
    if (t == 0) {
        int z = 0;
        while (z < m && s_sig[m - 1 - z] <= gap) ++z;
        s_z = z;
        const int lead_end = m - z;
        int ng = 0;
        for (int i = 0; i < lead_end;) {
            int end = i;
            while (end + 1 < lead_end && s_sig[end] - s_sig[end + 1] <= gap) ++end;
            if (end > i) {
                s_groups[ng][0] = i;
                s_groups[ng][1] = end;
                ++ng;
            }
            i = end + 1;
        }
        s_ngroups = ng;
    }
    __syncthreads();
    const int z = s_z;
    const int lead = m - z;

    if (z > 0) {
        if (lead > 0) {
            form_whitened(a.r + (size_t)blk * mm, a.kinv + (size_t)bin * mm, m, Ab);
            if (a.refine) {
                // T1 = A^H E_lead  (X[j][i] = sum_k conj(A(k,i)) E(k,j))
                cgemm(
                    m, lead, m, [&](int i, int k) { return cconj(Ab[i * m + k]); },
                    [&](int k, int j) { return Es[j * m + k]; }, [&](int i, int j, double2 v) { X[j * m + i] = v; });
                // S = A T1 into Ab (in place: held in registers across the barrier)
                cgemm(
                    m, lead, m, [&](int i, int k) { return Ab[k * m + i]; },
                    [&](int k, int j) { return X[j * m + k]; }, [&](int i, int j, double2 v) { Ab[j * m + i] = v; });
                // two-pass Gram-Schmidt over the columns of S (gsvd.cpp:442-464)
                for (int j = 0; j < lead; ++j) {
                    for (int pass = 0; pass < 2; ++pass) {
                        {
                            const int k = t >> 2, part = t & 3;
                            double2 d = make_double2(0, 0);
                            if (k < j)
                                for (int i = part; i < m; i += 4) d = cadd(d, cmulc(Ab[k * m + i], Ab[j * m + i]));
                            d.x += __shfl_xor_sync(0xffffffffu, d.x, 1);
                            d.y += __shfl_xor_sync(0xffffffffu, d.y, 1);
                            d.x += __shfl_xor_sync(0xffffffffu, d.x, 2);
                            d.y += __shfl_xor_sync(0xffffffffu, d.y, 2);
                            if (k < j && part == 0) s_dots[k] = d;
                        }
                        __syncthreads();
                        {
                            const int i = t >> 2, part = t & 3;
                            double2 acc = make_double2(0, 0);
                            if (i < m)
                                for (int k = part; k < j; k += 4) acc = cadd(acc, cmul(s_dots[k], Ab[k * m + i]));
                            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
                            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
                            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
                            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
                            if (i < m && part == 0) Ab[j * m + i] = csub(Ab[j * m + i], acc);
                        }
                        __syncthreads();
                    }
                    if (t < kWarp) {
                        double v = 0;
                        for (int i = t; i < m; i += kWarp) v += cnorm(Ab[j * m + i]);
                        v = group_sum<kWarp>(v);
                        if (t == 0) s_nrm = sqrt(v);
                    }
                    __syncthreads();
                    double nrm = s_nrm;
                    if (!(nrm > 1e-200)) {
                        // refinement collapsed: keep the original vector, one pass
                        if (t < m) Ab[j * m + t] = Es[j * m + t];
                        __syncthreads();
                        for (int k = 0; k < j; ++k) {
                            if (t < kWarp) {
                                double2 d = make_double2(0, 0);
                                for (int i = t; i < m; i += kWarp) d = cadd(d, cmulc(Ab[k * m + i], Ab[j * m + i]));
                                d = group_sum2<kWarp>(d);
                                if (t == 0) s_dots[0] = d;
                            }
                            __syncthreads();
                            if (t < m) Ab[j * m + t] = csub(Ab[j * m + t], cmul(s_dots[0], Ab[k * m + t]));
                            __syncthreads();
                        }
                        if (t < kWarp) {
                            double v = 0;
                            for (int i = t; i < m; i += kWarp) v += cnorm(Ab[j * m + i]);
                            v = group_sum<kWarp>(v);
                            if (t == 0) s_nrm = sqrt(v);
                        }
                        __syncthreads();
                        nrm = s_nrm;
                        if (!(nrm > 0)) continue;
                    }
                    const double inv = 1.0 / nrm;
                    if (t < m) Ab[j * m + t] = cscale(inv, Ab[j * m + t]);
                    __syncthreads();
                }
            } else {
                // no refinement: the Jacobi lead vectors span the kept subspace
                for (int e = t; e < m * lead; e += blockDim.x) Ab[e] = Es[e];
                __syncthreads();
            }
            // P = I - B B^H into X; candidates P P e_j (two projection passes)
            cgemm(
                m, m, lead, [&](int i, int k) { return Ab[k * m + i]; },
                [&](int k, int j) { return cconj(Ab[k * m + j]); },
                [&](int i, int j, double2 v) {
                    X[j * m + i] = make_double2((i == j ? 1.0 : 0.0) - v.x, -v.y);
                });
            cgemm(
                m, m, m, [&](int i, int k) { return X[k * m + i]; }, [&](int k, int j) { return X[j * m + k]; },
                [&](int i, int j, double2 v) { Ab[j * m + i] = v; });
        } else {
            for (int e = t; e < mm; e += blockDim.x) Ab[e] = make_double2((e / m) == (e % m) ? 1.0 : 0.0, 0.0);
            __syncthreads();
        }
        pick_right_looking(Ab, m, z, Es, lead, ps, true);
    }

    // tied groups (gsvd.cpp:505-543)
    const int ng = s_ngroups;
    for (int gi = 0; gi < ng; ++gi) {
        const int i0 = s_groups[gi][0];
        const int kdim = s_groups[gi][1] - i0 + 1;
        // candidate j = sum_kk g_kk conj(g_kk[j])  -> column j of G G^H
        cgemm(
            m, m, kdim, [&](int r, int kk) { return Es[(i0 + kk) * m + r]; },
            [&](int kk, int j) { return cconj(Es[(i0 + kk) * m + j]); },
            [&](int r, int j, double2 v) { Ab[j * m + r] = v; });
        pick_right_looking(Ab, m, kdim, Es, i0, ps, false);
    }

    // phase rule (gsvd.cpp:545-564): warp per vector
    const int warp = t / kWarp, lane = t % kWarp;
    for (int j = warp; j < m; j += kCanThreads / kWarp) {
        double best = -1;
        int bi = 0;
        for (int i = lane; i < m; i += kWarp) {
            const double2 v = Es[j * m + i];
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
        if (!(best > 0)) continue;
        const double2 val = Es[j * m + bi];
        const double av = hypot(val.x, val.y);
        const double2 up = make_double2(val.x / av, -(val.y / av));
        __syncwarp();
        for (int i = lane; i < m; i += kWarp) Es[j * m + i] = cmul(Es[j * m + i], up);
    }
    __syncthreads();
    for (int e = t; e < mm; e += blockDim.x) eg[e] = Es[e];
    __syncthreads();
    }
}

size_t canonical_smem_bytes(int m) { return 3 * (size_t)m * m * sizeof(double2); }

void launch_canonical(const CanonArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = canonical_smem_bytes(a.m);
    cudaFuncSetAttribute(canonical_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = nblk * a.bins;
    if (grid > 148) grid = 148;  // persistent: one CTA per SM drains the worklist
    canonical_kernel<<<grid, kCanThreads, smem, s>>>(a);
}

}  // namespace sslg
