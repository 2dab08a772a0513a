// GSVD of small arrays (m <= 8: BASELINE config C1) with one WARP per
// (block, bin) instead of one CTA.
//
// At m = 8 an SVD is ~30 kFLOP; the CTA-wide solver (gsvd.cu) spent most of
// its time in block barriers and serial phases.  Here a warp owns a bin:
//   1. A = K^-1 R in FP64 (gsvd.cpp:596), column-major in warp-private
//      shared memory;
//   2. the reference's one-sided Jacobi on A (jacobi_svd, gsvd.cpp:622-695:
//      drop line 1e-20 max |w|^2, no-rotation test |a_pq|^2 <= tol2 |w_p|^2
//      |w_q|^2, the same rotation, at most max_sweeps sweeps) in round-robin
//      order: the m/2 pairs of a round in parallel, 64/MC lanes per pair
//      (dot products by shuffles), __syncwarp between rounds;
//   3. sigma = |w_j|, stable descending order with index tie-break
//      (gsvd.cpp:331-338), u_j = w_j / sigma_j;
//   4. canonicalization: a bin with no vanishing value, no tied group and a
//      converged solve needs only the phase rule (largest entry real
//      positive, gsvd.cpp:545-564), done here; any other bin is handed to
//      canonical_kernel through the worklist (its full-space restatement of
//      canonicalize_subspaces), exactly as the CTA solver does.
#include "common.cuh"
#include "jacobi_rot.cuh"
#include "kernels.cuh"

namespace sslg {

namespace {

constexpr int kSmallWarps = 4;  // warps (bins) per CTA

template <int MC>
struct SmallScratch {
    double2 w[MC * MC];  // column-major: w[j * MC + i] = A(i, j) (R widened, before the whitening)
    double2 k[MC * MC];  // K^-1 row-major (stride MC)
    double cn[MC];
    double sig[MC];
    int perm[MC];  // rank -> column
};

}  // namespace

template <int MC>
__global__ void __launch_bounds__(32 * kSmallWarps, 8) small_jacobi_kernel(GsvdArgs a, int nbins_total) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    constexpr int L = 64 / MC;  // lanes per column pair
    constexpr int RPL = MC / L; // rows per lane
    __shared__ SmallScratch<MC> sc[kSmallWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int blk = blockIdx.x * kSmallWarps + warp;  // (block, bin) index
    if (blk >= nbins_total) return;  // whole warp: no CTA barrier below
    SmallScratch<MC>& S = sc[warp];
    const int m = a.m, mm = m * m;
    const int bin = blk % a.bins;
    const float2* r = a.r + (size_t)blk * mm;
    const double2* kinv = a.kinv + (size_t)bin * mm;

    // 1. A = K^-1 R; padding rows / columns (m < MC) are zero.  R and K^-1
    //    are staged in shared memory by coalesced loads first
    for (int e = lane; e < MC * MC; e += 32) {
        const int i = e / MC, j = e % MC;
        const bool in = i < m && j < m;
        S.w[j * MC + i] = in ? f2d(r[i * m + j]) : make_double2(0, 0);  // R(i, j), column-major
        S.k[i * MC + j] = in ? kinv[i * m + j] : make_double2(0, 0);
    }
    __syncwarp();
    constexpr int EPL = MC * MC / 32;  // entries per lane
    double2 av[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
        const int e = lane + 32 * u;
        const int i = e % MC, j = e / MC;
        double2 acc = make_double2(0, 0);
#pragma unroll 4
        for (int k = 0; k < MC; ++k) acc = cadd(acc, cmul(S.k[i * MC + k], S.w[j * MC + k]));
        av[u] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
        const int e = lane + 32 * u;
        S.w[(e / MC) * MC + (e % MC)] = av[u];
    }
    __syncwarp();

    // 2. one-sided Jacobi sweeps
    const int g = lane / L, s = lane % L;
    const int n_even = (m + 1) & ~1;
    int sweep = 0;
    bool converged = false;
    double maxrel = 0.0;
    while (sweep < a.max_sweeps) {
        // fresh squared column norms (gsvd.cpp:633-637): lane j owns column j
        double mx = 0.0;
        if (lane < m) {
            double v = 0.0;
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                const double2 x = S.w[lane * MC + i];
                v = fma(x.x, x.x, fma(x.y, x.y, v));
            }
            S.cn[lane] = v;
            mx = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        __syncwarp();
        const double drop = 1e-20 * mx;
        bool rot = false;
        for (int rd = 0; rd < n_even - 1; ++rd) {
            int p, q;
            rr_pair(rd, g, n_even, p, q);
            if (g < n_even / 2 && q < m) {
                double2 P[RPL], Q[RPL];
#pragma unroll
                for (int u = 0; u < RPL; ++u) {
                    P[u] = S.w[p * MC + s + u * L];
                    Q[u] = S.w[q * MC + s + u * L];
                }
                double cp = S.cn[p], cq = S.cn[q];
                if (rotate_pair<RPL, L>(P, Q, cp, cq, drop, s, MC, maxrel, a.tol2)) {
#pragma unroll
                    for (int u = 0; u < RPL; ++u) {
                        S.w[p * MC + s + u * L] = P[u];
                        S.w[q * MC + s + u * L] = Q[u];
                    }
                    __syncwarp(group_mask<L>());  // every lane of the group read the norms
                    if (s == 0) {
                        S.cn[p] = cp;
                        S.cn[q] = cq;
                    }
                    rot = true;
                }
            }
            __syncwarp();
        }
        ++sweep;
        if (!__any_sync(0xffffffffu, rot)) {
            converged = true;
            break;
        }
    }

    // 3. values, stable descending order, normalized vectors
    if (lane < m) {
        double v = 0.0;
        for (int i = 0; i < m; ++i) {
            const double2 x = S.w[lane * MC + i];
            v = fma(x.x, x.x, fma(x.y, x.y, v));
        }
        S.sig[lane] = sqrt(v);
    }
    __syncwarp();
    if (lane < m) {
        const double sj = S.sig[lane];
        int rank = 0;
        for (int k = 0; k < m; ++k) {
            const double sk = S.sig[k];
            rank += (sk > sj || (sk == sj && k < lane)) ? 1 : 0;
        }
        S.perm[rank] = lane;
    }
    __syncwarp();
    // 4. structure of the sorted values (gsvd.cpp:475-505)
    bool special = !converged;
    {
        const double smax = S.sig[S.perm[0]] > 0 ? S.sig[S.perm[0]] : 0.0;
        const double gap = 1e-5 * smax;
        for (int k = 0; k < m; ++k) {
            const double sk = S.sig[S.perm[k]];
            if (sk <= gap) special = true;  // a vanishing value
            if (k + 1 < m && sk - S.sig[S.perm[k + 1]] <= gap) special = true;  // a tied pair (or vanishing tail)
        }
    }
    const bool phase = a.canonical && !special;
    double2* eb = a.e + (size_t)blk * mm;
    // lane = vector rank: normalize, phase (largest |entry| real positive), store
    if (lane < m) {
        const int j = S.perm[lane];
        const double nrm = S.sig[j];
        const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
        double2 up = make_double2(1.0, 0.0);
        if (phase) {
            double best = -1.0;
            double2 val = make_double2(0, 0);
            for (int i = 0; i < m; ++i) {
                const double2 x = cscale(inv, S.w[j * MC + i]);
                const double mg = hypot(x.x, x.y);
                if (mg > best) {
                    best = mg;
                    val = x;
                }
            }
            if (best > 0) {
                const double av = hypot(val.x, val.y);
                up = make_double2(val.x / av, -(val.y / av));
            }
        }
        for (int i = 0; i < m; ++i) eb[(size_t)lane * m + i] = cmul(cscale(inv, S.w[j * MC + i]), up);
        a.sigma[(size_t)blk * m + lane] = nrm;
    }
    if (lane == 0) {
        a.sweeps[blk] = (uint32_t)sweep;
        a.conv[blk] = converged ? 1 : 0;
        if (a.canonical && special) a.work[2 + atomicAdd(a.work, 1u)] = (uint32_t)blk;
    }
}

// m <= 8 only: at m = 16 (C2) the warp solver measured slower than the CTA
// solver (48 vs 30 us per block): without the QR preconditioning it needs
// 10.2 instead of 6.0 sweeps, and C2's bins often carry tied / vanishing
// groups that then take the separate canonical_kernel pass (0.49 ms per 32
// blocks) instead of the CTA solver's fused pickers
bool small_jacobi_supported(const GsvdArgs& a) { return a.m <= 8; }

void launch_small_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const int n = nblk * a.bins;
    const int grid = (n + kSmallWarps - 1) / kSmallWarps;
    small_jacobi_kernel<8><<<grid, 32 * kSmallWarps, 0, s>>>(a, n);
}

}  // namespace sslg
