// GSVD of small arrays (m <= 8: BASELINE config C1) with eight LANES per
// (block, bin) instead of a CTA: four bins per warp, lane j of a bin's
// quarter-warp holding column j of the Jacobi matrix in registers.
//
// At m = 8 an SVD is ~30 kFLOP and a C1 launch (32 blocks x 257 bins) fills
// the GPU only about once, so the solve is bound by its dependent chain per
// Jacobi round.  With the columns in registers a round is: the partner's
// column and norm by shuffle (no shared memory, no barriers), the dot product
// computed by both lanes of the pair bit-identically, the rotation parameters
// (jrot, also bit-identical on both lanes), and each lane updating only its
// own column.
//   1. A = K^-1 R in FP64 (gsvd.cpp:596), lane j forming column j;
//   2. the reference's one-sided Jacobi on A (jacobi_svd, gsvd.cpp:622-695:
//      drop line 1e-20 max |w|^2, no-rotation test |a_pq|^2 <= tol2 |w_p|^2
//      |w_q|^2, the same rotation (c, s), at most max_sweeps sweeps) in
//      round-robin order, the m/2 pairs of a round at once;
//   3. sigma = |w_j|, stable descending order with index tie-break
//      (gsvd.cpp:331-338), u_j = w_j / sigma_j;
//   4. canonicalization: a bin with no vanishing value, no tied group and a
//      converged solve needs only the phase rule (largest entry real
//      positive, gsvd.cpp:545-564), done here; any other bin is handed to
//      canonical_kernel through the worklist (its full-space restatement of
//      canonicalize_subspaces), exactly as the CTA solver does.
//
// The q column of a pair is stored multiplied by the unit phase ph =
// a_pq / |a_pq| (Q' ph instead of Q' = s P + c conj(ph) Q), which gives both
// lanes the same update form  w' = c w + beta t  (t the partner column) and
// costs six DFMA per entry instead of eight.  Column phases are arbitrary in
// the one-sided Jacobi -- they change neither any |a_pq| nor any norm -- and
// step 4 fixes them (the phase rule, or canonical_kernel's projector-based
// picker for special bins).
#include "common.cuh"
#include "jacobi_rot.cuh"
#include "kernels.cuh"

namespace sslg {

namespace {

constexpr int kMC = 8;            // channel capacity = lanes per bin
constexpr int kSmallWarps = 4;    // warps per CTA
constexpr int kBinsPerWarp = 32 / kMC;

// partner of column j in round r of the circle method over n = 8 columns
// (rr_pair: pair 0 = (n-1, r), pair g = (r+g, r-g) mod n-1)
__device__ __forceinline__ int rr_partner(int j, int r) {
    if (j == kMC - 1) return r;
    if (j == r) return kMC - 1;
    int p = 2 * r - j;
    if (p < 0) p += kMC - 1;
    if (p >= kMC - 1) p -= kMC - 1;
    return p;
}

}  // namespace

__global__ void __launch_bounds__(32 * kSmallWarps) small_jacobi_kernel(GsvdArgs a, int nbins_total) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    const int lane = threadIdx.x & 31;
    const int quarter = lane / kMC, j = lane % kMC;  // j: this lane's column
    const unsigned qm = 0xFFu << (kMC * quarter);
    const int base = kMC * quarter;  // first lane of the quarter
    const int blk = (blockIdx.x * kSmallWarps + (threadIdx.x >> 5)) * kBinsPerWarp + quarter;  // (block, bin)
    if (blk >= nbins_total) return;  // a whole quarter: only quarter-scoped synchronization below
    const int m = a.m, mm = m * m;
    const int bin = blk % a.bins;
    const float2* r = a.r + (size_t)blk * mm;
    const double2* kinv = a.kinv + (size_t)bin * mm;

    // 1. column j of A = K^-1 R; rows / columns >= m (m < 8) are zero
    double2 w[kMC];
    {
        double2 rc[kMC];
#pragma unroll
        for (int k = 0; k < kMC; ++k) rc[k] = (k < m && j < m) ? f2d(r[k * m + j]) : make_double2(0, 0);
#pragma unroll
        for (int i = 0; i < kMC; ++i) {
            double2 acc = make_double2(0, 0);
            if (i < m) {
#pragma unroll
                for (int k = 0; k < kMC; ++k)
                    if (k < m) acc = cadd(acc, cmul(__ldg(kinv + i * m + k), rc[k]));
            }
            w[i] = acc;
        }
    }

    // 2. one-sided Jacobi sweeps
    int sweep = 0;
    bool converged = false;
    while (sweep < a.max_sweeps) {
        // fresh squared column norms (gsvd.cpp:633-637) and the drop line
        double cn = 0.0;
#pragma unroll
        for (int i = 0; i < kMC; ++i) cn = fma(w[i].x, w[i].x, fma(w[i].y, w[i].y, cn));
        double mx = cn;
#pragma unroll
        for (int o = kMC / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(qm, mx, o));
        const double drop = 1e-20 * mx;
        bool rot = false;
#pragma unroll 1
        for (int rd = 0; rd < kMC - 1; ++rd) {
            const int pj = rr_partner(j, rd);
            const int src = base + pj;
            double2 t[kMC];
#pragma unroll
            for (int i = 0; i < kMC; ++i) {
                t[i].x = __shfl_sync(qm, w[i].x, src);
                t[i].y = __shfl_sync(qm, w[i].y, src);
            }
            const double ct = __shfl_sync(qm, cn, src);
            // conj(w) t: the real part and the two halves of the imaginary
            // part are symmetric under swapping w and t, so the partner lane
            // forms the conjugate bit for bit
            double re0 = 0, re1 = 0, s10 = 0, s11 = 0, s20 = 0, s21 = 0;
#pragma unroll
            for (int i = 0; i < kMC; i += 2) {
                re0 = fma(w[i].x, t[i].x, fma(w[i].y, t[i].y, re0));
                s10 = fma(w[i].x, t[i].y, s10);
                s20 = fma(w[i].y, t[i].x, s20);
                re1 = fma(w[i + 1].x, t[i + 1].x, fma(w[i + 1].y, t[i + 1].y, re1));
                s11 = fma(w[i + 1].x, t[i + 1].y, s11);
                s21 = fma(w[i + 1].y, t[i + 1].x, s21);
            }
            const bool lower = j < pj;  // this lane holds the pair's p column
            const double re = re0 + re1, s1 = s10 + s11, s2 = s20 + s21;
            // a_pq = conj(w_p) w_q and the pair's norms, the same on both lanes
            const double dx = re, dy = lower ? s1 - s2 : s2 - s1;
            const double cp = lower ? cn : ct, cq = lower ? ct : cn;
            const double mag2 = fma(dx, dx, dy * dy);
            if (pj < m && j < m && !(cp <= drop || cq <= drop || mag2 <= a.tol2 * cp * cq)) {
                const JRot q = jrot(dx, dy, cp, cq);
                // p: w' = c w - s conj(ph) t;  q: w' ph = c w + s ph t
                const double bx = lower ? -q.alx : q.alx, by = -q.aly;
#pragma unroll
                for (int i = 0; i < kMC; ++i) {
                    const double2 x = w[i], y = t[i];
                    w[i].x = fma(q.c, x.x, fma(bx, y.x, -by * y.y));
                    w[i].y = fma(q.c, x.y, fma(bx, y.y, by * y.x));
                }
                cn = lower ? q.c * q.c * cp - q.cs2 + q.sn * q.sn * cq : q.sn * q.sn * cp + q.cs2 + q.c * q.c * cq;
                rot = true;
            }
        }
        ++sweep;
        if (!__any_sync(qm, rot)) {
            converged = true;
            break;
        }
    }

    // 3. values, stable descending order (padding columns are exactly zero
    //    and rank after every real column), normalized vectors
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < kMC; ++i) v = fma(w[i].x, w[i].x, fma(w[i].y, w[i].y, v));
    const double sig = sqrt(v);
    int rank = 0;
    double smax = 0.0;
    bool special = !converged;
#pragma unroll
    for (int k = 0; k < kMC; ++k) {
        const double sk = __shfl_sync(qm, sig, base + k);
        rank += (sk > sig || (sk == sig && k < j)) ? 1 : 0;
        if (k < m) smax = fmax(smax, sk);
    }
    // 4. structure of the sorted values (gsvd.cpp:475-505): a vanishing value,
    //    or two values within the gap (then some adjacent pair is)
    const double gap = 1e-5 * smax;
    if (j < m && sig <= gap) special = true;
#pragma unroll
    for (int k = 0; k < kMC; ++k) {  // every lane shuffles (quarter-wide mask)
        const double sk = __shfl_sync(qm, sig, base + k);
        if (j < m && k != j && k < m && fabs(sk - sig) <= gap) special = true;
    }
    special = __any_sync(qm, special);
    const bool phase = a.canonical && !special;
    if (j < m) {
        const double inv = sig > 0 ? 1.0 / sig : 0.0;
        double2 up = make_double2(1.0, 0.0);
        if (phase) {  // largest |entry| real positive (first on ties)
            double best = -1.0;
            double2 val = make_double2(0, 0);
#pragma unroll
            for (int i = 0; i < kMC; ++i) {
                if (i < m) {
                    const double2 x = cscale(inv, w[i]);
                    const double mg = hypot(x.x, x.y);
                    if (mg > best) {
                        best = mg;
                        val = x;
                    }
                }
            }
            if (best > 0) {
                const double av2 = hypot(val.x, val.y);
                up = make_double2(val.x / av2, -(val.y / av2));
            }
        }
        double2* eb = a.e + (size_t)blk * mm + (size_t)rank * m;
#pragma unroll
        for (int i = 0; i < kMC; ++i)
            if (i < m) eb[i] = cmul(cscale(inv, w[i]), up);
        a.sigma[(size_t)blk * m + rank] = sig;
    }
    if (j == 0) {
        a.sweeps[blk] = (uint32_t)sweep;
        a.conv[blk] = converged ? 1 : 0;
        if (a.canonical && special) a.work[2 + atomicAdd(a.work, 1u)] = (uint32_t)blk;
    }
}

// m <= 8 only: at m = 16 (C2) a warp-sized solver measured slower than the
// CTA solver (48 vs 30 us per block): without the QR preconditioning it needs
// 10.2 instead of 6.0 sweeps, and C2's bins often carry tied / vanishing
// groups that then take the separate canonical_kernel pass (0.49 ms per 32
// blocks) instead of the CTA solver's fused pickers
bool small_jacobi_supported(const GsvdArgs& a) { return a.m <= kMC; }

void launch_small_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const int n = nblk * a.bins;
    const int per_cta = kSmallWarps * kBinsPerWarp;
    small_jacobi_kernel<<<(n + per_cta - 1) / per_cta, 32 * kSmallWarps, 0, s>>>(a, n);
}

}  // namespace sslg
