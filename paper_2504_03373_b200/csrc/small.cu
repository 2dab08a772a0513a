// GSVD of small arrays (m <= 16: BASELINE configs C1 and C2) with MC lanes
// per (block, bin) instead of a CTA: 32 / MC bins per warp, lane j of a bin's
// lane group holding column j of the Jacobi matrix in registers.
//
// At m = 8 an SVD is ~30 kFLOP and a C1 launch (32 blocks x 257 bins) fills
// the GPU about once, so the solve is bound by its dependent chain per Jacobi
// round.  With the columns in registers a round is: the partner's column and
// norm by shuffle (no shared memory, no barriers), the dot product computed
// by both lanes of the pair bit-identically, the rotation parameters (jrot,
// also bit-identical on both lanes), and each lane updating only its own
// column.
//   1. A = K^-1 R in FP64 (gsvd.cpp:596), lane j forming column j;
//   2. the reference's one-sided Jacobi on A (jacobi_svd, gsvd.cpp:622-695:
//      drop line 1e-20 max |w|^2, no-rotation test |a_pq|^2 <= tol2 |w_p|^2
//      |w_q|^2, the same rotation (c, s), at most max_sweeps sweeps) in
//      round-robin order, the m/2 pairs of a round at once;
//   3. sigma = |w_j|, stable descending order with index tie-break
//      (gsvd.cpp:331-338), u_j = w_j / sigma_j;
//   4. canonicalization (canonicalize_subspaces, gsvd.cpp:470-565) in the
//      lane group: the vanishing block (sigma <= 1e-5 sigma_max) rebuilt from
//      the candidates e_j projected twice against the lead vectors, each
//      tied group from the candidates N N^H e_j, both with the reference's
//      picker (pick_orthonormal, gsvd.cpp:404-436: index order, thresholds
//      {0.05, 1e-8, 0}, two projection passes against every accepted
//      vector), lane j owning candidate j; then the phase rule (largest entry
//      real positive, gsvd.cpp:545-564) on every vector (a bin that did not
//      converge within max_sweeps is canonicalized from its last iterate, as
//      canonical_kernel would).  Only refine_leading (the A A^H refinement)
//      sends bins to canonical_kernel through the worklist, so without it the
//      engine skips that launch.
//
// The q column of a pair is stored multiplied by the unit phase ph =
// a_pq / |a_pq| (Q' ph instead of Q' = s P + c conj(ph) Q), which gives both
// lanes the same update form  w' = c w + beta t  (t the partner column) and
// costs six DFMA per entry instead of eight.  Column phases are arbitrary in
// the one-sided Jacobi -- they change neither any |a_pq| nor any norm -- and
// step 4 fixes them.
#include "common.cuh"
#include "jacobi_rot.cuh"
#include "kernels.cuh"

namespace sslg {

namespace {

constexpr int kSmallWarps = 4;  // warps per CTA

// partner of column j in round r of the circle method over n columns
// (rr_pair: pair 0 = (n-1, r), pair g = (r+g, r-g) mod n-1)
template <int N>
__device__ __forceinline__ int rr_partner(int j, int r) {
    if (j == N - 1) return r;
    if (j == r) return N - 1;
    int p = 2 * r - j;
    if (p < 0) p += N - 1;
    if (p >= N - 1) p -= N - 1;
    return p;
}

// the lane (within the bin's group) whose vector has rank r (r uniform)
__device__ __forceinline__ int lane_of_rank(unsigned gm, int base, int rank, int r) {
    return __ffs(__ballot_sync(gm, rank == r) >> base) - 1;
}

// c -= (v^H c) v, twice, v a vector staged in shared memory (broadcast
// reads); only `active` lanes update c
template <int MC>
__device__ __forceinline__ void project_out(double2 (&c)[MC], const double2* v, bool active) {
    for (int pass = 0; pass < 2; ++pass) {
        double dx = 0, dy = 0;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            const double2 vv = v[i];
            dx = fma(vv.x, c[i].x, fma(vv.y, c[i].y, dx));
            dy = fma(vv.x, c[i].y, fma(-vv.y, c[i].x, dy));
        }
        if (active) {
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                const double2 vv = v[i];
                c[i].x -= fma(dx, vv.x, -dy * vv.y);
                c[i].y -= fma(dx, vv.y, dy * vv.x);
            }
        }
    }
}

// The reference's picker (pick_orthonormal) over the candidates c (lane j:
// the image of e_j), right-looking: an accepted candidate is normalized,
// staged in sq for the projections, and stored as the vector of rank
// i0 + taken in the row sv[lane of that rank] (that lane's snapshot belongs to
// this group and is not read again); every remaining candidate is projected
// against it twice.  Slots left unfilled get zero vectors (the reference's
// zero-initialized output); the caller reloads every lane's vector from its
// row once all groups are picked.
template <int MC>
__device__ __forceinline__ void pick_group(double2 (&c)[MC], double2 (*sv)[MC], double2* sq, double n0, int i0,
                                           int need, int m, int j, int rank, unsigned gm, int base) {
    bool used = j >= m;
    int taken = 0;
    const double thresholds[3] = {0.05, 1e-8, 0.0};
    __syncwarp(gm);  // the caller's reads of the group's rows precede the first accepted vector's store
    for (int tp = 0; tp < 3 && taken < need; ++tp) {
        const double thr = thresholds[tp];
        int start = 0;
        while (taken < need) {
            double n2 = 0;
#pragma unroll
            for (int i = 0; i < MC; ++i) n2 = fma(c[i].x, c[i].x, fma(c[i].y, c[i].y, n2));
            const double nr = sqrt(n2);
            const bool ok = !used && j >= start && (n0 > 1e-140) && (nr > thr * n0) && (nr > 0);
            const unsigned bal = __ballot_sync(gm, ok) >> base;
            if (!bal) break;
            const int sel = __ffs(bal) - 1;
            const int dl = lane_of_rank(gm, base, rank, i0 + taken);
            if (j == sel) {
                used = true;
                const double inv = 1.0 / nr;
#pragma unroll
                for (int i = 0; i < MC; ++i) {
                    c[i] = cscale(inv, c[i]);
                    sq[i] = c[i];
                    sv[dl][i] = c[i];
                }
            }
            __syncwarp(gm);
            project_out<MC>(c, sq, !used);
            __syncwarp(gm);  // every lane has read sq before the next accepted vector
            start = sel + 1;
            ++taken;
        }
    }
    if (rank >= i0 + taken && rank < i0 + need)
#pragma unroll
        for (int i = 0; i < MC; ++i) sv[j][i] = make_double2(0, 0);
    __syncwarp(gm);
}

}  // namespace

// resident CTAs per SM: the register budget of the solve (the canonicalization
// path is rare and may spill)
template <int MC>
constexpr int small_ctas() { return MC <= 8 ? 4 : 3; }

template <int MC>
__global__ void __launch_bounds__(32 * kSmallWarps, small_ctas<MC>()) small_jacobi_kernel(GsvdArgs a, int nbins_total) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    constexpr int kBins = 32 / MC;    // bins per warp
    const int lane = threadIdx.x & 31;
    const int slot = lane / MC, j = lane % MC;  // j: this lane's column
    const int base = MC * slot;                 // first lane of the bin's group
    const unsigned gm = ((1u << MC) - 1u) << base;
    const int blk = (blockIdx.x * kSmallWarps + (threadIdx.x >> 5)) * kBins + slot;  // (block, bin)
    if (blk >= nbins_total) return;  // a whole group: only group-scoped synchronization below
    const int m = a.m, mm = m * m;
    const int bin = blk % a.bins;
    const float2* r = a.r + (size_t)blk * mm;
    const double2* kinv = a.kinv + (size_t)bin * mm;

    // 1. column j of A = K^-1 R; rows / columns >= m are zero
    double2 w[MC];
    {
        double2 rc[MC];
#pragma unroll
        for (int k = 0; k < MC; ++k) rc[k] = (k < m && j < m) ? f2d(r[k * m + j]) : make_double2(0, 0);
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            double2 acc = make_double2(0, 0);
            if (i < m) {
#pragma unroll
                for (int k = 0; k < MC; ++k)
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
        for (int i = 0; i < MC; ++i) cn = fma(w[i].x, w[i].x, fma(w[i].y, w[i].y, cn));
        double mx = cn;
#pragma unroll
        for (int o = MC / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(gm, mx, o));
        const double drop = 1e-20 * mx;
        bool rot = false;
#pragma unroll 1
        for (int rd = 0; rd < MC - 1; ++rd) {
            const int pj = rr_partner<MC>(j, rd);
            const int src = base + pj;
            double2 t[MC];
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                t[i].x = __shfl_sync(gm, w[i].x, src);
                t[i].y = __shfl_sync(gm, w[i].y, src);
            }
            const double ct = __shfl_sync(gm, cn, src);
            // conj(w) t: the real part and the two halves of the imaginary
            // part are symmetric under swapping w and t, so the partner lane
            // forms the conjugate bit for bit
            double re0 = 0, re1 = 0, s10 = 0, s11 = 0, s20 = 0, s21 = 0;
#pragma unroll
            for (int i = 0; i < MC; i += 2) {
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
                for (int i = 0; i < MC; ++i) {
                    const double2 x = w[i], y = t[i];
                    w[i].x = fma(q.c, x.x, fma(bx, y.x, -by * y.y));
                    w[i].y = fma(q.c, x.y, fma(bx, y.y, by * y.x));
                }
                cn = lower ? q.c * q.c * cp - q.cs2 + q.sn * q.sn * cq : q.sn * q.sn * cp + q.cs2 + q.c * q.c * cq;
                rot = true;
            }
        }
        ++sweep;
        if (!__any_sync(gm, rot)) {
            converged = true;
            break;
        }
    }

    // 3. values, stable descending order (padding columns are exactly zero
    //    and rank after every real column), normalized vectors
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < MC; ++i) v = fma(w[i].x, w[i].x, fma(w[i].y, w[i].y, v));
    const double sig = sqrt(v);
    int rank = 0;
    double smax = 0.0;
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        const double sk = __shfl_sync(gm, sig, base + k);
        rank += (sk > sig || (sk == sig && k < j)) ? 1 : 0;
        if (k < m) smax = fmax(smax, sk);
    }
    {
        const double inv = sig > 0 ? 1.0 / sig : 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) w[i] = cscale(inv, w[i]);
    }
    // 4. structure of the sorted values (gsvd.cpp:475-505): the vanishing
    //    block (a suffix of the ranks) and the tied runs above it
    const double gap = 1e-5 * smax;
    const int z = __popc(__ballot_sync(gm, j < m && sig <= gap));
    const int lead = m - z;
    double snext = 0.0;  // the value of rank + 1
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        const double sk = __shfl_sync(gm, sig, base + k);
        const int rk = __shfl_sync(gm, rank, base + k);
        if (rk == rank + 1) snext = sk;
    }
    const bool tie = rank + 1 < lead && sig - snext <= gap;  // rank ties with rank + 1
    unsigned tie_rank = 0;                                   // bit r: rank r ties with rank r + 1
    for (unsigned tl = __ballot_sync(gm, tie) >> base; tl; tl &= tl - 1)
        tie_rank |= 1u << __shfl_sync(gm, rank, base + __ffs(tl) - 1);
    bool special = z > 0 || tie_rank != 0;
    if (a.canonical && special && !a.refine) {
        // the group's vectors (by lane) and one accepted-vector slot in shared
        // memory: the projections and candidate sums read them by broadcast
        __shared__ double2 s_vec[kSmallWarps * kBins][MC][MC];
        __shared__ double2 s_acc[kSmallWarps * kBins][MC];
        const int gsl = (threadIdx.x >> 5) * kBins + slot;
        double2(*sv)[MC] = s_vec[gsl];
#pragma unroll
        for (int i = 0; i < MC; ++i) sv[j][i] = w[i];
        __syncwarp(gm);
        if (z > 0) {
            // candidates e_j projected twice against every lead vector
            double2 c[MC];
#pragma unroll
            for (int i = 0; i < MC; ++i) c[i] = make_double2(i == j ? 1.0 : 0.0, 0.0);
            for (int k = 0; k < lead; ++k) project_out<MC>(c, sv[lane_of_rank(gm, base, rank, k)], true);
            pick_group<MC>(c, sv, s_acc[gsl], 1.0, lead, z, m, j, rank, gm, base);
        }
        // tied runs in rank order: ranks i0 .. i1 with bits i0 .. i1-1 set
        for (unsigned rest = tie_rank; rest;) {
            const int i0 = __ffs(rest) - 1;
            int i1 = i0;
            while ((rest >> i1) & 1u) ++i1;
            rest &= ~((1u << i1) - 1u);
            const int d = i1 - i0 + 1;
            // candidate j = N N^H e_j = sum_k u_k conj(u_k[j])
            double2 c[MC];
#pragma unroll
            for (int i = 0; i < MC; ++i) c[i] = make_double2(0, 0);
            for (int k = i0; k <= i1; ++k) {
                // the group's vectors above the vanishing block are unchanged
                // since the snapshot (the pickers only rewrite their own ranks)
                const double2* uk = sv[lane_of_rank(gm, base, rank, k)];
                const double2 ukj = make_double2(uk[j].x, -uk[j].y);  // conj(u_k[j])
#pragma unroll
                for (int i = 0; i < MC; ++i) c[i] = cadd(c[i], cmul(uk[i], ukj));
            }
            double n2 = 0;
#pragma unroll
            for (int i = 0; i < MC; ++i) n2 = fma(c[i].x, c[i].x, fma(c[i].y, c[i].y, n2));
            pick_group<MC>(c, sv, s_acc[gsl], sqrt(n2), i0, d, m, j, rank, gm, base);
        }
#pragma unroll
        for (int i = 0; i < MC; ++i) w[i] = sv[j][i];  // picked vectors, or the snapshot
        special = false;
    }
    const bool phase = a.canonical && !special;
    if (j < m) {
        double2 up = make_double2(1.0, 0.0);
        if (phase) {  // largest |entry| real positive (first on ties)
            double best = -1.0;
            double2 val = make_double2(0, 0);
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                if (i < m) {
                    const double mg = hypot(w[i].x, w[i].y);
                    if (mg > best) {
                        best = mg;
                        val = w[i];
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
        for (int i = 0; i < MC; ++i)
            if (i < m) eb[i] = cmul(w[i], up);
        a.sigma[(size_t)blk * m + rank] = sig;
    }
    if (j == 0) {
        a.sweeps[blk] = (uint32_t)sweep;
        a.conv[blk] = converged ? 1 : 0;
        if (a.canonical && special) a.work[2 + atomicAdd(a.work, 1u)] = (uint32_t)blk;
    }
}

// m <= 16: lane groups of 8 (C1) or 16 (C2) lanes
bool small_jacobi_supported(const GsvdArgs& a) { return a.m <= 16; }
bool small_jacobi_selected(const GsvdArgs& a) { return small_jacobi_supported(a) && !a.phase_clk && !a.force_cta; }

void launch_small_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const int n = nblk * a.bins;
    if (a.m <= 8) {
        constexpr int per_cta = kSmallWarps * 4;
        small_jacobi_kernel<8><<<(n + per_cta - 1) / per_cta, 32 * kSmallWarps, 0, s>>>(a, n);
    } else {
        constexpr int per_cta = kSmallWarps * 2;
        small_jacobi_kernel<16><<<(n + per_cta - 1) / per_cta, 32 * kSmallWarps, 0, s>>>(a, n);
    }
}

}  // namespace sslg
