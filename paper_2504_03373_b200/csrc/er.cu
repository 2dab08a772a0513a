// Right factor E_r and reconstruction residual of the GSVD (GsvdBinResult::e_r
// and recon_residual, reference include/ssl/gsvd.hpp:52-60).
//
// The solver (gsvd.cu) never forms the right singular vectors: its Jacobi
// runs on the QR-preconditioned R^H and the left vectors come from one
// back-multiplication.  E_r is therefore rebuilt here from the final,
// canonicalized left factor E, one CTA per (block, bin), only when a caller
// asks for it (sslg_gsvd_ex; it is not on the localization hot path):
//
//   A = K^-1 R (FP64), Y = E^H A.
//   Lead groups (gsvd.cpp:381-565 rules: values above 1e-5 sigma_max, runs
//   whose consecutive gaps are <= 1e-5 sigma_max):
//     the reference's rows are V^H of its Jacobi (gsvd.cpp:713-716), rotated
//     by W^H = (B^H U_g) inside a tied group (gsvd.cpp:535-543) and phased
//     with the left vector (gsvd.cpp:545-564).  With B the final basis that
//     is B^H U_g V_g^H, the unitary polar factor of Y_g = B^H A = (B^H U_g)
//     Sigma_g V_g^H: independent of how the group's basis was mixed, so it
//     is computed from Y_g alone -- a single row is normalized, a tied group
//     runs Newton-Schulz iterations X <- (3X - X X^H X) / 2 in FP64.
//   Vanishing block: the reference keeps its Jacobi's arbitrary V^H rows
//     there; these rows are the canonical completion of the lead rows to a
//     unitary matrix (standard-basis candidates in index order, two
//     projection passes, thresholds {0.05, 1e-8, 0}: pick_orthonormal,
//     gsvd.cpp:402-436), so E_r is unitary like the reference's.
//   resid = ||A - E diag(sigma) E_r||_F / ||A||_F (gsvd.cpp:573-585).
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

constexpr int kErThreads = 256;

namespace {

// A[i][j] = sum_k kinv[i][k] * R[k][j] into `a` (row-major); R is staged
// (widened) in `tmp`
__device__ void form_a(double2* a, double2* tmp, const float2* __restrict__ r, const double2* __restrict__ kinv,
                       int m) {
    const int mm = m * m;
    for (int e = threadIdx.x; e < mm; e += blockDim.x) tmp[e] = f2d(r[e]);
    __syncthreads();
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
        const int i = e / m, j = e % m;
        double2 acc = make_double2(0, 0);
        for (int k = 0; k < m; ++k) {
            const double2 x = kinv[i * m + k], y = tmp[k * m + j];
            acc.x = fma(x.x, y.x, fma(-x.y, y.y, acc.x));
            acc.y = fma(x.x, y.y, fma(x.y, y.x, acc.y));
        }
        a[e] = acc;
    }
    __syncthreads();
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double t = 0;
    for (int i = 0; i < nw; ++i) t += red[i];
    __syncthreads();
    return t;
}

}  // namespace

__global__ void __launch_bounds__(kErThreads) er_kernel(ErArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m, mm = m * m;
    double2* A = reinterpret_cast<double2*>(smem_raw);  // [m][m]: A, then Newton-Schulz scratch, then A again
    double2* Y = A + mm;                                // [m][m]: rows of E^H A, then E_r
    double2* G = Y + mm;                                // [m][m]: E (vector-major), Gram, then E again
    __shared__ double sig[kMaxM];
    __shared__ double red[kErThreads / 32];
    __shared__ int s_grp[kMaxM + 2];  // polar group starts, s_grp[ng] = end of the polar rows
    __shared__ int s_ng, s_z;
    __shared__ double2 s_x[kMaxM];
    __shared__ double2 s_d[kMaxM];
    __shared__ int s_src[kMaxM];  // standard-basis index each completion row came from

    if (a.abort && *a.abort) return;
    const int blk = blockIdx.x / a.bins, b = blockIdx.x % a.bins;
    const size_t base = ((size_t)blk * a.bins + b) * mm;
    const float2* r = a.r + base;
    const double2* kinv = a.kinv + (size_t)b * mm;
    const double2* e = a.e + base;  // [vector][row]
    const int t = threadIdx.x;

    for (int i = t; i < m; i += blockDim.x) sig[i] = a.sigma[((size_t)blk * a.bins + b) * m + i];
    form_a(A, G, r, kinv, m);
    for (int x = t; x < mm; x += blockDim.x) G[x] = e[x];
    __syncthreads();
    // Y[i][c] = sum_r conj(E[r][i]) A[r][c]
    for (int x = t; x < mm; x += blockDim.x) {
        const int i = x / m, c = x % m;
        double2 acc = make_double2(0, 0);
        for (int k = 0; k < m; ++k) {
            const double2 u = G[i * m + k], v = A[k * m + c];
            acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
            acc.y = fma(u.x, v.y, fma(-u.y, v.x, acc.y));
        }
        Y[x] = acc;
    }
    if (t == 0) {  // group structure (gsvd.cpp:475-497)
        const double smax = sig[0] > 0 ? sig[0] : 0.0;
        const double gap = 1e-5 * smax;
        int z = 0;
        while (z < m && sig[m - 1 - z] <= gap) ++z;
        const int lead = m - z;
        int ng = 0;
        for (int i = 0; i < lead;) {
            int end = i;
            while (end + 1 < lead && sig[end] - sig[end + 1] <= gap) ++end;
            s_grp[ng++] = i;
            i = end + 1;
        }
        // the vanishing values above the Jacobi's drop line (1e-10 sigma_max:
        // 1e-20 of the squared column norms, gsvd.cpp:639) form one more polar
        // group -- Y_v = Q^H Sigma_v V_v^H for the canonical basis E_v = E_old Q,
        // so its polar factor Q^H V_v^H keeps the residual down to the block's
        // value spread; rows below the line get the canonical completion
        int z1 = 0;
        while (z1 < z && sig[lead + z1] > 1e-10 * smax) ++z1;
        if (z1) s_grp[ng++] = lead;
        s_grp[ng] = lead + z1;
        s_ng = ng;
        s_z = z - z1;
    }
    __syncthreads();
    const int ng = s_ng, lead = m - s_z;  // rows [0, lead) by polar factors, [lead, m) by completion

    // Polar groups in rank order.  A row e_i^H A carries the residual error of
    // e_i towards larger-value vectors amplified by sigma_j / sigma_i; the
    // reference's rows (accumulated Jacobi rotations) are orthonormal to
    // round-off, so each group's rows are first projected off every earlier
    // row (two classical Gram-Schmidt passes), then normalized (one value)
    // or replaced by their polar factor (tied group: Newton-Schulz, the rows
    // scaled so their extreme singular values straddle 1 inside (0, sqrt 3)).
    for (int gi = 0; gi < ng; ++gi) {
        const int i0 = s_grp[gi], k = s_grp[gi + 1] - i0;
        double2* X = Y + i0 * m;
        for (int rep = 0; rep < 2 && i0 > 0; ++rep) {
            // G[p][q] = X_p . conj(Y_q) for q < i0, then X_p -= sum_q G[p][q] Y_q
            for (int x = t; x < k * i0; x += blockDim.x) {
                const int p = x / i0, q = x % i0;
                double2 acc = make_double2(0, 0);
                for (int c = 0; c < m; ++c) {
                    const double2 u = X[p * m + c], v = Y[q * m + c];
                    acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
                    acc.y = fma(u.y, v.x, fma(-u.x, v.y, acc.y));
                }
                G[x] = acc;
            }
            __syncthreads();
            for (int x = t; x < k * m; x += blockDim.x) {
                const int p = x / m, c = x % m;
                double2 v = X[x];
                for (int q = 0; q < i0; ++q) v = csub(v, cmul(G[p * i0 + q], Y[q * m + c]));
                X[x] = v;
            }
            __syncthreads();
        }
        if (k == 1) {
            if (t < 32) {
                double s2 = 0;
                for (int c = t; c < m; c += 32) s2 += cnorm(X[c]);
                for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                const double inv = s2 > 0 ? 1.0 / sqrt(s2) : 0.0;
                for (int c = t; c < m; c += 32) X[c] = cscale(inv, X[c]);
            }
            __syncthreads();
            continue;
        }
        const double s_hi = sig[i0], s_lo = sig[i0 + k - 1];
        const double sc = sqrt(2.0 / (s_hi * s_hi + s_lo * s_lo));
        for (int x = t; x < k * m; x += blockDim.x) X[x] = cscale(sc, X[x]);
        __syncthreads();
        bool last = false;
        for (int it = 0; it < 100; ++it) {  // ~log1.5(sigma_hi / sigma_lo) + 6 steps
            // G = X X^H (k x k); once max |G - I| <= 1e-12 one more step
            // (quadratic convergence) leaves only round-off
            bool off = false;
            for (int x = t; x < k * k; x += blockDim.x) {
                const int p = x / k, q = x % k;
                double2 acc = make_double2(0, 0);
                for (int c = 0; c < m; ++c) {
                    const double2 u = X[p * m + c], v = X[q * m + c];
                    acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
                    acc.y = fma(-u.x, v.y, fma(u.y, v.x, acc.y));
                }
                G[x] = acc;
                const double dx = acc.x - (p == q ? 1.0 : 0.0);
                if (fabs(dx) > 1e-12 || fabs(acc.y) > 1e-12) off = true;
            }
            const bool conv = __syncthreads_or(off) == 0;
            if (last) break;
            last = conv;
            // A <- G X, X <- (3 X - G X) / 2
            for (int x = t; x < k * m; x += blockDim.x) {
                const int p = x / m, c = x % m;
                double2 acc = make_double2(0, 0);
                for (int q = 0; q < k; ++q) {
                    const double2 u = G[p * k + q], v = X[q * m + c];
                    acc.x = fma(u.x, v.x, fma(-u.y, v.y, acc.x));
                    acc.y = fma(u.x, v.y, fma(u.y, v.x, acc.y));
                }
                A[x] = acc;
            }
            __syncthreads();
            for (int x = t; x < k * m; x += blockDim.x)
                X[x] = make_double2(1.5 * X[x].x - 0.5 * A[x].x, 1.5 * X[x].y - 0.5 * A[x].y);
            __syncthreads();
        }
        __syncthreads();
    }

    // vanishing block: canonical completion of the rows taken so far
    int taken = lead;
    const double thr[3] = {0.05, 1e-8, 0.0};
    for (int pass = 0; pass < 3 && taken < m; ++pass) {
        for (int j = 0; j < m && taken < m; ++j) {
            // candidate row delta_j, skipped if an earlier pass took it
            bool used = false;
            for (int q = lead; q < taken; ++q) used |= (s_src[q - lead] == j);
            if (used) continue;
            for (int c = t; c < m; c += blockDim.x) s_x[c] = make_double2(c == j ? 1.0 : 0.0, 0.0);
            __syncthreads();
            for (int rep = 0; rep < 2; ++rep) {
                // d_q = x . conj(row_q), then x -= sum_q d_q row_q
                for (int q = t; q < taken; q += blockDim.x) {
                    double2 acc = make_double2(0, 0);
                    for (int c = 0; c < m; ++c) {
                        const double2 u = s_x[c], v = Y[q * m + c];
                        acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
                        acc.y = fma(u.y, v.x, fma(-u.x, v.y, acc.y));
                    }
                    s_d[q] = acc;
                }
                __syncthreads();
                for (int c = t; c < m; c += blockDim.x) {
                    double2 x = s_x[c];
                    for (int q = 0; q < taken; ++q) x = csub(x, cmul(s_d[q], Y[q * m + c]));
                    s_x[c] = x;
                }
                __syncthreads();
            }
            double n2 = 0;
            for (int c = 0; c < m; ++c) n2 += cnorm(s_x[c]);  // every thread: uniform decision
            const double nrm = sqrt(n2);
            if (!(nrm > thr[pass]) || !(nrm > 0)) {
                __syncthreads();
                continue;
            }
            const double inv = 1.0 / nrm;
            for (int c = t; c < m; c += blockDim.x) Y[taken * m + c] = cscale(inv, s_x[c]);
            __syncthreads();
            if (t == 0) s_src[taken - lead] = j;
            __syncthreads();
            ++taken;
        }
    }

    if (a.er) {
        double2* out = a.er + base;
        for (int x = t; x < mm; x += blockDim.x) out[x] = Y[x];
    }
    if (a.resid) {
        __syncthreads();
        form_a(A, G, r, kinv, m);
        for (int x = t; x < mm; x += blockDim.x) G[x] = e[x];
        __syncthreads();
        double err = 0, ref = 0;
        for (int x = t; x < mm; x += blockDim.x) {
            const int row = x / m, col = x % m;
            double2 acc = A[x];
            ref += cnorm(acc);
            for (int i = 0; i < m; ++i) acc = csub(acc, cmul(cscale(sig[i], G[i * m + row]), Y[i * m + col]));
            err += cnorm(acc);
        }
        err = block_sum(err, red);
        ref = block_sum(ref, red);
        if (t == 0) a.resid[(size_t)blk * a.bins + b] = ref > 0 ? sqrt(err / ref) : sqrt(err);
    }
}

void launch_er(const ErArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = (size_t)3 * a.m * a.m * sizeof(double2);
    cudaFuncSetAttribute(er_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    er_kernel<<<nblk * a.bins, kErThreads, smem, s>>>(a);
}

}  // namespace sslg
