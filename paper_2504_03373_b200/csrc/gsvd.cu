// Kernel (2): batched complex GSVD, one CTA per (block, frequency bin).
//
//   A = K^-1 R                    (gsvd.cpp:596 / 702, here in FP64)
//   one-sided Jacobi on A         (jacobi_svd, gsvd.cpp:622-695)
//   sigma_j = |w_j|, u_j = w_j / sigma_j, stable descending sort
//   canonical bases for vanishing / tied groups + phase rule
//                                 (canonicalize_subspaces, gsvd.cpp:470-565)
//
// The solver is the reference's own FP64 oracle algorithm (gsvd_reference),
// re-organized for the GPU: the Jacobi pairs of one sweep are scheduled by the
// round-robin (circle) ordering, so the M/2 disjoint pairs of a round rotate
// concurrently, one 8-lane group per pair, with the inner products reduced by
// warp shuffles.  W = A V lives in shared memory (M x M complex double,
// column-major, 57.6 KB at M = 60).  Rotation angle, skip tests (drop
// 1e-20 * max|w|^2, |a_pq|^2 <= 1e-28 |w_p|^2 |w_q|^2), convergence (a sweep
// without rotations) and the 60-sweep cap are the reference's.
//
// Outputs per (block, bin): sigma [M] descending, E [M vectors][M rows]
// (vector-major: the [bin][vector][mic] gather of music.cpp:127-135),
// sweep count and convergence flag.
#include "common.cuh"
#include "kernels.cuh"
#include "whiten.cuh"

namespace sslg {

constexpr int kJacThreads = 256;
constexpr int kLPP = 8;                    // lanes per column pair
constexpr int kRows = kMaxM / kLPP;        // rows per lane (8)

__global__ void __launch_bounds__(kJacThreads, 2) jacobi_kernel(GsvdArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);  // [m cols][m rows]
    __shared__ double cn[kMaxM];
    __shared__ double s_drop;
    __shared__ int s_perm[kMaxM];
    __shared__ double s_sig[kMaxM];

    const int blk = blockIdx.x;
    const int bin = blk % a.bins;
    const int m = a.m;
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
                    if (row < m) v += cnorm(W[j * m + row]);
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
                    double2 d0 = make_double2(0, 0), d1 = make_double2(0, 0);
#pragma unroll
                    for (int u = 0; u < kRows; ++u) {
                        const int row = s + u * kLPP;
                        if (row < m) {
                            wp[u] = W[p * m + row];
                            wq[u] = W[q * m + row];
                            if (u & 1) d1 = cadd(d1, cmulc(wp[u], wq[u]));
                            else d0 = cadd(d0, cmulc(wp[u], wq[u]));
                        }
                    }
                    double2 dot = group_sum2<kLPP>(cadd(d0, d1));
                    const double cp = cn[p], cq = cn[q];
                    const double mag2 = dot.x * dot.x + dot.y * dot.y;
                    if (!(cp <= drop || cq <= drop) && !(mag2 <= 1e-28 * cp * cq)) {
                        const double mag = sqrt(mag2);
                        const double inv_mag = 1.0 / mag;
                        const double2 ph = make_double2(dot.x * inv_mag, dot.y * inv_mag);
                        const double tau = (cq - cp) * (0.5 * inv_mag);
                        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        const double c = 1.0 / sqrt(1.0 + t * t);
                        const double sn = t * c;
                        const double2 al = make_double2(sn * ph.x, -sn * ph.y);  // s * conj(ph)
                        const double2 be = make_double2(c * ph.x, -c * ph.y);    // c * conj(ph)
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            if (row < m) {
                                W[p * m + row] = csub(cscale(c, wp[u]), cmul(al, wq[u]));
                                W[q * m + row] = cadd(cscale(sn, wp[u]), cmul(be, wq[u]));
                            }
                        }
                        if (s == 0) {
                            cn[p] = c * c * cp - 2.0 * c * sn * mag + sn * sn * cq;
                            cn[q] = sn * sn * cp + 2.0 * c * sn * mag + c * c * cq;
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

    // sigma_j = |w_j| (gsvd.cpp:677-686)
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        const int j = 2 * g + cc;
        if (j < m) {
            double v = 0;
#pragma unroll
            for (int u = 0; u < kRows; ++u) {
                const int row = s + u * kLPP;
                if (row < m) v += cnorm(W[j * m + row]);
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
    __syncthreads();
    const size_t base = (size_t)blk * m;
    if (tid < m) a.sigma[base + tid] = s_sig[s_perm[tid]];
    double2* eb = a.e + (size_t)blk * m * m;
    for (int e = tid; e < m * m; e += blockDim.x) {
        const int rank = e / m, row = e % m;
        const int j = s_perm[rank];
        const double nrm = s_sig[j];
        double2 v = make_double2(0, 0);
        if (nrm > 0) v = cscale(1.0 / nrm, W[j * m + row]);
        eb[e] = v;
    }
    if (tid == 0) {
        a.sweeps[blk] = (uint32_t)sweep;
        a.conv[blk] = converged ? 1 : 0;
    }
}

size_t jacobi_smem_bytes(int m) { return (size_t)m * m * sizeof(double2); }

void launch_jacobi(const GsvdArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = jacobi_smem_bytes(a.m);
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    jacobi_kernel<<<nblk * a.bins, kJacThreads, smem, s>>>(a);
}

}  // namespace sslg
