// One-time noise-model setup on the device: per-bin inverse K^-1 and the
// Hermitian / positive-definite gate.
//
// Inverse: Gauss-Jordan elimination with partial pivoting and the pivot floor
// scale * eps(T) * n of mat_inverse<T> (reference proj/src/gsvd.cpp:21-62).
// NoiseModel::prepare_inverses builds a float and a double inverse per bin
// (gsvd.cpp:756-768) and either may throw "singular at bin b"; both are run
// here so the error behaviour matches, and the FP64 inverse is kept for the
// solver.  One CTA per bin, the augmented [K | I] block resident in SMEM.
//
// PD gate (NoiseModel::check_positive_definite, gsvd.cpp:736-754): the
// Hermitian test is reproduced as written; "smallest eigenvalue > 0" is
// decided by an FP64 Cholesky (a Hermitian matrix is positive definite iff
// its Cholesky pivots are all positive) instead of a full Jacobi
// eigensolve.
#include "common.cuh"

namespace sslg {

template <typename T>
struct cplx_t;
template <>
struct cplx_t<float> {
    using type = float2;
};
template <>
struct cplx_t<double> {
    using type = double2;
};

template <typename T>
__device__ __forceinline__ T cabs_t(T re, T im);
template <>
__device__ __forceinline__ float cabs_t<float>(float re, float im) { return hypotf(re, im); }
template <>
__device__ __forceinline__ double cabs_t<double>(double re, double im) { return hypot(re, im); }

template <typename T>
__device__ __forceinline__ T eps_t();
template <>
__device__ __forceinline__ float eps_t<float>() { return 1.1920928955078125e-07f; }
template <>
__device__ __forceinline__ double eps_t<double>() { return 2.220446049250313080847e-16; }

constexpr int kInvThreads = 256;

// aug: [m][2m] complex T (left half K, right half the running inverse)
template <typename T>
__global__ void __launch_bounds__(kInvThreads) gauss_jordan_kernel(const float2* __restrict__ k, int m,
                                                                    double2* __restrict__ inv_out,
                                                                    unsigned int* bad_bin) {
    using C = typename cplx_t<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* aug = reinterpret_cast<C*>(smem_raw);
    __shared__ T s_scale;
    __shared__ int s_piv;
    __shared__ int s_fail;
    __shared__ C s_f[kMaxM];
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int w = 2 * m;
    const float2* kb = k + (size_t)b * m * m;

    for (int e = tid; e < m * w; e += blockDim.x) {
        const int i = e / w, j = e % w;
        C v;
        if (j < m) {
            v.x = (T)kb[i * m + j].x;
            v.y = (T)kb[i * m + j].y;
        } else {
            v.x = (j - m == i) ? (T)1 : (T)0;
            v.y = (T)0;
        }
        aug[e] = v;
    }
    if (tid == 0) s_fail = 0;
    __syncthreads();
    // scale = max |k_ij|
    if (tid < 32) {
        T mx = 0;
        for (int e = tid; e < m * m; e += 32) {
            const C v = aug[(e / m) * w + (e % m)];
            const T a = cabs_t<T>(v.x, v.y);
            mx = a > mx ? a : mx;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const T other = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = other > mx ? other : mx;
        }
        if (tid == 0) s_scale = mx;
    }
    __syncthreads();
    const T floor_ = s_scale * eps_t<T>() * (T)m;

    for (int col = 0; col < m; ++col) {
        // partial pivoting: first row with the largest magnitude
        if (tid < 32) {
            T best = -1;
            int bi = col;
            for (int r = col + tid; r < m; r += 32) {
                const C v = aug[r * w + col];
                const T a = cabs_t<T>(v.x, v.y);
                if (a > best) {
                    best = a;
                    bi = r;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const T ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (tid == 0) {
                s_piv = bi;
                if (!(best > floor_)) s_fail = 1;
            }
        }
        __syncthreads();
        if (s_fail) break;
        const int piv = s_piv;
        if (piv != col)
            for (int j = tid; j < w; j += blockDim.x) {
                const C t0 = aug[col * w + j];
                aug[col * w + j] = aug[piv * w + j];
                aug[piv * w + j] = t0;
            }
        __syncthreads();
        // d = 1 / a(col, col) with the textbook complex division
        const C p = aug[col * w + col];
        const T den = p.x * p.x + p.y * p.y;
        C d;
        d.x = p.x / den;
        d.y = -p.y / den;
        __syncthreads();
        for (int j = tid; j < w; j += blockDim.x) {
            const C v = aug[col * w + j];
            C r;
            r.x = v.x * d.x - v.y * d.y;
            r.y = v.x * d.y + v.y * d.x;
            aug[col * w + j] = r;
        }
        for (int r = tid; r < m; r += blockDim.x) s_f[r] = aug[r * w + col];
        __syncthreads();
        for (int e = tid; e < m * w; e += blockDim.x) {
            const int r = e / w, j = e % w;
            if (r == col) continue;
            const C f = s_f[r];
            if (f.x == (T)0 && f.y == (T)0) continue;
            const C pv = aug[col * w + j];
            C v = aug[e];
            v.x -= f.x * pv.x - f.y * pv.y;
            v.y -= f.x * pv.y + f.y * pv.x;
            aug[e] = v;
        }
        __syncthreads();
    }
    if (s_fail) {
        if (tid == 0) atomicMin(bad_bin, (unsigned)b);
        return;
    }
    if (inv_out)
        for (int e = tid; e < m * m; e += blockDim.x) {
            const int i = e / m, j = e % m;
            const C v = aug[i * w + m + j];
            inv_out[(size_t)b * m * m + e] = make_double2((double)v.x, (double)v.y);
        }
}

// Hermitian test + FP64 Cholesky.  bad_herm / bad_pd receive the first bad bin.
__global__ void __launch_bounds__(kInvThreads) pd_check_kernel(const float2* __restrict__ k, int m,
                                                                unsigned int* bad_herm, unsigned int* bad_pd,
                                                                double* min_pivot) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* a = reinterpret_cast<double2*>(smem_raw);  // [m][m]
    __shared__ int s_fail;
    __shared__ double s_piv;
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const float2* kb = k + (size_t)b * m * m;
    if (tid < 32) {
        double scale = 0, herm = 0;
        for (int e = tid; e < m * m; e += 32) {
            const int i = e / m, j = e % m;
            const float2 v = kb[i * m + j];
            const float2 u = kb[j * m + i];
            scale = fmax(scale, (double)hypotf(v.x, v.y));
            herm = fmax(herm, (double)hypotf(v.x - u.x, v.y + u.y));
        }
        for (int o = 16; o > 0; o >>= 1) {
            scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
            herm = fmax(herm, __shfl_xor_sync(0xffffffffu, herm, o));
        }
        if (tid == 0) s_fail = herm > 1e-5 * scale + 1e-30 ? 1 : 0;
    }
    for (int e = tid; e < m * m; e += blockDim.x) a[e] = f2d(kb[e]);
    __syncthreads();
    if (s_fail) {
        if (tid == 0) atomicMin(bad_herm, (unsigned)b);
        return;
    }
    // right-looking Cholesky on the lower triangle
    for (int c = 0; c < m; ++c) {
        if (tid == 0) {
            const double d = a[c * m + c].x;
            s_piv = d;
            if (!(d > 0)) s_fail = 1;
        }
        __syncthreads();
        if (s_fail) break;
        const double rs = rsqrt(s_piv);
        for (int r = c + 1 + tid; r < m; r += blockDim.x) a[r * m + c] = cscale(rs, a[r * m + c]);
        __syncthreads();
        const int n = m - c - 1;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int r = c + 1 + e / n, j = c + 1 + e % n;
            if (j > r) continue;
            // a(r, j) -= l(r, c) * conj(l(j, c))
            const double2 lr = a[r * m + c], lj = a[j * m + c];
            a[r * m + j] = csub(a[r * m + j], cmul(lr, cconj(lj)));
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (s_fail) atomicMin(bad_pd, (unsigned)b);
        if (min_pivot) min_pivot[b] = s_piv;
    }
}

void launch_gauss_jordan(const float2* k, int m, int bins, double2* inv_out, unsigned int* bad_f,
                         unsigned int* bad_d, cudaStream_t s) {
    const size_t smem_f = (size_t)m * 2 * m * sizeof(float2);
    const size_t smem_d = (size_t)m * 2 * m * sizeof(double2);
    cudaFuncSetAttribute(gauss_jordan_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
    cudaFuncSetAttribute(gauss_jordan_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
    gauss_jordan_kernel<float><<<bins, kInvThreads, smem_f, s>>>(k, m, nullptr, bad_f);
    gauss_jordan_kernel<double><<<bins, kInvThreads, smem_d, s>>>(k, m, inv_out, bad_d);
}

void launch_pd_check(const float2* k, int m, int bins, unsigned int* bad_herm, unsigned int* bad_pd,
                     double* min_pivot, cudaStream_t s) {
    const size_t smem = (size_t)m * m * sizeof(double2);
    cudaFuncSetAttribute(pd_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pd_check_kernel<<<bins, kInvThreads, smem, s>>>(k, m, bad_herm, bad_pd, min_pivot);
}

}  // namespace sslg
