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
// The elimination's arithmetic is the reference's, operation for operation:
// std::complex products and the division 1/a(col,col) in the limited-range
// textbook form the reference is built with (-fcx-limited-range), every
// product and sum rounded on its own (no FMA contraction: x86-64 baseline
// code has none), so both inverses are bit-identical to mat_inverse<T>.
//
// PD gate (NoiseModel::check_positive_definite, gsvd.cpp:736-754): the
// Hermitian test as written, then the smallest eigenvalue of the FP64
// widening from the reference's own cyclic complex Jacobi
// (hermitian_eigenvalues, eig.cpp:11-84: same pair order, same stop rule,
// same rotation formulas and rounding), one warp per bin.
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
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T sub_rn(T a, T b);
template <>
__device__ __forceinline__ float sub_rn<float>(float a, float b) { return __fsub_rn(a, b); }
template <>
__device__ __forceinline__ double sub_rn<double>(double a, double b) { return __dsub_rn(a, b); }

// std::complex<T> product, limited-range form (a*c - b*d, a*d + b*c)
template <typename C, typename T>
__device__ __forceinline__ C cmul_rn(C a, C b) {
    C r;
    r.x = sub_rn<T>(mul_rn<T>(a.x, b.x), mul_rn<T>(a.y, b.y));
    r.y = add_rn<T>(mul_rn<T>(a.x, b.y), mul_rn<T>(a.y, b.x));
    return r;
}

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
                                                                    unsigned int* bad_bin, int pivoting) {
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
        if (!pivoting) {  // Pivoting::none: the diagonal entry or give up (gsvd.cpp:33-39)
            if (tid == 0) {
                const C v = aug[col * w + col];
                s_piv = col;
                if (!(cabs_t<T>(v.x, v.y) > floor_)) s_fail = 1;
            }
        } else if (tid < 32) {
            // partial pivoting: first row with the largest magnitude
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
        // d = (1, 0) / a(col, col), limited-range division:
        // ((1*x + 0*y) / den, (0*x - 1*y) / den), den = x*x + y*y
        const C p = aug[col * w + col];
        const T den = add_rn<T>(mul_rn<T>(p.x, p.x), mul_rn<T>(p.y, p.y));
        C d;
        d.x = add_rn<T>(p.x, mul_rn<T>((T)0, p.y)) / den;
        d.y = sub_rn<T>(mul_rn<T>((T)0, p.x), p.y) / den;
        __syncthreads();
        for (int j = tid; j < w; j += blockDim.x) aug[col * w + j] = cmul_rn<C, T>(aug[col * w + j], d);
        for (int r = tid; r < m; r += blockDim.x) s_f[r] = aug[r * w + col];
        __syncthreads();
        for (int e = tid; e < m * w; e += blockDim.x) {
            const int r = e / w, j = e % w;
            if (r == col) continue;
            const C f = s_f[r];
            if (f.x == (T)0 && f.y == (T)0) continue;
            const C pr = cmul_rn<C, T>(f, aug[col * w + j]);
            C v = aug[e];
            v.x = sub_rn<T>(v.x, pr.x);
            v.y = sub_rn<T>(v.y, pr.y);
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

// Hermitian test + hermitian_eigenvalues (eig.cpp:11-84) on the FP64
// widening, one warp per bin (the matrix in shared memory).  The rotation
// sequence is the reference's -- pairs (p, q) in row-major order, skipped
// when |a_pq| <= 1e-14 max|a|, at most 60 sweeps -- and within a rotation the
// column pair is updated for every row, then the row pair for every column,
// each element with the reference's rounding; lanes split the rows/columns.
// bad_herm / bad_pd receive the first bad bin, min_eig[b] the smallest
// eigenvalue (NaN when the Hermitian test fails).
__device__ __forceinline__ double2 cmul_d(double2 a, double2 b) { return cmul_rn<double2, double>(a, b); }
__device__ __forceinline__ double2 rscale_d(double s, double2 a) {  // real * complex
    return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}

__global__ void __launch_bounds__(32) pd_check_kernel(const float2* __restrict__ k, int m, unsigned int* bad_herm,
                                                      unsigned int* bad_pd, double* min_eig) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* a = reinterpret_cast<double2*>(smem_raw);  // [m][m] row-major
    const int b = blockIdx.x;
    const int lane = threadIdx.x;
    const float2* kb = k + (size_t)b * m * m;
    double scale = 0, herm = 0, amax = 0;
    for (int e = lane; e < m * m; e += 32) {
        const int i = e / m, j = e % m;
        const float2 v = kb[i * m + j];
        const float2 u = kb[j * m + i];
        scale = fmax(scale, (double)hypotf(v.x, v.y));
        herm = fmax(herm, (double)hypotf(v.x - u.x, v.y + u.y));
        a[e] = f2d(v);
        amax = fmax(amax, hypot((double)v.x, (double)v.y));
    }
    for (int o = 16; o > 0; o >>= 1) {
        scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
        herm = fmax(herm, __shfl_xor_sync(0xffffffffu, herm, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    __syncwarp();
    if (herm > 1e-5 * scale + 1e-30) {
        if (lane == 0) {
            atomicMin(bad_herm, (unsigned)b);
            if (min_eig) min_eig[b] = __longlong_as_double(0x7ff8000000000000ll);
        }
        return;
    }
    const double stop = 1e-14 * (amax > 0 ? amax : 1.0);
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p + 1 < m; ++p) {
            for (int q = p + 1; q < m; ++q) {
                const double2 apq = a[p * m + q];
                const double mag = hypot(apq.x, apq.y);
                if (mag <= stop) continue;  // warp-uniform (every lane reads the same entry)
                rotated = true;
                const double2 ph = make_double2(apq.x / mag, apq.y / mag);
                const double app = a[p * m + p].x;
                const double aqq = a[q * m + q].x;
                const double tau = __dsub_rn(aqq, app) / __dmul_rn(2.0, mag);
                const double t = (tau >= 0 ? 1.0 : -1.0) /
                                 __dadd_rn(fabs(tau), sqrt(__dadd_rn(1.0, __dmul_rn(tau, tau))));
                const double c = 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(t, t)));
                const double s = __dmul_rn(t, c);
                const double2 sphc = rscale_d(s, cconj(ph));  // s * conj(ph)
                const double2 sph = rscale_d(s, ph);          // s * ph
                __syncwarp();
                for (int i = lane; i < m; i += 32) {  // columns p, q
                    const double2 aip = a[i * m + p], aiq = a[i * m + q];
                    const double2 x = rscale_d(c, aip), y = cmul_d(sphc, aiq);
                    const double2 u = cmul_d(sph, aip), v = rscale_d(c, aiq);
                    a[i * m + p] = make_double2(__dsub_rn(x.x, y.x), __dsub_rn(x.y, y.y));
                    a[i * m + q] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
                }
                __syncwarp();
                for (int j = lane; j < m; j += 32) {  // rows p, q
                    const double2 apj = a[p * m + j], aqj = a[q * m + j];
                    const double2 x = rscale_d(c, apj), y = cmul_d(sph, aqj);
                    const double2 u = cmul_d(sphc, apj), v = rscale_d(c, aqj);
                    a[p * m + j] = make_double2(__dsub_rn(x.x, y.x), __dsub_rn(x.y, y.y));
                    a[q * m + j] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
                }
                __syncwarp();
                if (lane == 0) {
                    a[p * m + p].y = 0.0;
                    a[q * m + q].y = 0.0;
                }
                __syncwarp();
            }
        }
        if (!rotated) break;
    }
    double mn = INFINITY;
    for (int i = lane; i < m; i += 32) mn = fmin(mn, a[i * m + i].x);
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) {
        if (!(mn > 0)) atomicMin(bad_pd, (unsigned)b);  // eig.back() > 0 (gsvd.cpp:746-747)
        if (min_eig) min_eig[b] = mn;
    }
}

void launch_gauss_jordan(const float2* k, int m, int bins, double2* inv_out, unsigned int* bad_f,
                         unsigned int* bad_d, cudaStream_t s, int pivoting, double2* inv_f_out) {
    const size_t smem_f = (size_t)m * 2 * m * sizeof(float2);
    const size_t smem_d = (size_t)m * 2 * m * sizeof(double2);
    cudaFuncSetAttribute(gauss_jordan_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
    cudaFuncSetAttribute(gauss_jordan_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
    gauss_jordan_kernel<float><<<bins, kInvThreads, smem_f, s>>>(k, m, inv_f_out, bad_f, pivoting);
    gauss_jordan_kernel<double><<<bins, kInvThreads, smem_d, s>>>(k, m, inv_out, bad_d, pivoting);
}

void launch_pd_check(const float2* k, int m, int bins, unsigned int* bad_herm, unsigned int* bad_pd,
                     double* min_eig, cudaStream_t s) {
    const size_t smem = (size_t)m * m * sizeof(double2);
    cudaFuncSetAttribute(pd_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pd_check_kernel<<<bins, 32, smem, s>>>(k, m, bad_herm, bad_pd, min_eig);
}

}  // namespace sslg
