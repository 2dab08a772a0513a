// Single-warp QRCP experiment (development aid): one warp factors a 60x60
// complex matrix stored ROW-major in shared memory (lanes own columns j and
// j+32, so a row of the trailing matrix is one contiguous warp access);
// compares the R diagonal with the block-wide column-resident qrcp_to_rh.
#include "../../paper_2504_03373_b200/csrc/gsvd.cu"
#include <cstdio>
#include <cstdlib>
using namespace sslg;

__device__ void qrcp_warp(double2* Wr, int m, int* piv, double* rdiag) {
    const int lane = threadIdx.x & 31;
    __shared__ double2 u[kMaxM];
    double n2[2] = {0, 0};
    int cidx[2] = {lane, lane + 32};
    for (int h = 0; h < 2; ++h)
        if (cidx[h] < m)
            for (int i = 0; i < m; ++i) n2[h] += cnorm(Wr[i * m + cidx[h]]);
    int pos[2] = {-1, -1};
    for (int k = 0; k < m; ++k) {
        // pivot: largest remaining norm, lowest column on ties
        unsigned key = 0;
        for (int h = 0; h < 2; ++h)
            if (cidx[h] < m && pos[h] < 0) key = max(key, pivot_key(n2[h], cidx[h]));
        const unsigned kk = __reduce_max_sync(0xffffffffu, key);
        const int p = 63 - (int)((kk - 1u) & 63u);
        // Householder vector of column p, rows k..m-1 (two rows per lane)
        double2 x0 = Wr[k * m + p];
        double a2 = 0;
        for (int i = k + lane; i < m; i += 32) a2 += cnorm(Wr[i * m + p]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        const double alpha = fast_sqrt(a2);
        const double ax2 = cnorm(x0);
        double2 ph = make_double2(1, 0);
        double ax0 = 0;
        if (ax2 > 0) {
            const double ri = fast_rsqrt(ax2);
            ax0 = ax2 * ri;
            ph = make_double2(x0.x * ri, x0.y * ri);
        }
        const double tau = alpha > 0 ? fast_rcp(alpha * (alpha + ax0)) : 0.0;
        for (int i = k + lane; i < m; i += 32) u[i] = i == k ? make_double2(x0.x + ph.x * alpha, x0.y + ph.y * alpha) : Wr[i * m + p];
        __syncwarp();
        if (lane == 0) {
            piv[k] = p;
            rdiag[k] = alpha;
        }
        for (int h = 0; h < 2; ++h)
            if (cidx[h] == p) pos[h] = k;
        // trailing update of every unpivoted column (lane-owned)
        for (int h = 0; h < 2; ++h) {
            const int j = cidx[h];
            if (j >= m || pos[h] >= 0) continue;
            double sx = 0, sy = 0;
            for (int i = k; i < m; ++i) {
                const double2 uu = u[i], y = Wr[i * m + j];
                sx = fma(uu.x, y.x, fma(uu.y, y.y, sx));
                sy = fma(uu.x, y.y, fma(-uu.y, y.x, sy));
            }
            const double fx = tau * sx, fy = tau * sy;
            double nn = 0;
            for (int i = k; i < m; ++i) {
                const double2 uu = u[i];
                double2 y = Wr[i * m + j];
                y.x = fma(-fx, uu.x, fma(fy, uu.y, y.x));
                y.y = fma(-fx, uu.y, fma(-fy, uu.x, y.y));
                Wr[i * m + j] = y;
                if (i > k) nn += cnorm(y);
            }
            n2[h] = nn;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256, 2) qrw_bench(const double2* a, long long* clk, int* piv, double* rd, int m, int nwarps_active) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {  // a is column-major: row-major copy
        const int j = e / m, i = e % m;
        W[i * m + j] = a[e];
    }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x < 32) qrcp_warp(W, m, piv, rd);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
int main() {
    const int m = 60;
    static double2 h[3600];
    srand(1);
    for (int i = 0; i < m * m; ++i) h[i] = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    double2* a; long long* clk; int* piv; double* rd;
    cudaMalloc(&a, sizeof h); cudaMalloc(&clk, 8); cudaMalloc(&piv, 256); cudaMalloc(&rd, 512);
    cudaMemcpy(a, h, sizeof h, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(qrw_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
    for (int r = 0; r < 3; ++r) {
        qrw_bench<<<1, 256, 60000>>>(a, clk, piv, rd, m, 1);
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        double rdh[64]; int ph[64];
        cudaMemcpy(rdh, rd, 60 * 8, cudaMemcpyDeviceToHost); cudaMemcpy(ph, piv, 60 * 4, cudaMemcpyDeviceToHost);
        printf("single-warp qrcp: %lld cycles (%s); |R00| %.6f |R59| %.3e piv0 %d\n", c, cudaGetErrorString(cudaGetLastError()), rdh[0], rdh[59], ph[0]);
    }
    return 0;
}
