// Standalone latency harness for the QRCP phase (development aid): one CTA,
// random 60x60 complex matrix, clock64 around the factorization.
#include "../../paper_2504_03373_b200/csrc/gsvd.cu"
#include <cstdio>
#include <cstdlib>
using namespace sslg;
__global__ void __launch_bounds__(256, 2) qr_bench(const double2* a, double2* out, long long* clk, int m) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    __shared__ QrScratch qs;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) W[e] = a[e];
    __syncthreads();
    long long t0 = clock64();
    qrcp_to_rh<60>(W, m, qs);
    long long t1 = clock64();
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) out[e] = W[e];
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
int main() {
    const int m = 60;
    static double2 h[3600];
    srand(1);
    for (int i = 0; i < m * m; ++i) h[i] = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    double2 *a, *o; long long* clk; long long c;
    cudaMalloc(&a, sizeof h); cudaMalloc(&o, sizeof h); cudaMalloc(&clk, 8);
    cudaMemcpy(a, h, sizeof h, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(qr_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
    for (int r = 0; r < 2; ++r) {
        qr_bench<<<1, 256, 60000>>>(a, o, clk, m);
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        printf("qrcp_to_rh<60>: %lld cycles (%s)\n", c, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
