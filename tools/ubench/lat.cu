// Latency microbenchmarks (development aid): DFMA chain, SHFL chain (f64),
// sqrt(f64), LDS.64 chain, __syncthreads with 8 warps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* clk, double a, int n) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* clk, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_sqrt(double* out, long long* clk, int n) {
    double x = 2.0 + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = sqrt(x) + 1.5; }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_div(double* out, long long* clk, int n) {
    double x = 2.0 + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = 1.0 / x + 1.5; }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_lds(double* out, long long* clk, int n) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t1 = clock64();
    out[threadIdx.x] = j; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_bar(double* out, long long* clk, int n) {
    __shared__ double s[256];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncthreads(); x += s[(threadIdx.x + 1) & 255]; __syncthreads(); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
// DFMA throughput with 8 warps, 8 independent chains each
__global__ void k_dfma_tp(double* out, long long* clk, double a, int n) {
    double x[8];
    for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-3 + u;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, 1e-3);
    long long t1 = clock64();
    double s = 0; for (int u = 0; u < 8; ++u) s += x[u];
    out[threadIdx.x] = s; if (threadIdx.x == 0) clk[0] = t1 - t0;
}
int main() {
    double* out; long long* clk; long long h;
    cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 64);
    const int n = 1000;
    auto run = [&](const char* name, auto launch, double per) {
        launch(); cudaDeviceSynchronize(); launch(); cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %8.2f cycles/op\n", name, (double)h / per);
    };
    run("dfma latency", [&] { k_dfma<<<1, 32>>>(out, clk, 0.999, n); }, 4.0 * n);
    run("shfl.f64 xor (+dadd) lat", [&] { k_shfl<<<1, 32>>>(out, clk, n); }, 2.0 * n);
    run("sqrt f64 latency", [&] { k_sqrt<<<1, 32>>>(out, clk, n); }, 1.0 * n);
    run("1/x f64 latency", [&] { k_div<<<1, 32>>>(out, clk, n); }, 1.0 * n);
    run("lds chain latency", [&] { k_lds<<<1, 32>>>(out, clk, n); }, 1.0 * n);
    run("2x bar+sts/lds 8 warps", [&] { k_bar<<<1, 256>>>(out, clk, n); }, 1.0 * n);
    run("dfma tp 1 warp (cyc/instr)", [&] { k_dfma_tp<<<1, 32>>>(out, clk, 0.999, n); }, 8.0 * n);
    run("dfma tp 4 warps/SM", [&] { k_dfma_tp<<<1, 128>>>(out, clk, 0.999, n); }, 8.0 * n);
    run("dfma tp 8 warps/SM", [&] { k_dfma_tp<<<1, 256>>>(out, clk, 0.999, n); }, 8.0 * n);
    run("dfma tp 16 warps/SM", [&] { k_dfma_tp<<<1, 512>>>(out, clk, 0.999, n); }, 8.0 * n);
    return 0;
}
