// Throughput of FP64 warp MMA (mma.sync m8n8k4 f64, DMMA) against DFMA on
// this B200 (development aid): every warp runs independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5 + threadIdx.x * 1e-7;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5 + threadIdx.x * 1e-7;
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fma(a, c[j], b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256, iters = 4096;
    double* d;
    cudaMalloc(&d, (size_t)blocks * threads * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        k_dmma<<<blocks, threads>>>(d, 16);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        // one m8n8k4 = 8*8*4 FMA = 512 FLOP per warp-instruction
        const double fl_mma = (double)blocks * (threads / 32) * iters * 8 * 512.0;
        printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl_mma / ms / 1e9);
        k_dfma<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl_fma = (double)blocks * threads * iters * 8 * 2.0;
        printf("DFMA:        %.2f TFLOP/s\n", fl_fma / ms / 1e9);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
