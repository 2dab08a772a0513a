// FP64 FMA throughput probe: the roofline denominator for the FP64 solver
// kernels (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
// Every thread runs 8 independent DFMA chains; the grid covers every SM
// several times over.
#include "../../include/sslgpu.h"
#include "common.cuh"

#include <cuda_runtime.h>

namespace sslg {

__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 123.456) out[0] = s;  // keep the chains live
}

// FP32 counterpart (the ceiling a float Jacobi would have: SURVEY's
// "FP32 pipe utilisation" framing of the solver)
__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-6f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 123.456f) out[0] = s;
}

template <class T, class K>
static int probe_tflops(int device, K kern, T a, T b, double* tflops) {
    if (cudaSetDevice(device) != cudaSuccess) return SSLG_DEVICE;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    T* d = nullptr;
    if (cudaMalloc(&d, sizeof(T)) != cudaSuccess) return SSLG_DEVICE;
    const int iters = 4096, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(d, 64, a, b);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(d, iters, a, b);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
    *tflops = flops / (best * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? SSLG_OK : SSLG_DEVICE;
}

}  // namespace sslg

extern "C" int sslg_probe_fp32_tflops(int device, double* tflops) {
    return sslg::probe_tflops<float>(device, sslg::ffma_probe_kernel, 0.999999f, 1e-6f, tflops);
}

extern "C" int sslg_probe_fp64_tflops(int device, double* tflops) {
    return sslg::probe_tflops<double>(device, sslg::dfma_probe_kernel, 0.999999, 1e-9, tflops);
}
