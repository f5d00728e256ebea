// probe.cu — FP64 peak microbenchmark (roofline denominator, SURVEY §8d:
// "P_FP64 must be measured with a DFMA-chain microbenchmark on the box").
#include <cuda_runtime.h>

#include "ignis_b200.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma_chain(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains live
}

}  // namespace

extern "C" int ign_probe_fp64_peak(int device, double* tflops) {
    if (cudaSetDevice(device) != cudaSuccess) return IGN_CUDA_ERROR;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, 64 * 1024 * sizeof(double)) != cudaSuccess) return IGN_CUDA_ERROR;
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        k_dfma_chain<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
        if (rep > 0 && ms > 0.f) best = best > flops / (ms * 1e9) ? best : flops / (ms * 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return IGN_CUDA_ERROR;
    *tflops = best;
    return IGN_OK;
}
