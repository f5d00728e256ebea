// Dev microbenchmark: FP64 dependent-chain latency and throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void chain(double* out, int iters, double a, double b, long long* cyc) {
    double x = threadIdx.x * 1e-9 + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = x + a;            // DADD
        else if (OP == 1) x = x * a;       // DMUL
        else if (OP == 2) x = fma(x, a, b);// DFMA
        else x = b / x;                    // DIV
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (x == 1234.5) out[0] = x;
}
template <int OP, int ILP>
__global__ void tput(double* out, int iters, double a, double b) {
    double x[ILP];
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            if (OP == 0) x[k] = x[k] + a; else if (OP == 1) x[k] = x[k] * a; else if (OP == 2) x[k] = fma(x[k], a, b); else x[k] = b / x[k];
        }
    double s = 0; for (int k = 0; k < ILP; ++k) s += x[k];
    if (s == 1234.5) out[0] = s;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024);
    const char* nm[4] = {"DADD", "DMUL", "DFMA", "DIV"};
    int iters = 4096;
    for (int op = 0; op < 4; ++op) {
        long long h;
        if (op == 0) chain<0><<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc);
        if (op == 1) chain<1><<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc);
        if (op == 2) chain<2><<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc);
        if (op == 3) chain<3><<<1, 32>>>(out, iters, 1.0000001, 1.0, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%s dependent latency: %.2f cycles\n", nm[op], (double)h / iters);
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int op = 0; op < 4; ++op) for (int warps = 4; warps <= 32; warps *= 2) {
        int it = op == 3 ? 256 : 4096;
        cudaEventRecord(e0);
        if (op == 0) tput<0, 4><<<sms, 32 * warps>>>(out, it, 1.0000001, 1e-9);
        if (op == 1) tput<1, 4><<<sms, 32 * warps>>>(out, it, 1.0000001, 1e-9);
        if (op == 2) tput<2, 4><<<sms, 32 * warps>>>(out, it, 1.0000001, 1e-9);
        if (op == 3) tput<3, 4><<<sms, 32 * warps>>>(out, it, 1.0000001, 1.0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * 32 * warps * it * 4;
        printf("%s ILP4 warps/SM=%2d: %.2f Gop/s  (%.1f lane-ops/clk/SM at %d MHz)\n", nm[op], warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
