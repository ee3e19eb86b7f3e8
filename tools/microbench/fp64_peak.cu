// DFMA throughput microbenchmark (B200 FP64 roofline denominator): every
// thread runs 8 independent FMA chains for ITERS iterations; all SMs, enough
// warps to cover the FP64 latency.  Prints TFLOP/s (FMA = 2 FLOP).
#include <cstdio>
#include <cuda_runtime.h>

template <int ITERS>
__global__ void __launch_bounds__(256) k_dfma(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out;
    cudaMalloc(&out, sizeof(double));
    constexpr int ITERS = 1 << 16;
    const int blocks = sms * 8, threads = 256;
    k_dfma<ITERS><<<blocks, threads>>>(out, 0.999999, 1e-6);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<ITERS><<<blocks, threads>>>(out, 0.999999, 1e-6);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flop = 2.0 * 8.0 * ITERS * (double)blocks * threads;
    printf("{\"fp64_dfma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f}\n", flop / (best * 1e-3) / 1e12,
           sms, best);
    return 0;
}
