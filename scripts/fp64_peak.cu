// FP64 FMA-pipe peak on this GPU (the ALU roofline denominator of bench.py):
// every thread runs 8 independent DFMA chains; grid = 4 x SMs x 512 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 512, blocks = sms * 4, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, \"best_ms\": %.3f, "
           "\"dfma_per_clk_per_sm_at_max_clock\": %.1f}\n",
           flops / (best * 1e-3) / 1e12, sms, clk / 1e3, best, flops / (best * 1e-3) / (sms * clk * 1e3) / 2);
    return cudaGetLastError() != cudaSuccess;
}
