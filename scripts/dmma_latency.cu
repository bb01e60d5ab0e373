// DMMA (mma.sync m8n8k4 f64) throughput vs warps/SM and independent accumulator chains
// per warp — how much independent MMA work the cell-group kernel must keep in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_latency dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NACC>
__global__ void chains(double* out, int iters) {
    double acc[NACC][2];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k][0] = acc[k][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) dmma(acc[k][0], acc[k][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += acc[k][0] + acc[k][1];
    if (s == 12345.678) out[0] = s;
}

template <int NACC>
void run(int wps, int sms, int clk, double* out) {
    const int threads = 128, blocks = sms * wps / 4;
    const int iters = (1 << 15) / NACC;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<NACC><<<blocks, threads>>>(out, 4);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        chains<NACC><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fma = 256.0 * NACC * iters * (double)blocks * threads / 32;
    printf("warps/SM %2d  chains %2d  %.1f TF  (%.1f FMA/clk/SM)\n", wps, NACC, 2 * fma / (best * 1e-3) / 1e12,
           fma / (best * 1e-3) / (sms * (clk * 1e3)));
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    for (int wps : {4, 8, 16, 32}) {
        run<1>(wps, sms, clk, out);
        run<2>(wps, sms, clk, out);
        run<4>(wps, sms, clk, out);
        run<8>(wps, sms, clk, out);
    }
    return 0;
}
