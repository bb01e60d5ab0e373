// Probe: FP64 tensor-core MMA (mma.sync.m8n8k4.f64, SASS DMMA) throughput on this GPU,
// alone and interleaved with DFMA streams — decides whether the cell-group spread/gather
// (small 16x32x256 GEMMs per chunk) should move to DMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NMMA, int NFMA>
__global__ void mix(double* out, int iters) {
    double acc[8][2];
    double f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k][0] = acc[k][1] = 0.0; f[k] = threadIdx.x + k; }
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NMMA; ++k) dmma(acc[k % 8][0], acc[k % 8][1], a, b);
#pragma unroll
        for (int k = 0; k < NFMA; ++k) f[k % 8] = fma(f[k % 8], 0.999999, 1e-7);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1] + f[k];
    if (s == 12345.678) out[0] = s;
}

template <int NMMA, int NFMA>
void run(int sms, int clk_khz, double* out) {
    const int iters = 1 << 13, threads = 256, blocks = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mix<NMMA, NFMA><<<blocks, threads>>>(out, 16);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        mix<NMMA, NFMA><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warps = (double)blocks * threads / 32;
    const double mma_flops = 2.0 * 256 * NMMA * (double)iters * warps;   // m8n8k4 = 256 FMA per warp
    const double fma_flops = 2.0 * 32 * NFMA * (double)iters * warps;
    const double t = best * 1e-3;
    printf("NMMA=%2d NFMA=%2d  dmma %.2f TF  dfma %.2f TF  total %.2f TF  (fma-equivalent lanes/clk/SM %.1f)\n", NMMA,
           NFMA, mma_flops / t / 1e12, fma_flops / t / 1e12, (mma_flops + fma_flops) / t / 1e12,
           (mma_flops + fma_flops) / 2 / t / (sms * (clk_khz * 1e3)));
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    run<8, 0>(sms, clk, out);
    run<16, 0>(sms, clk, out);
    run<0, 8>(sms, clk, out);
    run<8, 8>(sms, clk, out);
    run<8, 16>(sms, clk, out);
    run<4, 32>(sms, clk, out);
    run<2, 32>(sms, clk, out);
    return 0;
}
