// DMMA.8x8x4 throughput vs warps per SM (W) and independent accumulator chains per warp (C):
// how many chains a warp needs to keep the FP64 tensor pipe busy.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe scripts/dmma_chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void probe(double* out, int iters) {
    double acc[C][2];
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(int W, double* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 8192 / C * 16;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<C><<<sms, 32 * W>>>(out, iters);
    cudaEventRecord(e0);
    probe<C><<<sms, 32 * W>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flop = (double)sms * W * iters * C * 512.0;
    printf("{\"warps_per_sm\": %d, \"chains\": %d, \"tflops\": %.2f}\n", W, C, flop / ms * 1e-9);
}
int main() {
    double* out; cudaMalloc(&out, 148 * 1024 * 8);
    for (int W : {4, 8, 12, 16, 32}) { run<2>(W, out); run<4>(W, out); run<8>(W, out); run<16>(W, out); }
    return 0;
}
