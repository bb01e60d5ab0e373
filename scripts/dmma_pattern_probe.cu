// DMMA.8x8x4 throughput vs the operand pattern of 8 consecutive DMMAs into 8 accumulators:
// NA distinct A registers x NB distinct B registers (NA * NB = 8, B index inner), operands
// from registers (opaque, no loads).  Found: which fragment layouts the gather / spread
// loops should use.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p scripts/dmma_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NA, int NB, bool BOUTER>
__global__ void probe(double* out, int iters) {
    const int lane = threadIdx.x & 31;
    double A[NA], B[NB], S[8][2] = {};
    for (int i = 0; i < NA; ++i) { A[i] = 1.0 + (lane + i) * 1e-9; asm volatile("mov.b64 %0, %0;" : "+d"(A[i])); }
    for (int j = 0; j < NB; ++j) { B[j] = 1.0 - (lane + j) * 1e-9; asm volatile("mov.b64 %0, %0;" : "+d"(B[j])); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = (NA * NB == 64) ? k : (BOUTER ? k % NA : k / NB), j = (NA * NB == 64) ? k : (BOUTER ? k / NA : k % NB);
                dmma(S[k][0], S[k][1], A[i], B[j]);
            }
        }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += S[k][0] + S[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NA, int NB, bool BOUTER>
void run(double* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1024, W = 16;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<NA, NB, BOUTER><<<sms, 32 * W>>>(out, iters);
    cudaEventRecord(e0);
    probe<NA, NB, BOUTER><<<sms, 32 * W>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flop = (double)sms * W * iters * 64 * 512.0;
    printf("{\"distinct_A\": %d, \"distinct_B\": %d, \"b_outer\": %d, \"tflops\": %.2f}\n", NA, NB, (int)BOUTER, flop / ms * 1e-9);
}
int main() {
    double* out; cudaMalloc(&out, 148 * 512 * 8);
    run<1, 8, false>(out); run<2, 4, false>(out); run<4, 2, false>(out); run<8, 1, false>(out);
    run<1, 8, true>(out); run<2, 4, true>(out); run<4, 2, true>(out); run<8, 1, true>(out);
    run<8, 8, false>(out);
    return 0;
}
