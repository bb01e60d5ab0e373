// How many warps per SM (and independent chains per warp) the FP64 FMA pipe needs to
// saturate on this GPU — design input for the cell-group kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_occupancy fp64_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}

// DFMA stream with a shared-memory broadcast operand every `ratio` FMAs (like the spread loop)
template <int CH>
__global__ void chains_lds(double* out, int iters, double b) {
    __shared__ double w[256];
    w[threadIdx.x % 256] = 0.999 + threadIdx.x * 1e-9;
    __syncthreads();
    double x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(&w[(i * 2) & 254]);
#pragma unroll
        for (int k = 0; k < CH; k += 2) {
            x[k] = fma(x[k], v.x, b);
            x[k + 1] = fma(x[k + 1], v.y, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}

template <class K>
float run(K kern, int blocks, int threads, int iters, double* out, bool lds) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        if (lds) ((void (*)(double*, int, double))kern)<<<blocks, threads>>>(out, iters, 1e-7);
        else ((void (*)(double*, int, double, double))kern)<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 14;
    printf("warps_per_sm chains lds lane_dfma_per_clk_per_sm(at %d MHz)\n", clk / 1000);
    for (int wps : {4, 8, 12, 16, 24, 32}) {
        const int threads = 128, blocks = sms * wps / 4;
        struct { const void* k; int ch; bool lds; } ks[] = {
            {(const void*)chains<2>, 2, false}, {(const void*)chains<4>, 4, false},
            {(const void*)chains<8>, 8, false}, {(const void*)chains<16>, 16, false},
            {(const void*)chains_lds<8>, 8, true}, {(const void*)chains_lds<32>, 32, true}};
        for (auto& k : ks) {
            float ms = run(k.k, blocks, threads, iters, out, k.lds);
            double lane_ops = (double)k.ch * iters * threads * blocks;
            printf("%2d %2d %d %.1f\n", wps, k.ch, (int)k.lds, lane_ops / (ms * 1e-3) / (sms * (clk * 1e3)));
        }
    }
    return 0;
}
