// Probe: latency of cudaMallocAsync from the default pool (release threshold = max)
// when allocation sizes alternate like the library's per-call buffers.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <vector>
int main() {
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaStream_t s;
    cudaStreamCreate(&s);
    double worst = 0, total = 0;
    int slow = 0;
    for (int rep = 0; rep < 40; ++rep) {
        std::vector<void*> ps;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 6; ++i) { void* p; cudaMallocAsync(&p, (64u << 20) + i * 4096, s); ps.push_back(p); }
        auto t1 = std::chrono::steady_clock::now();
        void* big; cudaMallocAsync(&big, (size_t)4 << 30, s); cudaMemsetAsync(big, 0, 1 << 20, s);
        for (void* p : ps) cudaFreeAsync(p, s);
        cudaFreeAsync(big, s);
        cudaStreamSynchronize(s);
        double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        total += ms; if (ms > worst) worst = ms; if (ms > 5) ++slow;
    }
    printf("6 x 64 MB cudaMallocAsync: mean %.3f ms worst %.3f ms, %d of 40 > 5 ms\n", total / 40, worst, slow);
    return 0;
}
