// Checks the fragment layout of mma.sync.aligned.m8n8k4.row.col.f64 assumed by the
// DMMA cell-group kernel:  A[8x4] a0 = A[lane>>2][lane&3];  B[4x8] b0 = B[lane&3][lane>>2];
// D[8x8] {d0,d1} = D[lane>>2][2*(lane&3) + {0,1}].
//   nvcc -gencode arch=compute_100a,code=sm_100a -o dmma_layout dmma_layout.cu && ./dmma_layout
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* D) {
    const int l = threadIdx.x;
    double a = A[(l >> 2) * 4 + (l & 3)];
    double b = B[(l & 3) * 8 + (l >> 2)];
    double d0 = C[(l >> 2) * 8 + 2 * (l & 3)], d1 = C[(l >> 2) * 8 + 2 * (l & 3) + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
    D[(l >> 2) * 8 + 2 * (l & 3)] = d0;
    D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}

int main() {
    double A[32], B[32], C[64], D[64];
    for (int i = 0; i < 32; ++i) { A[i] = 1.0 + i * 0.5; B[i] = 2.0 - i * 0.25; }
    for (int i = 0; i < 64; ++i) C[i] = i * 0.125;
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512); cudaMalloc(&dD, 512);
    cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C, 512, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC, dD);
    cudaMemcpy(D, dD, 512, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
            double r = C[i * 8 + j];
            for (int kk = 0; kk < 4; ++kk) r += A[i * 4 + kk] * B[kk * 8 + j];
            double e = D[i * 8 + j] - r;
            if (e < 0) e = -e;
            if (e > maxerr) maxerr = e;
        }
    printf("dmma m8n8k4.f64 layout check: max abs err %.3e -> %s\n", maxerr, maxerr == 0.0 ? "OK" : "MISMATCH");
    return maxerr != 0.0;
}
