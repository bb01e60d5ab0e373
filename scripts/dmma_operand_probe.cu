// DMMA.8x8x4 throughput with the operand patterns of the spread loops (spread3d_fly_k,
// sinkhorn3d_ws_k): per k-step each warp loads its fragments from shared memory, forms the
// A operand by a DMUL, and issues 8 DMMAs into 8 accumulators (2 per A fragment, 4 A x 2 B).
//   mode 0: fixed registers (the chain probe)          mode 1: 4 A x 2 B operands per step, from registers
//   mode 2: + operands loaded from shared memory       mode 3: + the A operand formed by a DMUL
// The half-step's loops (sinkhorn3d_ws_k), 16 DMMAs per step into 16 accumulators:
//   mode 4: spread warp, w_p on x (12 DMUL per step)   mode 5: w_p on y (10 DMUL per step)
//   mode 6: gather warp: B fragments in registers, 4 k-steps of 8 DMMAs per m-tile, then the
//           (a, b) contraction (16 DFMA per m-tile)
//   mode 7: mode 6 without the contraction (accumulators carried)
//   mode 9: mode 7 with the operands swapped (the footprint fragment as A, the window as B)
//   mode 8: mode 6 with the contraction of m-tile mt after the DMMAs of m-tile mt + 1
//           (two accumulator sets)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_operand_probe scripts/dmma_operand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void probe(double* out, int iters) {
    __shared__ double ww[2][3][32][20];
    for (int i = threadIdx.x; i < 2 * 3 * 32 * 20; i += blockDim.x) (&ww[0][0][0][0])[i] = 1.0 + i * 1e-9;
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3, a0 = 2 * ((threadIdx.x >> 5) & 7);
    double S[4][2][2] = {};
    double ra[8], rb[2];
    for (int i = 0; i < 8; ++i) ra[i] = 1.0 + (lane + i) * 1e-9;
    rb[0] = 1.0 - lane * 1e-9; rb[1] = 1.0 + lane * 2e-9;
    for (int it = 0; it < iters; ++it) {
        const double(*w)[32][20] = ww[it & 1];  // operands change every iteration (no hoisting)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int p = 4 * ks + tq;
            double am[4], b0, b1;
            if (MODE == 0) {
                am[0] = am[1] = am[2] = am[3] = ra[0]; b0 = b1 = rb[0];
            } else if (MODE == 1) {
                am[0] = ra[ks & 7]; am[1] = ra[(ks + 1) & 7]; am[2] = ra[(ks + 2) & 7]; am[3] = ra[(ks + 3) & 7];
                b0 = rb[ks & 1]; b1 = rb[(ks + 1) & 1];
            } else {
                b0 = w[2][p][gq]; b1 = w[2][p][8 + gq];
                const double2 xa = *reinterpret_cast<const double2*>(&w[0][p][a0]);
                const double ylo = w[1][p][gq], yhi = w[1][p][8 + gq];
                if (MODE == 2) { am[0] = xa.x; am[1] = ylo; am[2] = xa.y; am[3] = yhi; }
                else { am[0] = xa.x * ylo; am[1] = xa.x * yhi; am[2] = xa.y * ylo; am[3] = xa.y * yhi; }
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                dmma(S[mt][0][0], S[mt][0][1], am[mt], b0);
                dmma(S[mt][1][0], S[mt][1][1], am[mt], b1);
            }
        }
    }
    double s = 0;
    for (int mt = 0; mt < 4; ++mt) for (int n = 0; n < 2; ++n) s += S[mt][n][0] + S[mt][n][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// modes 4-5: 64 DMMAs per iteration (4 k-steps x 16); modes 6-9: 128 (4 m-tiles x 4 k-steps x 8)
template <int MODE>
__global__ void probe_ws(double* out, int iters) {
    __shared__ double ww[2][3][32][20];
    __shared__ double wsc2[2][32];
    for (int i = threadIdx.x; i < 2 * 3 * 32 * 20; i += blockDim.x) (&ww[0][0][0][0])[i] = 1.0 + i * 1e-9;
    if (threadIdx.x < 64) (&wsc2[0][0])[threadIdx.x] = 1.0 - threadIdx.x * 1e-9;
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3, a0 = 4 * ((threadIdx.x >> 5) & 3);
    double S[8][2][2] = {};
    double Fb[8][4];
    for (int nt = 0; nt < 8; ++nt)
        for (int k = 0; k < 4; ++k) {
            Fb[nt][k] = 1.0 + (nt * 4 + k + lane) * 1e-9;
            asm volatile("mov.b64 %0, %0;" : "+d"(Fb[nt][k]));  // opaque: no rematerialisation in the loop
        }
    double part = 0.0;
    for (int it = 0; it < iters; ++it) {
        const double(*w)[32][20] = ww[it & 1];  // operands change every iteration (no hoisting)
        const double* wsc = wsc2[it & 1];
        if (MODE == 9) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double az = w[2][p][4 * ks + tq];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) dmma(S[nt][0][0], S[nt][0][1], Fb[nt][ks], az);
                }
            }
        } else if (MODE == 7) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double az = w[2][p][4 * ks + tq];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) dmma(S[nt][0][0], S[nt][0][1], az, Fb[nt][ks]);
                }
            }
        } else if (MODE == 8) {
            double acc[2][8][2];
            auto contract = [&](int mt, double (&a)[8][2]) {
                const int p = 8 * mt + gq;
                const double2 ylo = *reinterpret_cast<const double2*>(&w[1][p][2 * tq]);
                const double2 yhi = *reinterpret_cast<const double2*>(&w[1][p][8 + 2 * tq]);
                const double2 xa = *reinterpret_cast<const double2*>(&w[0][p][a0]);
                const double2 xb = *reinterpret_cast<const double2*>(&w[0][p][a0 + 2]);
                const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
                for (int al = 0; al < 4; ++al) {
                    double q = a[2 * al][0] * ylo.x;
                    q = fma(a[2 * al][1], ylo.y, q);
                    q = fma(a[2 * al + 1][0], yhi.x, q);
                    q = fma(a[2 * al + 1][1], yhi.y, q);
                    part = fma(q, xv[al], part);
                }
            };
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
                double (&a)[8][2] = acc[mt & 1];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) a[nt][0] = a[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double az = w[2][p][4 * ks + tq];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) dmma(a[nt][0], a[nt][1], az, Fb[nt][ks]);
                }
                if (mt > 0) contract(mt - 1, acc[(mt - 1) & 1]);
            }
            contract(3, acc[1]);
        } else if (MODE == 6) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
                double acc[8][2];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double az = w[2][p][4 * ks + tq];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) dmma(acc[nt][0], acc[nt][1], az, Fb[nt][ks]);
                }
                const double2 ylo = *reinterpret_cast<const double2*>(&w[1][p][2 * tq]);
                const double2 yhi = *reinterpret_cast<const double2*>(&w[1][p][8 + 2 * tq]);
                const double2 xa = *reinterpret_cast<const double2*>(&w[0][p][a0]);
                const double2 xb = *reinterpret_cast<const double2*>(&w[0][p][a0 + 2]);
                const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
                for (int al = 0; al < 4; ++al) {
                    double q = acc[2 * al][0] * ylo.x;
                    q = fma(acc[2 * al][1], ylo.y, q);
                    q = fma(acc[2 * al + 1][0], yhi.x, q);
                    q = fma(acc[2 * al + 1][1], yhi.y, q);
                    part = fma(q, xv[al], part);
                }
            }
        } else {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const int p = 4 * ks + tq;
                const double b0 = w[2][p][gq], b1 = w[2][p][8 + gq];
                const double wv = wsc[p];
                const double2 xa = *reinterpret_cast<const double2*>(&w[0][p][a0]);
                const double2 xb = *reinterpret_cast<const double2*>(&w[0][p][a0 + 2]);
                double xv[4], ylo, yhi;
                if (MODE == 4) {
                    xv[0] = wv * xa.x; xv[1] = wv * xa.y; xv[2] = wv * xb.x; xv[3] = wv * xb.y;
                    ylo = w[1][p][gq]; yhi = w[1][p][8 + gq];
                } else {
                    xv[0] = xa.x; xv[1] = xa.y; xv[2] = xb.x; xv[3] = xb.y;
                    ylo = wv * w[1][p][gq]; yhi = wv * w[1][p][8 + gq];
                }
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const double am = xv[mt >> 1] * ((mt & 1) ? yhi : ylo);
                    dmma(S[mt][0][0], S[mt][0][1], am, b0);
                    dmma(S[mt][1][0], S[mt][1][1], am, b1);
                }
            }
        }
    }
    double s = part;
    for (int mt = 0; mt < 8; ++mt) for (int n = 0; n < 2; ++n) s += S[mt][n][0] + S[mt][n][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run_ws(int W, int ctas, double* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe_ws<MODE><<<sms * ctas, 32 * W>>>(out, iters);
    cudaEventRecord(e0);
    probe_ws<MODE><<<sms * ctas, 32 * W>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const int dmma_per_iter = MODE >= 6 ? 128 : 64;  // gather pattern: 4 m-tiles x 4 k-steps x 8
    const double flop = (double)sms * ctas * W * iters * dmma_per_iter * 512.0;
    printf("{\"mode\": %d, \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", MODE, W, ctas, flop / ms * 1e-9);
}
template <int MODE>
void run(int W, int ctas, double* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<MODE><<<sms * ctas, 32 * W>>>(out, iters);
    cudaEventRecord(e0);
    probe<MODE><<<sms * ctas, 32 * W>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flop = (double)sms * ctas * W * iters * 8 * 8 * 512.0;
    printf("{\"mode\": %d, \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", MODE, W, ctas, flop / ms * 1e-9);
}
int main() {
    double* out; cudaMalloc(&out, 148 * 4 * 1024 * 8);
    for (int c : {1, 2}) { run<0>(8, c, out); run<1>(8, c, out); run<2>(8, c, out); run<3>(8, c, out); }
    for (int c : {1, 2}) { run_ws<4>(4, c, out); run_ws<5>(4, c, out); run_ws<6>(4, c, out); }
    for (int c : {1, 2}) { run_ws<4>(8, c, out); run_ws<5>(8, c, out); run_ws<6>(8, c, out); }
    for (int c : {1, 2}) { run_ws<7>(4, c, out); run_ws<8>(4, c, out); run_ws<7>(8, c, out); run_ws<8>(8, c, out); }
    for (int c : {1, 2}) { run_ws<9>(4, c, out); run_ws<9>(8, c, out); }
    return 0;
}
