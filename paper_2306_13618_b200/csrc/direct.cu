// K6: direct tiled kernel sum, Eq. (4.3) / the dense mat-vecs of Algorithm 1
// (P:506):  t_i = sum_j k(||tgt_i - src_j||) w_j  in fp64, no approximation.
// Targets live in registers, source tiles are staged in shared memory; the source
// range is split over blockIdx.y when there are too few targets to fill the GPU,
// with partial sums combined in a fixed order (deterministic) before the epilogue.
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"

namespace uotk {

namespace {

constexpr int kDT = 128;   // threads per block = targets per block
constexpr int kTile = 128; // sources per shared-memory tile

template <int D>
__device__ __forceinline__ double pair_sum_tile(const double (*sp)[kTile], const double* sw, int cnt,
                                                const double* xi, int kind, double inv_or_c2) {
    double acc = 0.0;
    if (kind == UOTK_GAUSS) {
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) {
            double r2 = 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - sp[t][j];
                r2 = fma(v, v, r2);
            }
            acc = fma(exp(-r2 * inv_or_c2), sw[j], acc);
        }
    } else if (kind == UOTK_GAUSS_R2) {
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) {
            double r2 = 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - sp[t][j];
                r2 = fma(v, v, r2);
            }
            acc = fma(r2 * exp(-r2 * inv_or_c2), sw[j], acc);
        }
    } else if (kind == UOTK_LAP || kind == UOTK_ENERGY) {
        // Laplace exp(-r/l) (inv_or_c2 = 1/l) and the energy kernel -r (Eq. 4.2; Table 1)
        const bool lap = kind == UOTK_LAP;
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) {
            double r2 = 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - sp[t][j];
                r2 = fma(v, v, r2);
            }
            const double r = sqrt(r2);
            acc = fma(lap ? exp(-r * inv_or_c2) : -r, sw[j], acc);
        }
    } else {
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) {
            double r2 = inv_or_c2;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - sp[t][j];
                r2 = fma(v, v, r2);
            }
            acc = fma(1.0 / sqrt(r2), sw[j], acc);
        }
    }
    return acc;
}

// partial[y][i] = sum over this block's source slice; if nsplit == 1 the epilogue runs here
template <int D, class Epi>
__global__ void __launch_bounds__(kDT) direct_k(int64_t n_src, const double* __restrict__ src,
                                                const double* __restrict__ w, int64_t n_tgt,
                                                const double* __restrict__ tgt, int kind, double inv_or_c2,
                                                int64_t slice, double* __restrict__ partial, Epi epi,
                                                unsigned long long* dmax) {
    __shared__ double sp[D][kTile];
    __shared__ double sw[kTile];
    const int64_t i = blockIdx.x * (int64_t)kDT + threadIdx.x;
    double xi[D];
    for (int t = 0; t < D; ++t) xi[t] = i < n_tgt ? tgt[i * D + t] : 0.0;
    const int64_t j0 = blockIdx.y * slice;
    const int64_t j1 = min(n_src, j0 + slice);
    double acc = 0.0;
    for (int64_t jt = j0; jt < j1; jt += kTile) {
        const int cnt = (int)((j1 - jt) < kTile ? (j1 - jt) : kTile);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += kDT) {
            for (int t = 0; t < D; ++t) sp[t][k] = src[(jt + k) * D + t];
            sw[k] = w[jt + k];
        }
        __syncthreads();
        acc += pair_sum_tile<D>(sp, sw, cnt, xi, kind, inv_or_c2);  // two-level summation
    }
    double dd = 0.0;
    if (i < n_tgt) {
        if (partial) partial[blockIdx.y * n_tgt + i] = acc;
        else dd = epi(i, acc);
    }
    if (!partial) warp_max_atomic(dmax, dd);
}

template <class Epi>
__global__ void combine_k(const double* __restrict__ partial, int nsplit, int64_t n, Epi epi,
                          unsigned long long* dmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double dd = 0.0;
    if (i < n) {
        double acc = 0.0;
        for (int y = 0; y < nsplit; ++y) acc += partial[y * n + i];
        dd = epi(i, acc);
    }
    warp_max_atomic(dmax, dd);
}

// Few targets (C1: 1000 x 1000): one warp per target over ALL sources (lanes stride the
// source tile in shared memory, then a shuffle reduction), the epilogue in the same launch
// — one kernel per half-step instead of a source-split kernel plus a combine kernel, so the
// CUDA-graph-replayed iteration is two short launches (C1: 38k -> 47k iterations/s; a CTA
// of 256 threads per target measured slower, 31k).
constexpr int kWTile = 1024;  // sources per shared-memory tile
template <int D, int WT, class Epi>
__global__ void __launch_bounds__(WT) direct_warp_k(int64_t n_src, const double* __restrict__ src,
                                                    const double* __restrict__ w, int64_t n_tgt,
                                                    const double* __restrict__ tgt, int kind, double inv_or_c2,
                                                    Epi epi, unsigned long long* dmax) {
    __shared__ double sp[D][kWTile];
    __shared__ double sw[kWTile];
    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)(WT / 32) + (threadIdx.x >> 5);
    double xi[D];
    for (int t = 0; t < D; ++t) xi[t] = i < n_tgt ? tgt[i * D + t] : 0.0;
    // the epilogue's per-target inputs, loaded now (their latency hides behind the pair loop)
    typename Epi::In ein{};
    if (lane == 0 && i < n_tgt) ein = epi.load(i);
    double acc = 0.0;
    for (int64_t jt = 0; jt < n_src; jt += kWTile) {
        const int cnt = (int)((n_src - jt) < kWTile ? (n_src - jt) : kWTile);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += WT) {
            for (int t = 0; t < D; ++t) sp[t][k] = src[(jt + k) * D + t];
            sw[k] = w[jt + k];
        }
        __syncthreads();
        double part = 0.0;
        for (int j = lane; j < cnt; j += 32) {
            double r2 = kind == UOTK_IMQ ? inv_or_c2 : 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - sp[t][j];
                r2 = fma(v, v, r2);
            }
            double kv;
            if (kind == UOTK_GAUSS) kv = exp(-r2 * inv_or_c2);
            else if (kind == UOTK_GAUSS_R2) kv = r2 * exp(-r2 * inv_or_c2);
            else if (kind == UOTK_LAP) kv = exp(-sqrt(r2) * inv_or_c2);
            else if (kind == UOTK_ENERGY) kv = -sqrt(r2);
            else kv = 1.0 / sqrt(r2);
            part = fma(kv, sw[j], part);
        }
        acc += part;  // two-level summation: per tile, then over tiles
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    double dd = 0.0;
    double wn;
    if (lane == 0 && i < n_tgt) dd = epi.apply(i, acc, ein, wn);
    warp_max_atomic(dmax, dd);
}

}  // namespace

template <class Epi>
void direct_sum_epi(int d, int64_t n_src, const double* src, const double* w, int64_t n_tgt, const double* tgt,
                    int kind, double param, const Epi& epi, unsigned long long* dmax, cudaStream_t s) {
    if (n_tgt == 0) return;
    const int64_t tb = (n_tgt + kDT - 1) / kDT;
    // split the sources over blockIdx.y until the grid has ~8 blocks per SM, keeping
    // slices of >= 64 sources (small problems, e.g. C1's 1000 x 1000, are latency-bound:
    // a long per-thread loop over all sources would leave the GPU idle)
    int sms = 148;
    {
        int dev = 0;
        UOTK_CUDA(cudaGetDevice(&dev));
        UOTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const double arg0 = kind == UOTK_IMQ ? param * param : 1.0 / param;
    static const bool warp_env = [] {  // UOTK_DIRECT_WARP=0: always the source-split kernel
        const char* e = getenv("UOTK_DIRECT_WARP");
        return !(e && e[0] == '0');
    }();
    // a warp per target: when the targets alone leave the GPU underfilled and a warp's
    // pass over all sources stays short
    if (warp_env && n_tgt <= 64LL * sms && n_src <= 16384 && tb < 2LL * sms) {
#define UOTK_WARP_LAUNCH(WT)                                                                                     \
    do {                                                                                                        \
        const unsigned blocks = (unsigned)((n_tgt + WT / 32 - 1) / (WT / 32));                                  \
        if (d == 1) direct_warp_k<1, WT, Epi><<<blocks, WT, 0, s>>>(n_src, src, w, n_tgt, tgt, kind, arg0, epi, dmax); \
        else if (d == 2) direct_warp_k<2, WT, Epi><<<blocks, WT, 0, s>>>(n_src, src, w, n_tgt, tgt, kind, arg0, epi, dmax); \
        else direct_warp_k<3, WT, Epi><<<blocks, WT, 0, s>>>(n_src, src, w, n_tgt, tgt, kind, arg0, epi, dmax); \
    } while (0)
        ProfScope ps_(kProfDirect, s);
        UOTK_WARP_LAUNCH(256);  // 128-thread CTAs measured the same
#undef UOTK_WARP_LAUNCH
        UOTK_LAUNCHED();
        return;
    }
    const int64_t want = (8LL * sms + tb - 1) / tb;
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(want, n_src / 64));
    if (nsplit > 65535) nsplit = 65535;
    const int64_t slice = n_src == 0 ? 1 : (n_src + nsplit - 1) / nsplit;
    const double arg = kind == UOTK_IMQ ? param * param : 1.0 / param;
    DevBuf<double> partial;
    if (nsplit > 1) partial.alloc((size_t)nsplit * n_tgt, s);
    dim3 grid((unsigned)tb, (unsigned)nsplit);
    ProfScope ps_(kProfDirect, s);
#define UOTK_DIRECT_LAUNCH(DD)                                                                           \
    direct_k<DD, Epi><<<grid, kDT, 0, s>>>(n_src, src, w, n_tgt, tgt, kind, arg, slice, partial.p, epi, dmax)
    if (d == 1) UOTK_DIRECT_LAUNCH(1);
    else if (d == 2) UOTK_DIRECT_LAUNCH(2);
    else UOTK_DIRECT_LAUNCH(3);
#undef UOTK_DIRECT_LAUNCH
    UOTK_LAUNCHED();
    if (nsplit > 1) {
        combine_k<Epi><<<(unsigned)((n_tgt + 255) / 256), 256, 0, s>>>(partial.p, (int)nsplit, n_tgt, epi, dmax);
        UOTK_LAUNCHED();
    }
}

template void direct_sum_epi<EpiStore>(int, int64_t, const double*, const double*, int64_t, const double*, int,
                                       double, const EpiStore&, unsigned long long*, cudaStream_t);
template void direct_sum_epi<EpiSinkhorn>(int, int64_t, const double*, const double*, int64_t, const double*, int,
                                          double, const EpiSinkhorn&, unsigned long long*, cudaStream_t);
template void direct_sum_epi<EpiDot>(int, int64_t, const double*, const double*, int64_t, const double*, int,
                                     double, const EpiDot&, unsigned long long*, cudaStream_t);

}  // namespace uotk
