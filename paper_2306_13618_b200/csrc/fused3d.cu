// Tuned d = 3 NFFT passes.
//
// Points are sorted by grid cell (points.cu), so every run of equal keys shares one
// (2m)^3 window footprint on the oversampled grid.  Runs are cut into chunks of <= 32
// points and the window values of every chunk (3 axes x 32 slots x 2m taps, zero for
// empty slots) are computed ONCE per point set (fused3d_prepare) — the points do not
// move between Sinkhorn iterations.  A 128-thread CTA then walks a contiguous,
// chunk-balanced range of chunks, streaming each chunk's 12 KB window block into
// shared memory with a TMA bulk copy (cp.async.bulk + mbarrier, double buffered).
// For each cell group the threads own fixed footprint columns (b, c) x all 2m values
// of a, so that
//   gather  (outer sum of (4.6)):  t_p = sum_abc g[a,b,c] X_p[a] Y_p[b] Z_p[c]
//   spread  (inner sum of (4.6)):  S[a,b,c] += w_p X_p[a] Y_p[b] Z_p[c]
// are register-blocked FMA loops (window values broadcast from shared memory).  The
// per-point partial gathers are reduced with a transposing warp butterfly and a
// 4-warp shared-memory sum, the Sinkhorn update (3.3)/(3.4) runs on t_p, and the new
// weight w_p = mass_p u_p is spread into registers at once — one pass over the points
// per half-step; the footprint is read once and flushed once (fp64 RED) per group.
#include <cub/cub.cuh>

#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "window.cuh"

namespace uotk {

namespace {

constexpr int kM = 8;                  // window half-width of the tuned kernels
constexpr int kT = 2 * kM;             // taps per axis
constexpr int kThreads = 128;          // 4 warps
constexpr int kChunk = 32;             // points per chunk (one per lane in the butterfly)
constexpr int kNJ = kT * kT / kThreads;  // owned (b, c) columns per thread
constexpr int kWinDoubles = 3 * kChunk * kT;
constexpr uint32_t kWinBytes = kWinDoubles * sizeof(double);  // 12 KB
constexpr int kBlocksPerSM = 2;

struct __align__(128) Smem {
    double win[2][3][kChunk][kT];  // double-buffered window blocks (TMA destination)
    double wn[kChunk];             // spread weights of the chunk
    double red[kThreads / 32][kChunk];
    unsigned long long bar[2];     // mbarriers of the two buffers
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion signalled on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// MODE: 0 = gather -> epilogue -> spread (Sinkhorn half-step), 1 = spread only, 2 = gather only
template <int MODE, class Epi>
__global__ void __launch_bounds__(kThreads, kBlocksPerSM)
chunked3d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
            int64_t nchunks, int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out,
            const double* __restrict__ w_in, Epi epi, unsigned long long* dmax) {
    constexpr bool GATHER = MODE != 1;
    constexpr bool SPREAD = MODE != 2;
    __shared__ Smem sm;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // owned columns: (b, c) for b in {cb0, cb0 + 1} (one 16-byte load of Y_p[b..b+1])
    const int cc = tid % kT;
    const int cb0 = kNJ * (tid / kT);
    int cb[kNJ];
#pragma unroll
    for (int j = 0; j < kNJ; ++j) cb[j] = cb0 + j;

    // cost-balanced contiguous chunk range of this CTA (fused3d_prepare)
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t cend = bounds[blockIdx.x + 1];
    const int64_t ng2 = (int64_t)ng * ng;
    (void)nchunks;

    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < 2 && cbeg + k < cend; ++k) {
            mbar_expect_tx(&sm.bar[k], kWinBytes);
            bulk_g2s(&sm.win[k][0][0][0], win + (cbeg + k) * kWinDoubles, kWinBytes, &sm.bar[k]);
        }
    }

    double g[kNJ][kT];  // footprint of the current group (gather source)
    double s[kNJ][kT];  // spread accumulators of the current group
    int32_t cur_key = -1;
    int64_t gbase = 0;
    double ddmax = 0.0;

    for (int64_t c = cbeg; c < cend; ++c) {
        const int k = (int)(c - cbeg);
        const int buf = k & 1;
        const int4 dsc = desc[c];  // {first point, count, key, 0}
        const int64_t p0 = dsc.x;
        const int cnt = dsc.y;
        const int32_t key = dsc.z;

        if (key != cur_key) {
            if (SPREAD && cur_key >= 0) {
#pragma unroll
                for (int j = 0; j < kNJ; ++j) {
                    const int64_t col = gbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
                    for (int a = 0; a < kT; ++a)
                        if (s[j][a] != 0.0) atomicAdd(grid_out + col + a * ng2, s[j][a]);
                }
            }
            cur_key = key;
            const int c2 = key % ng;
            const int c1 = (key / ng) % ng;
            const int c0 = key / ng2;
            gbase = ((int64_t)(c0 - kM + 1) * ng + (c1 - kM + 1)) * ng + (c2 - kM + 1);
#pragma unroll
            for (int j = 0; j < kNJ; ++j) {
                const int64_t col = gbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
                for (int a = 0; a < kT; ++a) {
                    if (GATHER) g[j][a] = __ldg(grid_in + col + a * ng2);
                    if (SPREAD) s[j][a] = 0.0;
                }
            }
        }
        if (GATHER) {
            // warm L1 with the epilogue's per-point inputs and, at a group boundary, with
            // the next group's footprint columns (hides their latency behind this chunk)
            if (lane < cnt) epi.prefetch(p0 + lane);
            if (c + 1 < cend) {
                const int32_t nkey = desc[c + 1].z;
                if (nkey != key) {
                    const int n2 = nkey % ng, n1 = (nkey / ng) % ng, n0 = nkey / ng2;
                    const int64_t nbase = ((int64_t)(n0 - kM + 1) * ng + (n1 - kM + 1)) * ng + (n2 - kM + 1);
#pragma unroll
                    for (int j = 0; j < kNJ; ++j) {
                        const double* colp = grid_in + nbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
                        for (int a = 0; a < kT; ++a)
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(colp + a * ng2));
                    }
                }
            }
        }
        double wn_reg;  // spread weight of slot `lane` (broadcast by shuffles in the spread)
        mbar_wait(&sm.bar[buf], (k >> 1) & 1);
        const double(*wx)[kT] = sm.win[buf][0];
        const double(*wy)[kT] = sm.win[buf][1];
        const double(*wz)[kT] = sm.win[buf][2];

        if (GATHER) {
            double r[kChunk];
#pragma unroll
            for (int p = 0; p < kChunk; p += 2) {
                double e[2][kNJ][2];
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int j = 0; j < kNJ; ++j) e[q][j][0] = e[q][j][1] = 0.0;
#pragma unroll
                for (int a = 0; a < kT; a += 2) {
                    const double2 x0 = *reinterpret_cast<const double2*>(&wx[p][a]);
                    const double2 x1 = *reinterpret_cast<const double2*>(&wx[p + 1][a]);
#pragma unroll
                    for (int j = 0; j < kNJ; ++j) {
                        e[0][j][0] = fma(g[j][a], x0.x, e[0][j][0]);
                        e[0][j][1] = fma(g[j][a + 1], x0.y, e[0][j][1]);
                        e[1][j][0] = fma(g[j][a], x1.x, e[1][j][0]);
                        e[1][j][1] = fma(g[j][a + 1], x1.y, e[1][j][1]);
                    }
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double2 yv = *reinterpret_cast<const double2*>(&wy[p + q][cb0]);
                    const double v = fma(e[q][0][0] + e[q][0][1], yv.x, (e[q][1][0] + e[q][1][1]) * yv.y);
                    r[p + q] = v * wz[p + q][cc];
                }
            }
            // transposing butterfly: lane l ends with this warp's sum for slot l
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) {
                const bool upper = lane & sh;
#pragma unroll
                for (int kk = 0; kk < sh; ++kk) {
                    const double send = upper ? r[kk] : r[kk + sh];
                    const double keep = upper ? r[kk + sh] : r[kk];
                    r[kk] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
                }
            }
            sm.red[warp][lane] = r[0];
            __syncthreads();
            // every warp sums the 4 warp partials of slot `lane`; warp 0 applies the
            // epilogue (writes), the others evaluate the same update to obtain the
            // spread weight in registers — no second barrier
            double wn = 0.0;
            if (lane < cnt) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; ++w) t += sm.red[w][lane];
                if (warp == 0) {
                    const double dd = epi(p0 + lane, t);
                    ddmax = fmax(ddmax, dd);
                    if (SPREAD) wn = epi.w_next[p0 + lane];
                } else if (SPREAD) {
                    wn = epi.weight(p0 + lane, t);
                }
            }
            wn_reg = wn;
        } else {
            wn_reg = (lane < cnt) ? w_in[p0 + lane] : 0.0;
        }

        if (SPREAD) {
#pragma unroll 2
            for (int p = 0; p < kChunk; ++p) {
                const double wzp = __shfl_sync(0xffffffffu, wn_reg, p) * wz[p][cc];
                const double2 yv = *reinterpret_cast<const double2*>(&wy[p][cb0]);
                double wj[kNJ];
                wj[0] = wzp * yv.x;
                wj[1] = wzp * yv.y;
#pragma unroll
                for (int a = 0; a < kT; a += 2) {
                    const double2 xv = *reinterpret_cast<const double2*>(&wx[p][a]);
#pragma unroll
                    for (int j = 0; j < kNJ; ++j) {
                        s[j][a] = fma(wj[j], xv.x, s[j][a]);
                        s[j][a + 1] = fma(wj[j], xv.y, s[j][a + 1]);
                    }
                }
            }
        }
        __syncthreads();  // every thread is done with win[buf] and wn
        if (tid == 0 && c + 2 < cend) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.bar[buf], kWinBytes);
            bulk_g2s(&sm.win[buf][0][0][0], win + (c + 2) * kWinDoubles, kWinBytes, &sm.bar[buf]);
        }
    }
    if (SPREAD && cur_key >= 0) {
#pragma unroll
        for (int j = 0; j < kNJ; ++j) {
            const int64_t col = gbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
            for (int a = 0; a < kT; ++a)
                if (s[j][a] != 0.0) atomicAdd(grid_out + col + a * ng2, s[j][a]);
        }
    }
    if (GATHER && warp == 0) warp_max_atomic(dmax, ddmax);
}

// ---------------------------------------------------------------- chunk preparation
__global__ void chunk_count_k(const int32_t* __restrict__ run_len, const int32_t* __restrict__ nruns,
                              int32_t* __restrict__ nchunk) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < *nruns) nchunk[r] = (run_len[r] + kChunk - 1) / kChunk;
}

__global__ void chunk_desc_k(const int32_t* __restrict__ run_key, const int32_t* __restrict__ run_len,
                             const int32_t* __restrict__ run_start, const int32_t* __restrict__ chunk_off,
                             const int32_t* __restrict__ nruns, int4* __restrict__ desc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *nruns) return;
    const int len = run_len[r];
    const int nc = (len + kChunk - 1) / kChunk;
    for (int k = 0; k < nc; ++k)
        desc[chunk_off[r] + k] = make_int4(run_start[r] + k * kChunk, min(kChunk, len - k * kChunk), run_key[r], 0);
}

// window values of every chunk: [chunk][axis][slot][tap], zero for empty slots
__global__ void chunk_window_k(const int4* __restrict__ desc, const double* __restrict__ u, int64_t n,
                               KBWindow w, double* __restrict__ out) {
    const int64_t c = blockIdx.x;
    const int4 dsc = desc[c];
    const int a = threadIdx.x % kT;
    const int q = threadIdx.x / kT;
    double* o = out + c * kWinDoubles;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int pp = 0; pp < kChunk / (kThreads / kT); ++pp) {
            const int p = q + pp * (kThreads / kT);
            double val = 0.0;
            if (p < dsc.y) {
                const double ut = u[ax * n + dsc.x + p];
                val = kb_phi(ut - floor(ut) + (double)(kM - 1 - a), w);
            }
            o[(ax * kChunk + p) * kT + a] = val;
        }
    }
}

// cost of a chunk for the static partition: 8 per chunk + 2 when it opens a cell group
// (footprint load and flush), in units of 1/8 chunk
__global__ void chunk_cost_k(const int4* __restrict__ desc, int64_t nchunks, int32_t* __restrict__ cost) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < nchunks) cost[c] = 8 + ((c == 0 || desc[c].z != desc[c - 1].z) ? 2 : 0);
}

// bounds[b] = first chunk whose inclusive cost prefix exceeds b * total / nb
__global__ void chunk_bounds_k(const int32_t* __restrict__ prefix, int64_t nchunks, int nb,
                               int32_t* __restrict__ bounds) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    if (b == nb) {
        bounds[b] = (int32_t)nchunks;
        return;
    }
    const double target = (double)prefix[nchunks - 1] * b / nb;
    int64_t lo = 0, hi = nchunks;  // first c with prefix[c] > target
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if ((double)prefix[mid] > target) hi = mid;
        else lo = mid + 1;
    }
    bounds[b] = (int32_t)(b == 0 ? 0 : lo);
}

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

// The Sinkhorn epilogue exposes w_next / weight(); the plain gathers do not spread.
struct EpiNone {
    double* w_next = nullptr;
    __device__ double operator()(int64_t, double) const { return 0.0; }
    __device__ double weight(int64_t, double) const { return 0.0; }
    __device__ void prefetch(int64_t) const {}
};
template <class Epi>
struct EpiGatherOnly : Epi {
    double* w_next = nullptr;
    __device__ double weight(int64_t, double) const { return 0.0; }
};

template <int MODE, class Epi>
void launch(const PointSet& ps, const double* gin, double* gout, const double* w, const FastParams& fp,
            const Epi& epi, unsigned long long* dmax, cudaStream_t s, int tag) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    ProfScope prof(tag, s);
    chunked3d_k<MODE, Epi><<<ps.chunk_blocks, kThreads, 0, s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                ps.chunk_bounds.p, ps.nchunks, fp.ng, gin, gout,
                                                                w, epi, dmax);
    UOTK_LAUNCHED();
}

}  // namespace

bool fused3d_available(const FastParams& fp) { return fp.d == 3 && fp.m == kM; }

// Build the chunk list and the per-chunk window blocks (once per point set).  Chunks
// pad runs to multiples of 32 slots; when the padding would waste more than 3/4 of the
// work (sparse clouds) the point set stays on the generic kernels (ps.chunked = false).
void fused3d_prepare(PointSet& ps, const FastParams& fp, cudaStream_t s) {
    ps.chunked = false;
    ps.nchunks = 0;
    if (!fused3d_available(fp) || ps.n == 0) return;
    const int n = (int)ps.n;
    DevBuf<int32_t> run_key(n, s), run_len(n, s), run_start(n, s), nchunk(n, s), chunk_off(n, s), cnt(2, s);
    size_t tmp_bytes = 0, t2 = 0, t3 = 0;
    UOTK_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp_bytes, ps.key.p, run_key.p, run_len.p, cnt.p, n, s));
    UOTK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, run_len.p, run_start.p, n, s));
    tmp_bytes = std::max(tmp_bytes, t2);
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    UOTK_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, tmp_bytes, ps.key.p, run_key.p, run_len.p, cnt.p, n, s));
    add_launches(2);
    int32_t nruns = 0;
    UOTK_CUDA(cudaMemcpyAsync(&nruns, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaStreamSynchronize(s));
    t3 = tmp_bytes;
    UOTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t3, run_len.p, run_start.p, nruns, s));
    chunk_count_k<<<blocks_for(nruns, 256), 256, 0, s>>>(run_len.p, cnt.p, nchunk.p);
    UOTK_LAUNCHED();
    UOTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t3, nchunk.p, chunk_off.p, nruns, s));
    add_launches(2);
    int32_t last[2];
    UOTK_CUDA(cudaMemcpyAsync(&last[0], chunk_off.p + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaMemcpyAsync(&last[1], nchunk.p + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaStreamSynchronize(s));
    const int64_t nchunks = (int64_t)last[0] + last[1];
    if ((double)n < 0.25 * kChunk * (double)nchunks) return;  // too sparse for the chunked kernel
    ps.chunk_desc.alloc(nchunks, s);
    ps.chunk_win.alloc((size_t)nchunks * kWinDoubles, s);
    chunk_desc_k<<<blocks_for(nruns, 256), 256, 0, s>>>(run_key.p, run_len.p, run_start.p, chunk_off.p, cnt.p,
                                                        ps.chunk_desc.p);
    UOTK_LAUNCHED();
    const KBWindow win = make_window(fp.b, kM);
    {
        ProfScope prof(kProfSetup, s);
        chunk_window_k<<<(unsigned)nchunks, kThreads, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.n, win, ps.chunk_win.p);
        UOTK_LAUNCHED();
    }
    // cost-balanced static partition of the chunks over the CTAs
    int sms = 148;
    {
        int dev = 0;
        UOTK_CUDA(cudaGetDevice(&dev));
        UOTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int nb = (int)std::min<int64_t>((int64_t)sms * kBlocksPerSM, nchunks);
    DevBuf<int32_t> cost(nchunks, s), prefix(nchunks, s);
    chunk_cost_k<<<blocks_for(nchunks, 256), 256, 0, s>>>(ps.chunk_desc.p, nchunks, cost.p);
    UOTK_LAUNCHED();
    size_t t4 = 0;
    UOTK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t4, cost.p, prefix.p, (int)nchunks, s));
    DevBuf<uint8_t> tmp2(t4, s);
    UOTK_CUDA(cub::DeviceScan::InclusiveSum(tmp2.p, t4, cost.p, prefix.p, (int)nchunks, s));
    add_launches(1);
    ps.chunk_bounds.alloc(nb + 1, s);
    chunk_bounds_k<<<blocks_for(nb + 1, 256), 256, 0, s>>>(prefix.p, nchunks, nb, ps.chunk_bounds.p);
    UOTK_LAUNCHED();
    ps.chunk_blocks = nb;
    ps.nchunks = nchunks;
    ps.chunked = true;
}

void fused3d_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s) {
    launch<0, EpiSinkhorn>(ps, grid_in, grid_out, nullptr, fp, epi, dmax, s, kProfFused);
}

void fused3d_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    launch<1, EpiNone>(ps, nullptr, grid, w, fp, EpiNone{}, nullptr, s, kProfSpread);
}

void fused3d_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s) {
    EpiGatherOnly<EpiStore> e;
    static_cast<EpiStore&>(e) = epi;
    launch<2, EpiGatherOnly<EpiStore>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

void fused3d_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s) {
    EpiGatherOnly<EpiDot> e;
    static_cast<EpiDot&>(e) = epi;
    launch<2, EpiGatherOnly<EpiDot>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

}  // namespace uotk
