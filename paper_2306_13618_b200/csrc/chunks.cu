// Chunk preparation for the tuned cell-group kernels (layout: chunks.cuh): run-length
// encoding of the sorted cell keys, chunk descriptors, the precomputed window blocks
// (Kaiser-Bessel values of (4.6)'s phi at every tap), and a cost-balanced static
// partition of the chunks over the kernels' work units (CTAs for d = 3, warps for d <= 2).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "chunks.cuh"
#include "common.cuh"
#include "profile.cuh"
#include "window.cuh"
#include "window_fit.h"

namespace uotk {

namespace {

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

// over all n run slots: chunks per run, zero (run length and chunks) past the last run, so
// the scans can run over n items without the host knowing the run count
__global__ void chunk_count_k(int32_t* __restrict__ run_len, const int32_t* __restrict__ nruns,
                              int32_t* __restrict__ nchunk, int n) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (r < *nruns) {
        nchunk[r] = (run_len[r] + kChunk - 1) / kChunk;
    } else {
        run_len[r] = 0;
        nchunk[r] = 0;
    }
}

// cnt[1] = total number of chunks (chunk_off is the exclusive sum of nchunk over n slots)
__global__ void chunk_total_k(const int32_t* __restrict__ chunk_off, const int32_t* __restrict__ nchunk, int n,
                              int32_t* __restrict__ cnt) {
    cnt[1] = chunk_off[n - 1] + nchunk[n - 1];
}

__global__ void chunk_desc_k(const int32_t* __restrict__ run_key, const int32_t* __restrict__ run_len,
                             const int32_t* __restrict__ run_start, const int32_t* __restrict__ chunk_off,
                             const int32_t* __restrict__ nruns, int4* __restrict__ desc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *nruns) return;
    const int len = run_len[r];
    const int nc = (len + kChunk - 1) / kChunk;
    for (int k = 0; k < nc; ++k)
        desc[chunk_off[r] + k] = make_int4(run_start[r] + k * kChunk, min(kChunk, len - k * kChunk), run_key[r],
                                           r + 1 < *nruns ? run_key[r + 1] : -1);  // .w: the next group's key
}

// Window blocks (layout per d: chunks.cuh).  One warp per (chunk, axis): lane p loads
// its point's coordinate once and evaluates its row of taps phi(f + m - 1 - a); the rows
// are staged in shared memory and written out coalesced.  KZ (d = 3 only): width of the
// z rows (16, or 24 for z-segment groups: the 16 taps sit at the cell's offset; 12 for
// m = 6, whose 12 taps fill the whole row).
constexpr int kWinWarps = 4;
constexpr int kMaxRow = 44;  // widest row stride (d = 3, KZ = 40)

// widest row of a (D, KZ) block: the staging buffer is sized by it (not by kMaxRow), so
// the common blocks leave room for more resident warps
__host__ __device__ constexpr int win_row_max(int d, int kz) {
    return d == 3 ? (chunk_zstride3(kz) > chunk_xstride3(kz) ? chunk_zstride3(kz) : chunk_xstride3(kz))
                  : (d == 2 ? (chunk_ystride2(kz) > kChunkT ? chunk_ystride2(kz) : kChunkT) : kChunkT);
}
template <int D, int KZ>
__global__ void __launch_bounds__(kWinWarps * 32)
chunk_window_rows_k(const int4* __restrict__ desc, const double* __restrict__ u, const int32_t* __restrict__ key,
                    int64_t n, int64_t nchunks, KBHorner hc, double* __restrict__ out) {
    static_assert(win_row_max(D, KZ) <= kMaxRow, "window row wider than the staging bound");
    __shared__ double stage[kWinWarps][kChunk * win_row_max(D, KZ)];
    constexpr int kW = D == 3 ? chunk_win3_doubles(KZ) : (D == 2 ? chunk_win2_doubles(KZ) : chunk_win_doubles(D));
    constexpr bool YSEG = D == 2 && KZ == 24;  // d = 2 y-segment rows (chunks.cuh)
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t job = blockIdx.x * (int64_t)kWinWarps + warp;  // (chunk, axis)
    if (job >= nchunks * D) return;
    const int64_t c = job / D;
    const int ax = (int)(job - c * D);
    const int4 dsc = desc[c];
    // row stride and offset of this axis' matrix inside the chunk block
    const int stride = D == 3 ? (ax == 2 ? chunk_zstride3(KZ) : chunk_xstride3(KZ))
                              : (D == 2 && ax == 1 ? chunk_ystride2(KZ) : kChunkT);
    const int64_t base = c * kW + (int64_t)ax * kChunk * (D == 3 ? chunk_xstride3(KZ) : kChunkT);
    double* st = stage[warp];
    const int p = lane;
    double f = 0.0;
    int off = 0;  // first column of the taps in this row
    const bool live = p < dsc.y;
    if (live) {
        const double ut = u[ax * n + dsc.x + p];
        f = ut - floor(ut);
        if (D == 3 && ax == 2 && (KZ == 24 || KZ == 40)) off = key[dsc.x + p] - dsc.z;
        if (YSEG && ax == 1) off = key[dsc.x + p] - dsc.z;
    }
    // the row: zeros (empty slots, padding columns), then the 2m taps of a live point,
    // each a degree-14 polynomial in f - 1/2 (window_fit.h)
    for (int col = 0; col < stride; ++col) st[p * stride + col] = 0.0;
    if (live) {
        // mirror pairs a, TAPS - 1 - a: phi is even, so the mirror tap is tap a's polynomial
        // at -t — the even and odd halves in t^2 give both (15 FMA per pair instead of 28)
        constexpr int TAPS = (D == 3 && KZ == 12) ? 12 : kChunkT;
        const double t = f - 0.5, t2 = t * t;
        auto col = [&](int a) { return (D == 2 && !(YSEG && ax == 1)) ? swz2(p, a) : a + off; };
#pragma unroll
        for (int a = 0; a < TAPS / 2; ++a) {
            double e = hc.c[a][kHornerDeg], o = hc.c[a][kHornerDeg - 1];
#pragma unroll
            for (int j = kHornerDeg - 2; j >= 0; j -= 2) e = fma(e, t2, hc.c[a][j]);
#pragma unroll
            for (int j = kHornerDeg - 3; j >= 1; j -= 2) o = fma(o, t2, hc.c[a][j]);
            st[p * stride + col(a)] = fma(t, o, e);
            st[p * stride + col(TAPS - 1 - a)] = fma(-t, o, e);
        }
    }
    __syncwarp();
    double* o = out + base;
    for (int e = lane; e < kChunk * stride; e += 32) o[e] = st[e];
}

// group key of a z-segment: the cell key with its z index rounded down to a multiple of kSegZ
__global__ void segment_key_k(const int32_t* __restrict__ key, int64_t n, int ng, int segz,
                              int32_t* __restrict__ gk) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const int32_t k = key[i];
        gk[i] = k - (k % ng) % segz;
    }
}

// hybrid group keys (chunks.cuh) straight from the sorted cell keys.  A point's cell is
// dense (>= minpts points) iff the run holds the minpts-window [f, f + minpts) around its
// start f: if key[i - minpts + 1] == key[i] the run already spans minpts points up to i,
// else f lies in the last minpts slots (binary search) and key[f + minpts - 1] decides.
// Dense cells keep their key, the others take their z-segment's key with kSegFlag.  Each
// run's first point also adds the run's one-cell chunk count (galloping to the run's end)
// to *onecell (the layout the hybrid one replaces).
__global__ void hybrid_key_k(const int32_t* __restrict__ key, int n, int ng, int segz, int minpts,
                             int32_t* __restrict__ gk, int32_t* __restrict__ onecell) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int add = 0;
    if (i < n) {
        const int32_t k = key[i];
        bool dense;
        int first;
        if (i - minpts + 1 >= 0 && key[i - minpts + 1] == k) {
            dense = true;
            first = -1;  // not the run's first point
        } else {
            int lo = i - minpts + 1 < 0 ? 0 : i - minpts + 1, hi = i;  // first index with key == k
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (key[mid] < k) lo = mid + 1;
                else hi = mid;
            }
            first = lo;
            dense = first + minpts - 1 < n && key[first + minpts - 1] == k;
        }
        gk[i] = dense ? k : ((k - (k % ng) % segz) | kSegFlag);
        if (first == i) {  // the run's end by galloping, then a binary search in the last step
            int step = 1, lo = i;  // key[lo] == k
            while (lo + step < n && key[lo + step] == k) {
                lo += step;
                step <<= 1;
            }
            int hi = lo + step > n ? n : lo + step;
            while (lo < hi) {  // first index with key > k
                const int mid = (lo + hi) >> 1;
                if (key[mid] <= k) lo = mid + 1;
                else hi = mid;
            }
            add = (lo - i + kChunk - 1) / kChunk;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) add += __shfl_xor_sync(0xffffffffu, add, off);
    if ((threadIdx.x & 31) == 0 && add) atomicAdd(onecell, add);
}

// cost of a chunk for the static partition: fix per chunk + step per 4-point k-step of its
// points (the kernels skip the steps past a chunk's count) + group when it opens a cell
// group (footprint load and flush)
__global__ void chunk_cost_k(const int4* __restrict__ desc, int64_t nchunks, int fix, int step, int group,
                             int32_t* __restrict__ cost) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < nchunks)
        cost[c] = fix + step * ((desc[c].y + 3) >> 2) + ((c == 0 || desc[c].z != desc[c - 1].z) ? group : 0);
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

}  // namespace

bool chunked_available(const FastParams& fp) {
    return (fp.m == kChunkM && fp.d >= 1 && fp.d <= 3) || (fp.m == 6 && fp.d == 3);
}

// Build the chunk list and the per-chunk window blocks (once per point set).  Chunks pad
// runs to multiples of 32 slots; when the padding would waste too much work (sparse
// clouds: d = 3 below ~3 points per chunk, d = 2 below 2) or the window blocks would not fit
// comfortably in free device memory, the point set stays on the generic kernels
// (ps.chunked = false).
void chunked_prepare(PointSet& ps, const FastParams& fp, cudaStream_t s, PointUse use) {
    ps.chunked = false;
    ps.nchunks = 0;
    if (!chunked_available(fp) || ps.n == 0 || (fp.flags & UOTK_FLAG_GENERIC)) return;
    const int d = fp.d;
    const int n = (int)ps.n;
    trace_mark("chunks: start");
    DevBuf<int32_t> run_key(n, s), run_len(n, s), run_start(n, s), nchunk(n, s), chunk_off(n, s), cnt(3, s);
    cnt.zero();  // cnt[2] (the hybrid pass's one-cell count) is read back by every encode
    trace_mark("chunks: 6 scratch allocations");
    size_t tmp_bytes = 0, t2 = 0;
    UOTK_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp_bytes, ps.key.p, run_key.p, run_len.p, cnt.p, n, s));
    UOTK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, run_len.p, run_start.p, n, s));
    trace_mark("chunks: cub size queries");
    tmp_bytes = std::max(tmp_bytes, t2);
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    trace_mark("chunks: temp allocation");
    int32_t nruns = 0;
    int32_t onecell_chunks = 0;  // cnt[2]: written by hybrid_key_k only
    // runs of equal group keys -> chunks of <= 32 points; returns the number of chunks.
    // One host synchronisation per encode: the scans run over all n run slots (the slots
    // past the last run zeroed on the device), and the run and chunk counts come back
    // together.
    auto encode = [&](const int32_t* keys) -> int64_t {
        size_t t = tmp_bytes;
        UOTK_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, t, keys, run_key.p, run_len.p, cnt.p, n, s));
        add_launches(2);
        chunk_count_k<<<blocks_for(n, 256), 256, 0, s>>>(run_len.p, cnt.p, nchunk.p, n);
        UOTK_LAUNCHED();
        t = tmp_bytes;
        UOTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, run_len.p, run_start.p, n, s));
        t = tmp_bytes;
        UOTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, nchunk.p, chunk_off.p, n, s));
        add_launches(4);
        chunk_total_k<<<1, 1, 0, s>>>(chunk_off.p, nchunk.p, n, cnt.p);
        UOTK_LAUNCHED();
        int32_t h[3];
        UOTK_CUDA(cudaMemcpyAsync(h, cnt.p, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        UOTK_CUDA(cudaStreamSynchronize(s));
        trace_mark("chunks: run-length encode + scans");
        nruns = h[0];
        onecell_chunks = h[2];
        return (int64_t)h[1];
    };
    const bool forced = fp.flags & UOTK_FLAG_CHUNKED;
    // spread-only d = 3 sets whose windows the spread evaluates (spread3d_fly_k): when the
    // one-cell chunks are only partly filled (but not sparse enough for the all-segment
    // layouts below), hybrid groups — dense cells alone, sparse cells in z-segments — cut
    // the chunk count (MMD^2 at 1M: 89k -> 73k chunks, 39k -> 20k footprint flushes).  The
    // hybrid keys and the one-cell chunk count come from one pass over the sorted keys, so
    // a set that takes the hybrid layout needs one run-length encode, not two.
    static const bool fly_env = [] {
        const char* e = getenv("UOTK_SPREAD_FLY");
        return !(e && e[0] == '0');
    }();
    static const bool hybrid_env = [] {
        const char* e = getenv("UOTK_HYBRID");
        return !(e && e[0] == '0');
    }();
    bool hybrid = false;
    DevBuf<int32_t> gk;
    int64_t nchunks = 0;
    if (fly_env && hybrid_env && d == 3 && fp.m == kChunkM && use == kUseSpreadOnly &&
        std::pow((double)fp.ng, 3) < (double)kSegFlag) {
        gk.alloc(n, s);
        UOTK_CUDA(cudaMemsetAsync(cnt.p + 2, 0, sizeof(int32_t), s));
        hybrid_key_k<<<blocks_for(n, 256), 256, 0, s>>>(ps.key.p, n, fp.ng, kSegZ, kHybridMin, gk.p, cnt.p + 2);
        UOTK_LAUNCHED();
        // the one-cell chunk count decides which layouts to encode: partly filled sets try the
        // hybrid one; sparser ones go straight to the z-segment layouts below (their choice
        // needs only this count), dense ones to the one-cell layout
        int32_t n1h = 0;
        UOTK_CUDA(cudaMemcpyAsync(&n1h, cnt.p + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        UOTK_CUDA(cudaStreamSynchronize(s));
        const double n1 = (double)n1h;
        if ((double)n >= 0.5 * kChunk * n1 && (double)n < 0.95 * kChunk * n1) {
            const int64_t nh = encode(gk.p);
            if ((double)nh < 0.95 * n1) {
                hybrid = true;
                nchunks = nh;
            }
        }
        if (!hybrid && (double)n < 0.5 * kChunk * n1) nchunks = n1h;  // the z-segment branch encodes
        trace_mark("chunks: hybrid groups");
    }
    if (!hybrid && nchunks == 0) nchunks = encode(ps.key.p);
    trace_mark("chunks: encode");
    // d = 3 sparse clouds: group z-segments of kSegZ cells when that needs sufficiently
    // fewer chunks (each costs 1.5x a one-cell chunk: 24 instead of 16 z-columns)
    int kz = fp.m == 6 ? 12 : 16;
    double chunk_cost = 1.0;
    if (!hybrid && d == 3 && fp.m == kChunkM && (double)n < 0.5 * kChunk * (double)nchunks) {
        gk.alloc(n, s);
        segment_key_k<<<blocks_for(n, 256), 256, 0, s>>>(ps.key.p, ps.n, fp.ng, kSegZ, gk.p);
        UOTK_LAUNCHED();
        const int64_t nseg = encode(gk.p);
        if (1.5 * (double)nseg < (double)nchunks) {
            kz = 24;
            chunk_cost = 1.5;
            nchunks = nseg;
        } else {
            nchunks = encode(ps.key.p);  // back to one-cell groups
        }
        static const bool seg40_env = [] {
            const char* e = getenv("UOTK_SEG40");
            return !(e && e[0] == '0');
        }();
        // a spread-only set still below 1/4 fill: 25-cell segments if they merge groups
        if (kz == 24 && use == kUseSpreadOnly && seg40_env && (double)n < 0.25 * kChunk * (double)nchunks) {
            segment_key_k<<<blocks_for(n, 256), 256, 0, s>>>(ps.key.p, ps.n, fp.ng, kSegZ40, gk.p);
            UOTK_LAUNCHED();
            const int64_t nseg40 = encode(gk.p);
            if ((double)nseg40 < 0.7 * (double)nchunks) {
                kz = 40;
                chunk_cost = 2.5;
                nchunks = nseg40;
            } else {  // back to the 9-cell segments
                segment_key_k<<<blocks_for(n, 256), 256, 0, s>>>(ps.key.p, ps.n, fp.ng, kSegZ, gk.p);
                UOTK_LAUNCHED();
                nchunks = encode(gk.p);
            }
        }
        trace_mark("chunks: z-segments");
    }
    // d = 2 sparse clouds: y-segments of kSegY cells (one 16 x 24 footprint) when that needs
    // sufficiently fewer chunks; the footprint flushes (fp64 RED) bind those sets
    static const bool yseg_env = [] {
        const char* e = getenv("UOTK_YSEG");
        return !(e && e[0] == '0');
    }();
    if (d == 2 && fp.m == kChunkM && yseg_env && (double)n < 0.5 * kChunk * (double)nchunks) {
        gk.alloc(n, s);
        segment_key_k<<<blocks_for(n, 256), 256, 0, s>>>(ps.key.p, ps.n, fp.ng, kSegY, gk.p);
        UOTK_LAUNCHED();
        const int64_t nseg = encode(gk.p);
        if (1.5 * (double)nseg < (double)nchunks) {
            kz = 24;
            chunk_cost = 1.5;
            nchunks = nseg;
        } else {
            nchunks = encode(ps.key.p);  // back to one-cell groups
        }
        trace_mark("chunks: y-segments");
    }
    // minimum mean fill of the 32-slot chunks (per unit of chunk cost): below it the padded
    // GEMM work and the per-group footprint flush cost more than the generic kernels'
    // per-tap atomics (d = 3: ~3 points per chunk, measured on C5/C2 clouds; d = 2: ~2;
    // d = 1: any)
    const double min_fill = d == 3 ? 0.09 : (d == 2 ? 1.0 / 16 : 0.0);
    if (!forced && (double)n < min_fill * chunk_cost * kChunk * (double)nchunks) return;
    // a gather-only set this sparse is gathered by the generic kernel anyway (nfft.cu)
    if (!forced && use == kUseGatherOnly && d == 3 && (double)n < kGatherMinFill3 * kChunk * (double)nchunks) return;
    const int wd = d == 3 ? chunk_win3_doubles(kz) : (d == 2 ? chunk_win2_doubles(kz) : chunk_win_doubles(d));
    // spread-only d = 3 one-cell (or hybrid) sets: the spread evaluates the windows itself
    const bool fly = fly_env && d == 3 && kz == 16 && fp.m == kChunkM && use == kUseSpreadOnly;
    const size_t win_bytes = fly ? 0 : (size_t)nchunks * wd * sizeof(double);
    // cudaMemGetInfo can stall the host (milliseconds, and seconds when the stream-ordered
    // pool caches tens of GB): ask it only for blocks that are a noticeable fraction of the
    // device and that the pool's cached (reserved but unused) memory cannot hold already
    static size_t total_b = 0;
    if (total_b == 0) {
        size_t f0 = 0;
        UOTK_CUDA(cudaMemGetInfo(&f0, &total_b));
    }
    size_t free_b = total_b;
    if (win_bytes > total_b / 16) {
        int dev = 0;
        cudaMemPool_t pool = nullptr;
        UOTK_CUDA(cudaGetDevice(&dev));
        if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) pool = nullptr;
        cudaGetLastError();
        // memory the pool keeps reserved but unused is reusable
        auto pool_cached = [&]() -> size_t {
            unsigned long long reserved = 0, used = 0;
            if (pool && cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
                cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
                return (size_t)(reserved - used);
            cudaGetLastError();
            return 0;
        };
        size_t cached = pool_cached();
        // the library's block cache holds freed blocks as "used": give them back first
        if (cached < win_bytes && block_cache_bytes() > 0) {
            block_cache_release();
            cached = pool_cached();
        }
        if (cached < win_bytes) {
            size_t t0 = 0;
            UOTK_CUDA(cudaMemGetInfo(&free_b, &t0));
            free_b += cached;
        }
        trace_mark("chunks: memory check");
    }
    if (win_bytes > free_b / 2) {  // keep the generic path rather than exhaust HBM
        if (forced) fail(UOTK_ENOMEM, "UOTK_FLAG_CHUNKED: window blocks do not fit in device memory");
        return;
    }
    ps.chunk_desc.alloc(nchunks, s);
    if (!fly) ps.chunk_win.alloc((size_t)nchunks * wd, s);
    chunk_desc_k<<<blocks_for(nruns, 256), 256, 0, s>>>(run_key.p, run_len.p, run_start.p, chunk_off.p, cnt.p,
                                                        ps.chunk_desc.p);
    UOTK_LAUNCHED();
    // the polynomial fit costs ~0.1 ms of host time: keep the last few (b, m) fits
    static std::mutex fit_mu;
    static std::vector<std::pair<std::pair<double, int>, KBHorner>> fits;
    KBHorner win;
    {
        std::lock_guard<std::mutex> lk(fit_mu);
        auto it = std::find_if(fits.begin(), fits.end(), [&](const auto& e) {
            return e.first.first == fp.b && e.first.second == fp.m;
        });
        if (it != fits.end()) {
            win = it->second;
        } else {
            win = kb_horner_fit(fp.b, fp.m);
            if (fits.size() >= 8) fits.erase(fits.begin());
            fits.push_back({{fp.b, fp.m}, win});
        }
    }
    ps.win_fly = fly;
    if (fly) ps.win_coef = win;
    if (!fly) {
        ProfScope prof(kProfSetup, s);
        const unsigned wb = (unsigned)((nchunks * d + kWinWarps - 1) / kWinWarps);
        if (d == 3 && kz == 12)
            chunk_window_rows_k<3, 12><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else if (d == 3 && kz == 40)
            chunk_window_rows_k<3, 40><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else if (d == 3 && kz == 24)
            chunk_window_rows_k<3, 24><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else if (d == 3)
            chunk_window_rows_k<3, 16><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else if (d == 2 && kz == 24)
            chunk_window_rows_k<2, 24><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else if (d == 2)
            chunk_window_rows_k<2, 16><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        else
            chunk_window_rows_k<1, 16><<<wb, kWinWarps * 32, 0, s>>>(ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, nchunks,
                                                                      win, ps.chunk_win.p);
        UOTK_LAUNCHED();
    }
    // cost-balanced static partition of the chunks over the work units
    int sms = 148;
    {
        int dev = 0;
        UOTK_CUDA(cudaGetDevice(&dev));
        UOTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const bool m6 = d == 3 && fp.m == 6;
    const int nb = (int)std::min<int64_t>(
        (int64_t)sms * (m6 ? kCtas3M6 : (fly ? kCtasFly3 : chunk_units_per_sm(d))), nchunks);
    DevBuf<int32_t> cost(nchunks, s), prefix(nchunks, s);
    int cfix = 8, cstep = 0, cgroup = d == 3 ? 2 : 1;
    if (const char* e = getenv("UOTK_COST")) sscanf(e, "%d,%d,%d", &cfix, &cstep, &cgroup);  // A/B only
    chunk_cost_k<<<blocks_for(nchunks, 256), 256, 0, s>>>(ps.chunk_desc.p, nchunks, cfix, cstep, cgroup, cost.p);
    UOTK_LAUNCHED();
    size_t t4 = 0;
    UOTK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t4, cost.p, prefix.p, (int)nchunks, s));
    DevBuf<uint8_t> tmp2(t4, s);
    UOTK_CUDA(cub::DeviceScan::InclusiveSum(tmp2.p, t4, cost.p, prefix.p, (int)nchunks, s));
    add_launches(1);
    ps.chunk_bounds.alloc(nb + 1, s);
    chunk_bounds_k<<<blocks_for(nb + 1, 256), 256, 0, s>>>(prefix.p, nchunks, nb, ps.chunk_bounds.p);
    if (d == 2 || m6) {
        const int nw = (int)std::min<int64_t>((int64_t)sms * (m6 ? kCtasWS3M6 : kUnitsWS2 * kCtasWS2), nchunks);
        ps.chunk_bounds_ws.alloc(nw + 1, s);
        chunk_bounds_k<<<blocks_for(nw + 1, 256), 256, 0, s>>>(prefix.p, nchunks, nw, ps.chunk_bounds_ws.p);
        UOTK_LAUNCHED();
        ps.chunk_units_ws = nw;
    }
    UOTK_LAUNCHED();
    trace_mark("chunks: windows + bounds");
    ps.chunk_blocks = nb;
    ps.chunk_kz = hybrid ? kGroupsHybrid : kz;
    ps.chunk_fill = (double)n / ((double)kChunk * (double)nchunks);
    ps.nchunks = nchunks;
    ps.chunked = true;
}

}  // namespace uotk
