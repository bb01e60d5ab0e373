// Tuned d = 2 and d = 1 NFFT passes: cell-group kernels with one warp per work unit
// (DESIGN.md §7).  Same chunked layout as the d = 3 kernels (chunks.cuh): points sorted by
// cell, runs of equal keys cut into chunks of <= 32 points, window values precomputed per
// chunk.  A warp walks a contiguous, cost-balanced range of chunks; the footprint of the
// current cell group — (2m)^d grid values, 16 x 16 in d = 2 — lives in the warp's
// registers: the gather operand F is loaded once per group and the spread accumulators S
// are flushed once per group (fp64 RED), so the grid sees one read and one atomic flush
// per group instead of (2m)^d atomics per point.
//
// d = 2, with X_p, Y_p the windows of point p along the two axes (outer / inner sums of
// (4.6)):
//   gather  G[p, b] = sum_a X_p[a] F[a, b]         (32x16x16 GEMM on DMMA, mma.sync f64)
//           t_p     = sum_b G[p, b] Y_p[b]          (per point, quad shuffle reduction)
//   spread  S[a, b] += sum_p (w_p X_p[a]) Y_p[b]   (16x16x32 GEMM on DMMA)
// The window block of a chunk (8 KB) is streamed into the warp's shared-memory ring by a
// TMA bulk copy; its swizzle (tap a of slot p at column (a + 4p) & 15) makes every
// fragment load hit the minimum number of shared-memory wavefronts.
//
// d = 1: lane p holds the 16 window values of point p in registers (loaded straight from
// the chunk's block); t_p = sum_a X_p[a] F[a] in-lane, and the spread accumulates
// w_p X_p[a] per lane, reduced across the warp by a transpose-reduction only when the
// group is flushed.
#include <cstdlib>

#include "chunks.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "ptx.cuh"

namespace uotk {

bool chunked_available(const FastParams& fp);  // chunks.cu
// d = 3 kernels (fused3d.cu)
void fused3d_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s);
void fused3d_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s);
void fused3d_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s);
void fused3d_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s);

namespace {

constexpr int kM = kChunkM;
// d = 2 window blocks: X [slot 32][16 taps, swizzled], then Y: one-cell groups (KY = 16)
// [slot 32][16 taps, swizzled]; y-segment groups of sparse clouds (KY = 24: kSegY cells
// along y share one 16 x 24 footprint) [slot 32][24 columns, stride 28], the 16 taps at
// the point's cell offset in the segment (chunks.cuh)
template <int KY>
struct Lay2 {
    static constexpr int NT = KY / 8;                           // 8-wide column tiles along y
    static constexpr int YS = KY == 16 ? kChunkT : chunk_ystride2(KY);
    static constexpr int W = chunk_win2_doubles(KY);            // doubles per chunk block
    static constexpr uint32_t Bytes = W * sizeof(double);
    // column c of slot p's Y row
    __device__ static __forceinline__ int y(int p, int c) { return KY == 16 ? p * kChunkT + swz2(p, c) : p * YS + c; }
};
constexpr int kW1 = chunk_win_doubles(1);  // 512 doubles per chunk
template <int KY>
struct Ring2 {
    static constexpr int N = KY == 16 ? 3 : 2;  // window blocks in flight per warp (3 CTAs per SM)
};

template <int KY>
struct __align__(128) Smem2 {
    double win[kWarps2][Ring2<KY>::N][Lay2<KY>::W];  // per-warp TMA ring of window blocks
    double red[kWarps2][kChunk];                       // per-warp gathered t of the current chunk
    unsigned long long bar[kWarps2][Ring2<KY>::N];
};

// chunk descriptors of a warp's range, batched: lane L holds the descriptor of chunk
// base + L of the current batch (cur) and of the next batch (nxt, in flight)
struct DescBatch {
    int4 cur, nxt;
    const int4* desc;
    int64_t cbeg, cend;
    __device__ __forceinline__ int4 fetch(int64_t c) const {
        return c < cend ? desc[c] : make_int4(0, 0, -1, 0);
    }
    __device__ __forceinline__ void init(const int4* d, int64_t b, int64_t e, int lane) {
        desc = d;
        cbeg = b;
        cend = e;
        cur = fetch(b + lane);
        nxt = fetch(b + 32 + lane);
    }
    // descriptor of chunk cbeg + k (warp-uniform k); advances the batches at k % 32 == 0
    __device__ __forceinline__ int4 get(int64_t k, int lane) {
        if (k > 0 && (k & 31) == 0) {
            cur = nxt;
            nxt = fetch(cbeg + k + 32 + lane);
        }
        const int src = (int)(k & 31);
        return make_int4(__shfl_sync(0xffffffffu, cur.x, src), __shfl_sync(0xffffffffu, cur.y, src),
                         __shfl_sync(0xffffffffu, cur.z, src), 0);
    }
    // descriptor of chunk cbeg + k + 1 without advancing
    __device__ __forceinline__ int4 peek_next(int64_t k) const {
        const int src = (int)((k + 1) & 31);
        const bool in_nxt = ((k + 1) & 31) == 0;
        const int4 v = in_nxt ? nxt : cur;
        return make_int4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                         __shfl_sync(0xffffffffu, v.z, src), 0);
    }
};

// MODE: 0 = gather -> epilogue -> spread (Sinkhorn half-step), 1 = spread only, 2 = gather only
template <int MODE, class Epi, int KY>
__global__ void __launch_bounds__(kWarps2 * 32, kCtas2)
chunked2d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
            int nunits, int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out,
            const double* __restrict__ w_in, Epi epi, unsigned long long* dmax) {
    constexpr bool GATHER = MODE != 1;
    constexpr bool SPREAD = MODE != 2;
    using In = typename Epi::In;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using L = Lay2<KY>;
    constexpr int NT = L::NT;
    constexpr int R = Ring2<KY>::N;
    Smem2<KY>& sm = *reinterpret_cast<Smem2<KY>*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gq = lane >> 2;  // fragment group: row of A / D, column of B
    const int tq = lane & 3;   // thread in group
    const int unit = blockIdx.x * kWarps2 + warp;
    if (unit >= nunits) return;  // warps are independent: no CTA-wide barrier below
    const int64_t cbeg = bounds[unit];
    const int64_t nck = bounds[unit + 1] - cbeg;
    if (nck <= 0) return;
    double* swin = &sm.win[warp][0][0];
    unsigned long long* bar = sm.bar[warp];
    if (lane == 0) {
        for (int r = 0; r < R; ++r) mbar_init(&bar[r], 1);
        mbar_init_fence();
    }
    __syncwarp();
    if (lane == 0) {
        for (int k = 0; k < R && k < nck; ++k) {
            mbar_expect_tx(&bar[k], L::Bytes);
            bulk_g2s(swin + k * L::W, win + (cbeg + k) * L::W, L::Bytes, &bar[k]);
        }
    }
    DescBatch db;
    db.init(desc, cbeg, cbeg + nck, lane);

    double Fb[NT][4];     // Fb[nt][ks] = F[4ks + tq][8nt + gq]          (gather B operand)
    double S[2][NT][2];   // S[mt][nt][i] = S[8mt + gq][8nt + 2tq + i]  (spread accumulators)
    int32_t cur_key = -1;
    int64_t org = 0;  // grid index of footprint (0, 0) of the current group
    double ddmax = 0.0;
    auto origin = [&](int32_t kk) -> int64_t { return (int64_t)(kk / ng - kM + 1) * ng + (kk % ng - kM + 1); };
    auto flush = [&]() {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            double* row = grid_out + org + (int64_t)(8 * mt + gq) * ng + 2 * tq;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (S[mt][nt][i] != 0.0) atomicAdd(row + 8 * nt + i, S[mt][nt][i]);
        }
    };

    int4 dsc = db.get(0, lane);
    In in_cur{};
    double w_cur = 0.0;  // spread-only: source weight of slot `lane`
    if (GATHER && lane < dsc.y) in_cur = epi.load(dsc.x + lane);
    if (!GATHER && lane < dsc.y) w_cur = w_in[dsc.x + lane];
    for (int64_t k = 0; k < nck; ++k) {
        const int64_t c = cbeg + k;
        const int slot = (int)(k % R);
        const int64_t p0 = dsc.x;
        const int cnt = dsc.y;
        // next chunk's descriptor and per-point inputs, in flight during this chunk
        const int4 dnext = db.peek_next(k);
        In in_next{};
        double w_nxt = 0.0;
        if (k + 1 < nck && lane < dnext.y) {
            if (GATHER) in_next = epi.load(dnext.x + lane);
            else w_nxt = w_in[dnext.x + lane];
        }
        if (dsc.z != cur_key) {
            if (SPREAD && cur_key >= 0) flush();
            cur_key = dsc.z;
            org = origin(cur_key);
            if (GATHER) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double* row = grid_in + org + (int64_t)(4 * ks + tq) * ng + gq;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) Fb[nt][ks] = __ldg(row + 8 * nt);
                }
            }
            if (SPREAD) {
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) S[mt][nt][0] = S[mt][nt][1] = 0.0;
            }
        }
        if (GATHER && k + 1 < nck && dnext.z != cur_key && lane < 16) {
            // warm L1 with the next group's footprint rows
            asm volatile("prefetch.global.L1 [%0];" ::"l"(grid_in + origin(dnext.z) + (int64_t)lane * ng));
        }
        mbar_wait(&bar[slot], (uint32_t)((k / R) & 1));
        const double* X = swin + slot * L::W;
        const double* Y = X + kChunk * kChunkT;

        double wn = 0.0;  // spread weight of slot `lane`
        if (GATHER) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
                const double* xr = X + p * kChunkT;
                double acc[NT][2];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double a = xr[swz2(p, 4 * ks + tq)];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a, Fb[nt][ks]);
                }
                // acc[nt][i] = G[p][8nt + 2tq + i]
                double part = 0.0;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const double2 y = *reinterpret_cast<const double2*>(Y + L::y(p, 8 * nt + 2 * tq));
                    part = fma(acc[nt][0], y.x, part);
                    part = fma(acc[nt][1], y.y, part);
                }
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                if (tq == 0) sm.red[warp][p] = part;
            }
            __syncwarp();
            const double t = sm.red[warp][lane];
            if (lane < cnt) ddmax = fmax(ddmax, epi.apply(p0 + lane, t, in_cur, wn));
        } else {
            wn = w_cur;
        }

        if (SPREAD) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {  // 4 points per k-step
                const int p = 4 * ks + tq;
                const double wp = __shfl_sync(0xffffffffu, wn, p);
                const double* xr = X + p * kChunkT;
                const double xa0 = wp * xr[swz2(p, gq)];
                const double xa1 = wp * xr[swz2(p, 8 + gq)];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const double yb = Y[L::y(p, 8 * nt + gq)];
                    dmma(S[0][nt][0], S[0][nt][1], xa0, yb);
                    dmma(S[1][nt][0], S[1][nt][1], xa1, yb);
                }
            }
        }
        __syncwarp();  // the warp is done with window slot `slot` and red
        if (lane == 0 && k + R < nck) {
            fence_proxy_async();
            mbar_expect_tx(&bar[slot], L::Bytes);
            bulk_g2s(swin + slot * L::W, win + (c + R) * L::W, L::Bytes, &bar[slot]);
        }
        if (k + 1 < nck) dsc = db.get(k + 1, lane);
        in_cur = in_next;
        w_cur = w_nxt;
    }
    if (SPREAD && cur_key >= 0) flush();
    if (GATHER) warp_max_atomic(dmax, ddmax);
}

// ---------------------------------------------------------------- warp-specialised d = 2 half-step
// One work unit = three warps: gather/update warps G0 and G1 take the even and the odd
// chunks of the unit's range (gather = 32 DMMAs + the Sinkhorn update (3.3)/(3.4)), and
// publish the 32 new weights; the spread warp S spreads every chunk in order (32 DMMAs)
// from those weights.  The gather side carries about twice the instructions of the
// spread side (the update's log/exp), hence two G warps per S warp.  The window ring
// (TMA, refilled by S when it releases a slot) and the weight hand-offs are per-unit
// mbarriers: the units of a CTA never synchronise after the start.
template <int KY>
struct RingWS2 {
    static constexpr int N = KY == 16 ? 5 : 4;  // 2 CTAs per SM: 2 x 2 units x N x (8 | 11) KB
};
template <int KY>
struct __align__(128) Smem2WS {
    double win[kUnitsWS2][RingWS2<KY>::N][Lay2<KY>::W];
    double w[kUnitsWS2][2][kChunk];  // published weights of the even / odd chunk
    unsigned long long win_full[kUnitsWS2][RingWS2<KY>::N];
    unsigned long long w_full[kUnitsWS2][2];
    unsigned long long w_empty[kUnitsWS2][2];
};

template <int KY>
__global__ void __launch_bounds__(3 * kUnitsWS2 * 32, kCtasWS2)
sinkhorn2d_ws_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
                int nunits, int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out,
                EpiSinkhorn epi, unsigned long long* dmax) {
    using In = EpiSinkhorn::In;
    using L = Lay2<KY>;
    constexpr int NT = L::NT;
    constexpr int kRingWS2 = RingWS2<KY>::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem2WS<KY>& sm = *reinterpret_cast<Smem2WS<KY>*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int u = warp / 3;     // unit within the CTA
    const int role = warp % 3;  // 0, 1: gather warps (chunk parity), 2: spread warp
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int unit = blockIdx.x * kUnitsWS2 + u;
    const bool active = unit < nunits;
    const int64_t cbeg = active ? bounds[unit] : 0;
    const int64_t nck = active ? bounds[unit + 1] - cbeg : 0;
    double* swin = &sm.win[u][0][0];
    unsigned long long* win_full = sm.win_full[u];
    unsigned long long* w_full = sm.w_full[u];
    unsigned long long* w_empty = sm.w_empty[u];
    if (role == 2 && lane == 0) {
        for (int r = 0; r < kRingWS2; ++r) mbar_init(&win_full[r], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&w_full[i], 32);
            mbar_init(&w_empty[i], 1);
        }
        mbar_init_fence();
    }
    __syncthreads();  // the only CTA-wide synchronisation (barrier initialisation)
    if (nck <= 0) return;
    if (role == 2 && lane == 0) {
        for (int k = 0; k < kRingWS2 && k < nck; ++k) {
            mbar_expect_tx(&win_full[k], L::Bytes);
            bulk_g2s(swin + k * L::W, win + (cbeg + k) * L::W, L::Bytes, &win_full[k]);
        }
    }
    auto origin = [&](int32_t kk) -> int64_t { return (int64_t)(kk / ng - kM + 1) * ng + (kk % ng - kM + 1); };

    if (role < 2) {
        double Fb[NT][4];  // Fb[nt][ks] = F[4ks + tq][8nt + gq]
        int32_t cur_key = -1;
        double ddmax = 0.0;
        int64_t k = role;
        auto fetch = [&](int64_t kk) { return kk < nck ? desc[cbeg + kk] : make_int4(0, 0, -1, 0); };
        // this warp's chunks k, k + 2 (descriptor ready) and k + 4 (descriptor in flight)
        int4 dsc = fetch(k);
        int4 dnext = fetch(k + 2);
        In in_cur{};
        if (k < nck && lane < dsc.y) in_cur = epi.load(dsc.x + lane);
        for (; k < nck; k += 2) {
            const int slot = (int)(k % kRingWS2);
            const int64_t p0 = dsc.x;
            const int cnt = dsc.y;
            const int4 dnext2 = fetch(k + 4);
            if (dsc.z != cur_key) {
                cur_key = dsc.z;
                const int64_t org = origin(cur_key);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double* row = grid_in + org + (int64_t)(4 * ks + tq) * ng + gq;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) Fb[nt][ks] = __ldg(row + 8 * nt);
                }
            }
            mbar_wait(&win_full[slot], (uint32_t)((k / kRingWS2) & 1));
            const double* X = swin + slot * L::W;
            const double* Y = X + kChunk * kChunkT;
            double t = 0.0;  // t of slot `lane`, assembled from the 4 m-tiles
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int p = 8 * mt + gq;
                const double* xr = X + p * kChunkT;
                double acc[NT][2];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double a = xr[swz2(p, 4 * ks + tq)];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a, Fb[nt][ks]);
                }
                double part = 0.0;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const double2 y = *reinterpret_cast<const double2*>(Y + L::y(p, 8 * nt + 2 * tq));
                    part = fma(acc[nt][0], y.x, part);
                    part = fma(acc[nt][1], y.y, part);
                }
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                // slot p = 8 mt + gq lives on lanes 4 gq .. 4 gq + 3; move it to lane p
                const double tp = __shfl_sync(0xffffffffu, part, 4 * (lane & 7));
                if ((lane >> 3) == mt) t = tp;
            }
            // the next chunk's epilogue inputs, issued after this chunk's DMMAs (a load
            // issued before them would share their wait on the long scoreboard)
            In in_next{};
            if (k + 2 < nck && lane < dnext.y) in_next = epi.load(dnext.x + lane);
            double wn = 0.0;
            if (lane < cnt) ddmax = fmax(ddmax, epi.apply(p0 + lane, t, in_cur, wn));
            // weights of chunk k go to buffer `role` (= k & 1); its previous content was
            // chunk k - 2, released by S
            if (k >= 2) mbar_wait(&w_empty[role], (uint32_t)(((k >> 1) - 1) & 1));
            sm.w[u][role][lane] = wn;
            mbar_arrive(&w_full[role]);
            dsc = dnext;
            dnext = dnext2;
            in_cur = in_next;
        }
        warp_max_atomic(dmax, ddmax);
    } else {
        double S[2][NT][2];  // S[mt][nt][i] = S[8mt + gq][8nt + 2tq + i]
        int32_t cur_key = -1;
        int64_t org = 0;
        auto flush = [&]() {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                double* row = grid_out + org + (int64_t)(8 * mt + gq) * ng + 2 * tq;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        if (S[mt][nt][i] != 0.0) atomicAdd(row + 8 * nt + i, S[mt][nt][i]);
            }
        };
        DescBatch db;
        db.init(desc, cbeg, cbeg + nck, lane);
        for (int64_t k = 0; k < nck; ++k) {
            const int64_t c = cbeg + k;
            const int slot = (int)(k % kRingWS2);
            const int b = (int)(k & 1);
            const int4 dsc = db.get(k, lane);
            if (dsc.z != cur_key) {
                if (cur_key >= 0) flush();
                cur_key = dsc.z;
                org = origin(cur_key);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) S[mt][nt][0] = S[mt][nt][1] = 0.0;
            }
            mbar_wait(&w_full[b], (uint32_t)((k >> 1) & 1));
            mbar_wait(&win_full[slot], (uint32_t)((k / kRingWS2) & 1));
            const double* X = swin + slot * L::W;
            const double* Y = X + kChunk * kChunkT;
            const double wl = sm.w[u][b][lane];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int p = 4 * ks + tq;
                const double wp = __shfl_sync(0xffffffffu, wl, p);
                const double* xr = X + p * kChunkT;
                const double xa0 = wp * xr[swz2(p, gq)];
                const double xa1 = wp * xr[swz2(p, 8 + gq)];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const double yb = Y[L::y(p, 8 * nt + gq)];
                    dmma(S[0][nt][0], S[0][nt][1], xa0, yb);
                    dmma(S[1][nt][0], S[1][nt][1], xa1, yb);
                }
            }
            __syncwarp();  // S is done with window slot `slot` and w[b]
            if (lane == 0) {
                mbar_arrive(&w_empty[b]);
                if (k + kRingWS2 < nck) {
                    fence_proxy_async();
                    mbar_expect_tx(&win_full[slot], L::Bytes);
                    bulk_g2s(swin + slot * L::W, win + (c + kRingWS2) * L::W, L::Bytes, &win_full[slot]);
                }
            }
        }
        if (cur_key >= 0) flush();
    }
}

// transpose-reduction of v[0..15] over the 32 lanes: returns sum_lanes v[lane >> 1]
__device__ __forceinline__ double warp_transpose_reduce16(double (&v)[16], int lane) {
    double v8[8], v4[4], v2[2];
    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4, h2 = lane & 2;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double send = h16 ? v[j] : v[j + 8];
        const double keep = h16 ? v[j + 8] : v[j];
        v8[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double send = h8 ? v8[j] : v8[j + 4];
        const double keep = h8 ? v8[j + 4] : v8[j];
        v4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const double send = h4 ? v4[j] : v4[j + 2];
        const double keep = h4 ? v4[j + 2] : v4[j];
        v2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const double send = h2 ? v2[0] : v2[1];
    double r = (h2 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

template <int MODE, class Epi>
__global__ void __launch_bounds__(kWarps1 * 32, kCtas1)
chunked1d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
            int nunits, const double* __restrict__ grid_in, double* __restrict__ grid_out,
            const double* __restrict__ w_in, Epi epi, unsigned long long* dmax) {
    constexpr bool GATHER = MODE != 1;
    constexpr bool SPREAD = MODE != 2;
    const int lane = threadIdx.x & 31;
    const int unit = blockIdx.x * kWarps1 + (threadIdx.x >> 5);
    if (unit >= nunits) return;
    const int64_t cbeg = bounds[unit];
    const int64_t cend = bounds[unit + 1];
    double F[kChunkT], S[kChunkT];
    int32_t cur_key = -1;
    double ddmax = 0.0;
    auto flush = [&]() {
        const double v = warp_transpose_reduce16(S, lane);
        if (!(lane & 1) && v != 0.0) atomicAdd(grid_out + (cur_key - kM + 1) + (lane >> 1), v);
    };
    for (int64_t c = cbeg; c < cend; ++c) {
        const int4 dsc = desc[c];
        const int64_t p0 = dsc.x;
        const int cnt = dsc.y;
        if (dsc.z != cur_key) {
            if (SPREAD && cur_key >= 0) flush();
            cur_key = dsc.z;
            if (GATHER) {
                const double* f = grid_in + (cur_key - kM + 1);
#pragma unroll
                for (int a = 0; a < kChunkT; ++a) F[a] = __ldg(f + a);
            }
            if (SPREAD) {
#pragma unroll
                for (int a = 0; a < kChunkT; ++a) S[a] = 0.0;
            }
        }
        // this lane's window row (zero for empty slots)
        double X[kChunkT];
        const double2* xr = reinterpret_cast<const double2*>(win + c * kW1 + lane * kChunkT);
#pragma unroll
        for (int a = 0; a < kChunkT / 2; ++a) {
            const double2 v = __ldg(xr + a);
            X[2 * a] = v.x;
            X[2 * a + 1] = v.y;
        }
        double wn = 0.0;
        if (GATHER) {
            double t = 0.0;
#pragma unroll
            for (int a = 0; a < kChunkT; ++a) t = fma(X[a], F[a], t);
            if (lane < cnt) {
                ddmax = fmax(ddmax, epi(p0 + lane, t));
                if (SPREAD) wn = epi.w_next[p0 + lane];
            }
        } else {
            wn = lane < cnt ? w_in[p0 + lane] : 0.0;
        }
        if (SPREAD) {
#pragma unroll
            for (int a = 0; a < kChunkT; ++a) S[a] = fma(wn, X[a], S[a]);
        }
    }
    if (SPREAD && cur_key >= 0) flush();
    if (GATHER) warp_max_atomic(dmax, ddmax);
}

template <int MODE, class Epi>
void launch12(const PointSet& ps, const double* gin, double* gout, const double* w, const FastParams& fp,
              const Epi& epi, unsigned long long* dmax, cudaStream_t s, int tag) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    const int nunits = ps.chunk_blocks;
    ProfScope prof(tag, s);
    if (fp.d == 2) {
        const int blocks = (nunits + kWarps2 - 1) / kWarps2;
        if (ps.chunk_kz == 24) {
            set_smem_attr((const void*)chunked2d_k<MODE, Epi, 24>, (int)sizeof(Smem2<24>));
            chunked2d_k<MODE, Epi, 24><<<blocks, kWarps2 * 32, sizeof(Smem2<24>), s>>>(
                ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds.p, nunits, fp.ng, gin, gout, w, epi, dmax);
        } else {
            set_smem_attr((const void*)chunked2d_k<MODE, Epi, 16>, (int)sizeof(Smem2<16>));
            chunked2d_k<MODE, Epi, 16><<<blocks, kWarps2 * 32, sizeof(Smem2<16>), s>>>(
                ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds.p, nunits, fp.ng, gin, gout, w, epi, dmax);
        }
    } else {
        const int blocks = (nunits + kWarps1 - 1) / kWarps1;
        chunked1d_k<MODE, Epi><<<blocks, kWarps1 * 32, 0, s>>>(ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds.p,
                                                                nunits, gin, gout, w, epi, dmax);
    }
    UOTK_LAUNCHED();
}

}  // namespace

// ------------------------------------------------------------ dispatch over d (nfft.cu, api.cu)
void chunked_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    if (fp.d == 3) return fused3d_spread(ps, w, grid, fp, s);
    launch12<1, EpiNone>(ps, nullptr, grid, w, fp, EpiNone{}, nullptr, s, kProfSpread);
}

void chunked_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s) {
    if (fp.d == 3) return fused3d_gather_store(ps, grid, fp, epi, s);
    EpiGatherOnly<EpiStore> e;
    static_cast<EpiStore&>(e) = epi;
    launch12<2, EpiGatherOnly<EpiStore>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

void chunked_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s) {
    if (fp.d == 3) return fused3d_gather_dot(ps, grid, fp, epi, s);
    EpiGatherOnly<EpiDot> e;
    static_cast<EpiDot&>(e) = epi;
    launch12<2, EpiGatherOnly<EpiDot>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

// one Sinkhorn half-step at the points of ps: gather from grid_in, update (3.3)/(3.4),
// spread the new weights into grid_out
void chunked_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s) {
    if (fp.d == 3) return fused3d_gather_spread(ps, grid_in, grid_out, fp, epi, dmax, s);
    static const bool ws = [] {
        const char* e = getenv("UOTK_FUSED_WS");
        return !(e && e[0] == '0');
    }();
    if (fp.d == 2 && ws) {
        if (ps.n == 0 || ps.nchunks == 0) return;
        const int nunits = ps.chunk_units_ws;
        const int blocks = (nunits + kUnitsWS2 - 1) / kUnitsWS2;
        ProfScope prof(kProfFused, s);
        if (ps.chunk_kz == 24) {
            set_smem_attr((const void*)sinkhorn2d_ws_k<24>, (int)sizeof(Smem2WS<24>));
            sinkhorn2d_ws_k<24><<<blocks, 3 * kUnitsWS2 * 32, sizeof(Smem2WS<24>), s>>>(
                ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds_ws.p, nunits, fp.ng, grid_in, grid_out, epi, dmax);
        } else {
            set_smem_attr((const void*)sinkhorn2d_ws_k<16>, (int)sizeof(Smem2WS<16>));
            sinkhorn2d_ws_k<16><<<blocks, 3 * kUnitsWS2 * 32, sizeof(Smem2WS<16>), s>>>(
                ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds_ws.p, nunits, fp.ng, grid_in, grid_out, epi, dmax);
        }
        UOTK_LAUNCHED();
        return;
    }
    launch12<0, EpiSinkhorn>(ps, grid_in, grid_out, nullptr, fp, epi, dmax, s, kProfFused);
}

}  // namespace uotk
