// d = 3 cell-group kernels for the window half-width m = 6 (12 taps per axis), DESIGN.md §7.
//
// Same method as fused3d.cu (points sorted by cell, chunks of <= 32 points sharing one
// footprint, window blocks precomputed once per point set and streamed by TMA, the c- and
// point-contractions on DMMA), for the 12^3 footprint of m = 6.  With sigma = 3 the
// Kaiser-Bessel error of m = 6 (4 pi (sqrt m + m)(1 - 1/sigma)^{1/4} e^{-2 pi m sqrt(1 - 1/sigma)}
// ~ 4e-12, footnote P:653's window) is within the 1e-9 kernel-sum bar with (12/16)^3 = 0.42
// of the taps of m = 8, sigma = 2.
//
// Window blocks: chunks.cuh's KZ = 12 layout (3 axes x 32 slots x 12 taps, 9 KB).  The 144
// (a, b) pairs of the footprint are
// taken in a-pairs: a-pair r = {2r, 2r+1} owns the 24 pairs (a, b) in a-major order, i.e.
// three 8-wide tiles
//   tile 0: (2r, b = 0..7)   tile 1: (2r, b = 8..11), (2r+1, b = 0..3)   tile 2: (2r+1, b = 4..11)
// gather  G[p, (a,b)] = sum_c Z_p[c] F[a,b,c]    (M = 32 points, N = 3 tiles per a-pair, K = 12)
//         t_p = sum_(a,b) X_p[a] Y_p[b] G[p, (a,b)]    (in registers + quad shuffles)
// spread  S[(a,b), c] += sum_p X_p[a] Y_p[b] (w_p Z_p[c])  (M = 3 tiles per a-pair, N = 16
//         columns of which c = 0..11 are live, K = 32 points)
// i.e. 216 + 288 DMMA per chunk against 1024 for m = 8.
#include "chunks.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "ptx.cuh"

namespace uotk {

namespace {

constexpr int kM = 6;
constexpr int kPairs = 6;             // a-pairs of the 12-tap footprint
constexpr int kStride = 12;           // window row stride (doubles), chunks.cuh KZ = 12
constexpr int kWD = chunk_win3_doubles(12);
constexpr int kNP = 2;                // a-pairs per warp: the Y/Z fragment loads serve two pairs
constexpr int kWarpsA = kPairs / kNP; // warps per footprint pass
constexpr uint32_t kWB = kWD * sizeof(double);

// (a-offset within the pair, b) of column j of tile t of an a-pair
__device__ __forceinline__ void tile_ab(int t, int j, int& al, int& b) {
    const int f = 8 * t + j;
    al = f >= 12;
    b = f - 12 * al;
}

__device__ __forceinline__ int64_t footprint_origin(int32_t kk, int ng) {
    const int64_t ng2 = (int64_t)ng * ng;
    const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
    return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
}

// gather B operand of the NP a-pairs starting at pair r0: Fb[3i + t][ks] = F[a][b][4ks + tq]
template <int NP>
__device__ __forceinline__ void load_footprint(double (&Fb)[3 * NP][3], const double* __restrict__ grid, int64_t org,
                                               int ng, int r0, int gq, int tq) {
    const int64_t ng2 = (int64_t)ng * ng;
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            int al, b;
            tile_ab(t, gq, al, b);
            const double* row = grid + org + (int64_t)(2 * (r0 + i) + al) * ng2 + (int64_t)b * ng;
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) Fb[3 * i + t][ks] = __ldg(row + 4 * ks + tq);
        }
}

template <int NP>
__device__ __forceinline__ void prefetch_footprint(const double* __restrict__ grid, int64_t org, int ng, int r0,
                                                   int gq, int tq) {
    const int64_t ng2 = (int64_t)ng * ng;
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            int al, b;
            tile_ab(t, gq, al, b);
            const double* row = grid + org + (int64_t)(2 * (r0 + i) + al) * ng2 + (int64_t)b * ng;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(row + 4 * tq));
        }
}

// the partial t_p of the NP a-pairs for the 8 points of m-tile mt (valid on tq == 0 lanes
// after the quad reduction)
template <int NP>
__device__ __forceinline__ double gather_mtile(const double (&Fb)[3 * NP][3], const double (*wx)[kStride],
                                               const double (*wy)[kStride], const double (*wz)[kStride], int mt, int r0,
                                               int gq, int tq) {
    const int p = 8 * mt + gq;
    double acc[3 * NP][2];
#pragma unroll
    for (int t = 0; t < 3 * NP; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
        const double az = wz[p][4 * ks + tq];
#pragma unroll
        for (int t = 0; t < 3 * NP; ++t) dmma(acc[t][0], acc[t][1], az, Fb[t][ks]);
    }
    // lane columns j = 2tq, 2tq+1 of each tile: b of tile 0 / 1 / 2
    const double2 y0 = *reinterpret_cast<const double2*>(&wy[p][2 * tq]);
    const double2 y1 = *reinterpret_cast<const double2*>(&wy[p][tq < 2 ? 8 + 2 * tq : 2 * tq - 4]);
    const double2 y2 = *reinterpret_cast<const double2*>(&wy[p][4 + 2 * tq]);
    double part = 0.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const double2 x = *reinterpret_cast<const double2*>(&wx[p][2 * (r0 + i)]);
        const double q0 = fma(acc[3 * i][1], y0.y, acc[3 * i][0] * y0.x);
        const double q1 = fma(acc[3 * i + 1][1], y1.y, acc[3 * i + 1][0] * y1.x);
        const double q2 = fma(acc[3 * i + 2][1], y2.y, acc[3 * i + 2][0] * y2.x);
        part = fma(x.x, q0, part);
        part = fma(tq < 2 ? x.x : x.y, q1, part);
        part = fma(x.y, q2, part);
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    return part;
}

// spread of one chunk into the accumulators of the NP a-pairs: A = xr[p][a] Y_p[b]
// (xr = X, or the weighted rows w X), B = zr[p][c] (Z or w Z); wscale multiplies B
template <int NP, bool WEIGHTED_B>
__device__ __forceinline__ void spread_chunk(double (&S)[3 * NP][2][2], const double (*xr)[kStride],
                                             const double (*wy)[kStride], const double (*wz)[kStride], double w_lane,
                                             int cnt, int r0, int gq, int tq) {
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        if (4 * ks >= cnt) break;  // k-steps past the chunk's points add zero windows
        const int p = 4 * ks + tq;
        double b0 = wz[p][gq];
        double b1 = gq < 4 ? wz[p][8 + gq] : 0.0;  // columns c = 12..15 do not exist
        if (WEIGHTED_B) {
            const double wp = __shfl_sync(0xffffffffu, w_lane, p);
            b0 *= wp;
            b1 *= wp;
        }
        const double yA = wy[p][gq];
        const double yB = wy[p][gq < 4 ? 8 + gq : gq - 4];
        const double yC = wy[p][4 + gq];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const double2 x = *reinterpret_cast<const double2*>(&xr[p][2 * (r0 + i)]);
            const double a0 = x.x * yA;
            const double a1 = (gq < 4 ? x.x : x.y) * yB;
            const double a2 = x.y * yC;
            dmma(S[3 * i][0][0], S[3 * i][0][1], a0, b0);
            dmma(S[3 * i][1][0], S[3 * i][1][1], a0, b1);
            dmma(S[3 * i + 1][0][0], S[3 * i + 1][0][1], a1, b0);
            dmma(S[3 * i + 1][1][0], S[3 * i + 1][1][1], a1, b1);
            dmma(S[3 * i + 2][0][0], S[3 * i + 2][0][1], a2, b0);
            dmma(S[3 * i + 2][1][0], S[3 * i + 2][1][1], a2, b1);
        }
    }
}

template <int NP>
__device__ __forceinline__ void flush_footprint(double (&S)[3 * NP][2][2], double* __restrict__ grid, int64_t org,
                                                int ng, int r0, int gq, int tq) {
    const int64_t ng2 = (int64_t)ng * ng;
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            int al, b;
            tile_ab(t, gq, al, b);
            double* row = grid + org + (int64_t)(2 * (r0 + i) + al) * ng2 + (int64_t)b * ng;
#pragma unroll
            for (int nz = 0; nz < 2; ++nz)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * nz + 2 * tq + e;
                    const double v = S[3 * i + t][nz][e];
                    if (c < 12 && v != 0.0) atomicAdd(row + c, v);
                }
        }
}

template <int NP>
__device__ __forceinline__ void zero_acc(double (&S)[3 * NP][2][2]) {
#pragma unroll
    for (int t = 0; t < 3 * NP; ++t)
#pragma unroll
        for (int nz = 0; nz < 2; ++nz) S[t][nz][0] = S[t][nz][1] = 0.0;
}

// ---------------------------------------------------------------- spread only, ring
// kWarpsA warps, warp w owns a-pairs 2w, 2w+1; window blocks stream through a ring of
// kRingS slots released by per-slot mbarriers (as spread3d_k).
constexpr int kRingS = 4;
struct __align__(128) SmemS6 {
    double win[kRingS][kWD];
    unsigned long long full[kRingS];
    unsigned long long empty[kRingS];
};

__global__ void __launch_bounds__(kWarpsA * 32, kCtas3M6)
spread3d_m6_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds, int ng,
              double* __restrict__ grid_out, const double* __restrict__ w_in) {
    extern __shared__ __align__(128) unsigned char s6_raw[];
    SmemS6& sm = *reinterpret_cast<SmemS6*>(s6_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    if (tid == 0) {
        for (int r = 0; r < kRingS; ++r) {
            mbar_init(&sm.full[r], 1);
            mbar_init(&sm.empty[r], kWarpsA);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < kRingS && k < nck; ++k) {
            mbar_expect_tx(&sm.full[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.full[k]);
        }
    double S[3 * kNP][2][2];
    const int r0 = kNP * warp;
    int32_t cur_key = -1;
    int64_t org = 0;
    int4 d0 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);
    int4 d1 = nck > 1 ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
    double w_cur = lane < d0.y ? w_in[d0.x + lane] : 0.0;
    for (int64_t k = 0; k < nck; ++k) {
        const int slot = (int)(k % kRingS);
        const int4 dsc = d0;
        d0 = d1;
        if (k + 2 < nck) d1 = desc[cbeg + k + 2];
        const double w_nxt = (k + 1 < nck && lane < d0.y) ? w_in[d0.x + lane] : 0.0;
        if (dsc.z != cur_key) {
            if (cur_key >= 0) flush_footprint<kNP>(S, grid_out, org, ng, r0, gq, tq);
            cur_key = dsc.z;
            org = footprint_origin(cur_key, ng);
            zero_acc<kNP>(S);
        }
        mbar_wait(&sm.full[slot], (uint32_t)((k / kRingS) & 1));
        const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[slot][0]);
        spread_chunk<kNP, true>(S, wx, wx + kChunk, wx + 2 * kChunk, w_cur, dsc.y, r0, gq, tq);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[slot]);
        if (tid == 0 && k + kRingS < nck) {
            mbar_wait(&sm.empty[slot], (uint32_t)((k / kRingS) & 1));
            fence_proxy_async();
            mbar_expect_tx(&sm.full[slot], kWB);
            bulk_g2s(&sm.win[slot][0], win + (cbeg + k + kRingS) * kWD, kWB, &sm.full[slot]);
        }
        w_cur = w_nxt;
    }
    if (cur_key >= 0) flush_footprint<kNP>(S, grid_out, org, ng, r0, gq, tq);
}

// ---------------------------------------------------------------- gather only, ring
// warp w contracts a-pair w; the warp k mod 6 reduces chunk k, applies the epilogue and
// refills the slot (as gather3d_k).
constexpr int kRingG = 4;
struct __align__(128) SmemG6 {
    double win[kRingG][kWD];
    double red[kRingG][kWarpsA][kChunk];
    unsigned long long full[kRingG];
    unsigned long long red_full[kRingG];
};

template <class Epi>
__global__ void __launch_bounds__(kWarpsA * 32, kCtas3M6)
gather3d_m6_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds, int ng,
              const double* __restrict__ grid_in, Epi epi, unsigned long long* dmax) {
    extern __shared__ __align__(128) unsigned char g6_raw[];
    SmemG6& sm = *reinterpret_cast<SmemG6*>(g6_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    if (tid == 0) {
        for (int r = 0; r < kRingG; ++r) {
            mbar_init(&sm.full[r], 1);
            mbar_init(&sm.red_full[r], kWarpsA);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < kRingG && k < nck; ++k) {
            mbar_expect_tx(&sm.full[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.full[k]);
        }
    double Fb[3 * kNP][3];
    const int r0 = kNP * warp;
    int32_t cur_key = -1;
    double ddmax = 0.0;
    int4 d0 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);
    int4 d1 = nck > 1 ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
    for (int64_t k = 0; k < nck; ++k) {
        const int slot = (int)(k % kRingG);
        const int4 dsc = d0;
        d0 = d1;
        if (k + 2 < nck) d1 = desc[cbeg + k + 2];
        if (dsc.z != cur_key) {
            cur_key = dsc.z;
            load_footprint<kNP>(Fb, grid_in, footprint_origin(cur_key, ng), ng, r0, gq, tq);
        }
        if (k + 1 < nck && d0.z != cur_key) prefetch_footprint<kNP>(grid_in, footprint_origin(d0.z, ng), ng, r0, gq, tq);
        mbar_wait(&sm.full[slot], (uint32_t)((k / kRingG) & 1));
        const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[slot][0]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            if (8 * mt >= dsc.y) break;  // m-tiles past the chunk's points hold no point
            const double part = gather_mtile<kNP>(Fb, wx, wx + kChunk, wx + 2 * kChunk, mt, r0, gq, tq);
            if (tq == 0) sm.red[slot][warp][8 * mt + gq] = part;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.red_full[slot]);
        if (warp == (int)(k % kWarpsA)) {
            mbar_wait(&sm.red_full[slot], (uint32_t)((k / kRingG) & 1));
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kWarpsA; ++w) t += sm.red[slot][w][lane];
            if (lane < dsc.y) ddmax = fmax(ddmax, epi(dsc.x + lane, t));
            __syncwarp();
            if (lane == 0 && k + kRingG < nck) {
                fence_proxy_async();
                mbar_expect_tx(&sm.full[slot], kWB);
                bulk_g2s(&sm.win[slot][0], win + (cbeg + k + kRingG) * kWD, kWB, &sm.full[slot]);
            }
        }
    }
    if (dmax) warp_max_atomic(dmax, ddmax);
}

// ---------------------------------------------------------------- warp-specialised half-step
// kGW gather warps (warp g owns a-pairs NPG g ...) and kSW spread warps.  Chunk k's
// partial gathers go to red[k % kRingR]; the gather warp k mod kGW reduces them, runs the
// update (3.3)/(3.4) for the 32 slots and publishes the weighted rows xw[p][a] = w_p X_p[a]
// (all 12 a) of chunk k; the spread warps spread chunk k from xw while the gather warps
// already work on chunk k+1.  All hand-offs are mbarriers:
//   win_full[kRingW]   TMA ring of window blocks (refilled by the first spread warp)
//   red_full/red_empty partial gathers of a chunk complete / consumed by its reducer
//   xw_full/xw_empty   weighted rows of a chunk published / consumed by the spread warps
constexpr int kNPG = kNP, kNPS = kNP;
constexpr int kGW = kPairs / kNPG, kSW = kPairs / kNPS;
constexpr int kThreadsWS = 32 * (kGW + kSW);
constexpr int kRingW = 4, kRingR = 4;
struct __align__(128) SmemWS6 {
    double win[kRingW][kWD];
    double xw[2][kChunk][kStride];
    double red[kRingR][kGW][kChunk];
    unsigned long long win_full[kRingW];
    unsigned long long red_full[kRingR];
    unsigned long long red_empty[kRingR];
    unsigned long long xw_full[2];
    unsigned long long xw_empty[2];
};

__global__ void __launch_bounds__(kThreadsWS, kCtasWS3M6)
sinkhorn3d_m6_ws_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
                   int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out, EpiSinkhorn epi,
                   unsigned long long* dmax) {
    extern __shared__ __align__(128) unsigned char w6_raw[];
    SmemWS6& sm = *reinterpret_cast<SmemWS6*>(w6_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    if (tid == 0) {
        for (int i = 0; i < kRingW; ++i) mbar_init(&sm.win_full[i], 1);
        for (int i = 0; i < kRingR; ++i) {
            mbar_init(&sm.red_full[i], kGW);
            mbar_init(&sm.red_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.xw_full[i], 1);
            mbar_init(&sm.xw_empty[i], 1);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < kRingW && k < nck; ++k) {
            mbar_expect_tx(&sm.win_full[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.win_full[k]);
        }

    if (warp < kGW) {
        // ------------------------------------------------------------ gather + update
        const int g = warp;
        const int r0 = kNPG * g;
        double Fb[3 * kNPG][3];
        int32_t cur_key = -1;
        double ddmax = 0.0;
        int4 d0 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);
        int4 d1 = nck > 1 ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
        for (int64_t k = 0; k < nck; ++k) {
            const int wslot = (int)(k % kRingW);
            const int rslot = (int)(k % kRingR);
            const int4 dsc = d0;
            d0 = d1;
            if (k + 2 < nck) d1 = desc[cbeg + k + 2];
            const bool reducer = g == (int)(k % kGW);
            EpiSinkhorn::In in{};
            if (reducer && lane < dsc.y) in = epi.load(dsc.x + lane);  // consumed after the DMMAs
            if (dsc.z != cur_key) {
                cur_key = dsc.z;
                load_footprint<kNPG>(Fb, grid_in, footprint_origin(cur_key, ng), ng, r0, gq, tq);
            }
            if (k + 1 < nck && d0.z != cur_key)
                prefetch_footprint<kNPG>(grid_in, footprint_origin(d0.z, ng), ng, r0, gq, tq);
            mbar_wait(&sm.win_full[wslot], (uint32_t)((k / kRingW) & 1));
            const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[wslot][0]);
            const double(*wy)[kStride] = wx + kChunk;
            const double(*wz)[kStride] = wx + 2 * kChunk;
            if (k >= kRingR) mbar_wait(&sm.red_empty[rslot], (uint32_t)(((k / kRingR) - 1) & 1));
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                if (8 * mt >= dsc.y) break;  // m-tiles past the chunk's points hold no point
                const double part = gather_mtile<kNPG>(Fb, wx, wy, wz, mt, r0, gq, tq);
                if (tq == 0) sm.red[rslot][g][8 * mt + gq] = part;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.red_full[rslot]);
            if (reducer) {
                mbar_wait(&sm.red_full[rslot], (uint32_t)((k / kRingR) & 1));
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < kGW; ++w) t += sm.red[rslot][w][lane];
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.red_empty[rslot]);
                double wp = 0.0;
                if (lane < dsc.y) ddmax = fmax(ddmax, epi.apply(dsc.x + lane, t, in, wp));
                // publish the weighted rows of chunk k (slot k & 1)
                if (k >= 2) mbar_wait(&sm.xw_empty[k & 1], (uint32_t)(((k >> 1) - 1) & 1));
                const double2* xs = reinterpret_cast<const double2*>(&wx[lane][0]);
                double2* xd = reinterpret_cast<double2*>(&sm.xw[k & 1][lane][0]);
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const double2 v = xs[q];
                    xd[q] = make_double2(wp * v.x, wp * v.y);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.xw_full[k & 1]);
            }
        }
        warp_max_atomic(dmax, ddmax);
    } else {
        // ------------------------------------------------------------ spread
        const int sw = warp - kGW;
        const int r0 = kNPS * sw;
        double S[3 * kNPS][2][2];
        int32_t cur_key = -1;
        int64_t org = 0;
        int4 dk1 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);  // descriptors two chunks ahead
        int4 dk2 = nck > 1 ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
        for (int64_t k = 0; k < nck; ++k) {
            const int wslot = (int)(k % kRingW);
            const int32_t key = dk1.z;
            const int cnt = dk1.y;
            dk1 = dk2;
            if (k + 2 < nck) dk2 = desc[cbeg + k + 2];
            if (key != cur_key) {
                if (cur_key >= 0) flush_footprint<kNPS>(S, grid_out, org, ng, r0, gq, tq);
                cur_key = key;
                org = footprint_origin(key, ng);
                zero_acc<kNPS>(S);
            }
            mbar_wait(&sm.xw_full[k & 1], (uint32_t)((k >> 1) & 1));
            // the window slot is complete: the reducer read it before publishing xw
            const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[wslot][0]);
            spread_chunk<kNPS, false>(S, sm.xw[k & 1], wx + kChunk, wx + 2 * kChunk, 0.0, cnt, r0, gq, tq);
            group_sync(1, 32 * kSW);  // all spread warps are done with xw[k & 1] and the window slot
            if (sw == 0 && lane == 0) {
                mbar_arrive(&sm.xw_empty[k & 1]);
                if (k + kRingW < nck) {
                    fence_proxy_async();
                    mbar_expect_tx(&sm.win_full[wslot], kWB);
                    bulk_g2s(&sm.win[wslot][0], win + (cbeg + k + kRingW) * kWD, kWB, &sm.win_full[wslot]);
                }
            }
        }
        if (cur_key >= 0) flush_footprint<kNPS>(S, grid_out, org, ng, r0, gq, tq);
    }
}

}  // namespace

void fused3d_m6_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s);
template <class Epi>
static void gather_m6(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi, cudaStream_t s,
                      unsigned long long* dmax);

// The Sinkhorn half-step: the warp-specialised single launch; UOTK_M6_WS=0 runs the two
// stand-alone kernels instead (gather with the update as its epilogue, then the spread of
// the new weights) — C3 solve 190 ms vs 218 ms (A/B on one box).
void fused3d_m6_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                              const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    static const bool ws = [] {
        const char* e = getenv("UOTK_M6_WS");
        return !(e && e[0] == '0');
    }();
    if (!ws) {
        gather_m6(ps, grid_in, fp, epi, s, dmax);
        fused3d_m6_spread(ps, epi.w_next, grid_out, fp, s);
        return;
    }
    set_smem_attr((const void*)sinkhorn3d_m6_ws_k, (int)sizeof(SmemWS6));
    ProfScope prof(kProfFused, s);
    sinkhorn3d_m6_ws_k<<<ps.chunk_units_ws, kThreadsWS, sizeof(SmemWS6), s>>>(
        ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds_ws.p, fp.ng, grid_in, grid_out, epi, dmax);
    UOTK_LAUNCHED();
}

void fused3d_m6_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    set_smem_attr((const void*)spread3d_m6_k, (int)sizeof(SmemS6));
    ProfScope prof(kProfSpread, s);
    spread3d_m6_k<<<ps.chunk_blocks, kWarpsA * 32, sizeof(SmemS6), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                       ps.chunk_bounds.p, fp.ng, grid, w);
    UOTK_LAUNCHED();
}

template <class Epi>
static void gather_m6(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi, cudaStream_t s,
                      unsigned long long* dmax) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    set_smem_attr((const void*)gather3d_m6_k<Epi>, (int)sizeof(SmemG6));
    ProfScope prof(kProfGather, s);
    gather3d_m6_k<Epi><<<ps.chunk_blocks, kWarpsA * 32, sizeof(SmemG6), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                            ps.chunk_bounds.p, fp.ng, grid, epi, dmax);
    UOTK_LAUNCHED();
}

void fused3d_m6_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                             cudaStream_t s) {
    gather_m6(ps, grid, fp, epi, s, nullptr);
}

void fused3d_m6_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                           cudaStream_t s) {
    gather_m6(ps, grid, fp, epi, s, nullptr);
}

}  // namespace uotk
