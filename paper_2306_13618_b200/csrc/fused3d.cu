// Tuned d = 3 NFFT passes on the FP64 tensor cores (DESIGN.md §7 "cell-group kernel").
//
// Points are sorted by grid cell (points.cu), so every run of equal keys shares one
// 16^3 window footprint on the oversampled grid (m = 8, 2m taps per axis).  Runs are cut
// into chunks of <= 32 points and the window values of every chunk (3 axes x 32 slots x
// 16 taps, zero for empty slots) are computed ONCE per point set (chunks.cu,
// chunked_prepare) — points do not move between Sinkhorn iterations.  A 256-thread CTA
// walks a contiguous, cost-balanced range of chunks, streaming each chunk's window block
// into shared memory with a TMA bulk copy (cp.async.bulk + mbarrier, double buffered in
// chunked3d_k, a ring of 4 in the warp-specialised sinkhorn3d_ws_k).  Sparse clouds use
// z-segment groups (KZ = 24: 9 cells along z share one 16 x 16 x 24 footprint).  Sets
// that are only ever spread (kernel-sum sources, MMD^2's z) evaluate their window blocks
// inside the spread (spread3d_fly_k) and, when their one-cell chunks are partly filled,
// take hybrid groups (dense cells alone, the sparser cells of a z-segment together).
//
// Per chunk, with X_p, Y_p, Z_p the windows of point p along the three axes and F the
// group's footprint (outer / inner sums of (4.6)):
//   gather  t_p = sum_a X_p[a] sum_b Y_p[b] sum_c F[a,b,c] Z_p[c]
//           -> the c-contraction is a GEMM  G[p,(a,b)] = sum_c Z[p,c] F[(a,b),c]  (32x256x16)
//              on DMMA (mma.sync.m8n8k4.f64); b and a are contracted per point in registers
//   spread  S[(a,b),c] += sum_p (X_p[a] Y_p[b]) (w_p Z_p[c])        (GEMM 256x16x32 on DMMA)
// Warp w owns the a-pair {2w, 2w+1}: its F (gather B operand) and S (spread
// accumulators) stay in registers for the whole cell group — the footprint is read once
// and flushed once (fp64 RED) per group.  Between the two GEMMs the per-warp partial
// gathers are summed in shared memory, every warp evaluates the Sinkhorn update (3.3)/
// (3.4) for the 32 slots (warp 0 writes the potentials), and the new weights are
// broadcast by shuffles into the spread's B operand: one pass over the points per
// half-step.  On B200 DMMA runs at the full FP64 rate (37 TFLOP/s measured,
// scripts/dmma_probe.cu) from 1/8 of the instructions of a DFMA formulation.
#include <cub/cub.cuh>

#include <type_traits>

#include "chunks.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "ptx.cuh"
#include "window.cuh"
#include "window_fit.h"

namespace uotk {

namespace {

constexpr int kM = kChunkM;          // window half-width of the tuned kernels
constexpr int kThreads = 256;        // 8 warps
constexpr int kStride = kStride3;    // padded row stride (doubles) of a window matrix: conflict-free fragments
constexpr int kWinDoubles = chunk_win_doubles(3);
constexpr uint32_t kWinBytes = kWinDoubles * sizeof(double);  // 15 KB
constexpr int kBlocksPerSM = kCtas3;

// Shared-memory copy of one chunk's window block with a z-row width KZ (chunks.cuh:
// 16 for one-cell groups, 24 for z-column segments of sparse clouds).
template <int KZ>
struct __align__(128) SmemK {
    double win[2][chunk_win3_doubles(KZ)];  // double-buffered window blocks (TMA destination)
    double red[kThreads / 32][kChunk];      // per-warp partial gathers
    unsigned long long bar[2];              // mbarriers of the two buffers
};

// MODE: 0 = gather -> epilogue -> spread (Sinkhorn half-step), 1 = spread only, 2 = gather only.
// KZ: footprint extent along z (16: the group is one cell; 24: a segment of kSegZ cells
// along z, each point's z-window placed at its cell's offset in the segment).
template <int MODE, class Epi, int KZ>
__global__ void __launch_bounds__(kThreads, kBlocksPerSM)
chunked3d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
            int64_t nchunks, int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out,
            const double* __restrict__ w_in, Epi epi, unsigned long long* dmax) {
    constexpr bool GATHER = MODE != 1;
    constexpr bool SPREAD = MODE != 2;
    constexpr int KS = KZ / 4;  // k-steps of the gather GEMM (contraction over z)
    constexpr int NZ = KZ / 8;  // n-tiles of the spread GEMM (output columns along z)
    constexpr int ZS = chunk_zstride3(KZ);
    constexpr int kWD = chunk_win3_doubles(KZ);
    constexpr uint32_t kWB = kWD * sizeof(double);
    __shared__ SmemK<KZ> sm;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;  // fragment "group" (row of A / D, column of B)
    const int tq = lane & 3;   // thread in group
    const int a0 = 2 * warp;   // this warp's a-pair

    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t cend = bounds[blockIdx.x + 1];
    const int64_t ng2 = (int64_t)ng * ng;
    (void)nchunks;

    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < 2 && cbeg + k < cend; ++k) {
            mbar_expect_tx(&sm.bar[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.bar[k]);
        }
    }

    // gather B operand: Fb[nt][ks] = F[a0 + (nt>>1)][8(nt&1) + gq][4ks + tq]
    double Fb[4][KS];
    // spread accumulators: S[mt][nz] = {S[a0 + (mt>>1)][8(mt&1) + gq][8nz + 2tq + i]}
    double S[4][NZ][2];
    int32_t cur_key = -1;
    int64_t gorg = 0;  // grid index of footprint (0,0,0) for the current group
    double ddmax = 0.0;

    auto origin = [&](int32_t kk) -> int64_t {
        const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
        return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
    };
    auto flush = [&]() {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int64_t row = gorg + (int64_t)(a0 + (mt >> 1)) * ng2 + (int64_t)(8 * (mt & 1) + gq) * ng;
#pragma unroll
            for (int nz = 0; nz < NZ; ++nz)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (S[mt][nz][i] != 0.0) atomicAdd(grid_out + row + 8 * nz + 2 * tq + i, S[mt][nz][i]);
        }
    };

    // descriptors two chunks ahead; the spread-only mode's source weights one chunk ahead
    int4 dsc_next = cbeg < cend ? desc[cbeg] : make_int4(0, 0, -1, 0);
    int4 dsc_next2 = cbeg + 1 < cend ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
    double w_cur = (!GATHER && lane < dsc_next.y) ? w_in[dsc_next.x + lane] : 0.0;
    for (int64_t c = cbeg; c < cend; ++c) {
        const int k = (int)(c - cbeg);
        const int buf = k & 1;
        const int4 dsc = dsc_next;  // {first point, count, group key, 0}
        dsc_next = dsc_next2;
        if (c + 2 < cend) dsc_next2 = desc[c + 2];
        double w_nxt = 0.0;
        if (!GATHER && c + 1 < cend && lane < dsc_next.y) w_nxt = w_in[dsc_next.x + lane];
        const int64_t p0 = dsc.x;
        const int cnt = dsc.y;
        const int32_t key = dsc.z;

        if (key != cur_key) {
            if (SPREAD && cur_key >= 0) flush();
            cur_key = key;
            gorg = origin(key);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int64_t row = gorg + (int64_t)(a0 + (nt >> 1)) * ng2 + (int64_t)(8 * (nt & 1) + gq) * ng;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
                    if (GATHER) Fb[nt][ks] = __ldg(grid_in + row + 4 * ks + tq);
            }
            if (SPREAD) {
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nz = 0; nz < NZ; ++nz) S[mt][nz][0] = S[mt][nz][1] = 0.0;
            }
        }
        if (GATHER) {
            // warm L1 with the epilogue's per-point inputs and, at a group boundary, with
            // the next group's footprint (hides their latency behind this chunk)
            if (lane < cnt) epi.prefetch(p0 + lane);
            if (c + 1 < cend) {
                const int32_t nkey = dsc_next.z;
                if (nkey != key) {
                    const int64_t norg = origin(nkey);
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) {
                        const double* rowp =
                            grid_in + norg + (int64_t)(a0 + (nt >> 1)) * ng2 + (int64_t)(8 * (nt & 1) + gq) * ng;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(rowp + 4 * tq));
                    }
                }
            }
        }
        mbar_wait(&sm.bar[buf], (k >> 1) & 1);
        const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[buf][0]);
        const double(*wy)[kStride] = wx + kChunk;
        const double(*wz)[ZS] = reinterpret_cast<const double(*)[ZS]>(&sm.win[buf][2 * kChunk * kStride]);

        double wn = 0.0;  // spread weight of slot `lane`
        if (GATHER) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {  // 8 points per m-tile
                if (8 * mt >= cnt) break;  // m-tiles past the chunk's points hold no point
                const int p = 8 * mt + gq;
                double acc[4][2];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const double az = wz[p][4 * ks + tq];  // A[p][c] = Z_p[c]
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], az, Fb[nt][ks]);
                }
                // acc[nt][i] = G[p][a = a0 + (nt>>1)][b = 8(nt&1) + 2tq + i]
                const double2 ylo = *reinterpret_cast<const double2*>(&wy[p][2 * tq]);
                const double2 yhi = *reinterpret_cast<const double2*>(&wy[p][8 + 2 * tq]);
                const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
                const double xv[2] = {xa.x, xa.y};
                double part = 0.0;
#pragma unroll
                for (int al = 0; al < 2; ++al) {
                    double q = acc[2 * al][0] * ylo.x;
                    q = fma(acc[2 * al][1], ylo.y, q);
                    q = fma(acc[2 * al + 1][0], yhi.x, q);
                    q = fma(acc[2 * al + 1][1], yhi.y, q);
                    part = fma(q, xv[al], part);
                }
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                if (tq == 0) sm.red[warp][p] = part;
            }
            __syncthreads();
            // every warp sums the 4 warp partials of slot `lane`; warp 0 applies the
            // epilogue (writes), the others evaluate the same update for the weights
            if (lane < cnt) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; ++w) t += sm.red[w][lane];
                if (warp == 0) {
                    const double dd = epi(p0 + lane, t);
                    ddmax = fmax(ddmax, dd);
                    if (SPREAD) wn = epi.weight(p0 + lane, t);
                } else if (SPREAD) {
                    wn = epi.weight(p0 + lane, t);
                }
            }
        } else {
            wn = w_cur;
        }

        if (SPREAD) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {  // 4 points per k-step
                if (4 * ks >= cnt) break;  // k-steps past the chunk's points add zero windows
                const int p = 4 * ks + tq;
                const double wp = __shfl_sync(0xffffffffu, wn, p);
                // B[p][c] = w_p Z_p[c] for c = 8 nz + gq
                double bz[NZ];
#pragma unroll
                for (int nz = 0; nz < NZ; ++nz) bz[nz] = wp * wz[p][8 * nz + gq];
                const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
                const double xv[2] = {xa.x, xa.y};
                const double ylo = wy[p][gq], yhi = wy[p][8 + gq];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    // A[(a,b)][p] = X_p[a] Y_p[b], a = a0 + (mt>>1), b = 8(mt&1) + gq
                    const double am = xv[mt >> 1] * ((mt & 1) ? yhi : ylo);
#pragma unroll
                    for (int nz = 0; nz < NZ; ++nz) dmma(S[mt][nz][0], S[mt][nz][1], am, bz[nz]);
                }
            }
        }
        __syncthreads();  // every thread is done with win[buf] and red
        if (tid == 0 && c + 2 < cend) {
            fence_proxy_async();
            mbar_expect_tx(&sm.bar[buf], kWB);
            bulk_g2s(&sm.win[buf][0], win + (c + 2) * kWD, kWB, &sm.bar[buf]);
        }
        w_cur = w_nxt;
    }
    if (SPREAD && cur_key >= 0) flush();
    if (GATHER && warp == 0) warp_max_atomic(dmax, ddmax);
}

// ---------------------------------------------------------------- warp-specialised half-step
// The Sinkhorn half-step with the gather and the spread on different warps of the CTA:
//   warps 0-3 ("G"): gather chunk k (DMMA GEMM over c + b/a contractions) and publish the
//                    four warp partials of t_p (red_full); no update, no barrier: G runs up
//                    to a window ring ahead of S;
//   warps 4-7 ("S"): the update (3.3)/(3.4) of chunk k+1 on ONE S warp (rotating, one chunk
//                    ahead: its log/exp chain overlaps the other S warps' DMMAs), then the
//                    spread of chunk k (A = w_p X_p Y_p, B = Z on DMMA).
// Each group's scalar phases then overlap DMMA streams instead of idling the FP64 pipe.
// Hand-offs are mbarriers: win_full[4] (TMA ring of window blocks, refilled by the last S
// warp to release a slot), red_full[4] (G partials), w_full / w_empty[4] (the weights);
// never __syncthreads.
constexpr int kRing = 4;
// Gather footprint staging: each G warp copies its 4 a-planes x 16 rows of the NEXT group's
// footprint (key = desc.w) into shared memory with 16-byte cp.async while the current group
// runs, and loads its B fragments from there at the group change (no global-latency stall
// at the first DMMAs of a group).  Rows start at the even double at or before the row
// (16-byte alignment): 18 doubles per row, the row's parity is the offset.
constexpr int kFootRow = 18;
struct __align__(128) SmemWS {
    double foot[4][4][16][kFootRow];
    double win[kRing][3][kChunk][kStride];
    double wsc[4][kChunk];     // the chunk's next weights w_p (the spread's A = w_p X_p Y_p)
    double red[4][4][kChunk];  // per-G-warp partial sums of t_p, 4 chunks in flight
    unsigned long long win_full[kRing];
    unsigned long long red_full[4];  // the four G partials of a chunk are in red[]
    unsigned long long w_full[4];    // a chunk's weights are in wsc[]
    unsigned long long w_empty[4];   // the four S warps are done with wsc[] of a chunk
    unsigned int slot_done[kRing];   // S warps done with a window slot (running count)
};

__global__ void __launch_bounds__(256, kBlocksPerSM)
sinkhorn3d_ws_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds,
                int ng, const double* __restrict__ grid_in, double* __restrict__ grid_out, EpiSinkhorn epi,
                unsigned long long* dmax) {
    extern __shared__ __align__(128) unsigned char ws_raw[];
    SmemWS& sm = *reinterpret_cast<SmemWS*>(ws_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const bool is_g = warp < 4;
    const int gw = warp & 3;  // warp index within its group
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int a0 = 4 * gw;  // the group-warp's a-quarter
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t cend = bounds[blockIdx.x + 1];
    const int64_t nck = cend - cbeg;
    const int64_t ng2 = (int64_t)ng * ng;

    if (tid == 0) {
        for (int i = 0; i < kRing; ++i) mbar_init(&sm.win_full[i], 1);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&sm.red_full[i], 4);
            mbar_init(&sm.w_full[i], 1);
            mbar_init(&sm.w_empty[i], 4);
        }
        for (int i = 0; i < kRing; ++i) sm.slot_done[i] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < kRing && k < nck; ++k) {
            mbar_expect_tx(&sm.win_full[k], kWinBytes);
            bulk_g2s(&sm.win[k][0][0][0], win + (cbeg + k) * kWinDoubles, kWinBytes, &sm.win_full[k]);
        }
    }
    auto origin = [&](int32_t kk) -> int64_t {
        const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
        return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
    };

    if (is_g) {
        // ------------------------------------------------------------ gather + update
        double Fb[8][4];  // Fb[nt][ks] = F[a0 + (nt>>1)][8(nt&1) + gq][4ks + tq]
        int32_t cur_key = -1;
        int4 dsc_next = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, -1);
        double(*foot)[16][kFootRow] = sm.foot[gw];
        // stage this warp's 64 footprint rows of group `key` (576 16-byte pieces, 18 per lane)
        auto stage = [&](int32_t key) {
            const int64_t org = origin(key);
#pragma unroll 6
            for (int t = 0; t < 18; ++t) {
                const int i = lane + 32 * t;
                const int row = i / 9, j = i - 9 * row;
                const int64_t rs = org + (int64_t)(a0 + (row >> 4)) * ng2 + (int64_t)(row & 15) * ng;
                const int sh = (int)(rs & 1);
                const uint32_t nb = j < 8 ? 16u : (sh ? 8u : 0u);
                cp_async16(&foot[row >> 4][row & 15][2 * j], grid_in + (rs - sh) + 2 * j, nb);
            }
            cp_async_commit();
        };
        if (nck > 0) stage(dsc_next.z);
        for (int64_t k = 0; k < nck; ++k) {
            const int64_t c = cbeg + k;
            const int slot = (int)(k % kRing);
            const int4 dsc = dsc_next;
            if (k + 1 < nck) dsc_next = desc[c + 1];
            const int cnt = dsc.y;
            if (dsc.z != cur_key) {
                cur_key = dsc.z;
                const int64_t org = origin(cur_key);
                cp_async_wait_all();
                __syncwarp();
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    const int64_t rs = org + (int64_t)(a0 + (nt >> 1)) * ng2 + (int64_t)(8 * (nt & 1) + gq) * ng;
                    const double* row = &foot[nt >> 1][8 * (nt & 1) + gq][rs & 1];
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) Fb[nt][ks] = row[4 * ks + tq];
                }
                __syncwarp();
                if (dsc.w >= 0) stage(dsc.w);  // the next group's rows, one group ahead
            }
            mbar_wait(&sm.win_full[slot], (uint32_t)((k / kRing) & 1));
            const double(*wx)[kStride] = sm.win[slot][0];
            const double(*wy)[kStride] = sm.win[slot][1];
            const double(*wz)[kStride] = sm.win[slot][2];
            double(*red)[kChunk] = sm.red[k & 3];
            double part[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                part[mt] = 0.0;
                if (8 * mt >= cnt) continue;  // m-tiles past the chunk's points hold no point
                const int p = 8 * mt + gq;
                double acc[8][2];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const double az = wz[p][4 * ks + tq];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) dmma(acc[nt][0], acc[nt][1], az, Fb[nt][ks]);
                }
                const double2 ylo = *reinterpret_cast<const double2*>(&wy[p][2 * tq]);
                const double2 yhi = *reinterpret_cast<const double2*>(&wy[p][8 + 2 * tq]);
                const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
                const double2 xb = *reinterpret_cast<const double2*>(&wx[p][a0 + 2]);
                const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
                for (int al = 0; al < 4; ++al) {
                    double q = acc[2 * al][0] * ylo.x;
                    q = fma(acc[2 * al][1], ylo.y, q);
                    q = fma(acc[2 * al + 1][0], yhi.x, q);
                    q = fma(acc[2 * al + 1][1], yhi.y, q);
                    part[mt] = fma(q, xv[al], part[mt]);
                }
            }
            // the four tiles' reductions over tq together (independent shuffles)
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) part[mt] += __shfl_xor_sync(0xffffffffu, part[mt], 1);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) part[mt] += __shfl_xor_sync(0xffffffffu, part[mt], 2);
            if (tq == 0) {
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) red[gw][8 * mt + gq] = part[mt];
            }
            // publish this warp's partials of chunk k; the update runs on the spread side.
            // Four partial-sum slots suffice: a G warp reaches chunk k+4 only after every S
            // warp released chunk k's window slot (ring of 4), i.e. after chunk k's update
            // (run by an S warp during chunk k-1) read them.
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.red_full[k & 3]);
        }
        cp_async_wait_all();  // a staged next group past this block's range
    } else {
        // ------------------------------------------------------------ spread
        double S[8][2][2];  // S[mt][nt] = S[a0 + (mt>>1)][8(mt&1) + gq][8nt + 2tq + i]
        int32_t cur_key = -1;
        int64_t org = 0;
        auto flush = [&]() {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                const int64_t row = org + (int64_t)(a0 + (mt >> 1)) * ng2 + (int64_t)(8 * (mt & 1) + gq) * ng;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        if (S[mt][nt][i] != 0.0) atomicAdd(grid_out + row + 8 * nt + 2 * tq + i, S[mt][nt][i]);
            }
        };
        // the update (3.3)/(3.4) of chunk j by one S warp (j mod 4), one chunk AHEAD of the
        // spread: lane p sums the four G partials, writes the potential, the next weight,
        // the sup-norm change, and publishes w_p in wsc[j & 3]
        double ddmax = 0.0;
        auto update = [&](int64_t j, const int4& dj) {
            if (lane < dj.y) epi.prefetch(dj.x + lane);
            mbar_wait(&sm.red_full[j & 3], (uint32_t)((j >> 2) & 1));
            double wp = 0.0;
            if (lane < dj.y) {
                const double(*red)[kChunk] = sm.red[j & 3];
                const double t = red[0][lane] + red[1][lane] + red[2][lane] + red[3][lane];
                ddmax = fmax(ddmax, epi.apply(dj.x + lane, t, epi.load(dj.x + lane), wp));
            }
            if (j >= 4) mbar_wait(&sm.w_empty[j & 3], (uint32_t)(((j >> 2) - 1) & 1));
            sm.wsc[j & 3][lane] = wp;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.w_full[j & 3]);
        };
        int4 dk_next = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, -1);
        if (nck > 0 && gw == 0) update(0, dk_next);
        for (int64_t k = 0; k < nck; ++k) {
            const int64_t c = cbeg + k;
            const int slot = (int)(k % kRing);
            const int4 dk = dk_next;
            if (k + 1 < nck) dk_next = desc[c + 1];
            if (k + 1 < nck && gw == (int)((k + 1) & 3)) update(k + 1, dk_next);
            const int32_t key = dk.z;
            const int cnt = dk.y;
            if (key != cur_key) {
                if (cur_key >= 0) flush();
                cur_key = key;
                org = origin(key);
#pragma unroll
                for (int mt = 0; mt < 8; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) S[mt][nt][0] = S[mt][nt][1] = 0.0;
            }
            mbar_wait(&sm.w_full[k & 3], (uint32_t)((k >> 2) & 1));
            mbar_wait(&sm.win_full[slot], (uint32_t)((k / kRing) & 1));
            const double(*wx)[kStride] = sm.win[slot][0];
            const double(*wy)[kStride] = sm.win[slot][1];
            const double(*wz)[kStride] = sm.win[slot][2];
            const double* wsc = sm.wsc[k & 3];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                if (4 * ks >= cnt) break;  // k-steps past the chunk's points add zero windows
                const int p = 4 * ks + tq;
                const double b0 = wz[p][gq];
                const double b1 = wz[p][8 + gq];
                const double wv = wsc[p];
                const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
                const double2 xb = *reinterpret_cast<const double2*>(&wx[p][a0 + 2]);
                const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
                // w_p folded into the two y values (2 DMUL per step instead of 4 on x)
                const double ylo = wv * wy[p][gq], yhi = wv * wy[p][8 + gq];
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const double am = xv[mt >> 1] * ((mt & 1) ? yhi : ylo);
                    dmma(S[mt][0][0], S[mt][0][1], am, b0);
                    dmma(S[mt][1][0], S[mt][1][1], am, b1);
                }
            }
            // release wsc[k & 3] (w_empty) and the window slot: no barrier among the S
            // warps (the update rotates over them); the last of the four refills the slot
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                mbar_arrive(&sm.w_empty[k & 3]);
                if ((atomicAdd(&sm.slot_done[slot], 1u) & 3u) == 3u && k + kRing < nck) {
                    __threadfence_block();
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&sm.win_full[slot], kWinBytes);
                    bulk_g2s(&sm.win[slot][0][0][0], win + (c + kRing) * kWinDoubles, kWinBytes, &sm.win_full[slot]);
                }
            }
        }
        if (cur_key >= 0) flush();
        warp_max_atomic(dmax, ddmax);
    }
}

// ---------------------------------------------------------------- spread only, ring
// The adjoint NFFT alone (kernel sums' sources, MMD^2): the same per-warp a-pair GEMMs as
// chunked3d_k<1>, but without a CTA barrier per chunk — window blocks stream through a
// ring of kRingS slots, each released by an mbarrier the eight warps arrive on, so the
// warps drift apart and the TMA refill overlaps the other warps' DMMAs.
constexpr int kRingS = 4;
template <int KZ>
struct __align__(128) SmemS {
    double win[kRingS][chunk_win3_doubles(KZ)];
    unsigned long long full[kRingS];
    unsigned long long empty[kRingS];
};

template <int KZ>
__global__ void __launch_bounds__(kThreads, kBlocksPerSM)
spread3d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds, int ng,
           double* __restrict__ grid_out, const double* __restrict__ w_in) {
    constexpr int NZ = KZ / 8;
    constexpr int ZS = chunk_zstride3(KZ);
    constexpr int kWD = chunk_win3_doubles(KZ);
    constexpr uint32_t kWB = kWD * sizeof(double);
    extern __shared__ __align__(128) unsigned char s_raw[];
    SmemS<KZ>& sm = *reinterpret_cast<SmemS<KZ>*>(s_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int a0 = 2 * warp;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    const int64_t ng2 = (int64_t)ng * ng;
    if (tid == 0) {
        for (int r = 0; r < kRingS; ++r) {
            mbar_init(&sm.full[r], 1);
            mbar_init(&sm.empty[r], kThreads / 32);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < kRingS && k < nck; ++k) {
            mbar_expect_tx(&sm.full[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.full[k]);
        }
    }
    double S[4][NZ][2];
    int32_t cur_key = -1;
    int64_t gorg = 0;
    auto origin = [&](int32_t kk) -> int64_t {
        const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
        return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
    };
    auto flush = [&]() {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int64_t row = gorg + (int64_t)(a0 + (mt >> 1)) * ng2 + (int64_t)(8 * (mt & 1) + gq) * ng;
#pragma unroll
            for (int nz = 0; nz < NZ; ++nz)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (S[mt][nz][i] != 0.0) atomicAdd(grid_out + row + 8 * nz + 2 * tq + i, S[mt][nz][i]);
        }
    };
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
            if (cur_key >= 0) flush();
            cur_key = dsc.z;
            gorg = origin(cur_key);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nz = 0; nz < NZ; ++nz) S[mt][nz][0] = S[mt][nz][1] = 0.0;
        }
        mbar_wait(&sm.full[slot], (uint32_t)((k / kRingS) & 1));
        const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[slot][0]);
        const double(*wy)[kStride] = wx + kChunk;
        const double(*wz)[ZS] = reinterpret_cast<const double(*)[ZS]>(&sm.win[slot][2 * kChunk * kStride]);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            if (4 * ks >= dsc.y) break;  // k-steps past the chunk's points add zero windows
            const int p = 4 * ks + tq;
            const double wp = __shfl_sync(0xffffffffu, w_cur, p);
            double bz[NZ];
#pragma unroll
            for (int nz = 0; nz < NZ; ++nz) bz[nz] = wp * wz[p][8 * nz + gq];
            const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
            const double xv[2] = {xa.x, xa.y};
            const double ylo = wy[p][gq], yhi = wy[p][8 + gq];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const double am = xv[mt >> 1] * ((mt & 1) ? yhi : ylo);
#pragma unroll
                for (int nz = 0; nz < NZ; ++nz) dmma(S[mt][nz][0], S[mt][nz][1], am, bz[nz]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[slot]);  // this warp is done with the slot
        if (tid == 0 && k + kRingS < nck) {
            // refill the slot once all eight warps released it
            mbar_wait(&sm.empty[slot], (uint32_t)((k / kRingS) & 1));
            fence_proxy_async();
            mbar_expect_tx(&sm.full[slot], kWB);
            bulk_g2s(&sm.win[slot][0], win + (cbeg + k + kRingS) * kWD, kWB, &sm.full[slot]);
        }
        w_cur = w_nxt;
    }
    if (cur_key >= 0) flush();
}

// ---------------------------------------------------------------- spread only, windows on the fly
// For a set that is only ever spread (kernel sums' sources, MMD^2's z = x u y) the window
// block of a chunk is used once: instead of precomputing it (a 15 KB HBM write and read
// per chunk) the CTA evaluates it in shared memory two chunks ahead of the DMMAs — every
// thread 6 of the 1536 taps (degree-14 polynomial per tap, window_fit.h; coefficients in
// shared memory), released by an mbarrier all 256 threads arrive on; the eight warps
// release a slot after their DMMAs (mbarrier, 8 arrivals) and the threads refill it.
// The source weight is folded into the z row (B = w_p Z_p) when the row is evaluated, so
// the DMMA loop forms only the A operand X_p[a] Y_p[b].  kCtasFly3 CTAs per SM (at most
// 85 registers per thread).
constexpr int kRingF = 4, kLeadF = 1;
#ifndef UOTK_DIAG_FLY
#define UOTK_DIAG_FLY 0  // timing diagnostics only: 1 skips the flushes, 2 the tap polynomials, 4 the DMMAs
#endif
// HYB: the set has hybrid groups (z rows 24 columns wide at stride 28, three z n-tiles of
// accumulators); one-cell sets keep 16-tap z rows at stride 20 and two n-tiles
template <bool HYB>
struct __align__(128) SmemF {
    static constexpr int kZS = HYB ? chunk_zstride3(24) : kStride;
    double win[kRingF][2][kChunk][kStride];  // x and y rows
    double winz[kRingF][kChunk][kZS];         // z rows (w_p folded in)
    // even / odd Horner coefficients of tap pair (a, 15 - a), in t^2; a row stride of 10
    // doubles puts the eight pairs' 16-byte reads in distinct banks
    double he[8][10];
    double ho[8][10];
    unsigned long long full[kRingF];
    unsigned long long empty[kRingF];
};

template <bool HYB>
__global__ void __launch_bounds__(kThreads, kCtasFly3)
spread3d_fly_k(const int4* __restrict__ desc, const double* __restrict__ u, const int32_t* __restrict__ key,
               int64_t n, const int32_t* __restrict__ bounds, int ng, double* __restrict__ grid_out,
               const double* __restrict__ w_in, KBHorner hcoef) {
    extern __shared__ __align__(128) unsigned char f_raw[];
    SmemF<HYB>& sm = *reinterpret_cast<SmemF<HYB>*>(f_raw);
    constexpr int NZT = HYB ? 3 : 2;  // z n-tiles of the accumulators
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int a0 = 2 * warp;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    const int64_t ng2 = (int64_t)ng * ng;
    if (tid == 0) {
        for (int r = 0; r < kRingF; ++r) {
            mbar_init(&sm.full[r], kThreads);
            mbar_init(&sm.empty[r], kThreads / 32);
        }
        mbar_init_fence();
    }
    if (tid < 64) {
        const int fa = tid >> 3, q = tid & 7;
        sm.he[fa][q] = hcoef.c[fa][2 * q];
        sm.ho[fa][q] = q < kHornerDeg / 2 ? hcoef.c[fa][2 * q + 1] : 0.0;
    }
    __syncthreads();
    // this thread's taps of a block: the mirror pair a = tid & 7 and 15 - a (phi is even, so
    // phi at tap 15 - a is tap a's polynomial at -t: the even and odd halves in t^2 give
    // both, 15 FMA per pair instead of 28) of point p = tid >> 3, all three axes
    // lanes 0-15 of a warp take rows r, r + 2 and lanes 16-31 rows r + 1, r + 3 of its four:
    // each half-warp's 8-byte stores then hit 16 distinct bank pairs (row stride 20)
    const int fa = tid & 7, frow = 4 * warp + 2 * ((lane >> 3) & 1) + (lane >> 4);
    // the coordinates and the weight of the next block to fill are loaded one fill ahead
    // (their L2 latency then overlaps a chunk of DMMAs instead of stalling the fill)
    double uf[3], wf = 0.0;
    int cntf = 0, offf = 0;
    bool segf = false;
    auto load_rows = [&](int64_t j) {
        const int4 dj = j < nck ? desc[cbeg + j] : make_int4(0, 0, 0, 0);
        cntf = dj.y;
        segf = HYB && (dj.z & kSegFlag) != 0;
        const bool live = frow < dj.y;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) uf[ax] = live ? u[(int64_t)ax * n + dj.x + frow] : 0.0;
        wf = live ? w_in[dj.x + frow] : 0.0;
        // a segment group's key is its first cell's: the point's z offset in the segment
        offf = (live && segf) ? key[dj.x + frow] - (dj.z & ~kSegFlag) : 0;
    };
    auto fill = [&](int64_t j) {
        const int slot = (int)(j % kRingF);
        double t[3];
        const int cnt = cntf;
        const double w = wf;
        const int off = offf;
        const bool seg = segf;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) t[ax] = uf[ax] - floor(uf[ax]) - 0.5;
        load_rows(j + 1);
        if (j >= kRingF) mbar_wait(&sm.empty[slot], (uint32_t)(((j - kRingF) / kRingF) & 1));
        if ((UOTK_DIAG_FLY & 2) == 0 && frow < cnt) {
            double t2[3], e[3], o[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                t2[ax] = t[ax] * t[ax];
                e[ax] = sm.he[fa][kHornerDeg / 2];
                o[ax] = sm.ho[fa][kHornerDeg / 2 - 1];
            }
#pragma unroll
            for (int q = kHornerDeg / 2 - 1; q >= 0; --q) {
                const double ce = sm.he[fa][q];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) e[ax] = fma(e[ax], t2[ax], ce);
            }
#pragma unroll
            for (int q = kHornerDeg / 2 - 2; q >= 0; --q) {
                const double co = sm.ho[fa][q];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) o[ax] = fma(o[ax], t2[ax], co);
            }
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                double v1 = fma(t[ax], o[ax], e[ax]);
                double v2 = fma(-t[ax], o[ax], e[ax]);
                if (ax == 2) {  // B = w_p Z_p, the 16 taps at the point's offset in the row
                    sm.winz[slot][frow][off + fa] = v1 * w;
                    sm.winz[slot][frow][off + kChunkT - 1 - fa] = v2 * w;
                } else {
                    sm.win[slot][ax][frow][fa] = v1;
                    sm.win[slot][ax][frow][kChunkT - 1 - fa] = v2;
                }
            }
        } else {
#pragma unroll
            for (int ax = 0; ax < 2; ++ax) {
                sm.win[slot][ax][frow][fa] = 0.0;
                sm.win[slot][ax][frow][kChunkT - 1 - fa] = 0.0;
            }
            sm.winz[slot][frow][off + fa] = 0.0;
            sm.winz[slot][frow][off + kChunkT - 1 - fa] = 0.0;
        }
        // a segment row's 8 columns outside the taps ([0, off) and [off + 16, 24)): one per thread
        if (HYB && seg) sm.winz[slot][frow][fa < off ? fa : fa + kChunkT] = 0.0;
        mbar_arrive(&sm.full[slot]);
    };
    load_rows(0);
    for (int64_t j = 0; j < kLeadF && j < nck; ++j) fill(j);

    double S[4][NZT][2];  // [m-tile][z n-tile][2]: n-tile 2 only for segment groups (24 z columns)
    int32_t cur_key = -1;
    int64_t gorg = 0;
    auto origin = [&](int32_t kk) -> int64_t {
        if (HYB) kk &= ~kSegFlag;
        const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
        return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
    };
    auto flush = [&]() {
        if (UOTK_DIAG_FLY & 1) {  // keep the accumulators alive without the atomics
            double acc = 0.0;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nz = 0; nz < 2; ++nz) acc += S[mt][nz][0] + S[mt][nz][1];
            acc += S[0][NZT - 1][0];
            if (acc == -1.2345e300) grid_out[0] = acc;
            return;
        }
        const int nzt = (HYB && (cur_key & kSegFlag)) ? 3 : 2;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int64_t row = gorg + (int64_t)(a0 + (mt >> 1)) * ng2 + (int64_t)(8 * (mt & 1) + gq) * ng;
#pragma unroll
            for (int nz = 0; nz < NZT; ++nz)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (nz < nzt && S[mt][nz][i] != 0.0) atomicAdd(grid_out + row + 8 * nz + 2 * tq + i, S[mt][nz][i]);
        }
    };
    int4 d0 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);
    for (int64_t k = 0; k < nck; ++k) {
        const int slot = (int)(k % kRingF);
        const int4 dsc = d0;
        if (k + 1 < nck) d0 = desc[cbeg + k + 1];
        if (k + kLeadF < nck) fill(k + kLeadF);  // windows of a later chunk while this one's are ready
        if (dsc.z != cur_key) {
            if (cur_key >= 0) flush();
            cur_key = dsc.z;
            gorg = origin(cur_key);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nz = 0; nz < NZT; ++nz) S[mt][nz][0] = S[mt][nz][1] = 0.0;
        }
        mbar_wait(&sm.full[slot], (uint32_t)((k / kRingF) & 1));
        const double(*wx)[kStride] = sm.win[slot][0];
        const double(*wy)[kStride] = sm.win[slot][1];
        const double(*wz)[SmemF<HYB>::kZS] = sm.winz[slot];
        // k-steps past the chunk's points add zero windows and are skipped.  A full chunk runs
        // its eight steps without a branch, so the compiler can load the operands of later
        // steps while the DMMAs of earlier ones run; a partial chunk stops after its last
        // occupied step.
        auto kstep = [&](int ks, auto nzt) {
            constexpr int NZ = decltype(nzt)::value;
            const int p = 4 * ks + tq;
            double bz[NZ];
#pragma unroll
            for (int nz = 0; nz < NZ; ++nz) bz[nz] = wz[p][8 * nz + gq];
            const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
            const double xv[2] = {xa.x, xa.y};
            const double ylo = wy[p][gq], yhi = wy[p][8 + gq];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const double am = xv[mt >> 1] * ((mt & 1) ? yhi : ylo);
#pragma unroll
                for (int nz = 0; nz < NZ; ++nz) dmma(S[mt][nz][0], S[mt][nz][1], am, bz[nz]);
            }
        };
        auto ksteps = [&](auto nzt) {
            if (dsc.y == kChunk) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) kstep(ks, nzt);
            } else {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    if (4 * ks >= dsc.y) break;
                    kstep(ks, nzt);
                }
            }
        };
        if (UOTK_DIAG_FLY & 4) {
        } else if (HYB && (dsc.z & kSegFlag)) {
            ksteps(std::integral_constant<int, NZT>{});
        } else {
            ksteps(std::integral_constant<int, 2>{});
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[slot]);  // this warp is done with the slot
    }
    if (cur_key >= 0) flush();
}

// ---------------------------------------------------------------- gather only, ring
// The forward NFFT alone (kernel sums' targets): per chunk every warp contracts its
// a-pair and writes 32 partial sums; the warp k mod 8 waits for all eight (mbarrier),
// reduces, applies the epilogue and — the slot being free then — refills it by TMA.
// No CTA barrier; the reduction duty rotates over the warps.
constexpr int kRingG = 4;
template <int KZ>
struct __align__(128) SmemG {
    double win[kRingG][chunk_win3_doubles(KZ)];
    double red[kRingG][kThreads / 32][kChunk];
    unsigned long long full[kRingG];
    unsigned long long red_full[kRingG];
};

template <int KZ, class Epi>
__global__ void __launch_bounds__(kThreads, kBlocksPerSM)
gather3d_k(const int4* __restrict__ desc, const double* __restrict__ win, const int32_t* __restrict__ bounds, int ng,
           const double* __restrict__ grid_in, Epi epi) {
    constexpr int KS = KZ / 4;
    constexpr int ZS = chunk_zstride3(KZ);
    constexpr int kWD = chunk_win3_doubles(KZ);
    constexpr uint32_t kWB = kWD * sizeof(double);
    constexpr int kW = kThreads / 32;
    extern __shared__ __align__(128) unsigned char g_raw[];
    SmemG<KZ>& sm = *reinterpret_cast<SmemG<KZ>*>(g_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gq = lane >> 2;
    const int tq = lane & 3;
    const int a0 = 2 * warp;
    const int64_t cbeg = bounds[blockIdx.x];
    const int64_t nck = bounds[blockIdx.x + 1] - cbeg;
    const int64_t ng2 = (int64_t)ng * ng;
    if (tid == 0) {
        for (int r = 0; r < kRingG; ++r) {
            mbar_init(&sm.full[r], 1);
            mbar_init(&sm.red_full[r], kW);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < kRingG && k < nck; ++k) {
            mbar_expect_tx(&sm.full[k], kWB);
            bulk_g2s(&sm.win[k][0], win + (cbeg + k) * kWD, kWB, &sm.full[k]);
        }
    }
    auto origin = [&](int32_t kk) -> int64_t {
        const int k2 = kk % ng, k1 = (kk / ng) % ng, k0 = kk / ng2;
        return ((int64_t)(k0 - kM + 1) * ng + (k1 - kM + 1)) * ng + (k2 - kM + 1);
    };
    double Fb[4][KS];
    int32_t cur_key = -1;
    int4 d0 = nck > 0 ? desc[cbeg] : make_int4(0, 0, -1, 0);
    int4 d1 = nck > 1 ? desc[cbeg + 1] : make_int4(0, 0, -1, 0);
    for (int64_t k = 0; k < nck; ++k) {
        const int slot = (int)(k % kRingG);
        const int4 dsc = d0;
        d0 = d1;
        if (k + 2 < nck) d1 = desc[cbeg + k + 2];
        if (dsc.z != cur_key) {
            cur_key = dsc.z;
            const int64_t gorg = origin(cur_key);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int64_t row = gorg + (int64_t)(a0 + (nt >> 1)) * ng2 + (int64_t)(8 * (nt & 1) + gq) * ng;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) Fb[nt][ks] = __ldg(grid_in + row + 4 * ks + tq);
            }
        }
        if (k + 1 < nck && d0.z != cur_key) {  // warm L1 with the next group's footprint
            const int64_t norg = origin(d0.z);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const double* rowp = grid_in + norg + (int64_t)(a0 + (nt >> 1)) * ng2 + (int64_t)(8 * (nt & 1) + gq) * ng;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(rowp + 4 * tq));
            }
        }
        mbar_wait(&sm.full[slot], (uint32_t)((k / kRingG) & 1));
        const double(*wx)[kStride] = reinterpret_cast<const double(*)[kStride]>(&sm.win[slot][0]);
        const double(*wy)[kStride] = wx + kChunk;
        const double(*wz)[ZS] = reinterpret_cast<const double(*)[ZS]>(&sm.win[slot][2 * kChunk * kStride]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            if (8 * mt >= dsc.y) break;  // m-tiles past the chunk's points hold no point
            const int p = 8 * mt + gq;
            double acc[4][2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const double az = wz[p][4 * ks + tq];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], az, Fb[nt][ks]);
            }
            const double2 ylo = *reinterpret_cast<const double2*>(&wy[p][2 * tq]);
            const double2 yhi = *reinterpret_cast<const double2*>(&wy[p][8 + 2 * tq]);
            const double2 xa = *reinterpret_cast<const double2*>(&wx[p][a0]);
            const double xv[2] = {xa.x, xa.y};
            double part = 0.0;
#pragma unroll
            for (int al = 0; al < 2; ++al) {
                double q = acc[2 * al][0] * ylo.x;
                q = fma(acc[2 * al][1], ylo.y, q);
                q = fma(acc[2 * al + 1][0], yhi.x, q);
                q = fma(acc[2 * al + 1][1], yhi.y, q);
                part = fma(q, xv[al], part);
            }
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            if (tq == 0) sm.red[slot][warp][p] = part;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.red_full[slot]);
        if (warp == (int)(k % kW)) {
            // reducer of chunk k: all eight partials, the epilogue, then the slot is free
            mbar_wait(&sm.red_full[slot], (uint32_t)((k / kRingG) & 1));
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kW; ++w) t += sm.red[slot][w][lane];
            if (lane < dsc.y) epi(dsc.x + lane, t);
            __syncwarp();
            if (lane == 0 && k + kRingG < nck) {
                fence_proxy_async();
                mbar_expect_tx(&sm.full[slot], kWB);
                bulk_g2s(&sm.win[slot][0], win + (cbeg + k + kRingG) * kWD, kWB, &sm.full[slot]);
            }
        }
    }
}

template <class Epi>
void launch_gather(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi, cudaStream_t s) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    if (ps.chunk_kz == 40) fail(UOTK_EUNSUPPORTED, "internal: gather on a spread-only point set");
    ProfScope prof(kProfGather, s);
    if (ps.chunk_kz == 24) {
        set_smem_attr((const void*)gather3d_k<24, Epi>, (int)sizeof(SmemG<24>));
        gather3d_k<24, Epi><<<ps.chunk_blocks, kThreads, sizeof(SmemG<24>), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                               ps.chunk_bounds.p, fp.ng, grid, epi);
    } else {
        set_smem_attr((const void*)gather3d_k<16, Epi>, (int)sizeof(SmemG<16>));
        gather3d_k<16, Epi><<<ps.chunk_blocks, kThreads, sizeof(SmemG<16>), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                               ps.chunk_bounds.p, fp.ng, grid, epi);
    }
    UOTK_LAUNCHED();
}

template <int MODE, class Epi>
void launch(const PointSet& ps, const double* gin, double* gout, const double* w, const FastParams& fp,
            const Epi& epi, unsigned long long* dmax, cudaStream_t s, int tag) {
    if (ps.n == 0 || ps.nchunks == 0) return;
    if (ps.chunk_kz == 40) fail(UOTK_EUNSUPPORTED, "internal: 25-cell segments on the phase-locked kernels");
    ProfScope prof(tag, s);
    if (ps.chunk_kz == 24)
        chunked3d_k<MODE, Epi, 24><<<ps.chunk_blocks, kThreads, 0, s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                        ps.chunk_bounds.p, ps.nchunks, fp.ng, gin,
                                                                        gout, w, epi, dmax);
    else
        chunked3d_k<MODE, Epi, 16><<<ps.chunk_blocks, kThreads, 0, s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                        ps.chunk_bounds.p, ps.nchunks, fp.ng, gin,
                                                                        gout, w, epi, dmax);
    UOTK_LAUNCHED();
}

}  // namespace

void fused3d_m6_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                              const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s);
void fused3d_m6_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s);
void fused3d_m6_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                             cudaStream_t s);
void fused3d_m6_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                           cudaStream_t s);

void fused3d_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s) {
    if (fp.m == 6) return fused3d_m6_gather_spread(ps, grid_in, grid_out, fp, epi, dmax, s);
    // warp-specialised kernel by default; UOTK_FUSED_WS=0 selects the phase-locked one
    static const bool ws = [] {
        const char* e = getenv("UOTK_FUSED_WS");
        return !(e && e[0] == '0');
    }();
    if (!ws || ps.chunk_kz != 16) {  // z-segment groups (sparse clouds) use the phase-locked kernel
        launch<0, EpiSinkhorn>(ps, grid_in, grid_out, nullptr, fp, epi, dmax, s, kProfFused);
        return;
    }
    if (ps.n == 0 || ps.nchunks == 0) return;
    set_smem_attr((const void*)sinkhorn3d_ws_k, (int)sizeof(SmemWS));
    ProfScope prof(kProfFused, s);
    sinkhorn3d_ws_k<<<ps.chunk_blocks, 256, sizeof(SmemWS), s>>>(ps.chunk_desc.p, ps.chunk_win.p, ps.chunk_bounds.p,
                                                                 fp.ng, grid_in, grid_out, epi, dmax);
    UOTK_LAUNCHED();
}

void fused3d_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    if (fp.m == 6) return fused3d_m6_spread(ps, w, grid, fp, s);
    static const bool ring = [] {
        const char* e = getenv("UOTK_SPREAD_RING");
        return !(e && e[0] == '0');
    }();
    if (!ring && !ps.win_fly) {
        launch<1, EpiNone>(ps, nullptr, grid, w, fp, EpiNone{}, nullptr, s, kProfSpread);
        return;
    }
    if (ps.n == 0 || ps.nchunks == 0) return;
    ProfScope prof(kProfSpread, s);
    if (ps.win_fly) {  // spread-only set without precomputed window blocks (one-cell or hybrid groups)
        auto go = [&](auto hyb) {
            constexpr bool H = decltype(hyb)::value;
            set_smem_attr((const void*)spread3d_fly_k<H>, (int)sizeof(SmemF<H>));
            spread3d_fly_k<H><<<ps.chunk_blocks, kThreads, sizeof(SmemF<H>), s>>>(
                ps.chunk_desc.p, ps.u.p, ps.key.p, ps.n, ps.chunk_bounds.p, fp.ng, grid, w, ps.win_coef);
            UOTK_LAUNCHED();
        };
        if (ps.chunk_kz == kGroupsHybrid) go(std::true_type{});
        else go(std::false_type{});
        return;
    }
    if (ps.chunk_kz == 40) {
        set_smem_attr((const void*)spread3d_k<40>, (int)sizeof(SmemS<40>));
        spread3d_k<40><<<ps.chunk_blocks, kThreads, sizeof(SmemS<40>), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                            ps.chunk_bounds.p, fp.ng, grid, w);
    } else if (ps.chunk_kz == 24) {
        set_smem_attr((const void*)spread3d_k<24>, (int)sizeof(SmemS<24>));
        spread3d_k<24><<<ps.chunk_blocks, kThreads, sizeof(SmemS<24>), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                            ps.chunk_bounds.p, fp.ng, grid, w);
    } else {
        set_smem_attr((const void*)spread3d_k<16>, (int)sizeof(SmemS<16>));
        spread3d_k<16><<<ps.chunk_blocks, kThreads, sizeof(SmemS<16>), s>>>(ps.chunk_desc.p, ps.chunk_win.p,
                                                                            ps.chunk_bounds.p, fp.ng, grid, w);
    }
    UOTK_LAUNCHED();
}

void fused3d_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s) {
    if (fp.m == 6) return fused3d_m6_gather_store(ps, grid, fp, epi, s);
    static const bool ring = [] {
        const char* e = getenv("UOTK_GATHER_RING");
        return !(e && e[0] == '0');
    }();
    if (ring) return launch_gather(ps, grid, fp, epi, s);
    EpiGatherOnly<EpiStore> e;
    static_cast<EpiStore&>(e) = epi;
    launch<2, EpiGatherOnly<EpiStore>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

void fused3d_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s) {
    if (fp.m == 6) return fused3d_m6_gather_dot(ps, grid, fp, epi, s);
    static const bool ring = [] {
        const char* e = getenv("UOTK_GATHER_RING");
        return !(e && e[0] == '0');
    }();
    if (ring) return launch_gather(ps, grid, fp, epi, s);
    EpiGatherOnly<EpiDot> e;
    static_cast<EpiDot&>(e) = epi;
    launch<2, EpiGatherOnly<EpiDot>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

}  // namespace uotk
