// Chunked point layout shared by the tuned cell-group kernels (fused3d.cu, fused12d.cu)
// and their preparation (chunks.cu).
//
// Points are sorted by grid cell (points.cu); every run of equal keys shares one (2m)^d
// window footprint.  Runs are cut into chunks of <= 32 points and the window values of
// every chunk are precomputed once per point set (points do not move between Sinkhorn
// iterations) into a fixed-size block per chunk, zero for empty slots:
//   d = 3: [axis 3][slot 32][tap, row stride 20]      (padded: conflict-free fragments);
//          z-segment groups: X, Y as above, Z [slot 32][24 placed taps, row stride 28]
//   d = 2: [axis 2][slot 32][16 taps, swizzled]       (tap a of slot p at (a + 4p) & 15)
//   d = 1: [slot 32][16 taps]                          (each lane reads its own row)
#pragma once
#include <cstdint>

namespace uotk {

constexpr int kChunkM = 8;              // window half-width of the tuned kernels
constexpr int kChunkT = 2 * kChunkM;    // taps per axis
constexpr int kChunk = 32;              // points per chunk
constexpr int kStride3 = 20;            // d = 3 padded row stride (doubles)
// work units of the kernels: d = 3 one CTA (8 warps) per unit, kCtas3 CTAs per SM;
// d <= 2 one warp per unit, kWarpsD warps per CTA, kCtasD CTAs per SM
constexpr int kCtas3 = 2;
// d = 3 spread-only sets with windows evaluated in the spread (fused3d.cu spread3d_fly_k)
constexpr int kCtasFly3 = 2;
constexpr int kWarps2 = 3, kCtas2 = 3;
constexpr int kWarps1 = 8, kCtas1 = 2;
// d = 2 warp-specialised Sinkhorn half-step: units of 2 gather warps + 1 spread warp,
// kUnitsWS2 units per CTA, kCtasWS2 CTAs per SM, its own chunk partition
constexpr int kUnitsWS2 = 2, kCtasWS2 = 2;
// d = 3, m = 6 (fused3d_m6.cu): stand-alone spread/gather CTAs of 3 warps, kCtas3M6 per SM
// (chunk_bounds); warp-specialised half-step CTAs of 3 + 3 warps, kCtasWS3M6 per SM (chunk_bounds_ws)
constexpr int kCtas3M6 = 5, kCtasWS3M6 = 3;
__host__ __device__ constexpr int chunk_units_per_sm(int d) {
    return d == 3 ? kCtas3 : (d == 2 ? kWarps2 * kCtas2 : kWarps1 * kCtas1);
}

// d = 3 z-column segments (sparse clouds): a group spans kSegZ cells along z, the
// footprint is 16 x 16 x KZ with KZ = 24 >= 15 + kSegZ, and each point's 16 z-taps are
// placed at its cell's offset in a KZ-wide row (stride 28: conflict-free fragments)
constexpr int kSegZ = 9;
// spread-only sets sparser still (kernel-sum sources, MMD^2): segments of 25 cells,
// footprint 16 x 16 x 40 — the group flushes (fp64 atomics), not the DMMAs, bind there
constexpr int kSegZ40 = 25;
// hybrid groups (d = 3 spread-only sets whose windows the spread evaluates, spread3d_fly_k):
// cells with at least kHybridMin points stay one-cell groups (16 x 16 x 16 footprints), the
// sparser cells of a kSegZ z-segment share a 16 x 16 x 24 footprint; the group key of such
// a segment is its first cell's key with kSegFlag set (keys < 2^30)
constexpr int kHybridMin = 24;
constexpr int32_t kSegFlag = 1 << 30;
constexpr int kGroupsHybrid = 1624;  // uotk_info.groups code of the hybrid layout
// KZ = 12: the one-cell layout of m = 6 (fused3d_m6.cu): all three axes [slot 32][12 taps],
// row stride 12 (no padding; 9 KB per chunk)
__host__ __device__ constexpr int chunk_zstride3(int kz) {
    return kz == 12 ? 12 : (kz == 16 ? kStride3 : (kz == 24 ? 28 : 44));
}
__host__ __device__ constexpr int chunk_xstride3(int kz) { return kz == 12 ? 12 : kStride3; }
__host__ __device__ constexpr int chunk_win3_doubles(int kz) {
    return kChunk * (2 * chunk_xstride3(kz) + chunk_zstride3(kz));
}

__host__ __device__ constexpr int chunk_win_doubles(int d) {
    return d == 3 ? chunk_win3_doubles(16) : d * kChunk * kChunkT;
}

// d = 2 y-segments (sparse clouds, e.g. C4's literal 4096^2 grid at ~5 points per cell):
// kSegY cells along y share one 16 x 24 footprint; X rows as for one cell (16 swizzled
// taps), Y rows 24 columns wide at stride 28 (conflict-free fragments), the 16 taps at the
// point's cell offset in the segment
constexpr int kSegY = 9;
__host__ __device__ constexpr int chunk_ystride2(int ky) { return ky == 16 ? kChunkT : 28; }
__host__ __device__ constexpr int chunk_win2_doubles(int ky) { return kChunk * (kChunkT + chunk_ystride2(ky)); }

// d = 3 stand-alone gathers on sets whose chunks are filled below this fraction use the
// generic per-point kernel (its per-point loads beat the padded GEMMs there; nfft.cu), and
// gather-only sets that sparse get no chunk list at all (chunks.cu)
constexpr double kGatherMinFill3 = 0.3;

// d = 2 swizzle: column of tap a in slot row p
__host__ __device__ __forceinline__ int swz2(int p, int a) { return (a + 4 * p) & 15; }

}  // namespace uotk
