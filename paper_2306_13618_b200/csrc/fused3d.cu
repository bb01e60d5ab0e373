// Tuned d = 3 NFFT passes.
//
// Points are sorted by grid cell (points.cu), so every run of equal keys shares one
// (2m)^3 window footprint on the oversampled grid.  A 128-thread CTA walks a
// contiguous range of sorted points; for each cell group the threads own fixed
// footprint columns (b, c) x all 2m values of a, so that
//   gather  (outer sum of (4.6)):  t_p = sum_abc g[a,b,c] X_p[a] Y_p[b] Z_p[c]
//   spread  (inner sum of (4.6)):  S[a,b,c] += w_p X_p[a] Y_p[b] Z_p[c]
// are register-blocked FMA loops over a chunk of <= 32 points whose window values sit
// in shared memory (broadcast reads).  The per-point partial gathers are reduced
// with a transposing warp butterfly and a 4-warp shared-memory sum, the Sinkhorn
// update (3.3)/(3.4) runs on the reduced t_p, and the new weight w_p = mass_p u_p is
// spread into registers immediately — one pass over the points per half-step, the
// grid footprint read once and flushed once (fp64 RED) per cell group.
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "window.cuh"

namespace uotk {

namespace {

constexpr int kThreads = 128;  // 4 warps; thread t owns columns (b, c) = (t>>4, t&15) and (b+8, c)
constexpr int kChunk = 32;     // points per chunk (one per lane in the butterfly)

template <int M>
struct Smem {
    static constexpr int T = 2 * M;
    double wx[kChunk][T];  // window along axis 0 (a)
    double wy[kChunk][T];  // axis 1 (b)
    double wz[kChunk][T];  // axis 2 (c)
    double wn[kChunk];     // spread weight of the chunk's points
    double red[kThreads / 32][kChunk];
};

// MODE: 0 = gather -> epilogue -> spread (Sinkhorn half-step), 1 = spread only, 2 = gather only
template <int M, int MODE, class Epi>
__global__ void __launch_bounds__(kThreads, 2)
cellgroup3d_k(const double* __restrict__ u, const int32_t* __restrict__ keys, int64_t n, int ng, KBWindow win,
              const double* __restrict__ grid_in, double* __restrict__ grid_out, const double* __restrict__ w_in,
              Epi epi, unsigned long long* dmax) {
    constexpr int T = 2 * M;          // taps per axis
    constexpr int NJ = T * T / kThreads;  // owned (b, c) columns per thread (2 for m = 8)
    constexpr bool GATHER = MODE != 1;
    constexpr bool SPREAD = MODE != 2;
    static_assert(T * T % kThreads == 0 || T * T < kThreads, "footprint / thread mapping");
    __shared__ __align__(16) Smem<M> sm;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // column ownership
    int cb[NJ > 0 ? NJ : 1], cc;
    cc = tid % T;
#pragma unroll
    for (int j = 0; j < NJ; ++j) cb[j] = tid / T + j * (kThreads / T);

    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t pb = (int64_t)blockIdx.x * per;
    const int64_t p_begin = pb < n ? pb : n;
    const int64_t p_end = p_begin + per < n ? p_begin + per : n;
    const double* u0 = u;
    const double* u1 = u + n;
    const double* u2 = u + 2 * n;
    const int64_t ng2 = (int64_t)ng * ng;

    double g[NJ][T];   // footprint values of the current group (gather source)
    double s[NJ][T];   // spread accumulators of the current group
    int32_t cur_key = -1;
    int64_t gbase = 0;  // linear index of footprint origin (a = b = c = 0)
    double ddmax = 0.0;

    auto flush = [&]() {
        if (SPREAD && cur_key >= 0) {
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int64_t col = gbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
                for (int a = 0; a < T; ++a)
                    if (s[j][a] != 0.0) atomicAdd(grid_out + col + a * ng2, s[j][a]);
            }
        }
    };

    for (int64_t p0 = p_begin; p0 < p_end;) {
        // ---- chunk = up to 32 points of one cell group (keys are sorted)
        const int32_t key = keys[p0];
        const bool same = (p0 + lane < p_end) && keys[p0 + lane] == key;
        const unsigned mask = __ballot_sync(0xffffffffu, same);
        const int cnt = (mask == 0xffffffffu) ? 32 : (__ffs(~mask) - 1);

        if (key != cur_key) {
            flush();
            cur_key = key;
            const int c2 = key % ng;
            const int c1 = (key / ng) % ng;
            const int c0 = key / ng2;
            gbase = ((int64_t)(c0 - M + 1) * ng + (c1 - M + 1)) * ng + (c2 - M + 1);
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int64_t col = gbase + (int64_t)cb[j] * ng + cc;
#pragma unroll
                for (int a = 0; a < T; ++a) {
                    if (GATHER) g[j][a] = grid_in[col + a * ng2];
                    if (SPREAD) s[j][a] = 0.0;
                }
            }
        }

        // ---- window values of the chunk (zero for unused slots)
        for (int e = tid; e < kChunk * 3 * T; e += kThreads) {
            const int p = e / (3 * T);
            const int r = e - p * 3 * T;
            const int ax = r / T;
            const int a = r - ax * T;
            double val = 0.0;
            if (p < cnt) {
                const double ut = (ax == 0 ? u0 : (ax == 1 ? u1 : u2))[p0 + p];
                const double f = ut - floor(ut);
                val = kb_phi(f + (double)(M - 1 - a), win);
            }
            if (ax == 0) sm.wx[p][a] = val;
            else if (ax == 1) sm.wy[p][a] = val;
            else sm.wz[p][a] = val;
        }
        if (!GATHER) {
            if (tid < kChunk) sm.wn[tid] = tid < cnt ? w_in[p0 + tid] : 0.0;
        }
        __syncthreads();

        if (GATHER) {
            // ---- partial gathers, one per point slot
            double r[kChunk];
#pragma unroll
            for (int p = 0; p < kChunk; ++p) {
                double acc[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    double e0 = 0.0, e1 = 0.0;
#pragma unroll
                    for (int a = 0; a < T; a += 2) {
                        const double2 xv = *reinterpret_cast<const double2*>(&sm.wx[p][a]);
                        e0 = fma(g[j][a], xv.x, e0);
                        e1 = fma(g[j][a + 1], xv.y, e1);
                    }
                    acc[j] = (e0 + e1) * sm.wy[p][cb[j]];
                }
                double v = acc[0];
#pragma unroll
                for (int j = 1; j < NJ; ++j) v += acc[j];
                r[p] = v * sm.wz[p][cc];
            }
            // ---- transposing butterfly: lane l ends with the warp sum for slot l
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) {
                const bool upper = lane & sh;
#pragma unroll
                for (int k = 0; k < sh; ++k) {
                    const double send = upper ? r[k] : r[k + sh];
                    const double keep = upper ? r[k + sh] : r[k];
                    r[k] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
                }
            }
            sm.red[warp][lane] = r[0];
            __syncthreads();
            if (warp == 0) {
                double dd = 0.0;
                double wn = 0.0;
                if (lane < cnt) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < kThreads / 32; ++w) t += sm.red[w][lane];
                    dd = epi(p0 + lane, t);
                    if (SPREAD) wn = epi.w_next[p0 + lane];
                }
                if (SPREAD) sm.wn[lane] = wn;
                ddmax = fmax(ddmax, dd);
            }
            __syncthreads();
        }

        if (SPREAD) {
#pragma unroll 4
            for (int p = 0; p < kChunk; ++p) {
                const double wz = sm.wn[p] * sm.wz[p][cc];
                double wj[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) wj[j] = wz * sm.wy[p][cb[j]];
#pragma unroll
                for (int a = 0; a < T; a += 2) {
                    const double2 xv = *reinterpret_cast<const double2*>(&sm.wx[p][a]);
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        s[j][a] = fma(wj[j], xv.x, s[j][a]);
                        s[j][a + 1] = fma(wj[j], xv.y, s[j][a + 1]);
                    }
                }
            }
        }
        __syncthreads();  // window buffers are rewritten by the next chunk
        p0 += cnt;
    }
    flush();
    if (GATHER && warp == 0) warp_max_atomic(dmax, ddmax);
}

// The Sinkhorn epilogue exposes w_next; the plain gathers do not spread.
struct EpiNone {
    double* w_next = nullptr;
    __device__ double operator()(int64_t, double) const { return 0.0; }
};

template <int M, int MODE, class Epi>
void launch(const PointSet& ps, const double* gin, double* gout, const double* w, const FastParams& fp,
            const Epi& epi, unsigned long long* dmax, cudaStream_t s, int tag) {
    if (ps.n == 0) return;
    KBWindow win = make_window(fp.b, M);
    int blocks = 148 * 2;
    const int64_t min_per = 64;
    if (ps.n < (int64_t)blocks * min_per) blocks = (int)std::max<int64_t>(1, (ps.n + min_per - 1) / min_per);
    ProfScope prof(tag, s);
    cellgroup3d_k<M, MODE, Epi><<<blocks, kThreads, 0, s>>>(ps.u.p, ps.key.p, ps.n, fp.ng, win, gin, gout, w, epi,
                                                            dmax);
    UOTK_LAUNCHED();
}

}  // namespace

bool fused3d_available(const FastParams& fp) { return fp.d == 3 && fp.m == 8; }

void fused3d_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s) {
    launch<8, 0, EpiSinkhorn>(ps, grid_in, grid_out, nullptr, fp, epi, dmax, s, kProfFused);
}

void fused3d_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    launch<8, 1, EpiNone>(ps, nullptr, grid, w, fp, EpiNone{}, nullptr, s, kProfSpread);
}

template <class Epi>
struct EpiGatherOnly : Epi {
    double* w_next = nullptr;
};

void fused3d_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s) {
    EpiGatherOnly<EpiStore> e;
    static_cast<EpiStore&>(e) = epi;
    launch<8, 2, EpiGatherOnly<EpiStore>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

void fused3d_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s) {
    EpiGatherOnly<EpiDot> e;
    static_cast<EpiDot&>(e) = epi;
    launch<8, 2, EpiGatherOnly<EpiDot>>(ps, grid, nullptr, nullptr, fp, e, nullptr, s, kProfGather);
}

}  // namespace uotk
