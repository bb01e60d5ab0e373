// Deterministic spread (uotk_opts.deterministic; DESIGN.md §7 "Deterministic mode"):
// the adjoint NFFT g_l = sum_j w_j prod_t phi(u_jt - l_t) (inner sum of (4.6))
// computed by PULLING at each grid point instead of pushing with fp64 atomics, so every
// g_l is summed in one fixed order — the points' cell-key order — whatever the launch
// configuration or scheduling: results are bitwise reproducible.
//
// One CTA per T^d tile of the footprint box.  The cells whose points reach the tile are
// the (T + 2m - 1)^d halo cells; with the points sorted by cell key (x-major), the halo
// cells of one (x[, y]) row form one contiguous point range, found by binary search.  The
// rows are visited in lexicographic order and their points in sorted order, in batches
// whose window values (d x 2m per point) are evaluated once into shared memory.
#include "common.cuh"
#include "profile.cuh"
#include "window.cuh"

namespace uotk {

namespace {

__device__ __forceinline__ int64_t lower_bound_key(const int32_t* __restrict__ key, int64_t n, int32_t k) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <int D>
struct PullCfg;
template <>
struct PullCfg<1> {
    static constexpr int T = 256;
};
template <>
struct PullCfg<2> {
    static constexpr int T = 16;
};
template <>
struct PullCfg<3> {
    static constexpr int T = 8;
};

template <int D, int M>
__global__ void __launch_bounds__(256 * (D == 3 ? 2 : 1))
    spread_pull_k(const double* __restrict__ u, const int32_t* __restrict__ key, const double* __restrict__ w,
                  int64_t n, int ng, int box_lo, int box_w, KBWindow win, double* __restrict__ grid) {
    constexpr int T = PullCfg<D>::T;
    constexpr int NT = D == 1 ? T : (D == 2 ? T * T : T * T * T);
    constexpr int H = T + 2 * M - 1;              // halo cells per axis
    constexpr int ROWS = D == 1 ? 1 : (D == 2 ? H : H * H);
    constexpr int B = 32;                         // points per batch
    __shared__ int64_t row_lo[ROWS], row_hi[ROWS];
    __shared__ double W[B][D][2 * M];
    __shared__ int base[B][D];
    __shared__ double wb[B];

    const int ntile = (box_w + T - 1) / T;
    int tl[3] = {0, 0, 0};
    {
        int b = blockIdx.x;
        for (int t = D - 1; t >= 0; --t) {
            tl[t] = box_lo + (b % ntile) * T;
            b /= ntile;
        }
    }
    // this thread's grid point
    int l[3] = {0, 0, 0};
    {
        int r = threadIdx.x;
        for (int t = D - 1; t >= 0; --t) {
            l[t] = tl[t] + r % T;
            r /= T;
        }
    }
    bool live = true;
    for (int t = 0; t < D; ++t) live = live && l[t] < box_lo + box_w;

    // halo cell range along each axis: cells c with c in [l - M, l + M - 1] for some l in the tile
    int c0[3], c1[3];
    for (int t = 0; t < D; ++t) {
        c0[t] = max(0, tl[t] - M);
        c1[t] = min(ng - 1, tl[t] + T - 1 + M - 1);
    }
    // contiguous point range of each row of halo cells (last axis runs contiguously)
    for (int r = threadIdx.x; r < ROWS; r += NT) {
        int64_t lo = 0, hi = 0;
        if (D == 1) {
            lo = lower_bound_key(key, n, c0[0]);
            hi = lower_bound_key(key, n, c1[0] + 1);
        } else {
            int cx = 0, cy = 0;
            bool ok;
            if (D == 2) {
                cx = c0[0] + r;
                ok = cx <= c1[0];
            } else {
                cx = c0[0] + r / H;
                cy = c0[1] + r % H;
                ok = cx <= c1[0] && cy <= c1[1];
            }
            if (ok) {
                const int32_t pre = D == 2 ? cx * ng : (cx * ng + cy) * ng;
                lo = lower_bound_key(key, n, pre + c0[D - 1]);
                hi = lower_bound_key(key, n, pre + c1[D - 1] + 1);
            }
        }
        row_lo[r] = lo;
        row_hi[r] = hi;
    }
    __syncthreads();

    double acc = 0.0;
    for (int r = 0; r < ROWS; ++r) {
        const int64_t p0 = row_lo[r], p1 = row_hi[r];  // uniform over the block
        for (int64_t pb = p0; pb < p1; pb += B) {
            const int cnt = (int)min((int64_t)B, p1 - pb);
            // window values of the batch: W[p][t][a] = phi(f + M - 1 - a), taps from cell - M + 1
            for (int e = threadIdx.x; e < cnt * D * 2 * M; e += NT) {
                const int p = e / (D * 2 * M), rem = e % (D * 2 * M), t = rem / (2 * M), a = rem % (2 * M);
                const double ut = u[(int64_t)t * n + pb + p];
                const double fl = floor(ut);
                W[p][t][a] = kb_phi(ut - fl + (M - 1 - a), win);
                if (a == 0) base[p][t] = (int)fl + ng / 2 - M + 1;
            }
            for (int p = threadIdx.x; p < cnt; p += NT) wb[p] = w[pb + p];
            __syncthreads();
            if (live) {
                for (int p = 0; p < cnt; ++p) {
                    double v = wb[p];
                    bool in = true;
#pragma unroll
                    for (int t = 0; t < D; ++t) {
                        const int a = l[t] - base[p][t];
                        in = in && a >= 0 && a < 2 * M;
                        v *= W[p][t][min(max(a, 0), 2 * M - 1)];
                    }
                    if (in) acc += v;
                }
            }
            __syncthreads();
        }
    }
    if (live) {
        int64_t gi = 0;
        for (int t = 0; t < D; ++t) gi = gi * ng + l[t];
        grid[gi] = acc;
    }
}

template <int D, int M>
void launch_pull(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    constexpr int T = PullCfg<D>::T;
    constexpr int NT = D == 1 ? T : (D == 2 ? T * T : T * T * T);
    const int ntile = (fp.box_w + T - 1) / T;
    int64_t blocks = 1;
    for (int t = 0; t < D; ++t) blocks *= ntile;
    KBWindow win = make_window(fp.b, M);
    ProfScope ps_(kProfSpread, s);
    spread_pull_k<D, M><<<(unsigned)blocks, NT, 0, s>>>(ps.u.p, ps.key.p, w, ps.n, fp.ng, fp.box_lo, fp.box_w, win,
                                                       grid);
    UOTK_LAUNCHED();
}

}  // namespace

// g = adjoint NFFT of w at the (sorted) point set, written (not added) on the footprint box;
// the caller zeroes the grid outside it as for every spread
void spread_deterministic(const PointSet& ps, const double* w_sorted, double* grid, const FastParams& fp,
                          cudaStream_t s) {
    if (ps.n == 0) return;
    switch (fp.d * 16 + fp.m) {
#define UOTK_PULL(DD, MM) \
    case DD * 16 + MM: launch_pull<DD, MM>(ps, w_sorted, grid, fp, s); break;
        UOTK_PULL(1, 2) UOTK_PULL(1, 3) UOTK_PULL(1, 4) UOTK_PULL(1, 5) UOTK_PULL(1, 6) UOTK_PULL(1, 7) UOTK_PULL(1, 8)
        UOTK_PULL(2, 2) UOTK_PULL(2, 3) UOTK_PULL(2, 4) UOTK_PULL(2, 5) UOTK_PULL(2, 6) UOTK_PULL(2, 7) UOTK_PULL(2, 8)
        UOTK_PULL(3, 2) UOTK_PULL(3, 3) UOTK_PULL(3, 4) UOTK_PULL(3, 5) UOTK_PULL(3, 6) UOTK_PULL(3, 7) UOTK_PULL(3, 8)
#undef UOTK_PULL
        default: fail(UOTK_EINVAL, "unsupported (d, m)");
    }
}

}  // namespace uotk
