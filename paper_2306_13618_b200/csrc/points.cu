// Point preparation (K1/K1b): bounding geometry, scaling into the torus (Eq. 4.7,
// P:594-596; Rem. 4.3 P:610), cell keys, radix sort by cell, permutations.
#include <cub/cub.cuh>

#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "profile.cuh"

namespace uotk {

void comm_allreduce_minmax(double* dmin, int nmin, double* dmax, int nmax, void* comm, cudaStream_t s);  // comm.cu
void chunked_prepare(PointSet& ps, const FastParams& fp, cudaStream_t s, PointUse use);  // chunks.cu

namespace {

constexpr int kGeomBlocks = 592;  // 4 x 148 SMs
constexpr int kGeomThreads = 256;

// per-block partial min / max per axis, plus a non-finite flag (as max)
// the last block to finish (a ticket on *done) reduces every block's partials into the
// final value and resets the ticket: no separate final launch.  min / max are exact in any
// order, so the result equals the two-launch reduction's.
__device__ __forceinline__ bool last_block(unsigned* done) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

template <int D>
__global__ void bbox_k(const double* __restrict__ p1, int64_t n1, const double* __restrict__ p2, int64_t n2,
                       double* __restrict__ pmin, double* __restrict__ pmax, double* out_min, double* out_max,
                       unsigned* done) {
    double lo[D], hi[D];
    double bad = 0;
    for (int t = 0; t < D; ++t) { lo[t] = DBL_MAX; hi[t] = -DBL_MAX; }
    const int64_t total = n1 + n2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const double* q = i < n1 ? p1 + i * D : p2 + (i - n1) * D;
        for (int t = 0; t < D; ++t) {
            double v = q[t];
            if (!isfinite(v)) bad = 1;
            else { lo[t] = fmin(lo[t], v); hi[t] = fmax(hi[t], v); }
        }
    }
    __shared__ double smin[D][kGeomThreads], smax[D + 1][kGeomThreads];
    for (int t = 0; t < D; ++t) { smin[t][threadIdx.x] = lo[t]; smax[t][threadIdx.x] = hi[t]; }
    smax[D][threadIdx.x] = bad;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            for (int t = 0; t < D; ++t) {
                smin[t][threadIdx.x] = fmin(smin[t][threadIdx.x], smin[t][threadIdx.x + w]);
                smax[t][threadIdx.x] = fmax(smax[t][threadIdx.x], smax[t][threadIdx.x + w]);
            }
            smax[D][threadIdx.x] = fmax(smax[D][threadIdx.x], smax[D][threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int t = 0; t < D; ++t) {
            pmin[blockIdx.x * D + t] = smin[t][0];
            pmax[blockIdx.x * (D + 1) + t] = smax[t][0];
        }
        pmax[blockIdx.x * (D + 1) + D] = smax[D][0];
    }
    if (last_block(done)) {
        __syncthreads();
        // the final reduction over the blocks' partials, by this block
        for (int t = 0; t < D; ++t) { smin[t][threadIdx.x] = DBL_MAX; smax[t][threadIdx.x] = -DBL_MAX; }
        smax[D][threadIdx.x] = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
            for (int t = 0; t < D; ++t) {
                smin[t][threadIdx.x] = fmin(smin[t][threadIdx.x], __ldcg(pmin + b * D + t));
                smax[t][threadIdx.x] = fmax(smax[t][threadIdx.x], __ldcg(pmax + b * (D + 1) + t));
            }
            smax[D][threadIdx.x] = fmax(smax[D][threadIdx.x], __ldcg(pmax + b * (D + 1) + D));
        }
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                for (int t = 0; t < D; ++t) {
                    smin[t][threadIdx.x] = fmin(smin[t][threadIdx.x], smin[t][threadIdx.x + w]);
                    smax[t][threadIdx.x] = fmax(smax[t][threadIdx.x], smax[t][threadIdx.x + w]);
                }
                smax[D][threadIdx.x] = fmax(smax[D][threadIdx.x], smax[D][threadIdx.x + w]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            for (int t = 0; t < D; ++t) { out_min[t] = smin[t][0]; out_max[t] = smax[t][0]; }
            out_max[D] = smax[D][0];
            *done = 0u;
        }
    }
}

// per-block partial max of ||p - c||^2 with c = (min + max)/2 read from device memory
template <int D>
__global__ void radius_k(const double* __restrict__ p1, int64_t n1, const double* __restrict__ p2, int64_t n2,
                         const double* __restrict__ gmin, const double* __restrict__ gmax, double* __restrict__ part,
                         double* out, unsigned* done) {
    double c[D];
    for (int t = 0; t < D; ++t) c[t] = 0.5 * (gmin[t] + gmax[t]);
    double r2 = 0;
    const int64_t total = n1 + n2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const double* q = i < n1 ? p1 + i * D : p2 + (i - n1) * D;
        double s = 0;
        for (int t = 0; t < D; ++t) { double v = q[t] - c[t]; s += v * v; }
        r2 = fmax(r2, s);
    }
    __shared__ double sm[kGeomThreads];
    sm[threadIdx.x] = r2;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
    if (last_block(done)) {  // the final reduction, by this block
        double v = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v = fmax(v, __ldcg(part + b));
        sm[threadIdx.x] = v;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            out[0] = sm[0];
            *done = 0u;
        }
    }
}

// the caller's point i of the set p1 (n1 points) u p2, row-major
template <int D>
__device__ __forceinline__ const double* point_ptr(const double* p1, int64_t n1, const double* p2, int64_t i) {
    return i < n1 ? p1 + i * D : p2 + (i - n1) * D;
}

// the cell key of a point: floor of its grid coordinate (x_t - c_t) * scale per axis,
// x-major.  gather_u_k writes u with the same expression, so the cell of u is
// the key.
template <int D>
__device__ __forceinline__ int32_t cell_key(const double* q, const double (&c)[3], double scale, int ng) {
    int32_t k = 0;
    for (int t = 0; t < D; ++t) {
        const double v = (q[t] - c[t]) * scale;
        const int cell = (int)floor(v) + ng / 2;
        k = k * ng + cell;
    }
    return k;
}

// scaled grid coordinates (SoA) + cell key + identity index
template <int D>
__global__ void scale_key_k(const double* __restrict__ p1, int64_t n1, const double* __restrict__ p2, int64_t n,
                            double c0, double c1, double c2, double scale, int ng, int32_t* __restrict__ key,
                            int32_t* __restrict__ idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c[3] = {c0, c1, c2};
    key[i] = cell_key<D>(point_ptr<D>(p1, n1, p2, i), c, scale, ng);
    idx[i] = (int32_t)i;
}

template <int D>
// sorted SoA torus coordinates, recomputed from the caller's row-major points (the same
// expression as scale_key_k, so the cell of u is the sorted key): one point's D contiguous
// doubles per random read instead of D scattered ones
__global__ void gather_u_k(const double* __restrict__ p1, int64_t n1, const double* __restrict__ p2,
                           const int32_t* __restrict__ perm, int64_t n, double c0, double c1, double c2, double scale,
                           double* __restrict__ u_out, SortedWeights sw) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c[3] = {c0, c1, c2};
    const int64_t j = perm[i];
    const double* q = point_ptr<D>(p1, n1, p2, j);
    for (int t = 0; t < D; ++t) u_out[t * n + i] = (q[t] - c[t]) * scale;
    // the set's weights in sorted order in the same pass (w1 for p1's points, sign2 * w2)
    if (sw.out) sw.out[i] = j < n1 ? sw.w1[j] : sw.sign2 * sw.w2[j - n1];
}

__global__ void permute_k(double* __restrict__ dst, const double* __restrict__ src, const int32_t* __restrict__ perm,
                          int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

__global__ void unpermute_k(double* __restrict__ dst, const double* __restrict__ src, const int32_t* __restrict__ perm,
                            int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[perm[i]] = src[i];
}

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

}  // namespace

Geometry compute_geometry(int d, const double* p1, int64_t n1, const double* p2, int64_t n2, cudaStream_t s,
                          void* comm) {
    Geometry g;
    g.d = d;
    const int nb = kGeomBlocks;
    DevBuf<double> pmin(nb * d, s), pmax(nb * (d + 1), s), fin(2 * d + 1 + 1, s), part(nb, s);
    DevBuf<unsigned> done(2, s);
    done.zero();
    double* gmin = fin.p;
    double* gmax = fin.p + d;  // d + 1 entries (last = non-finite flag)
    if (d == 1) bbox_k<1><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, pmin.p, pmax.p, gmin, gmax, done.p);
    else if (d == 2) bbox_k<2><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, pmin.p, pmax.p, gmin, gmax, done.p);
    else bbox_k<3><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, pmin.p, pmax.p, gmin, gmax, done.p);
    UOTK_LAUNCHED();
    if (comm) comm_allreduce_minmax(gmin, d, gmax, d + 1, comm, s);
    double* rfin = fin.p + 2 * d + 1;
    if (d == 1) radius_k<1><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, gmin, gmax, part.p, rfin, done.p + 1);
    else if (d == 2) radius_k<2><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, gmin, gmax, part.p, rfin, done.p + 1);
    else radius_k<3><<<nb, kGeomThreads, 0, s>>>(p1, n1, p2, n2, gmin, gmax, part.p, rfin, done.p + 1);
    UOTK_LAUNCHED();
    if (comm) comm_allreduce_minmax(nullptr, 0, rfin, 1, comm, s);
    double h[2 * kMaxD + 2];
    UOTK_CUDA(cudaMemcpyAsync(h, fin.p, (2 * d + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaStreamSynchronize(s));
    trace_mark("geometry: reductions + sync");
    if (h[2 * d] != 0) fail(UOTK_EDOMAIN, "non-finite point coordinate");
    // no point on any rank (a rank's own shard may be empty: the box is global)
    if (!(h[0] <= h[d])) return g;
    for (int t = 0; t < d; ++t) g.center[t] = 0.5 * (h[t] + h[d + t]);
    g.rmax = std::sqrt(h[2 * d + 1]);
    return g;
}

void make_pointset(PointSet& ps, const double* p1, int64_t n1, const double* p2, int64_t n2, const FastParams& fp,
                   cudaStream_t s, PointUse use, SortedWeights sw) {
    NvtxRange nvtx_("pointset");
    const int d = fp.d;
    const int64_t n = n1 + n2;
    ps.d = d;
    ps.n = n;
    ps.u.alloc((size_t)d * n, s);
    ps.key.alloc(n, s);
    ps.perm.alloc(n, s);
    if (n == 0) return;
    if (n > INT32_MAX) fail(UOTK_EUNSUPPORTED, "more than 2^31-1 points per call");
    const int tb = 256;
    const double scale = fp.ng / fp.h;
    const double* c = fp.center;
    const double cells = std::pow((double)fp.ng, d);
    {
        DevBuf<int32_t> key0(n, s), idx0(n, s);
        if (d == 1) scale_key_k<1><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, n, c[0], 0, 0, scale, fp.ng, key0.p, idx0.p);
        else if (d == 2) scale_key_k<2><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, n, c[0], c[1], 0, scale, fp.ng, key0.p, idx0.p);
        else scale_key_k<3><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, n, c[0], c[1], c[2], scale, fp.ng, key0.p, idx0.p);
        UOTK_LAUNCHED();
        int end_bit = 1;
        while ((double)(1ull << end_bit) < cells) ++end_bit;
        size_t tmp_bytes = 0;
        UOTK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key0.p, ps.key.p, idx0.p, ps.perm.p, (int)n, 0,
                                                  end_bit, s));
        DevBuf<uint8_t> tmp(tmp_bytes, s);
        UOTK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key0.p, ps.key.p, idx0.p, ps.perm.p, (int)n, 0,
                                                  end_bit, s));
        add_launches(1 + (end_bit + 7) / 8);  // CUB onesweep: histogram + one pass per 8 key bits
        trace_mark("pointset: sort");
        if (d == 1) gather_u_k<1><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, ps.perm.p, n, c[0], 0, 0, scale, ps.u.p, sw);
        else if (d == 2) gather_u_k<2><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, ps.perm.p, n, c[0], c[1], 0, scale, ps.u.p, sw);
        else gather_u_k<3><<<blocks_for(n, tb), tb, 0, s>>>(p1, n1, p2, ps.perm.p, n, c[0], c[1], c[2], scale, ps.u.p, sw);
        UOTK_LAUNCHED();
    }
    chunked_prepare(ps, fp, s, use);  // chunk list + precomputed windows (tuned cell-group kernels)
}

void permute_values(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    permute_k<<<blocks_for(n, 256), 256, 0, s>>>(dst, src, perm, n);
    UOTK_LAUNCHED();
}

void unpermute_values(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    unpermute_k<<<blocks_for(n, 256), 256, 0, s>>>(dst, src, perm, n);
    UOTK_LAUNCHED();
}

}  // namespace uotk
