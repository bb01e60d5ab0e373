// Near-field correction of the fast summation for kernels that are not smooth at the
// origin (Laplace exp(-r/l), energy -r; Eq. 4.2, Rem. 4.2 P:608, reading R24):
// the Fourier part sums the regularised K_R, which replaces K by the polynomial
// Q(||y||^2) on ||y|| < eps_I (torus units); the exact result is restored by
//     t_i += sum_{j : ||x_i - y_j|| < eps_I h} (K - K_R)(x_i - y_j) w_j ,
// a direct sum over the pairs closer than eps_I (a small fraction of all pairs: the
// ball of radius eps_I = p/N against the point cloud of torus radius <= 1/4).
//
// Buckets: a coarse grid of cells of B >= eps_I n_g grid cells per axis, so every
// partner of a target lies in the 3^d coarse cells around its own.  Each point set is
// sorted by coarse key once (CUB), its coordinates gathered in that order; a dense table
// holds the first point of every coarse cell.  The last axis varies fastest in the key,
// so the three cells of a neighbour row are one contiguous point range.  One thread per
// target (targets in coarse order: the threads of a warp read the same source points),
// partners visited in a fixed order: deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"

namespace uotk {

namespace {

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

template <int D>
__global__ void coarse_key_k(const double* __restrict__ u, int64_t n, int ng, int B, int nc, int32_t* __restrict__ key,
                             int32_t* __restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t k = 0;
    for (int t = 0; t < D; ++t) {
        const int cell = (int)floor(u[t * n + i]) + ng / 2;
        k = k * nc + min(nc - 1, max(0, cell / B));
    }
    key[i] = k;
    idx[i] = (int32_t)i;
}

template <int D>
__global__ void gather_coarse_k(const double* __restrict__ u, const int32_t* __restrict__ perm, int64_t n,
                                double* __restrict__ uc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = perm[i];
    for (int t = 0; t < D; ++t) uc[t * n + i] = u[t * n + j];
}

// start[c] = first position with key >= c, c = 0 .. ncells (binary search in the sorted keys)
__global__ void cell_start_k(const int32_t* __restrict__ key, int64_t n, int64_t ncells, int32_t* __restrict__ start) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c > ncells) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    start[c] = (int32_t)lo;
}

__global__ void permute_to_coarse_k(const double* __restrict__ w, const int32_t* __restrict__ perm, int64_t n,
                                    double* __restrict__ wc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) wc[i] = w[perm[i]];
}

struct NFCoef {
    int kind;        // UOTK_LAP / UOTK_ENERGY
    double h;        // torus scaling
    double inv_ell;  // Laplace 1/l
    double inv_ng;   // grid units -> torus units
    double sI;       // eps_I^2 (torus units)
    int npoly;
    double poly[16];  // Q in powers of (s - sI)
};

// out[map ? map[it] : it] += sum over partners closer than eps_I of (K - Q) w
template <int D>
__global__ void __launch_bounds__(128) nearfield_k(const double* __restrict__ ut, const int32_t* __restrict__ tperm,
                                                   const int32_t* __restrict__ tkey, int64_t nt,
                                                   const double* __restrict__ us, const double* __restrict__ ws,
                                                   const int32_t* __restrict__ sstart, int64_t ns, int nc, NFCoef c,
                                                   const int32_t* __restrict__ map, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nt) return;
    double xi[D];
    for (int t = 0; t < D; ++t) xi[t] = ut[t * nt + i];
    int cc[3] = {0, 0, 0};
    {
        int k = tkey[i];
        for (int t = D - 1; t >= 0; --t) {
            cc[t] = k % nc;
            k /= nc;
        }
    }
    const double r2max = c.sI / (c.inv_ng * c.inv_ng);  // eps_I^2 in grid units^2
    double acc = 0.0;
    const int z0 = max(0, cc[D - 1] - 1), z1 = min(nc - 1, cc[D - 1] + 1);
    const int nrow = D == 1 ? 1 : (D == 2 ? 3 : 9);
    for (int r = 0; r < nrow; ++r) {
        int pre = 0;
        bool ok = true;
        if (D == 2) {
            const int cx = cc[0] + r - 1;
            ok = cx >= 0 && cx < nc;
            pre = cx * nc;
        } else if (D == 3) {
            const int cx = cc[0] + r / 3 - 1, cy = cc[1] + r % 3 - 1;
            ok = cx >= 0 && cx < nc && cy >= 0 && cy < nc;
            pre = (cx * nc + cy) * nc;
        }
        if (!ok) continue;
        const int j0 = sstart[pre + z0], j1 = sstart[pre + z1 + 1];
        for (int j = j0; j < j1; ++j) {
            double r2 = 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const double v = xi[t] - us[t * ns + j];
                r2 = fma(v, v, r2);
            }
            if (r2 < r2max) {
                const double s = r2 * c.inv_ng * c.inv_ng;  // torus units
                const double hr = c.h * sqrt(s);
                const double k = c.kind == UOTK_LAP ? exp(-hr * c.inv_ell) : -hr;
                const double ds = s - c.sI;
                double q = 0.0;
                for (int m = c.npoly - 1; m >= 0; --m) q = fma(q, ds, c.poly[m]);
                acc = fma(k - q, ws[j], acc);
            }
        }
    }
    const int64_t it = tperm[i];
    out[map ? map[it] : it] += acc;
}

}  // namespace

bool nearfield_needed(const FastParams& fp) { return fp.eps_I > 0; }

// coarse buckets of one point set (its PointSet order -> coarse order)
void build_nearfield(NearField& nf, const PointSet& ps, const FastParams& fp, cudaStream_t s) {
    const int d = fp.d;
    const int64_t n = ps.n;
    nf.n = n;
    nf.B = std::max(1, (int)std::ceil(fp.eps_I * fp.ng * (1.0 + 1e-12)));
    nf.nc = (fp.ng + nf.B - 1) / nf.B;
    int64_t ncells = 1;
    for (int t = 0; t < d; ++t) ncells *= nf.nc;
    nf.perm.alloc(n, s);
    nf.key.alloc(n, s);
    nf.u.alloc((size_t)d * n, s);
    nf.start.alloc(ncells + 1, s);
    if (n > 0) {
        DevBuf<int32_t> key0(n, s), idx0(n, s);
        if (d == 1) coarse_key_k<1><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, n, fp.ng, nf.B, nf.nc, key0.p, idx0.p);
        else if (d == 2) coarse_key_k<2><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, n, fp.ng, nf.B, nf.nc, key0.p, idx0.p);
        else coarse_key_k<3><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, n, fp.ng, nf.B, nf.nc, key0.p, idx0.p);
        UOTK_LAUNCHED();
        int end_bit = 1;
        while ((int64_t(1) << end_bit) < ncells) ++end_bit;
        size_t tmp_bytes = 0;
        UOTK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key0.p, nf.key.p, idx0.p, nf.perm.p, (int)n, 0,
                                                  end_bit, s));
        DevBuf<uint8_t> tmp(tmp_bytes, s);
        UOTK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key0.p, nf.key.p, idx0.p, nf.perm.p, (int)n, 0,
                                                  end_bit, s));
        add_launches(1 + (end_bit + 7) / 8);
        if (d == 1) gather_coarse_k<1><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, nf.perm.p, n, nf.u.p);
        else if (d == 2) gather_coarse_k<2><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, nf.perm.p, n, nf.u.p);
        else gather_coarse_k<3><<<blocks_for(n, 256), 256, 0, s>>>(ps.u.p, nf.perm.p, n, nf.u.p);
        UOTK_LAUNCHED();
    }
    cell_start_k<<<blocks_for(ncells + 1, 256), 256, 0, s>>>(nf.key.p, n, ncells, nf.start.p);
    UOTK_LAUNCHED();
}

// out (indexed by the target PointSet order, or through `map` to caller order) +=
// near-field correction of the sum over the sources with weights w (source PointSet order)
void nearfield_apply(const NearField& src, const double* w, const NearField& tgt, const FastParams& fp,
                     const int32_t* map, double* out, cudaStream_t s) {
    if (src.n == 0 || tgt.n == 0) return;
    if (src.nc != tgt.nc) fail(UOTK_EINVAL, "internal: near-field bucket grids differ");
    DevBuf<double> wc(src.n, s);
    permute_to_coarse_k<<<blocks_for(src.n, 256), 256, 0, s>>>(w, src.perm.p, src.n, wc.p);
    UOTK_LAUNCHED();
    NFCoef c{};
    c.kind = fp.kind;
    c.h = fp.h;
    c.inv_ell = fp.kind == UOTK_LAP ? 1.0 / fp.param : 0.0;
    c.inv_ng = 1.0 / fp.ng;
    c.sI = fp.eps_I * fp.eps_I;
    c.npoly = (int)fp.poly_I.size();
    for (int k = 0; k < c.npoly && k < 16; ++k) c.poly[k] = fp.poly_I[k];
    ProfScope ps_(kProfGather, s);
    const int nb = blocks_for(tgt.n, 128);
    if (fp.d == 1)
        nearfield_k<1><<<nb, 128, 0, s>>>(tgt.u.p, tgt.perm.p, tgt.key.p, tgt.n, src.u.p, wc.p, src.start.p, src.n,
                                          src.nc, c, map, out);
    else if (fp.d == 2)
        nearfield_k<2><<<nb, 128, 0, s>>>(tgt.u.p, tgt.perm.p, tgt.key.p, tgt.n, src.u.p, wc.p, src.start.p, src.n,
                                          src.nc, c, map, out);
    else
        nearfield_k<3><<<nb, 128, 0, s>>>(tgt.u.p, tgt.perm.p, tgt.key.p, tgt.n, src.u.p, wc.p, src.start.p, src.n,
                                          src.nc, c, map, out);
    UOTK_LAUNCHED();
}

// dd = epi(i, t_i) for every point of a set (the Sinkhorn update applied to a kernel sum
// that was completed outside the gather, e.g. by the near-field correction)
template <class Epi>
__global__ void apply_epi_k(const double* __restrict__ t, int64_t n, Epi epi, unsigned long long* dmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double dd = 0.0;
    if (i < n) dd = epi(i, t[i]);
    warp_max_atomic(dmax, dd);
}

void apply_sinkhorn_update(const double* t, int64_t n, const EpiSinkhorn& epi, unsigned long long* dmax,
                           cudaStream_t s) {
    if (n == 0) return;
    apply_epi_k<EpiSinkhorn><<<blocks_for(n, 256), 256, 0, s>>>(t, n, epi, dmax);
    UOTK_LAUNCHED();
}

}  // namespace uotk
