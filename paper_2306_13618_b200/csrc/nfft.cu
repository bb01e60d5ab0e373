// Generic NFFT passes (any d, any m): window spreading (adjoint NFFT, inner sum of
// (4.6)), the FFT chain with the fused D_k multiplication, and interpolation
// (forward NFFT, outer sum of (4.6)) — P:590-592.  These are the simple
// thread-per-point kernels; the tuned cell-group kernels live in fused3d.cu / fused12d.cu.
#include <cstdlib>

#include <string>
#include <utility>

#include "chunks.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "window.cuh"

namespace uotk {

void comm_allreduce_spectrum(double2* buf, size_t count, void* comm, cudaStream_t s);  // comm.cu
// tuned cell-group passes for chunked point sets (fused12d.cu dispatches over d)
bool chunked_available(const FastParams& fp);
void chunked_spread(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s);
void chunked_gather_store(const PointSet& ps, const double* grid, const FastParams& fp, const EpiStore& epi,
                          cudaStream_t s);
void chunked_gather_dot(const PointSet& ps, const double* grid, const FastParams& fp, const EpiDot& epi,
                        cudaStream_t s);

namespace {

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

// g[l] += w_j prod_t phi(u_jt - l_t): one thread per point, global fp64 RED per tap.
template <int D, int M>
__global__ void spread_simple_k(const double* __restrict__ u, const double* __restrict__ w, int64_t n, int ng,
                                KBWindow win, double* __restrict__ grid) {
    constexpr int T = 2 * M;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double W[D][T];
    int base[D];
    for (int t = 0; t < D; ++t) {
        const double ut = u[t * n + i];
        const double fl = floor(ut);
        const double f = ut - fl;
        base[t] = (int)fl - M + 1 + ng / 2;
#pragma unroll
        for (int a = 0; a < T; ++a) W[t][a] = kb_phi(f + (M - 1 - a), win);
    }
    const double wi = w[i];
    if (D == 1) {
#pragma unroll
        for (int a = 0; a < T; ++a) atomicAdd(grid + base[0] + a, wi * W[0][a]);
    } else if (D == 2) {
        for (int a = 0; a < T; ++a) {
            const double wa = wi * W[0][a];
            double* row = grid + (int64_t)(base[0] + a) * ng + base[1];
#pragma unroll
            for (int b = 0; b < T; ++b) atomicAdd(row + b, wa * W[D - 1][b]);
        }
    } else {
        for (int a = 0; a < T; ++a) {
            for (int b = 0; b < T; ++b) {
                const double wab = wi * W[0][a] * W[1][b];
                double* row = grid + ((int64_t)(base[0] + a) * ng + (base[1] + b)) * ng + base[D - 1];
#pragma unroll
                for (int c = 0; c < T; ++c) atomicAdd(row + c, wab * W[D - 1][c]);
            }
        }
    }
}

// t_i = sum_l g[l] prod_t phi(u_it - l_t), then the epilogue.
template <int D, int M, class Epi>
__global__ void gather_simple_k(const double* __restrict__ u, int64_t n, int ng, KBWindow win,
                                const double* __restrict__ grid, Epi epi, unsigned long long* dmax) {
    constexpr int T = 2 * M;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double dd = 0.0;
    if (i < n) {
        double W[D][T];
        int base[D];
        for (int t = 0; t < D; ++t) {
            const double ut = u[t * n + i];
            const double fl = floor(ut);
            const double f = ut - fl;
            base[t] = (int)fl - M + 1 + ng / 2;
#pragma unroll
            for (int a = 0; a < T; ++a) W[t][a] = kb_phi(f + (M - 1 - a), win);
        }
        double acc = 0.0;
        if (D == 1) {
#pragma unroll
            for (int a = 0; a < T; ++a) acc += grid[base[0] + a] * W[0][a];
        } else if (D == 2) {
            for (int a = 0; a < T; ++a) {
                const double* row = grid + (int64_t)(base[0] + a) * ng + base[1];
                double r = 0.0;
#pragma unroll
                for (int b = 0; b < T; ++b) r += row[b] * W[D - 1][b];
                acc += r * W[0][a];
            }
        } else {
            for (int a = 0; a < T; ++a) {
                double ra = 0.0;
                for (int b = 0; b < T; ++b) {
                    const double* row = grid + ((int64_t)(base[0] + a) * ng + (base[1] + b)) * ng + base[D - 1];
                    double r = 0.0;
#pragma unroll
                    for (int c = 0; c < T; ++c) r += row[c] * W[D - 1][c];
                    ra += r * W[1][b];
                }
                acc += ra * W[0][a];
            }
        }
        dd = epi(i, acc);
    }
    warp_max_atomic(dmax, dd);
}

// H_k = G_k * D_k for |k_t| <= N/2 (k in I_N with the Nyquist split), 0 elsewhere.
// D_k layout: ((k_0 + N/2) (N+1) + (k_1 + N/2)) (N/2+1) + k_last  (last axis halved).
template <int D>
__global__ void scale_spectrum_k(double2* __restrict__ spec, const double* __restrict__ Dk, int ng, int N,
                                 int64_t total) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int nh = ng / 2 + 1;
    int64_t rem = i / nh;
    const int kl = (int)(i % nh);
    bool inside = kl <= N / 2;
    int64_t didx = kl;
    int64_t dstride = N / 2 + 1;
#pragma unroll
    for (int t = D - 2; t >= 0; --t) {
        const int q = (int)(rem % ng);
        rem /= ng;
        const int k = q < ng / 2 ? q : q - ng;
        inside = inside && (k >= -N / 2) && (k <= N / 2);
        didx += (int64_t)(k + N / 2) * dstride;
        dstride *= (N + 1);
    }
    if (!inside) {
        spec[i] = make_double2(0.0, 0.0);
        return;
    }
    const double f = Dk[didx];
    double2 v = spec[i];
    v.x *= f;
    v.y *= f;
    spec[i] = v;
}

// ---- the exchange step of the multi-rank path on the truncated spectrum only (SURVEY
// §8(e)): the ranks' partial coefficients are needed on I_N alone (D_k vanishes outside),
// so they are packed into the D_k layout ((N+1)^(d-1) (N/2+1) complex: 1/8 of the half
// spectrum in d = 3 at sigma = 2), all-reduced, and unpacked (zeros elsewhere).

// decode a D_k-layout index into the half-spectrum index of an n_g^d grid
template <int D>
__device__ __forceinline__ int64_t compact_to_spec(int64_t i, int ng, int N) {
    const int nh = N / 2 + 1;
    const int kl = (int)(i % nh);
    int64_t rem = i / nh;
    int64_t sidx = kl, sstride = ng / 2 + 1;
#pragma unroll
    for (int t = D - 2; t >= 0; --t) {
        const int k = (int)(rem % (N + 1)) - N / 2;
        rem /= (N + 1);
        sidx += (int64_t)(k < 0 ? k + ng : k) * sstride;
        sstride *= ng;
    }
    return sidx;
}

// compact[i] = spec[...] (* Dk[i] if Dk)
template <int D>
__global__ void pack_spectrum_k(const double2* __restrict__ spec, const double* __restrict__ Dk, int ng, int N,
                                int64_t ndk, double2* __restrict__ compact) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ndk; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = spec[compact_to_spec<D>(i, ng, N)];
        if (Dk) {
            const double f = Dk[i];
            v.x *= f;
            v.y *= f;
        }
        compact[i] = v;
    }
}

// spec = the compact values on I_N, zero elsewhere (the whole half spectrum is written)
template <int D>
__global__ void unpack_spectrum_k(const double2* __restrict__ compact, int ng, int N, int64_t total,
                                  double2* __restrict__ spec) {
    const int nh = ng / 2 + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = i / nh;
        const int kl = (int)(i % nh);
        bool inside = kl <= N / 2;
        int64_t didx = kl;
        int64_t dstride = N / 2 + 1;
#pragma unroll
        for (int t = D - 2; t >= 0; --t) {
            const int q = (int)(rem % ng);
            rem /= ng;
            const int k = q < ng / 2 ? q : q - ng;
            inside = inside && (k >= -N / 2) && (k <= N / 2);
            didx += (int64_t)(k + N / 2) * dstride;
            dstride *= (N + 1);
        }
        spec[i] = inside ? compact[didx] : make_double2(0.0, 0.0);
    }
}

// partial sums of sum_k D_k |G_k|^2 over the compact I_N values (weight 2 for k_last > 0:
// the conjugate-symmetric half; k_last <= N/2 < n_g/2)
__global__ void compact_energy_k(const double2* __restrict__ compact, const double* __restrict__ Dk, int N,
                                 int64_t ndk, double* __restrict__ part) {
    __shared__ double sm[256];
    const int nh = N / 2 + 1;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ndk; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = compact[i];
        acc += (i % nh == 0 ? 1.0 : 2.0) * Dk[i] * (v.x * v.x + v.y * v.y);
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// the pruned transform's layout t2c [ky' = ky + H][kz][qx (n)] <-> D_k layout [kx + H][ky + H][kz]
__global__ void pack_pruned_k(const double2* __restrict__ t2c, const double* __restrict__ Dk, int n, int N,
                              double2* __restrict__ compact) {
    const int H = N / 2;
    const int64_t total = (int64_t)(N + 1) * (N + 1) * (H + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int kz = (int)(i % (H + 1));
        const int64_t r = i / (H + 1);
        const int jy = (int)(r % (N + 1));
        const int jx = (int)(r / (N + 1));
        const int kx = jx - H;
        double2 v = t2c[((int64_t)jy * (H + 1) + kz) * n + (kx < 0 ? kx + n : kx)];
        if (Dk) {
            const double f = Dk[i];
            v.x *= f;
            v.y *= f;
        }
        compact[i] = v;
    }
}

__global__ void unpack_pruned_k(const double2* __restrict__ compact, int n, int N, double2* __restrict__ t2c) {
    const int H = N / 2;
    const int64_t total = (int64_t)(2 * H + 1) * (H + 1) * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int qx = (int)(i % n);
        const int64_t r = i / n;
        const int kz = (int)(r % (H + 1));
        const int jy = (int)(r / (H + 1));
        const int kx = qx < n / 2 ? qx : qx - n;
        t2c[i] = (kx < -H || kx > H) ? make_double2(0.0, 0.0)
                                      : compact[((int64_t)(kx + H) * (N + 1) + jy) * (H + 1) + kz];
    }
}

inline int64_t dk_elems(int d, int N) {
    int64_t e = N / 2 + 1;
    for (int t = 0; t < d - 1; ++t) e *= (N + 1);
    return e;
}

template <int D, int M>
void spread_dm(const PointSet& ps, const double* w, double* grid, const FastParams& fp, cudaStream_t s) {
    KBWindow win = make_window(fp.b, M);
    ProfScope ps_(kProfSpread, s);
    spread_simple_k<D, M><<<blocks_for(ps.n, 128), 128, 0, s>>>(ps.u.p, w, ps.n, fp.ng, win, grid);
    UOTK_LAUNCHED();
}

template <int D, int M, class Epi>
void gather_dm(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi,
               unsigned long long* dmax, cudaStream_t s) {
    KBWindow win = make_window(fp.b, M);
    ProfScope ps_(kProfGather, s);
    gather_simple_k<D, M, Epi><<<blocks_for(ps.n, 128), 128, 0, s>>>(ps.u.p, ps.n, fp.ng, win, grid, epi, dmax);
    UOTK_LAUNCHED();
}

}  // namespace

#define UOTK_DISPATCH_DM(d, m, CALL)                                              \
    do {                                                                          \
        switch ((d) * 16 + (m)) {                                                 \
            case 16 + 2: { constexpr int DD = 1, MM = 2; CALL; } break;            \
            case 16 + 3: { constexpr int DD = 1, MM = 3; CALL; } break;            \
            case 16 + 4: { constexpr int DD = 1, MM = 4; CALL; } break;            \
            case 16 + 5: { constexpr int DD = 1, MM = 5; CALL; } break;            \
            case 16 + 6: { constexpr int DD = 1, MM = 6; CALL; } break;            \
            case 16 + 7: { constexpr int DD = 1, MM = 7; CALL; } break;            \
            case 16 + 8: { constexpr int DD = 1, MM = 8; CALL; } break;            \
            case 32 + 2: { constexpr int DD = 2, MM = 2; CALL; } break;            \
            case 32 + 3: { constexpr int DD = 2, MM = 3; CALL; } break;            \
            case 32 + 4: { constexpr int DD = 2, MM = 4; CALL; } break;            \
            case 32 + 5: { constexpr int DD = 2, MM = 5; CALL; } break;            \
            case 32 + 6: { constexpr int DD = 2, MM = 6; CALL; } break;            \
            case 32 + 7: { constexpr int DD = 2, MM = 7; CALL; } break;            \
            case 32 + 8: { constexpr int DD = 2, MM = 8; CALL; } break;            \
            case 48 + 2: { constexpr int DD = 3, MM = 2; CALL; } break;            \
            case 48 + 3: { constexpr int DD = 3, MM = 3; CALL; } break;            \
            case 48 + 4: { constexpr int DD = 3, MM = 4; CALL; } break;            \
            case 48 + 5: { constexpr int DD = 3, MM = 5; CALL; } break;            \
            case 48 + 6: { constexpr int DD = 3, MM = 6; CALL; } break;            \
            case 48 + 7: { constexpr int DD = 3, MM = 7; CALL; } break;            \
            case 48 + 8: { constexpr int DD = 3, MM = 8; CALL; } break;            \
            default: fail(UOTK_EINVAL, "unsupported (d, m)");                     \
        }                                                                         \
    } while (0)

void spread_deterministic(const PointSet& ps, const double* w_sorted, double* grid, const FastParams& fp,
                          cudaStream_t s);  // determ.cu

void spread(const PointSet& ps, const double* w_sorted, double* grid, const FastParams& fp, cudaStream_t s) {
    if (ps.n == 0) return;
    if (fp.deterministic) {
        spread_deterministic(ps, w_sorted, grid, fp, s);
        return;
    }
    if (chunked_available(fp) && ps.chunked) {
        chunked_spread(ps, w_sorted, grid, fp, s);
        return;
    }
    UOTK_DISPATCH_DM(fp.d, fp.m, (spread_dm<DD, MM>(ps, w_sorted, grid, fp, s)));
}

// Stand-alone gathers (kernel sums, marginals) on sparse d = 3 clouds stay on the generic
// kernel: with few points per chunk its per-point loads beat the padded DMMA GEMMs (the
// spread still profits from the cell groups: footprint flushes instead of per-tap atomics).

template <class Epi>
void gather_epi(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi,
                unsigned long long* dmax, cudaStream_t s) {
    if (ps.n == 0) return;
    const bool sparse3 = fp.d == 3 && ps.chunk_fill < kGatherMinFill3 && !(fp.flags & UOTK_FLAG_CHUNKED);
    if constexpr (std::is_same<Epi, EpiStore>::value) {
        if (chunked_available(fp) && ps.chunked && !sparse3) {
            chunked_gather_store(ps, grid, fp, epi, s);
            return;
        }
    }
    if constexpr (std::is_same<Epi, EpiDot>::value) {
        if (chunked_available(fp) && ps.chunked && !sparse3) {
            chunked_gather_dot(ps, grid, fp, epi, s);
            return;
        }
    }
    UOTK_DISPATCH_DM(fp.d, fp.m, (gather_dm<DD, MM, Epi>(ps, grid, fp, epi, dmax, s)));
}

template void gather_epi<EpiStore>(const PointSet&, const double*, const FastParams&, const EpiStore&,
                                   unsigned long long*, cudaStream_t);
template void gather_epi<EpiSinkhorn>(const PointSet&, const double*, const FastParams&, const EpiSinkhorn&,
                                      unsigned long long*, cudaStream_t);
template void gather_epi<EpiDot>(const PointSet&, const double*, const FastParams&, const EpiDot&,
                                 unsigned long long*, cudaStream_t);

void gather(const PointSet& ps, const double* grid, double* out_sorted, const FastParams& fp, cudaStream_t s) {
    gather_epi(ps, grid, fp, EpiStore{out_sorted, nullptr}, nullptr, s);
}

int comm_nranks(void* comm);  // comm.cu

size_t separable_work_elems(const FastParams& fp, void* comm);  // circgemm.cu
// Separable chain (Gaussian kernel): circgemm.cu, hand-written DMMA GEMM passes on the box
double* separable_chain_dmma(const FastParams& fp, const double* Csep, double* grid, double* spare, double* work,
                             double* zero_next, cudaStream_t s, void* comm);
void comm_allreduce(double* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s);  // comm.cu

static double* fft_chain_pruned(SpectralPlan& sp, double* grid, double2* spec, cudaStream_t s, void* comm);

double* fft_chain(SpectralPlan& sp, double* grid, double2* spec, cudaStream_t s, void* comm, double* zero_next,
                  bool* zeroed) {
    const FastParams& fp = sp.fp;
    if (zeroed) *zeroed = false;
    if (sp.sep_chain) {
        const size_t wd = separable_work_elems(fp, comm);
        if (sp.work.n < wd) sp.work.alloc(wd, s);
        if (fp.d == 1 && zero_next == grid) zero_next = nullptr;  // d = 1: one pass, still reading it
        if (zeroed) *zeroed = zero_next != nullptr;
        return separable_chain_dmma(fp, sp.pd->Csep.p, grid, reinterpret_cast<double*>(spec), sp.work.p, zero_next, s,
                                    comm);
    }
    ProfScope ps_(kProfFft, s);
    {
        static const bool pruned_env = [] {
            const char* e = getenv("UOTK_PRUNED_FFT");
            return !(e && e[0] == '0');
        }();
        const size_t need = (size_t)fp.box_w * fp.ng * (fp.ng / 2 + 1) + (size_t)fp.box_w * (fp.N / 2 + 1) * fp.ng +
                            (size_t)(fp.N + 1) * (fp.N / 2 + 1) * fp.ng;
        if (pruned_env && fp.d == 3 && !(fp.flags & UOTK_FLAG_FFT) && need <= sp.spec_elems)
            return fft_chain_pruned(sp, grid, spec, s, comm);
    }
    if (!sp.r2c) get_fft_plans(fp.d, fp.ng, &sp.r2c, &sp.c2r);
    UOTK_CUFFT(cufftSetStream(sp.r2c, s));
    UOTK_CUFFT(cufftSetStream(sp.c2r, s));
    UOTK_CUFFT(cufftExecD2Z(sp.r2c, grid, (cufftDoubleComplex*)spec));
    const int64_t total = (int64_t)sp.spec_elems;
    if (comm) {
        // D_k . G on I_N packed, summed over ranks, unpacked (zero outside I_N)
        const int64_t ndk = dk_elems(fp.d, fp.N);
        DevBuf<double2> compact(ndk, s);
        const int gb = (int)std::min<int64_t>(2368, (ndk + 255) / 256);
        if (fp.d == 1) pack_spectrum_k<1><<<gb, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, ndk, compact.p);
        else if (fp.d == 2) pack_spectrum_k<2><<<gb, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, ndk, compact.p);
        else pack_spectrum_k<3><<<gb, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, ndk, compact.p);
        UOTK_LAUNCHED();
        comm_allreduce_spectrum(compact.p, ndk, comm, s);
        const int gu = (int)std::min<int64_t>(2368, (total + 255) / 256);
        if (fp.d == 1) unpack_spectrum_k<1><<<gu, 256, 0, s>>>(compact.p, fp.ng, fp.N, total, spec);
        else if (fp.d == 2) unpack_spectrum_k<2><<<gu, 256, 0, s>>>(compact.p, fp.ng, fp.N, total, spec);
        else unpack_spectrum_k<3><<<gu, 256, 0, s>>>(compact.p, fp.ng, fp.N, total, spec);
        UOTK_LAUNCHED();
    } else {
        if (fp.d == 1) scale_spectrum_k<1><<<blocks_for(total, 256), 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total);
        else if (fp.d == 2) scale_spectrum_k<2><<<blocks_for(total, 256), 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total);
        else scale_spectrum_k<3><<<blocks_for(total, 256), 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total);
        UOTK_LAUNCHED();
    }
    UOTK_CUFFT(cufftExecZ2D(sp.c2r, (cufftDoubleComplex*)spec, grid));
    return grid;
}

namespace {

// partial sums of  sum_k D_k |G_k|^2  over the half spectrum (weight 2 for the
// conjugate-symmetric interior of the last axis, 1 for k_last = 0 and n_g/2)
template <int D>
__global__ void spectrum_energy_k(const double2* __restrict__ spec, const double* __restrict__ Dk, int ng, int N,
                                  int64_t total, double* __restrict__ part) {
    __shared__ double sm[256];
    double acc = 0.0;
    const int nh = ng / 2 + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = i / nh;
        const int kl = (int)(i % nh);
        bool inside = kl <= N / 2;
        int64_t didx = kl;
        int64_t dstride = N / 2 + 1;
#pragma unroll
        for (int t = D - 2; t >= 0; --t) {
            const int q = (int)(rem % ng);
            rem /= ng;
            const int k = q < ng / 2 ? q : q - ng;
            inside = inside && (k >= -N / 2) && (k <= N / 2);
            didx += (int64_t)(k + N / 2) * dstride;
            dstride *= (N + 1);
        }
        if (inside) {
            const double2 v = spec[i];
            const double wgt = (kl == 0 || 2 * kl == ng) ? 1.0 : 2.0;
            acc += wgt * Dk[didx] * (v.x * v.x + v.y * v.y);
        }
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

}  // namespace

// <g', g> for g' = the NFFT interpolant of the spread grid g: the quadratic form
// sum_ij w_i w_j K_RK(z_i - z_j) of (3.5) in the Fourier domain, sum_k D_k |G_k|^2
// (identical to spreading, FFT, D_k, inverse FFT, gathering and summing w_i t_i).
namespace {

// T1 [x'][y][kz] (kz < n/2 + 1) -> T1c [x'][kz][y] for kz <= H (32 x 32 tiles per x')
__global__ void prune_t1_k(const double2* __restrict__ t1, int n, int H, double2* __restrict__ t1c) {
    __shared__ double2 tile[32][33];
    const int xp = blockIdx.z;
    const int y0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const int half = n / 2 + 1;
    const double2* src = t1 + (int64_t)xp * n * half;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int y = y0 + i, kz = k0 + threadIdx.x;
        tile[i][threadIdx.x] = (y < n && kz <= H) ? src[(int64_t)y * half + kz] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double2* dst = t1c + (int64_t)xp * (H + 1) * n;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int kz = k0 + i, y = y0 + threadIdx.x;
        if (kz <= H && y < n) dst[(int64_t)kz * n + y] = tile[threadIdx.x][i];
    }
}

// T2 [x'][kz][ky (all n)] -> T2c [ky' = ky + H][kz][o + x'] for |ky| <= H (tiles of (x', ky) per kz)
__global__ void prune_t2_k(const double2* __restrict__ t2, int n, int H, int w, int o, double2* __restrict__ t2c) {
    __shared__ double2 tile[32][33];
    const int kz = blockIdx.z;
    const int x0 = blockIdx.x * 32, j0 = blockIdx.y * 32;  // j = ky' in [0, 2H]
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int xp = x0 + i, j = j0 + threadIdx.x;
        double2 v = make_double2(0.0, 0.0);
        if (xp < w && j <= 2 * H) {
            const int ky = j - H;
            const int q = ky < 0 ? ky + n : ky;
            v = t2[((int64_t)xp * (H + 1) + kz) * n + q];
        }
        tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int j = j0 + i, xp = x0 + threadIdx.x;
        if (j <= 2 * H && xp < w) t2c[((int64_t)j * (H + 1) + kz) * n + o + xp] = tile[threadIdx.x][i];
    }
}

// partial sums of sum D_k |G_k|^2 over kx, ky in [-H, H], kz in [0, H] (weight 2 for kz > 0)
__global__ void pruned_energy_k(const double2* __restrict__ t3, const double* __restrict__ Dk, int n, int N,
                                double* __restrict__ part) {
    __shared__ double sm[256];
    const int H = N / 2;
    const int64_t total = (int64_t)(2 * H + 1) * (H + 1) * (2 * H + 1);
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int jx = (int)(i % (2 * H + 1));
        const int64_t r = i / (2 * H + 1);
        const int kz = (int)(r % (H + 1));
        const int jy = (int)(r / (H + 1));
        const int kx = jx - H;
        const int qx = kx < 0 ? kx + n : kx;
        const double2 v = t3[((int64_t)jy * (H + 1) + kz) * n + qx];
        const double d = Dk[((int64_t)jx * (N + 1) + jy) * (H + 1) + kz];
        acc += (kz == 0 ? 1.0 : 2.0) * d * (v.x * v.x + v.y * v.y);
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
        if (threadIdx.x < s2) sm[threadIdx.x] += sm[threadIdx.x + s2];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// the kernel-sum chain's inverse half of the pruned transform (fft_chain_pruned):
// t2c [ky'][kz][kx] *= D_k for |kx| <= H (zero beyond), in place
__global__ void prune_scale_k(double2* __restrict__ t3, const double* __restrict__ Dk, int n, int N) {
    const int H = N / 2;
    const int64_t total = (int64_t)(2 * H + 1) * (H + 1) * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int qx = (int)(i % n);
        const int64_t r = i / n;
        const int kz = (int)(r % (H + 1));
        const int jy = (int)(r / (H + 1));
        const int kx = qx < n / 2 ? qx : qx - n;
        double2 v = t3[i];
        if (kx < -H || kx > H) {
            v = make_double2(0.0, 0.0);
        } else {
            const double d = Dk[((int64_t)(kx + H) * (N + 1) + jy) * (H + 1) + kz];
            v.x *= d;
            v.y *= d;
        }
        t3[i] = v;
    }
}

// T2c [ky' = ky + H][kz][x (all n)] -> T2 [x'][kz][ky (all n)] for x = o + x', zero for |ky| > H
// (the inverse of prune_t2_k; T2 is zeroed first)
__global__ void unprune_t2_k(const double2* __restrict__ t2c, int n, int H, int w, int o, double2* __restrict__ t2) {
    __shared__ double2 tile[32][33];
    const int kz = blockIdx.z;
    const int x0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int j = j0 + i, xp = x0 + threadIdx.x;
        tile[i][threadIdx.x] = (j <= 2 * H && xp < w) ? t2c[((int64_t)j * (H + 1) + kz) * n + o + xp]
                                                      : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int xp = x0 + i, j = j0 + threadIdx.x;
        if (xp < w && j <= 2 * H) {
            const int ky = j - H;
            const int q = ky < 0 ? ky + n : ky;
            t2[((int64_t)xp * (H + 1) + kz) * n + q] = tile[threadIdx.x][i];
        }
    }
}

// T1c [x'][kz][y] -> T1 [x'][y][kz] (kz < n/2 + 1; zero for kz > H; the inverse of prune_t1_k)
__global__ void unprune_t1_k(const double2* __restrict__ t1c, int n, int H, double2* __restrict__ t1) {
    __shared__ double2 tile[32][33];
    const int xp = blockIdx.z;
    const int y0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const int half = n / 2 + 1;
    const double2* src = t1c + (int64_t)xp * (H + 1) * n;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int kz = k0 + i, y = y0 + threadIdx.x;
        tile[i][threadIdx.x] = (kz <= H && y < n) ? src[(int64_t)kz * n + y] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double2* dst = t1 + (int64_t)xp * n * half;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int y = y0 + i, kz = k0 + threadIdx.x;
        if (y < n && kz < half) dst[(int64_t)y * half + kz] = tile[threadIdx.x][i];
    }
}

}  // namespace

// sum_k D_k |G_k|^2 by a pruned 3-D transform: the grid is zero outside the footprint box
// [o, o + w)^3 and D_k vanishes outside |k_t| <= N/2, so the z-pass transforms only the
// w n rows of the box slab, the y-pass only the w (N/2 + 1) rows with kept kz, and the
// x-pass only the (N + 1)(N/2 + 1) rows with kept (ky, kz) (C2-IMQ: ~20% of the full
// transform's rows).  The intermediates live in `spec`.
static void spectrum_energy_pruned(SpectralPlan& sp, double* grid, double2* spec, double* part, int nparts,
                                   cudaStream_t s, void* comm) {
    const FastParams& fp = sp.fp;
    const int n = fp.ng, o = fp.box_lo, w = fp.box_w, N = fp.N, H = N / 2;
    cufftHandle pz, py, px, pzi;
    get_pruned_plans(n, w, H, &pz, &py, &px, &pzi);
    const int half = n / 2 + 1;
    double2* t1 = spec;                                           // w n half
    double2* t1c = t1 + (size_t)w * n * half;                     // w (H+1) n
    double2* t2c = t1c + (size_t)w * (H + 1) * n;                 // (2H+1)(H+1) n
    UOTK_CUFFT(cufftSetStream(pz, s));
    UOTK_CUFFT(cufftSetStream(py, s));
    UOTK_CUFFT(cufftSetStream(px, s));
    UOTK_CUFFT(cufftExecD2Z(pz, grid + (size_t)o * n * n, (cufftDoubleComplex*)t1));
    dim3 tb(32, 8);
    prune_t1_k<<<dim3((n + 31) / 32, (H + 32) / 32, w), tb, 0, s>>>(t1, n, H, t1c);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2Z(py, (cufftDoubleComplex*)t1c, (cufftDoubleComplex*)t1c, CUFFT_FORWARD));
    UOTK_CUDA(cudaMemsetAsync(t2c, 0, (size_t)(2 * H + 1) * (H + 1) * n * sizeof(double2), s));
    prune_t2_k<<<dim3((w + 31) / 32, (2 * H + 1 + 31) / 32, H + 1), tb, 0, s>>>(t1c, n, H, w, o, t2c);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2Z(px, (cufftDoubleComplex*)t2c, (cufftDoubleComplex*)t2c, CUFFT_FORWARD));
    add_launches(3);
    if (comm) {
        // the ranks' G on I_N (D_k layout), summed, then the energy of the sum
        const int64_t ndk = dk_elems(3, N);
        DevBuf<double2> compact(ndk, s);
        pack_pruned_k<<<(int)std::min<int64_t>(2368, (ndk + 255) / 256), 256, 0, s>>>(t2c, nullptr, n, N, compact.p);
        UOTK_LAUNCHED();
        comm_allreduce_spectrum(compact.p, ndk, comm, s);
        compact_energy_k<<<nparts, 256, 0, s>>>(compact.p, sp.pd->Dk.p, N, ndk, part);
        UOTK_LAUNCHED();
        return;
    }
    pruned_energy_k<<<nparts, 256, 0, s>>>(t2c, sp.pd->Dk.p, n, N, part);
    UOTK_LAUNCHED();
}

// The kernel-sum chain F^-1 (D . F g) by pruned transforms (d = 3, non-separable kernels,
// one rank): the forward half as in spectrum_energy_pruned, then D_k on the kept
// (kx, ky, kz), the inverse x-pass on the (N + 1)(N/2 + 1) kept rows, the inverse y-pass
// on the w (N/2 + 1) rows of the box slab, the inverse z-pass (C2R) on its w n rows —
// g' is produced on the box slab [o, o + w) x n x n of `grid` (all a gather reads).
static double* fft_chain_pruned(SpectralPlan& sp, double* grid, double2* spec, cudaStream_t s, void* comm) {
    const FastParams& fp = sp.fp;
    const int n = fp.ng, o = fp.box_lo, w = fp.box_w, N = fp.N, H = N / 2;
    cufftHandle pz, py, px, pzi;
    get_pruned_plans(n, w, H, &pz, &py, &px, &pzi);
    const int half = n / 2 + 1;
    double2* t1 = spec;                            // w n half
    double2* t1c = t1 + (size_t)w * n * half;      // w (H+1) n
    double2* t2c = t1c + (size_t)w * (H + 1) * n;  // (2H+1)(H+1) n
    for (cufftHandle h : {pz, py, px, pzi}) UOTK_CUFFT(cufftSetStream(h, s));
    double* slab = grid + (size_t)o * n * n;
    UOTK_CUFFT(cufftExecD2Z(pz, slab, (cufftDoubleComplex*)t1));
    dim3 tb(32, 8);
    prune_t1_k<<<dim3((n + 31) / 32, (H + 32) / 32, w), tb, 0, s>>>(t1, n, H, t1c);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2Z(py, (cufftDoubleComplex*)t1c, (cufftDoubleComplex*)t1c, CUFFT_FORWARD));
    UOTK_CUDA(cudaMemsetAsync(t2c, 0, (size_t)(2 * H + 1) * (H + 1) * n * sizeof(double2), s));
    prune_t2_k<<<dim3((w + 31) / 32, (2 * H + 1 + 31) / 32, H + 1), tb, 0, s>>>(t1c, n, H, w, o, t2c);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2Z(px, (cufftDoubleComplex*)t2c, (cufftDoubleComplex*)t2c, CUFFT_FORWARD));
    if (comm) {  // D_k . G on I_N packed, summed over ranks, unpacked
        const int64_t ndk = dk_elems(3, N);
        DevBuf<double2> compact(ndk, s);
        pack_pruned_k<<<(int)std::min<int64_t>(2368, (ndk + 255) / 256), 256, 0, s>>>(t2c, sp.pd->Dk.p, n, N,
                                                                                      compact.p);
        UOTK_LAUNCHED();
        comm_allreduce_spectrum(compact.p, ndk, comm, s);
        unpack_pruned_k<<<296, 256, 0, s>>>(compact.p, n, N, t2c);
        UOTK_LAUNCHED();
    } else {
        prune_scale_k<<<296, 256, 0, s>>>(t2c, sp.pd->Dk.p, n, N);
        UOTK_LAUNCHED();
    }
    UOTK_CUFFT(cufftExecZ2Z(px, (cufftDoubleComplex*)t2c, (cufftDoubleComplex*)t2c, CUFFT_INVERSE));
    UOTK_CUDA(cudaMemsetAsync(t1c, 0, (size_t)w * (H + 1) * n * sizeof(double2), s));
    unprune_t2_k<<<dim3((w + 31) / 32, (2 * H + 1 + 31) / 32, H + 1), tb, 0, s>>>(t2c, n, H, w, o, t1c);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2Z(py, (cufftDoubleComplex*)t1c, (cufftDoubleComplex*)t1c, CUFFT_INVERSE));
    unprune_t1_k<<<dim3((n + 31) / 32, (half + 31) / 32, w), tb, 0, s>>>(t1c, n, H, t1);
    UOTK_LAUNCHED();
    UOTK_CUFFT(cufftExecZ2D(pzi, (cufftDoubleComplex*)t1, slab));
    add_launches(6);
    return grid;
}

void spectrum_energy(SpectralPlan& sp, double* grid, double2* spec, double* part, int nparts, cudaStream_t s,
                     void* comm) {
    const FastParams& fp = sp.fp;
    static const bool pruned = [] {
        const char* e = getenv("UOTK_PRUNED_FFT");
        return !(e && e[0] == '0');
    }();
    const size_t need = (size_t)fp.box_w * fp.ng * (fp.ng / 2 + 1) + (size_t)fp.box_w * (fp.N / 2 + 1) * fp.ng +
                        (size_t)(fp.N + 1) * (fp.N / 2 + 1) * fp.ng;
    if (pruned && fp.d == 3 && !(fp.flags & UOTK_FLAG_FFT) && need <= sp.spec_elems) {
        ProfScope ps_(kProfFft, s);
        spectrum_energy_pruned(sp, grid, spec, part, nparts, s, comm);
        return;
    }
    ProfScope ps_(kProfFft, s);
    if (!sp.r2c) get_fft_plans(fp.d, fp.ng, &sp.r2c, &sp.c2r);
    UOTK_CUFFT(cufftSetStream(sp.r2c, s));
    UOTK_CUFFT(cufftExecD2Z(sp.r2c, grid, (cufftDoubleComplex*)spec));
    if (comm) {
        // the ranks' G on I_N (D_k layout), summed, then the energy of the sum
        const int64_t ndk = dk_elems(fp.d, fp.N);
        DevBuf<double2> compact(ndk, s);
        const int gb = (int)std::min<int64_t>(2368, (ndk + 255) / 256);
        if (fp.d == 1) pack_spectrum_k<1><<<gb, 256, 0, s>>>(spec, nullptr, fp.ng, fp.N, ndk, compact.p);
        else if (fp.d == 2) pack_spectrum_k<2><<<gb, 256, 0, s>>>(spec, nullptr, fp.ng, fp.N, ndk, compact.p);
        else pack_spectrum_k<3><<<gb, 256, 0, s>>>(spec, nullptr, fp.ng, fp.N, ndk, compact.p);
        UOTK_LAUNCHED();
        comm_allreduce_spectrum(compact.p, ndk, comm, s);
        compact_energy_k<<<nparts, 256, 0, s>>>(compact.p, sp.pd->Dk.p, fp.N, ndk, part);
        UOTK_LAUNCHED();
        return;
    }
    const int64_t total = (int64_t)sp.spec_elems;
    if (fp.d == 1) spectrum_energy_k<1><<<nparts, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total, part);
    else if (fp.d == 2) spectrum_energy_k<2><<<nparts, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total, part);
    else spectrum_energy_k<3><<<nparts, 256, 0, s>>>(spec, sp.pd->Dk.p, fp.ng, fp.N, total, part);
    UOTK_LAUNCHED();
}

}  // namespace uotk
