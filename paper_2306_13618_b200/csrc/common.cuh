// Internal definitions shared by the uotk CUDA sources (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/uotk.h"
#include "window_fit.h"

namespace uotk {

// ------------------------------------------------------------------ errors
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);
void check_cufft(cufftResult r, const char* what, const char* file, int line);

#define UOTK_CUDA(call) ::uotk::check_cuda((call), #call, __FILE__, __LINE__)
#define UOTK_CUFFT(call) ::uotk::check_cufft((call), #call, __FILE__, __LINE__)
#define UOTK_LAUNCHED() ::uotk::note_launch(__FILE__, __LINE__)

void note_launch(const char* file, int line);  // counts launches + checks launch errors
// cudaFuncSetAttribute(max dynamic shared memory) once per (kernel, device)
void set_smem_attr(const void* func, int bytes);
void add_launches(int k);                      // launches made by library code we call (CUB)

// host-side phase timing for diagnosis: with UOTK_TRACE=1 in the environment every
// trace_mark prints the host microseconds since the previous mark to stderr
void trace_mark(const char* what);

// Per-thread resource slot (comm.cu comm_slot): the rank of a loopback communicator whose
// ranks run concurrently on one device from several host threads, else 0.  The cuFFT
// plans and the cuBLAS handle are cached per (device, slot).
extern thread_local int g_slot;
struct SlotScope {
    int prev;
    explicit SlotScope(void* comm);
    ~SlotScope() { g_slot = prev; }
};

// ------------------------------------------------------------------ device buffers
// Device allocation through the library's block cache (context.cu), backed by the
// stream-ordered pool (cudaMallocAsync on the call's stream).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    bool pooled = false;  // allocated from the stream-ordered pool (inside graph capture)
    DevBuf() = default;
    DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    void alloc(size_t count, cudaStream_t stream);
    void zero() { if (n) UOTK_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
    ~DevBuf();
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), pooled(o.pooled) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept;
};

bool is_device_pointer(const void* ptr);
size_t block_cache_bytes();   // freed device blocks the library keeps for reuse (this device)
void block_cache_release();   // return them to the stream-ordered pool
void release_plan_cache();    // nfft_plan.cu: drop the cached D_k / circulant tables
void release_fft_plans();     // context.cu: destroy the cached cuFFT plans

// A caller array that may live on the host or the device: `d` is always a device
// pointer valid for the duration of the call.
struct InArr {
    const double* d = nullptr;
    bool host = false;  // staged from host memory (an async copy when the memory is pinned)
    DevBuf<double> staged;
    void bind(const double* user, size_t count, cudaStream_t s);
};
struct OutArr {
    double* d = nullptr;
    double* user = nullptr;
    size_t count = 0;
    bool host = false;
    DevBuf<double> staged;
    cudaStream_t s = nullptr;
    void bind(double* user_ptr, size_t cnt, cudaStream_t stream);
    void flush();  // device -> host copy if needed (async)
};

// ------------------------------------------------------------------ geometry / plan
constexpr int kMaxD = 3;

struct Geometry {
    int d = 0;
    double center[kMaxD] = {0, 0, 0};
    double rmax = 0;
};

// Parameters of one fast summation.
struct FastParams {
    int d = 0;
    int kind = 0;
    double param = 0;      // kernel parameter in original units
    int N = 0;             // bandwidth
    int ng = 0;            // oversampled grid size per axis
    int m = 8;             // window half width (taps = 2m)
    double b = 0;          // Kaiser-Bessel shape, pi (2 - 1/sigma)
    double h = 1;          // torus scaling
    double center[kMaxD] = {0, 0, 0};
    double eps_B = 0;      // IMQ boundary band
    int p = 0;             // IMQ boundary order
    std::vector<double> poly;  // boundary polynomial K_B in t = (r - r0)/eps_B (torus units), ascending
    // interior regularisation (Laplace, energy; reading R24): K_R = Q(r^2) on r < eps_I,
    // Q in powers of (r^2 - eps_I^2), torus units; the near-field correction adds K - K_R there
    double eps_I = 0;
    std::vector<double> poly_I;
    int flags = 0;         // uotk_opts.flags (kernel family policy)
    bool deterministic = false;  // uotk_opts.deterministic: spreads by the pull kernel (determ.cu)
    // grid box [box_lo, box_lo + box_w)^d holding every window footprint of the points
    // (both sets): the spread writes only inside it and the gathers read only inside it
    int box_lo = 0, box_w = 0;
};

// Sorted, scaled point set on device.
struct PointSet {
    int d = 0;
    int64_t n = 0;
    DevBuf<double> u;        // d * n, SoA, grid units: u_t = (x_t - c_t)/h * ng
    DevBuf<int32_t> key;     // n, linear cell key (sorted ascending)
    DevBuf<int32_t> perm;    // n, sorted position -> caller index
    // chunked layout of the cell-group kernels (chunks.cuh): runs of equal keys split
    // into chunks of <= 32 points, with the window values precomputed per chunk
    bool chunked = false;
    int64_t nchunks = 0;
    DevBuf<int4> chunk_desc;  // {first point, count, key, 0}
    DevBuf<double> chunk_win; // nchunks x chunk_win_doubles(d) window values (zero for empty slots)
    DevBuf<int32_t> chunk_bounds;  // chunk_blocks + 1 cost-balanced work-unit boundaries
    int chunk_blocks = 0;     // work units: CTAs (d = 3) or warps (d <= 2)
    DevBuf<int32_t> chunk_bounds_ws;  // d = 2: partition for the warp-specialised half-step
    int chunk_units_ws = 0;
    int chunk_kz = 16;        // d = 3: z extent of a group footprint (16 one cell, 24 z-segment)
    // d = 3 spread-only one-cell sets: no window blocks, the spread evaluates them on the
    // fly from the per-tap polynomials (fused3d.cu spread3d_fly_k)
    bool win_fly = false;
    KBHorner win_coef;
    double chunk_fill = 0;    // mean occupied fraction of the 32 chunk slots
};

// Coarse buckets of a point set for the near-field correction (nearfield.cu): the set
// re-sorted by a coarse key (cells of B >= eps_I n_g grid cells per axis, nc per axis)
struct NearField {
    int64_t n = 0;
    int B = 1, nc = 1;
    DevBuf<int32_t> perm;   // coarse order -> PointSet order
    DevBuf<int32_t> key;    // coarse key (sorted)
    DevBuf<int32_t> start;  // nc^d + 1: first point of each coarse cell
    DevBuf<double> u;       // d x n grid coordinates in coarse order
};
bool nearfield_needed(const FastParams& fp);
void build_nearfield(NearField& nf, const PointSet& ps, const FastParams& fp, cudaStream_t s);
void nearfield_apply(const NearField& src, const double* w, const NearField& tgt, const FastParams& fp,
                     const int32_t* map, double* out, cudaStream_t s);

// Kernel-dependent Fourier-side tables, cached across calls (nfft_plan.cu) by the
// parameters they depend on; `ready` marks the end of their construction on the stream
// that built them (other streams wait on it).
struct PlanData {
    DevBuf<double> Dk;       // (N+1)^(d-1) * (N/2+1)
    // Gaussian kernel: D_k = prod_t d1(k_t) is separable, so F^-1 D F is the tensor power
    // of one real symmetric circulant n_g x n_g matrix Csep (DESIGN.md §7 "separable")
    bool separable = false;
    DevBuf<double> Csep;
    cudaEvent_t ready = nullptr;
    // completion of the last use on each stream that used the tables (recorded when a
    // call's SpectralPlan ends): the destructor waits for exactly these, not the device
    std::mutex use_mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
    void note_use(cudaStream_t s);
    PlanData() = default;
    PlanData(const PlanData&) = delete;
    PlanData& operator=(const PlanData&) = delete;
    ~PlanData();
};

// Fourier-side plan: the D_k table and the cuFFT handles.
struct SpectralPlan {
    FastParams fp;
    std::shared_ptr<PlanData> pd;
    cufftHandle r2c = 0, c2r = 0;  // owned by the context cache
    size_t grid_elems = 0;   // ng^d
    size_t spec_elems = 0;   // ng^(d-1) * (ng/2+1)
    cudaStream_t use_stream = nullptr;  // the call's stream (build_spectral_plan)
    DevBuf<double> work;                // the separable chain's compact intermediate (w^d)
    // the spectral step runs as the separable chain (Gaussian, and cheaper than the cuFFT
    // chain for this box and grid; build_spectral_plan), else as cuFFT D2Z / D_k / Z2D
    bool sep_chain = false;
    ~SpectralPlan() {
        if (pd) pd->note_use(use_stream);
    }
};

// ------------------------------------------------------------------ library context
struct Context;
Context& ctx();
void get_fft_plans(int d, int n, cufftHandle* r2c, cufftHandle* c2r);

// ------------------------------------------------------------------ host plan (nfft_plan.cu)
FastParams choose_params(int d, int kind, double param, const Geometry& g, const uotk_opts& o);
void build_spectral_plan(SpectralPlan& sp, cudaStream_t s);

// ------------------------------------------------------------------ kernels (launchers)
// geometry: bbox + max radius over up to two point sets (row-major n x d)
struct GeomScratch;
Geometry compute_geometry(int d, const double* p1, int64_t n1, const double* p2, int64_t n2,
                          cudaStream_t s, void* comm);
// scale, key and sort one point set; weights are permuted separately by permute_values
// use: what the point set will be used for (the chunk layout is skipped where no kernel
// would use it: gather-only d = 3 sets below kGatherMinFill3)
enum PointUse { kUseBoth = 0, kUseGatherOnly = 1, kUseSpreadOnly = 2 };
// optional: the set's weights permuted into sorted order while the coordinates are
// (out[i] = w1[j] for the first n1 points, sign2 * w2[j - n1] for the others; j = perm[i])
struct SortedWeights {
    const double* w1 = nullptr;
    const double* w2 = nullptr;
    double sign2 = 1.0;
    double* out = nullptr;
};
// the set is p1 (n1 points) followed by p2 (n2 points; may be null when n2 = 0)
void make_pointset(PointSet& ps, const double* p1, int64_t n1, const double* p2, int64_t n2, const FastParams& fp,
                   cudaStream_t s, PointUse use = kUseBoth, SortedWeights sw = SortedWeights{});
inline void make_pointset(PointSet& ps, const double* pts, int64_t n, const FastParams& fp, cudaStream_t s,
                          PointUse use = kUseBoth, SortedWeights sw = SortedWeights{}) {
    make_pointset(ps, pts, n, nullptr, 0, fp, s, use, sw);
}
void permute_values(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s);
void unpermute_values(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s);

// NFFT passes
void spread(const PointSet& ps, const double* w_sorted, double* grid, const FastParams& fp, cudaStream_t s);
// g' = F^-1 (D .* F g): returns the buffer holding g' (grid itself, or spec's storage
// reinterpreted as n_g^d doubles on the separable path)
// zero_next (optional): a grid that is zero outside the footprint box; the separable chain
// zeroes its box as a side job (then *zeroed = true: the caller's memset is not needed)
double* fft_chain(SpectralPlan& sp, double* grid, double2* spec, cudaStream_t s, void* comm,
                  double* zero_next = nullptr, bool* zeroed = nullptr);
// cuFFT plans of the pruned 3-D forward transform (box width w, kept modes |k| <= H)
void get_pruned_plans(int n, int w, int H, cufftHandle* pz, cufftHandle* py, cufftHandle* px, cufftHandle* pzi);
void gather(const PointSet& ps, const double* grid, double* out_sorted, const FastParams& fp, cudaStream_t s);
template <class Epi>
void gather_epi(const PointSet& ps, const double* grid, const FastParams& fp, const Epi& epi,
                unsigned long long* dmax, cudaStream_t s);

// direct sums t_i = sum_j k(|tgt_i - src_j|) w_j (row-major points) followed by an epilogue
template <class Epi>
void direct_sum_epi(int d, int64_t n_src, const double* src, const double* w, int64_t n_tgt,
                    const double* tgt, int kind, double param, const Epi& epi,
                    unsigned long long* dmax, cudaStream_t s);

// small reductions: sums[k] = sum_i terms_k(i), deterministic order; see reduce.cu
void sum_columns(const double* vals, int64_t n, int ncols, double* out_dev, cudaStream_t s);

}  // namespace uotk
