// Host planning of the fast summation (Sec. 4) and the kernel-coefficient
// setup on the device:  torus scaling h (Eq. 4.7; Rem. 4.3), bandwidth N
// (Eq. 4.4; Rem. 4.4), regularised kernel K_R, its Fourier
// coefficients b_k, and the deconvolved multiplier
//     D_k = w_k b_k / (n_g^{2d} prod_t phihat(k_t)^2),   k in I_N,
// which turns "spread -> FFT -> *D_k -> inverse FFT -> interpolate" into the
// factorisation (4.5)-(4.6).  See DESIGN.md "Fast summation".
#include <tuple>
#include <mutex>
#include <list>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace uotk {

namespace {

// next integer >= v whose prime factors are all in {2,3,5,7}, and even
int nice_even(int v) {
    if (v < 2) v = 2;
    for (int x = v + (v & 1);; x += 2) {
        int y = x;
        for (int p : {2, 3, 5, 7})
            while (y % p == 0) y /= p;
        if (y == 1) return x;
    }
}

// Modified Bessel I_0 by its power series (all terms positive), long double.
long double bessel_i0(long double z) {
    long double q = z * z / 4.0L, term = 1.0L, sum = 1.0L;
    for (int k = 1; k < 400; ++k) {
        term *= q / ((long double)k * (long double)k);
        sum += term;
        if (term < sum * 1e-21L) break;
    }
    return sum;
}

// Taylor coefficients y_k = K^(k)(r0)/k! of K(r) = (h^2 r^2 + c^2)^(-1/2) at r0
// (power-series recurrence for g^alpha with g(s) = A + B s + C s^2).
std::vector<long double> imq_taylor(long double h, long double c, long double r0, int n) {
    long double g[3] = {h * h * r0 * r0 + c * c, 2 * h * h * r0, h * h};
    const long double alpha = -0.5L;
    std::vector<long double> y(n, 0.0L);
    y[0] = powl(g[0], alpha);
    for (int k = 1; k < n; ++k) {
        long double acc = 0;
        for (int i = 1; i <= 2 && i <= k; ++i) acc += ((alpha + 1) * i - k) * g[i] * y[k - i];
        y[k] = acc / (k * g[0]);
    }
    return y;
}

// Taylor coefficients y_k = K^(k)(r0)/k! (torus radius r0, physical radius h r0) of the
// Laplace kernel exp(-h r / l) and of the energy kernel -h r.
std::vector<long double> lap_taylor(long double h, long double ell, long double r0, int n) {
    std::vector<long double> y(n);
    const long double a = -h / ell;
    long double v = expl(a * r0);
    for (int k = 0; k < n; ++k) {
        y[k] = v;
        v *= a / (k + 1);
    }
    return y;
}
std::vector<long double> energy_taylor(long double h, long double r0, int n) {
    std::vector<long double> y(n, 0.0L);
    y[0] = -h * r0;
    if (n > 1) y[1] = -h;
    return y;
}

// Interior regularisation of the kernels that are not smooth at 0 (Laplace, energy;
// Rem. 4.2 P:608, reading R24): on ||y|| < eps_I (torus units) K_R(y) = Q(||y||^2) with Q
// the degree p-1 Taylor polynomial of f(s) = K(h sqrt(s)) at s_I = eps_I^2 — a polynomial
// in the coordinates inside the ball (smooth at 0) matching K to order p-1 on the sphere.
// Returns the coefficients of Q in powers of (s - s_I).  Power series: sqrt(s_I + t) by
// the binomial series, then exp of a series (Laplace) or a multiple (energy).
std::vector<double> interior_poly(int kind, long double h, long double ell, long double epsI, int p) {
    const long double sI = epsI * epsI;
    std::vector<long double> g(p);  // sqrt(s_I + t) = sum g_k t^k
    long double c = sqrtl(sI);
    for (int k = 0; k < p; ++k) {
        g[k] = c;
        c *= (0.5L - k) / ((k + 1) * sI);
    }
    std::vector<long double> f(p);
    if (kind == UOTK_ENERGY) {
        for (int k = 0; k < p; ++k) f[k] = -h * g[k];
    } else {  // exp(A(t)), A = -(h/l) g: E_0 = e^{A_0}, E_k = (1/k) sum_{j=1}^k j A_j E_{k-j}
        std::vector<long double> A(p);
        for (int k = 0; k < p; ++k) A[k] = -h / ell * g[k];
        f[0] = expl(A[0]);
        for (int k = 1; k < p; ++k) {
            long double acc = 0;
            for (int j = 1; j <= k; ++j) acc += j * A[j] * f[k - j];
            f[k] = acc / k;
        }
    }
    std::vector<double> out(p);
    for (int k = 0; k < p; ++k) out[k] = (double)f[k];
    return out;
}

// Boundary polynomial K_B on t = (r - r0)/eps_B in [0, 1], r0 = 1/2 - eps_B:
// P^(j)(0) = eps_B^j K^(j)(r0) for j < p (C^{p-1} match with K) and P^(j)(1) = 0 for
// 1 <= j < p (flat at the torus boundary r = 1/2, so the radial extension by the
// constant P(1) is smooth across the sphere ||y|| = 1/2 in every dimension; reading R10).
std::vector<double> boundary_poly(int kind, double h, double param, double eps_B, int p) {
    const long double r0 = 0.5L - eps_B;
    std::vector<long double> y = kind == UOTK_IMQ   ? imq_taylor(h, param, r0, p)
                                 : kind == UOTK_LAP ? lap_taylor(h, param, r0, p)
                                                    : energy_taylor(h, r0, p);
    std::vector<long double> a(p);
    long double e = 1;
    for (int j = 0; j < p; ++j) { a[j] = y[j] * e; e *= eps_B; }
    const int q = p - 1;  // unknown c_i, i = 0..p-2, for t^{p+i}
    std::vector<long double> M(q * q), rhs(q);
    auto ff = [](int n, int k) -> long double {  // n!/(n-k)!
        if (k > n) return 0;
        long double r = 1;
        for (int i = 0; i < k; ++i) r *= (n - i);
        return r;
    };
    for (int k = 1; k <= q; ++k) {
        long double s = 0;
        for (int j = k; j < p; ++j) s += a[j] * ff(j, k);
        rhs[k - 1] = -s;
        for (int i = 0; i < q; ++i) M[(k - 1) * q + i] = ff(p + i, k);
    }
    // Gaussian elimination with partial pivoting
    for (int col = 0; col < q; ++col) {
        int piv = col;
        for (int r = col + 1; r < q; ++r)
            if (fabsl(M[r * q + col]) > fabsl(M[piv * q + col])) piv = r;
        if (piv != col) {
            for (int k = 0; k < q; ++k) std::swap(M[col * q + k], M[piv * q + k]);
            std::swap(rhs[col], rhs[piv]);
        }
        for (int r = col + 1; r < q; ++r) {
            long double f = M[r * q + col] / M[col * q + col];
            for (int k = col; k < q; ++k) M[r * q + k] -= f * M[col * q + k];
            rhs[r] -= f * rhs[col];
        }
    }
    std::vector<long double> cc(q);
    for (int r = q - 1; r >= 0; --r) {
        long double s = rhs[r];
        for (int k = r + 1; k < q; ++k) s -= M[r * q + k] * cc[k];
        cc[r] = s / M[r * q + r];
    }
    std::vector<double> poly(2 * p - 1);
    for (int j = 0; j < p; ++j) poly[j] = (double)a[j];
    for (int i = 0; i < q; ++i) poly[p + i] = (double)cc[i];
    return poly;
}

}  // namespace

FastParams choose_params(int d, int kind, double param, const Geometry& g, const uotk_opts& o) {
    FastParams fp;
    fp.d = d;
    fp.kind = kind;
    fp.param = param;
    for (int t = 0; t < d; ++t) fp.center[t] = g.center[t];
    fp.m = o.m > 0 ? o.m : 8;
    if (fp.m < 2 || fp.m > 8) fail(UOTK_EINVAL, "opts.m must be in [2, 8]");
    fp.flags = o.flags;
    fp.deterministic = o.deterministic != 0;
    if ((fp.flags & UOTK_FLAG_CHUNKED) && !(fp.m == 8 || (fp.m == 6 && d == 3)))
        fail(UOTK_EINVAL, "UOTK_FLAG_CHUNKED needs m = 8 (or m = 6 in d = 3)");
    const double sigma = o.sigma > 0 ? o.sigma : 2.0;
    if (sigma < 1.25) fail(UOTK_EINVAL, "opts.sigma must be >= 1.25");
    const double tol = o.tol > 0 ? o.tol : 1e-16;
    const double L = std::log(1.0 / tol);
    const double rmax = g.rmax;

    double Rbar_max;  // largest torus radius the points may occupy
    double h_min;
    if (kind == UOTK_GAUSS || kind == UOTK_GAUSS_R2) {
        // pure periodisation: pair differences must stay inside the cell (|diff_t| < 1/2)
        Rbar_max = 0.24;
        const double h_decay = 2.0 * std::sqrt(param * L);  // K(h/2) <= tol K(0)
        h_min = h_decay;
        fp.eps_B = 0;
        fp.p = 0;
    } else {  // IMQ, Laplace, energy: boundary polynomial K_B (and for the latter two K_I)
        fp.p = o.p > 0 ? o.p : 12;
        if (fp.p < 2 || fp.p > 16) fail(UOTK_EINVAL, "opts.p must be in [2, 16]");
        fp.eps_B = o.eps_B > 0 ? o.eps_B : 0.1;
        if (fp.eps_B >= 0.25) fail(UOTK_EINVAL, "opts.eps_B must be < 0.25");
        Rbar_max = 0.25 - fp.eps_B / 2;  // pair distances <= 1/2 - eps_B (reading R11)
        h_min = 0;
    }
    double h = std::max(rmax / Rbar_max, h_min);
    if (o.h > 0) {
        if (o.h < rmax / Rbar_max * (1 - 1e-12)) fail(UOTK_EINVAL, "opts.h too small for the point cloud");
        h = o.h;
    }
    if (!(h > 0)) h = (kind == UOTK_IMQ || kind == UOTK_LAP) ? std::max(param, 1e-3) : 1.0;
    fp.h = h;

    int N = o.N;
    if (N <= 0) {
        if (kind == UOTK_GAUSS || kind == UOTK_GAUSS_R2) {
            const double eb = param / (h * h);  // kernel exp(-|y|^2/eb) in torus units
            N = (int)std::ceil(2.0 * std::sqrt(L / (M_PI * M_PI * eb)));
            N = nice_even(std::max(N, 8));
        } else if (kind == UOTK_IMQ) {
            N = (d == 3) ? 192 : 256;
        } else {
            N = 256;  // Laplace / energy: with p = 12, eps_I = p/N (reading R24)
        }
    }
    if (N % 2) fail(UOTK_EINVAL, "opts.N must be even");
    fp.N = N;
    int ng = nice_even((int)std::ceil(sigma * N - 1e-9));
    // the window footprint of every point must stay inside the grid without wrap
    const double Rbar = rmax / h;
    const int ng_min = (int)std::ceil((fp.m + 2) / (0.5 - Rbar));
    if (ng < ng_min) ng = nice_even(ng_min);
    if (ng < 2 * N) ng = nice_even(2 * N);  // keeps k = +-N/2 distinct on the grid
    double grid = std::pow((double)ng, d);
    if (grid > 2.0e9) fail(UOTK_EUNSUPPORTED, "oversampled grid too large");
    fp.ng = ng;
    fp.b = M_PI * (2.0 - (double)N / ng);  // b = pi (2 - 1/sigma_eff)
    {
        // grid coordinates u in [-Rc, Rc] around index n_g/2; taps floor(u) - m + 1 .. floor(u) + m
        const int Rc = (int)std::ceil(Rbar * ng) + 1;
        // even origin and width (ng is even): every box row starts 16-byte aligned, for the
        // chain's 16-byte operand loads (circgemm.cu)
        const int lo = std::max(0, ng / 2 - Rc - fp.m) & ~1;
        const int hi = std::min(ng, (ng / 2 + Rc + fp.m + 1 + 1) & ~1);
        fp.box_lo = lo;
        fp.box_w = hi - lo;
    }
    if (kind == UOTK_IMQ || kind == UOTK_LAP || kind == UOTK_ENERGY)
        fp.poly = boundary_poly(kind, h, param, fp.eps_B, fp.p);
    if (kind == UOTK_LAP || kind == UOTK_ENERGY) {
        fp.eps_I = (double)fp.p / N;
        if (fp.eps_I >= 0.5 - fp.eps_B) fail(UOTK_EINVAL, "eps_I = p/N must stay below 1/2 - eps_B");
        fp.poly_I = interior_poly(kind, h, param, fp.eps_I, fp.p);
    }
    return fp;
}

// ---------------------------------------------------------------------------- kernels
struct KernelCoef {
    int kind;
    double h2;      // h^2
    double param;
    double r0, eps_B;
    int npoly;
    double poly[32];
    double sI;      // eps_I^2 (interior regularisation, Laplace / energy)
    int npolyI;
    double polyI[16];
};

// Samples of the regularised kernel K_R on the N^d grid j/N, j in I_N (stored at j mod N).
template <int D>
__global__ void sample_kernel_k(double* out, int N, KernelCoef kc) {
    int64_t total = 1;
    for (int t = 0; t < D; ++t) total *= N;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t rem = i;
    double r2 = 0;
    for (int t = D - 1; t >= 0; --t) {
        int q = (int)(rem % N);
        rem /= N;
        int j = q < N / 2 ? q : q - N;
        double y = (double)j / N;
        r2 += y * y;
    }
    double v;
    if (kc.kind == UOTK_GAUSS) {
        v = exp(-kc.h2 * r2 / kc.param);
    } else if (kc.kind == UOTK_GAUSS_R2) {
        v = kc.h2 * r2 * exp(-kc.h2 * r2 / kc.param);  // physical r^2 = h^2 r^2 (torus units)
    } else {
        double r = sqrt(r2);
        if (kc.npolyI > 0 && r2 < kc.sI) {  // interior K_I: Q(r^2) (Laplace, energy)
            const double ds = r2 - kc.sI;
            double acc = 0;
            for (int k = kc.npolyI - 1; k >= 0; --k) acc = acc * ds + kc.polyI[k];
            v = acc;
        } else if (r <= kc.r0) {
            const double hr = sqrt(kc.h2) * r;
            v = kc.kind == UOTK_IMQ ? 1.0 / sqrt(kc.h2 * r2 + kc.param * kc.param)
                                    : (kc.kind == UOTK_LAP ? exp(-hr / kc.param) : -hr);
        } else {
            double tt = r >= 0.5 ? 1.0 : (r - kc.r0) / kc.eps_B;
            double acc = 0;
            for (int k = kc.npoly - 1; k >= 0; --k) acc = acc * tt + kc.poly[k];
            v = acc;
        }
    }
    out[i] = v;
}

// D_k on k in [-N/2, N/2]^(d-1) x [0, N/2]; b_k read from the N-point half spectrum.
template <int D>
__global__ void dk_kernel(double* Dk, const double2* bspec, const double* psi, int N) {
    const int nh = N / 2 + 1;     // last axis
    const int nf = N + 1;         // other axes
    int64_t total = nh;
    for (int t = 0; t < D - 1; ++t) total *= nf;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t rem = i;
    int kl = (int)(rem % nh);
    rem /= nh;
    double fac = psi[kl] * ((kl == N / 2) ? 0.5 : 1.0);
    int64_t bidx = kl;
    int64_t bstride = nh;
    for (int t = D - 2; t >= 0; --t) {
        int k = (int)(rem % nf) - N / 2;
        rem /= nf;
        int ak = k < 0 ? -k : k;
        fac *= psi[ak] * ((ak == N / 2) ? 0.5 : 1.0);
        int q = k < 0 ? k + N : k;   // N-periodic index (k = +-N/2 -> N/2)
        bidx += (int64_t)q * bstride;
        bstride *= N;
    }
    double invN = 1.0;
    for (int t = 0; t < D; ++t) invN /= N;
    Dk[i] = fac * bspec[bidx].x * invN;
}

cudaStream_t private_stream();  // context.cu

void PlanData::note_use(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(use_mu);
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return;  // (never inside a capture: plans end with their call)
    }
    for (auto& u : uses)
        if (u.first == s) {
            cudaEventRecord(u.second, s);
            cudaGetLastError();
            return;
        }
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess && cudaEventRecord(e, s) == cudaSuccess)
        uses.emplace_back(s, e);
    else if (e)
        cudaEventDestroy(e);
    cudaGetLastError();
}

// Separable Gaussian: D_k = prod_t d1(|k_t|) on k in [-N/2, N/2]^(d-1) x [0, N/2] (the same
// values dk_kernel forms from the N^d samples' DFT: b_k factors over the axes)
template <int D>
__global__ void dk_separable_k(double* Dk, const double* __restrict__ d1, int N) {
    const int nh = N / 2 + 1, nf = N + 1;
    int64_t total = nh;
    for (int t = 0; t < D - 1; ++t) total *= nf;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t rem = i;
    double f = d1[rem % nh];
    rem /= nh;
    for (int t = D - 2; t >= 0; --t) {
        const int k = (int)(rem % nf) - N / 2;
        rem /= nf;
        f *= d1[k < 0 ? -k : k];
    }
    Dk[i] = f;
}

PlanData::~PlanData() {
    // evicted tables may still be read by kernels queued on the streams that used them:
    // wait for those uses only (not the whole device: unrelated streams, NCCL's included,
    // keep running), then hand the buffers back on the library's own stream
    for (auto& u : uses) {
        cudaEventSynchronize(u.second);
        cudaEventDestroy(u.second);
    }
    if (ready) {
        cudaEventSynchronize(ready);
        cudaEventDestroy(ready);
    }
    cudaGetLastError();
    try {
        cudaStream_t ps = private_stream();
        Dk.s = ps;
        Csep.s = ps;
    } catch (...) {
    }
}

namespace {

// the tables depend on (device, d, kind, N, n_g, m, b, h, kernel parameter, IMQ boundary)
using PlanKey = std::tuple<int, int, int, int, int, int, uint64_t, uint64_t, uint64_t, uint64_t, int, int>;
uint64_t bits(double v) {
    uint64_t u;
    memcpy(&u, &v, sizeof u);
    return u;
}
std::mutex g_plan_mu;
std::list<std::pair<PlanKey, std::shared_ptr<PlanData>>> g_plans;  // most recent first
constexpr size_t kPlanCacheSize = 8;

void build_plan_data(PlanData& pd, const FastParams& fp, cudaStream_t s);

}  // namespace

void release_plan_cache() {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plans.clear();  // tables still referenced by a live SpectralPlan stay until it ends
}

void build_spectral_plan(SpectralPlan& sp, cudaStream_t s) {
    const FastParams& fp = sp.fp;
    const int d = fp.d, ng = fp.ng;
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    static const bool sep_env = [] {
        const char* e = getenv("UOTK_SEPARABLE");
        return !(e && e[0] == '0');
    }();
    const PlanKey key{dev, d, fp.kind, fp.N, ng, fp.m, bits(fp.b), bits(fp.h), bits(fp.param), bits(fp.eps_B), fp.p,
                      sep_env ? 1 : 0};
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        for (auto it = g_plans.begin(); it != g_plans.end(); ++it) {
            if (it->first == key) {
                sp.pd = it->second;
                g_plans.splice(g_plans.begin(), g_plans, it);
                break;
            }
        }
    }
    if (sp.pd) {
        UOTK_CUDA(cudaStreamWaitEvent(s, sp.pd->ready, 0));
    } else {
        auto pd = std::make_shared<PlanData>();
        build_plan_data(*pd, fp, s);
        trace_mark("plan: tables built");
        UOTK_CUDA(cudaEventCreateWithFlags(&pd->ready, cudaEventDisableTiming));
        UOTK_CUDA(cudaEventRecord(pd->ready, s));
        sp.pd = pd;
        std::lock_guard<std::mutex> lk(g_plan_mu);
        g_plans.emplace_front(key, pd);
        if (g_plans.size() > kPlanCacheSize) g_plans.pop_back();
    }
    // The separable chain costs d GEMM passes of w^(d+1) MACs on the footprint box (w =
    // box_w), the cuFFT chain ~ n_g^d grid traffic: the separable one wins on the compact
    // boxes of C3 / C4-auto (21 / 16 us vs 74 / 29 us), cuFFT on C4's literal 4096^2 grid
    // (0.36 ms vs 1.18 ms per chain, w = 1982; scripts/chain_probe.py).  Estimates from those
    // measurements (DMMA GEMMs at ~25 TFLOP/s + ~5 us per pass; cuFFT ~25 us + 20 ps per
    // grid point); the cuFFT chain only when it is clearly cheaper.
    sp.sep_chain = sp.pd->separable && !(fp.flags & UOTK_FLAG_FFT);
    if (sp.sep_chain) {
        const double w = fp.box_w, g = std::pow((double)ng, d);
        const double t_sep = 2.0 * d * std::pow(w, d + 1) / 25e12 + 5e-6 * d;
        const double t_fft = 25e-6 + 2e-11 * g;
        if (t_fft < 0.7 * t_sep) sp.sep_chain = false;
    }
    // the full-grid cuFFT plans only where the full chain runs (fft_chain also creates them
    // on first use: the separable Gaussian chain and the pruned MMD^2 transform never do)
    if (!sp.sep_chain) get_fft_plans(d, ng, &sp.r2c, &sp.c2r);
    sp.use_stream = s;
    sp.grid_elems = 1;
    for (int t = 0; t < d; ++t) sp.grid_elems *= ng;
    sp.spec_elems = sp.grid_elems / ng * (ng / 2 + 1);
}

namespace {

void build_plan_data_separable(PlanData& pd, const FastParams& fp, cudaStream_t s);
std::vector<double> deconv_psi(const FastParams& fp);

void build_plan_data(PlanData& pd, const FastParams& fp, cudaStream_t s) {
    static const bool sep_env0 = [] {
        const char* e = getenv("UOTK_SEPARABLE");
        return !(e && e[0] == '0');
    }();
    if (fp.kind == UOTK_GAUSS && sep_env0) return build_plan_data_separable(pd, fp, s);
    const int d = fp.d, N = fp.N, ng = fp.ng;
    // 1) samples of K_R and their DFT -> b_k (real: K_R is real and even)
    size_t nsamp = 1;
    for (int t = 0; t < d; ++t) nsamp *= N;
    size_t nspec = nsamp / N * (N / 2 + 1);
    DevBuf<double> samp(nsamp, s);
    DevBuf<double2> bspec(nspec, s);
    KernelCoef kc{};
    kc.kind = fp.kind;
    kc.h2 = fp.h * fp.h;
    kc.param = fp.param;
    kc.eps_B = fp.eps_B;
    kc.r0 = 0.5 - fp.eps_B;
    kc.npoly = (int)fp.poly.size();
    if (kc.npoly > 32) fail(UOTK_EINVAL, "boundary polynomial too long");
    for (int k = 0; k < kc.npoly; ++k) kc.poly[k] = fp.poly[k];
    kc.sI = fp.eps_I * fp.eps_I;
    kc.npolyI = (int)fp.poly_I.size();
    if (kc.npolyI > 16) fail(UOTK_EINVAL, "interior polynomial too long");
    for (int k = 0; k < kc.npolyI; ++k) kc.polyI[k] = fp.poly_I[k];
    const int tb = 256;
    int gb = (int)((nsamp + tb - 1) / tb);
    if (d == 1) sample_kernel_k<1><<<gb, tb, 0, s>>>(samp.p, N, kc);
    else if (d == 2) sample_kernel_k<2><<<gb, tb, 0, s>>>(samp.p, N, kc);
    else sample_kernel_k<3><<<gb, tb, 0, s>>>(samp.p, N, kc);
    UOTK_LAUNCHED();
    cufftHandle r2c, c2r;
    get_fft_plans(d, N, &r2c, &c2r);
    UOTK_CUFFT(cufftSetStream(r2c, s));
    UOTK_CUFFT(cufftExecD2Z(r2c, samp.p, (cufftDoubleComplex*)bspec.p));

    // 2) per-axis deconvolution psi(k) = 1/(n_g^2 phihat(k)^2), k = 0..N/2 (deconv_psi)
    const std::vector<double> psi = deconv_psi(fp);
    DevBuf<double> psi_d(psi.size(), s);
    UOTK_CUDA(cudaMemcpyAsync(psi_d.p, psi.data(), psi.size() * sizeof(double), cudaMemcpyHostToDevice, s));

    // 3) D_k table
    size_t ndk = (size_t)(N / 2 + 1);
    for (int t = 0; t < d - 1; ++t) ndk *= (N + 1);
    pd.Dk.alloc(ndk, s);
    gb = (int)((ndk + tb - 1) / tb);
    if (d == 1) dk_kernel<1><<<gb, tb, 0, s>>>(pd.Dk.p, bspec.p, psi_d.p, N);
    else if (d == 2) dk_kernel<2><<<gb, tb, 0, s>>>(pd.Dk.p, bspec.p, psi_d.p, N);
    else dk_kernel<3><<<gb, tb, 0, s>>>(pd.Dk.p, bspec.p, psi_d.p, N);
    UOTK_LAUNCHED();
    // psi_d / samp / bspec are freed stream-ordered after the kernels that use them

    pd.separable = false;
}

// Kaiser-Bessel pair  phi(v) = sinh(b sqrt(m^2 - v^2))/sqrt(m^2 - v^2) * m/sinh(b m) (v in grid
// units) and phihat(k) = (pi m / n_g) I0(m sqrt(b^2 - (2 pi k/n_g)^2)) / sinh(b m):
// psi(k) = 1/(n_g^2 phihat(k)^2), k = 0..N/2
std::vector<double> deconv_psi(const FastParams& fp) {
    const int N = fp.N, ng = fp.ng;
    std::vector<double> psi(N / 2 + 1);
    const long double m = fp.m, b = fp.b;
    const long double sinh_bm = sinhl(b * m);
    for (int k = 0; k <= N / 2; ++k) {
        long double w = 2.0L * M_PI * k / ng;
        long double z = m * sqrtl(b * b - w * w);
        long double ph = (long double)M_PI * m / ng * bessel_i0(z) / sinh_bm;
        psi[k] = (double)(1.0L / ((long double)ng * ng * ph * ph));
    }
    return psi;
}

// The Gaussian's tables without the N^d samples and their DFT (no cuFFT plan): the samples
// exp(-h^2 |j/N|^2 / eps) factor over the axes, hence so do b_k and D_k = prod_t d1(k_t),
// d1(k) = psi(k) w(k) b1(k) / N with b1 the 1-D DFT of the samples (the same factors
// dk_kernel multiplies).  The chain F^-1 (D .* F g) is then (Csep x ... x Csep) g with the
// real symmetric circulant Csep[l][l'] = c(l - l'),  c(D) = d1(0) + 2 sum_{k=1}^{N/2} d1(k)
// cos(2 pi k D / n_g)  (k = +-N/2 carry weight 1/2 each, as in the FFT path).
void build_plan_data_separable(PlanData& pd, const FastParams& fp, cudaStream_t s) {
    const int d = fp.d, N = fp.N, ng = fp.ng;
    const std::vector<double> psi = deconv_psi(fp);
    std::vector<long double> d1(N / 2 + 1);
    const long double h2e = (long double)fp.h * fp.h / fp.param;
    for (int k = 0; k <= N / 2; ++k) {
        long double b1 = 0;
        for (int j = -N / 2; j < N / 2; ++j) {
            const long double y = (long double)j / N;
            b1 += expl(-h2e * y * y) * cosl(2.0L * M_PI * k * j / N);
        }
        d1[k] = (long double)psi[k] * (k == N / 2 ? 0.5L : 1.0L) * b1 / N;
    }
    std::vector<double> d1d(N / 2 + 1), cvec(ng), C((size_t)ng * ng);
    for (int k = 0; k <= N / 2; ++k) d1d[k] = (double)d1[k];
    for (int D = 0; D < ng; ++D) {
        long double c = d1[0];
        for (int k = 1; k <= N / 2; ++k) c += 2.0L * d1[k] * cosl(2.0L * M_PI * k * D / ng);
        cvec[D] = (double)c;
    }
    for (int l = 0; l < ng; ++l)
        for (int lp = 0; lp < ng; ++lp) C[(size_t)l * ng + lp] = cvec[((l - lp) % ng + ng) % ng];
    pd.Csep.alloc(C.size(), s);
    UOTK_CUDA(cudaMemcpyAsync(pd.Csep.p, C.data(), C.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    DevBuf<double> d1_dev(d1d.size(), s);
    UOTK_CUDA(cudaMemcpyAsync(d1_dev.p, d1d.data(), d1d.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    size_t ndk = (size_t)(N / 2 + 1);
    for (int t = 0; t < d - 1; ++t) ndk *= (N + 1);
    pd.Dk.alloc(ndk, s);
    const int gb = (int)((ndk + 255) / 256);
    if (d == 1) dk_separable_k<1><<<gb, 256, 0, s>>>(pd.Dk.p, d1_dev.p, N);
    else if (d == 2) dk_separable_k<2><<<gb, 256, 0, s>>>(pd.Dk.p, d1_dev.p, N);
    else dk_separable_k<3><<<gb, 256, 0, s>>>(pd.Dk.p, d1_dev.p, N);
    UOTK_LAUNCHED();
    UOTK_CUDA(cudaStreamSynchronize(s));  // C, d1d live on the host stack frame
    pd.separable = true;
}

}  // namespace

}  // namespace uotk
