// Small per-point kernels and deterministic reductions used by the Sinkhorn and MMD
// drivers: objective terms of the recovered plan, mass
// validation, and column sums in a fixed order (two passes, no atomics).
#include "common.cuh"
#include "reduce.cuh"

namespace uotk {

namespace {

constexpr int kRB = 256;
constexpr int kRBlocks = 296;  // 2 x 148 SMs

__global__ void colsum_partial_k(const double* __restrict__ vals, int64_t n, int ncols, double* __restrict__ part) {
    __shared__ double sm[kRB];
    for (int c = 0; c < ncols; ++c) {
        double acc = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)kRB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRB)
            acc += vals[c * n + i];
        sm[threadIdx.x] = acc;
        __syncthreads();
        for (int w = kRB / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) part[c * gridDim.x + blockIdx.x] = sm[0];
        __syncthreads();
    }
}

__global__ void colsum_final_k(const double* __restrict__ part, int nb, int ncols, double* __restrict__ out) {
    __shared__ double sm[kRB];
    for (int c = 0; c < ncols; ++c) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < nb; b += kRB) acc += part[c * nb + b];
        sm[threadIdx.x] = acc;
        __syncthreads();
        for (int w = kRB / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[c] = sm[0];
        __syncthreads();
    }
}

// Terms of the objectives at one side of the plan, from pot (beta or gamma), the
// mass (mu or nu) and the kernel sum t against the other side's scaled masses:
//   p = mass e^{lam pot} t          (row / column marginal of pi)
//   col 0: p     col 1: pot * p     col 2: p log(p / mass)
//   col 3: mass e^{-pot/eta}        col 4: mass
__global__ void uot_terms_k(const double* __restrict__ pot, const double* __restrict__ mass,
                            const double* __restrict__ t, int64_t n, double lam, double eta,
                            double* __restrict__ cols) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double mu = mass[i], b = pot[i];
    const double p = mu * exp(lam * b) * t[i];
    cols[0 * n + i] = p;
    cols[1 * n + i] = b * p;
    cols[2 * n + i] = p > 0.0 ? p * log(p / mu) : 0.0;
    cols[3 * n + i] = mu * exp(-b / eta);
    cols[4 * n + i] = mu;
}

__global__ void check_mass_k(const double* __restrict__ a, int64_t n, int* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const double v = a[i];
        if (!(v > 0.0) || !isfinite(v)) atomicOr(flag, 4);
    }
}

__global__ void check_finite_k(const double* __restrict__ a, int64_t n, int* __restrict__ flag, int bit) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !isfinite(a[i])) atomicOr(flag, bit);
}

__global__ void multiply_k(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ prod) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) prod[i] = a[i] * b[i];
}

__global__ void split_bits_k(const int* __restrict__ flag, int32_t* __restrict__ bits) {
    if (threadIdx.x < 4) bits[threadIdx.x] = (*flag >> threadIdx.x) & 1;
}

__global__ void join_bits_k(const int32_t* __restrict__ bits, int* __restrict__ flag) {
    if (threadIdx.x == 0) *flag = bits[0] | (bits[1] << 1) | (bits[2] << 2) | (bits[3] << 3);
}

// w = mass * exp(lam * pot)
__global__ void scaled_mass_k(const double* __restrict__ mass, const double* __restrict__ pot, int64_t n, double lam,
                              double* __restrict__ w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) w[i] = pot ? mass[i] * exp(lam * pot[i]) : mass[i];
}

// ws[i] = w[perm[i]] with w = (a, -b): MMD^2's signed weights in sorted order, read from
// the caller's two arrays
__global__ void permute_signed_k(double* __restrict__ ws, const double* __restrict__ a, int64_t n,
                                 const double* __restrict__ b, const int32_t* __restrict__ perm, int64_t nz) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nz) return;
    const int64_t j = perm[i];
    ws[i] = j < n ? a[j] : -b[j - n];
}

__global__ void signed_concat_k(const double* __restrict__ a, int64_t n, const double* __restrict__ b, int64_t m,
                                double* __restrict__ w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) w[i] = a[i];
    else if (i < n + m) w[i] = -b[i - n];
}

// moment columns of one weighted point set (row-major n x d), around a centre c:
//   col 0: a_i   col 1: a_i ||x_i - c||^2   col 2 + t: a_i (x_it - c_t)
__global__ void moment_cols_k(const double* __restrict__ x, const double* __restrict__ a, int64_t n, int d,
                              const double* __restrict__ c, double* __restrict__ cols) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double ai = a[i];
    double r2 = 0.0;
    for (int t = 0; t < d; ++t) {
        const double v = x[i * d + t] - (c ? c[t] : 0.0);
        r2 = fma(v, v, r2);
        cols[(2 + t) * n + i] = ai * v;
    }
    cols[i] = ai;
    cols[n + i] = ai * r2;
}

// w_i t'_i with w = mass e^{lam pot}: the summands of <pi, d^2> (t' = the d^2 k sum)
__global__ void transport_k(const double* __restrict__ pot, const double* __restrict__ mass,
                            const double* __restrict__ tp, int64_t n, double lam, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = mass[i] * exp(lam * pot[i]) * tp[i];
}

inline int blocks_for(int64_t n, int tb) { return (int)std::max<int64_t>(1, (n + tb - 1) / tb); }

}  // namespace

void uot_transport(const double* pot, const double* mass, const double* tp, int64_t n, double lam, double* out,
                   cudaStream_t s) {
    if (n == 0) return;
    transport_k<<<blocks_for(n, 256), 256, 0, s>>>(pot, mass, tp, n, lam, out);
    UOTK_LAUNCHED();
}

void moment_cols(const double* x, const double* a, int64_t n, int d, const double* c, double* cols, cudaStream_t s) {
    if (n == 0) return;
    moment_cols_k<<<blocks_for(n, 256), 256, 0, s>>>(x, a, n, d, c, cols);
    UOTK_LAUNCHED();
}

void sum_columns(const double* vals, int64_t n, int ncols, double* out_dev, cudaStream_t s) {
    DevBuf<double> part((size_t)ncols * kRBlocks, s);
    colsum_partial_k<<<kRBlocks, kRB, 0, s>>>(vals, n, ncols, part.p);
    UOTK_LAUNCHED();
    colsum_final_k<<<1, kRB, 0, s>>>(part.p, kRBlocks, ncols, out_dev);
    UOTK_LAUNCHED();
}

void uot_terms(const double* pot, const double* mass, const double* t, int64_t n, double lam, double eta,
               double* cols, cudaStream_t s) {
    if (n == 0) return;
    uot_terms_k<<<blocks_for(n, 256), 256, 0, s>>>(pot, mass, t, n, lam, eta, cols);
    UOTK_LAUNCHED();
}

void check_mass(const double* a, int64_t n, int* flag, cudaStream_t s) {
    if (n == 0) return;
    check_mass_k<<<blocks_for(n, 256), 256, 0, s>>>(a, n, flag);
    UOTK_LAUNCHED();
}

void check_finite(const double* a, int64_t n, int* flag, int bit, cudaStream_t s) {
    if (n == 0) return;
    check_finite_k<<<blocks_for(n, 256), 256, 0, s>>>(a, n, flag, bit);
    UOTK_LAUNCHED();
}

void multiply(const double* a, const double* b, int64_t n, double* prod, cudaStream_t s) {
    if (n == 0) return;
    multiply_k<<<blocks_for(n, 256), 256, 0, s>>>(a, b, n, prod);
    UOTK_LAUNCHED();
}

void split_bits(const int* flag, int32_t* bits, cudaStream_t s) {
    split_bits_k<<<1, 32, 0, s>>>(flag, bits);
    UOTK_LAUNCHED();
}

void join_bits(const int32_t* bits, int* flag, cudaStream_t s) {
    join_bits_k<<<1, 32, 0, s>>>(bits, flag);
    UOTK_LAUNCHED();
}

void scaled_mass(const double* mass, const double* pot, int64_t n, double lam, double* w, cudaStream_t s) {
    if (n == 0) return;
    scaled_mass_k<<<blocks_for(n, 256), 256, 0, s>>>(mass, pot, n, lam, w);
    UOTK_LAUNCHED();
}

void permute_signed(double* ws, const double* a, int64_t n, const double* b, const int32_t* perm, int64_t nz,
                    cudaStream_t s) {
    if (nz == 0) return;
    permute_signed_k<<<blocks_for(nz, 256), 256, 0, s>>>(ws, a, n, b, perm, nz);
    UOTK_LAUNCHED();
}

void signed_concat(const double* a, int64_t n, const double* b, int64_t m, double* w, cudaStream_t s) {
    if (n + m == 0) return;
    signed_concat_k<<<blocks_for(n + m, 256), 256, 0, s>>>(a, n, b, m, w);
    UOTK_LAUNCHED();
}

}  // namespace uotk
