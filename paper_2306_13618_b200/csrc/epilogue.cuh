// Per-point epilogues applied to a freshly computed kernel sum t_i (K5 in DESIGN.md).
#pragma once
#include <cstdint>

namespace uotk {

// out[perm[i]] = t  (perm == nullptr -> out[i] = t): the plain kernel sum (4.3).
struct EpiStore {
    double* out;
    const int32_t* perm;
    __device__ __forceinline__ double operator()(int64_t i, double t) const {
        out[perm ? perm[i] : i] = t;
        return 0.0;
    }
    __device__ __forceinline__ void prefetch(int64_t) const {}
    // software-pipelined form used by the chunked kernels: load() the per-point inputs a
    // chunk ahead, apply() them; apply returns the sup-norm change and the next weight
    struct In {};
    __device__ __forceinline__ In load(int64_t) const { return {}; }
    __device__ __forceinline__ double apply(int64_t i, double t, const In&, double& w) const {
        w = 0.0;
        return (*this)(i, t);
    }
};

// One Sinkhorn half-step, (3.3) / (3.4) in scaling form:
//   pot_i   <- -c log t_i            (c = eta/(1 + eta*lambda))
//   w_next  <- mass_i * exp(lambda * pot_i)   (= mass_i * t_i^(-eta*lambda/(1+eta*lambda)))
// Returns |pot_new - pot_old| for the sup-norm change; flags t <= 0 or non-finite.
struct EpiSinkhorn {
    double* pot;
    const double* mass;
    double* w_next;
    double* t_store;  // optional copy of t (for the plan marginals)
    double c;
    double lam;
    int* flag;
    __device__ __forceinline__ double operator()(int64_t i, double t) const {
        if (!(t > 0.0) || !isfinite(t)) {
            atomicOr(flag, 1);
            t = 1.0;
        }
        const double pnew = -c * log(t);
        const double dd = fabs(pnew - pot[i]);
        pot[i] = pnew;
        const double w = mass[i] * exp(lam * pnew);
        if (!isfinite(w)) atomicOr(flag, 2);
        w_next[i] = w;
        if (t_store) t_store[i] = t;
        return dd;
    }
    __device__ __forceinline__ void prefetch(int64_t i) const {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(mass + i));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pot + i));
    }
    struct In {
        double pot, mass;
    };
    __device__ __forceinline__ In load(int64_t i) const { return {pot[i], mass[i]}; }
    // operator() with the inputs preloaded; also returns the next weight w (no re-read)
    __device__ __forceinline__ double apply(int64_t i, double t, const In& in, double& w) const {
        if (!(t > 0.0) || !isfinite(t)) {
            atomicOr(flag, 1);
            t = 1.0;
        }
        const double pnew = -c * log(t);
        pot[i] = pnew;
        w = in.mass * exp(lam * pnew);
        if (!isfinite(w)) atomicOr(flag, 2);
        w_next[i] = w;
        if (t_store) t_store[i] = t;
        return fabs(pnew - in.pot);
    }
    // the same next weight without side effects (bit-identical to operator()'s w_next)
    __device__ __forceinline__ double weight(int64_t i, double t) const {
        if (!(t > 0.0) || !isfinite(t)) t = 1.0;
        const double pnew = -c * log(t);
        return mass[i] * exp(lam * pnew);
    }
};

// prod[i] = w[i] * t (MMD^2 quadratic form sum_i w_i (K w)_i, reduced afterwards).
struct EpiDot {
    const double* w;
    double* prod;
    __device__ __forceinline__ double operator()(int64_t i, double t) const {
        prod[i] = w[i] * t;
        return 0.0;
    }
    __device__ __forceinline__ void prefetch(int64_t) const {}
    struct In {
        double w;
    };
    __device__ __forceinline__ In load(int64_t i) const { return {w[i]}; }
    __device__ __forceinline__ double apply(int64_t i, double t, const In& in, double& wn) const {
        wn = 0.0;
        prod[i] = in.w * t;
        return 0.0;
    }
};

// Chunked-kernel adaptors: the Sinkhorn epilogue exposes w_next / weight(); the plain
// gathers do not spread, and a spread-only pass has no epilogue at all.
struct EpiNone {
    double* w_next = nullptr;
    __device__ double operator()(int64_t, double) const { return 0.0; }
    __device__ double weight(int64_t, double) const { return 0.0; }
    __device__ void prefetch(int64_t) const {}
    struct In {};
    __device__ In load(int64_t) const { return {}; }
    __device__ double apply(int64_t, double, const In&, double& w) const {
        w = 0.0;
        return 0.0;
    }
};
template <class Epi>
struct EpiGatherOnly : Epi {
    double* w_next = nullptr;
    __device__ double weight(int64_t, double) const { return 0.0; }
};

// warp max of non-negative doubles, one atomicMax per warp on the uint64 bit pattern
__device__ __forceinline__ void warp_max_atomic(unsigned long long* dst, double v) {
    if (!dst) return;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(dst, (unsigned long long)__double_as_longlong(v));
}

}  // namespace uotk
