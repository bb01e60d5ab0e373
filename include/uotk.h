/*
 * uotk.h — C ABI of the B200 fast radial-kernel library for arXiv 2306.13618
 * ("Unbalanced Optimal Transport and Maximum Mean Discrepancies: Interconnections
 * and Rapid Evaluation", Lakshmanan & Pichler).
 *
 * Citations: "P:n" = line n of the paper text, with its section /
 * equation / algorithm; "S:n" = line n of SPEC.md (interfaces only, not binding).
 *
 * The library evaluates the radial-kernel product K v, K_ij = k(||x_i - y_j||),
 * by NFFT-based fast summation (Sec. 4; factorisation (4.5)-(4.6),
 * P:590-592) or by a direct O(n m) sum (Eq. 4.3), and uses it inside the
 * entropic unbalanced-OT Sinkhorn iteration (Algorithm 2) and the
 * MMD^2 sums (Eq. 3.5).  Every step runs in hand-written sm_100a kernels
 * except two library calls: cuFFT provides the equispaced FFT of (4.6) where the
 * cuFFT chain is chosen, and CUB provides the radix sort of the points by cell and
 * the run-length encode / scans of the chunk layout (setup, once per call).
 *
 * Conventions shared by all entry points
 * --------------------------------------
 *  - Points are row-major n x d arrays of double (x in R^{n x d}, Alg. 2 input,
 *    P:616), d in {1, 2, 3} (the paper restricts to d <= 3).
 *  - Every array argument may be DEVICE memory (cudaMalloc / torch cuda tensor)
 *    or HOST memory (pinned or pageable); the library detects which with
 *    cudaPointerGetAttributes.  Host inputs are copied to device workspaces and
 *    host outputs copied back, all on `cuda_stream`.  All arrays are caller-owned;
 *    the library never retains a pointer after the call returns.
 *  - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *    enqueued on it.  Calls that return host scalars (uot result, mmd2) or write
 *    host outputs synchronise the stream before returning; a call with only
 *    device outputs returns without synchronising.
 *  - Outputs are in the CALLER's point order (the library sorts internally).
 *  - `opts` may be NULL (defaults, see uotk_opts_init).
 *  - `comm` is a uotk_comm created by uotk_comm_create, or NULL for one GPU.
 *    With a communicator every rank passes its LOCAL shard of the points; the
 *    oversampled Fourier coefficients of each kernel sum are summed over ranks
 *    (NCCL all-reduce of the truncated I_N spectrum; for the Gaussian's separable
 *    chain a reduce-scatter of the first pass's blocks, the middle pass on 1/P of
 *    the box per rank and an all-gather: UOTK_DIST_CHAIN=0 keeps one all-reduce)
 *    so each rank obtains the sums at its own targets from all ranks' sources.  Scalar results (uot result, mmd2) are global and
 *    identical on all ranks.
 *    A rank's local shard may be empty (n = 0 or m = 0) with a multi-rank
 *    communicator: it still takes part in every collective.  Input and numeric
 *    errors (UOTK_EDOMAIN, UOTK_EOVERFLOW) are decided on flags or-ed over all ranks,
 *    so every rank returns the same status, and the stopping rule's sup-norm changes
 *    are maxed over ranks (all ranks stop at the same iteration).
 *  - Return value: UOTK_OK (0) or a negative status; uotk_last_error() returns a
 *    thread-local description of the last failure.  No C++ exception crosses
 *    the ABI.  Several host threads may call the library concurrently on one
 *    device only as the ranks of one loopback group (uotk_comm_create_loopback).
 */
#ifndef UOTK_H
#define UOTK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UOTK_ABI_VERSION 3

/* Status codes (mirroring SPEC's split of input vs numeric errors). */
enum {
    UOTK_OK = 0,
    UOTK_EINVAL = -1,       /* null pointer, d not in {1,2,3}, negative size, eps/lam/param <= 0, bad opts */
    UOTK_EDOMAIN = -2,      /* non-finite coordinate, or (UOT) a mass <= 0 or non-finite (KL needs mu_i > 0) */
    UOTK_EOVERFLOW = -3,    /* non-finite or non-positive intermediate t, u, v in Sinkhorn */
    UOTK_ENOMEM = -4,       /* device allocation failed */
    UOTK_ECUDA = -5,        /* CUDA runtime / kernel error */
    UOTK_ECUFFT = -6,       /* cuFFT error */
    UOTK_ENCCL = -7,        /* NCCL error or NCCL library not loadable */
    UOTK_EUNSUPPORTED = -8  /* parameter combination the library does not support (e.g. grid too large) */
};

/* Radial kernels of Eq. (4.2), P:560 (Table 1), as functions of r = ||x - y||:
 *   UOTK_GAUSS:  k(r) = exp(-r^2 / param)          (param = l^2 = eps in the configs' form)
 *   UOTK_IMQ:    k(r) = 1 / sqrt(r^2 + param^2)    (param = c)
 *   UOTK_LAP:    k(r) = exp(-r / param)            (param = l; Laplace kernel K^Lap)
 *   UOTK_ENERGY: k(r) = -r                         (Table 1's energy kernel k^e = -K^abs;
 *                                                   param is ignored, pass any value > 0)
 * LAP and ENERGY are not smooth at r = 0: their NFFT path regularises the kernel inside
 * ||y|| < eps_I (torus units, eps_I = p/N) and adds the exact near-field correction
 * sum_{||x_i - y_j|| < eps_I h} (k - K_R)(x_i - y_j) alpha_j (reading R24). */
typedef enum { UOTK_GAUSS = 0, UOTK_IMQ = 1, UOTK_GAUSS_R2 = 2, UOTK_LAP = 3, UOTK_ENERGY = 4 } uotk_kernel_kind;
/*   UOTK_GAUSS_R2: k(r) = r^2 exp(-r^2 / param)  (kernel sums only: the transport-cost
 *                  kernel of the Gibbs plan, d^2 k_ij, giving <pi, d^2> of P:462)    */

/* Evaluation method.  AUTO picks DIRECT when n_src * n_tgt is below a measured
 * crossover and NFFT otherwise. */
typedef enum { UOTK_AUTO = 0, UOTK_NFFT = 1, UOTK_DIRECT = 2 } uotk_method;

/* Fast-summation parameters (Rem. 4.4 P:612 and footnote P:653 leave them to the
 * implementation; defaults and auto rules are in DESIGN.md "Parameters").
 * A zero field means "automatic / default". */
typedef struct {
    int32_t method;   /* uotk_method                                                     */
    int32_t N;        /* bandwidth per axis of I_N (Eq. 4.4), even; 0 = auto       */
    double sigma;     /* oversampling: grid n_g = sigma * N per axis (even); 0 = 2.0      */
    int32_t m;        /* window half-width; 2m taps per axis (footnote P:653); 0 = 8.
                         Tuned cell-group kernels: m = 8 (d = 1..3) and m = 6 (d = 3; with
                         sigma = 3 its window error ~4e-12, R23); other m run on
                         the generic kernels                                              */
    int32_t p;        /* IMQ boundary polynomial order (K_B); 0 = 12          */
    double eps_B;     /* IMQ boundary band width in torus units; 0 = auto                 */
    double h;         /* torus scaling h (Eq. 4.7, Rem. 4.3 P:610); 0 = auto        */
    double tol;       /* target truncation tolerance of the auto rules; 0 = 1e-16        */
    int32_t flags;    /* UOTK_FLAG_* bits below; 0 = automatic                           */
    int32_t deterministic; /* 1 = bitwise reproducible results (run to run, any launch
                         configuration): every spread pulls each grid value in the points'
                         sorted order instead of accumulating with fp64 atomics, and the
                         fused half-steps run as gather + spread; slower.
                         0 = default (atomics; results reproducible to ~1e-15)            */
    /* Sinkhorn stopping rule (reading R20 of DESIGN.md; the paper's "while stopping
     * criteria"): with stop_tol > 0, after every check_every-th iteration the
     * loop ends once the sup-norm changes of beta and gamma within that iteration are
     * both <= stop_tol; `iters` is then the cap and uotk_uot_result.iters the count. */
    double stop_tol;     /* 0 = run exactly `iters` iterations                            */
    int32_t check_every; /* 0 = 10                                                        */
    int32_t reserved2;   /* must be 0                                                     */
} uotk_opts;

/* opts.flags: which spread/gather kernels the NFFT path may use (results agree to
 * rounding; for cross-checks and benchmarks).  By default the cell-group kernels
 * (points sorted by cell, chunks of <= 32 points sharing one window footprint,
 * DESIGN.md §7) run whenever m = 8 (or m = 6 in d = 3) and the point set is dense enough, else the
 * generic thread-per-point kernels.  At most one of the two bits may be set. */
#define UOTK_FLAG_GENERIC 1  /* always the generic thread-per-point kernels          */
#define UOTK_FLAG_CHUNKED 2  /* cell-group kernels at any density (m = 8; d = 3: or 6) */
#define UOTK_FLAG_TRANSPORT 4 /* uot: also evaluate the transport term <pi, d^2>    */
#define UOTK_FLAG_FFT 8       /* always the cuFFT chain (D2Z, D_k, Z2D), never the separable
                                 circulant GEMMs of the Gaussian (with a communicator those
                                 are slab-distributed: reduce-scatter / all-gather)        */
#define UOTK_FLAG_COST_R1 16  /* uot: cost d^1 instead of d^2, i.e. the Laplace Gibbs kernel
                                 exp(-||x - y|| / eps) (Algorithm 2's r = 1);
                                 not combinable with UOTK_FLAG_TRANSPORT                     */

/* What a call actually used (any pointer to it may be NULL). */
typedef struct {
    int32_t method_used; /* UOTK_NFFT or UOTK_DIRECT */
    int32_t N;           /* bandwidth (0 for DIRECT) */
    int32_t n_grid;      /* oversampled grid points per axis (0 for DIRECT) */
    int32_t m;           /* window half-width (0 for DIRECT) */
    double h;            /* torus scaling (0 for DIRECT) */
    /* Cell-group layout of the two point sets on the NFFT path: 0 = the
     * generic thread-per-point kernels; otherwise the z extent of a group's window
     * footprint: 16 = one-cell groups (m = 8; in d = 3 the warp-specialised half-step
     * sinkhorn3d_ws_k), 12 = one-cell groups with m = 6, 24 / 40 = z-segment groups of
     * sparse d = 3 clouds, 1624 = hybrid groups of a d = 3 spread-only set (cells with
     * >= 24 points alone, the sparser cells in 9-cell z-segments; windows evaluated in the
     * spread).  Set 1 = src (kernel sum), x (UOT) or z = x u y (MMD^2);
     * set 2 = tgt (kernel sum) or y (UOT), 0 for MMD^2. */
    int32_t groups1;
    int32_t groups2;
    int32_t nranks;      /* ranks of the communicator (1 without one) */
    int32_t reserved;
} uotk_info;

/* Result of uotk_uot_sinkhorn, all global over ranks.
 * Objective values of the plan pi = e^{lam beta} k e^{lam gamma} (.) (mu x nu) recovered
 * from the final potentials, lam = 1/eps:
 *   primal     discrete primal of (2.9), via the plan's marginals
 *   dual       dual function (3.1) of Theorem 3.1
 *   plan_mass  pi(X x X) = sum_i p_i
 *   mass_a     mu(X);  mass_b  nu(X)
 *   max_dbeta, max_dgamma   sup-norm change of beta / gamma in the last iteration */
typedef struct {
    double primal;
    double dual;
    double plan_mass;
    double mass_a;
    double mass_b;
    double max_dbeta;
    double max_dgamma;
    int32_t iters;
    int32_t reserved;
    uotk_info info;
    double transport;   /* <pi, d^2> = sum_ij pi_ij ||x_i - y_j||^2 with
                           UOTK_FLAG_TRANSPORT, else NaN */
} uotk_uot_result;

/* Fill *opts with the defaults (all automatic). */
void uotk_opts_init(uotk_opts* opts);

/*
 * Kernel sum, Eq. (4.3):
 *     out_i = sum_j k(||tgt_i - src_j||) alpha_j ,   i < n_tgt.
 * src: n_src x d, alpha: n_src (any sign), tgt: n_tgt x d, out: n_tgt.
 * n_src = 0 gives out = 0; n_tgt = 0 is a no-op.
 * NFFT path: adjoint NFFT of alpha at src (window spreading), FFT, multiplication
 * by the regularised kernel's Fourier coefficients b_k (Eq. 4.4-4.6), inverse FFT,
 * interpolation at tgt.  With `comm`, src/alpha/tgt/out are local shards.
 */
int uotk_kernel_sum(int d, int64_t n_src, const double* src, const double* alpha,
                    int64_t n_tgt, const double* tgt, int kind, double param,
                    double* out, const uotk_opts* opts, uotk_info* info,
                    void* comm, void* cuda_stream);

/*
 * Entropic unbalanced OT by Sinkhorn iterations, Algorithm 2 / Algorithm 1
 * with the Gibbs kernel k_ij = exp(-||x_i - y_j||^2 / eps) (r = 2).
 *   x: n x d, a: n masses (mu_i > 0);  y: m x d, b: m masses (nu_j > 0)
 *   eps   entropic regularisation = 1/lambda of the paper (Def. 2.7)
 *   lam1, lam2   marginal KL penalties eta_1, eta_2 (configs use lam1 = lam2)
 *   iters        number of iterations; one iteration = the beta-step (3.3) followed by
 *                the gamma-step (3.4), i.e. two kernel sums; iters >= 0
 *   gamma_init   starting gamma^0 (m values) or NULL for gamma^0 = 0
 *   beta, gamma  outputs: final dual potentials (n and m values)
 *   res          output: objective values (see uotk_uot_result); may be NULL
 * With iters = 0 the outputs are beta = 0, gamma = gamma^0.
 */
int uotk_uot_sinkhorn(int d, int64_t n, const double* x, const double* a,
                      int64_t m, const double* y, const double* b,
                      double eps, double lam1, double lam2, int iters,
                      const double* gamma_init, double* beta, double* gamma,
                      uotk_uot_result* res, const uotk_opts* opts,
                      void* comm, void* cuda_stream);

/*
 * MMD^2 of Eq. (3.5), V-statistic (diagonal terms included):
 *   sum_ij a_i a_j k(x_i,x_j) - 2 sum_ij a_i b_j k(x_i,y_j) + sum_ij b_i b_j k(y_i,y_j)
 * evaluated as one quadratic form over z = x u y with weights w = (a, -b).
 * x: n x d, a: n;  y: m x d, b: m (any sign);  *mmd2: host double (output).
 */
int uotk_mmd2(int d, int64_t n, const double* x, const double* a,
              int64_t m, const double* y, const double* b, int kind, double param,
              double* mmd2, const uotk_opts* opts, uotk_info* info,
              void* comm, void* cuda_stream);

/*
 * uotk_uot_sinkhorn plus the marginals of the recovered plan pi, in caller order:
 *   p_i = sum_j pi_ij (n values),  q_j = sum_i pi_ij (m values)  (device or host; either
 *   may be NULL).  With opts->flags & UOTK_FLAG_TRANSPORT, res->transport = <pi, d^2>,
 *   one extra kernel sum with k(r) = r^2 exp(-r^2/eps) (UOTK_GAUSS_R2).
 */
int uotk_uot_sinkhorn_ex(int d, int64_t n, const double* x, const double* a,
                         int64_t m, const double* y, const double* b,
                         double eps, double lam1, double lam2, int iters,
                         const double* gamma_init, double* beta, double* gamma,
                         double* p, double* q, uotk_uot_result* res, const uotk_opts* opts,
                         void* comm, void* cuda_stream);

/*
 * The constant c* of Prop. 2.9, Eq. (2.10), r = 2, lambda = 1/eps:
 *   c* = exp(-<mu x nu | d^2> / (mu(X) nu(X) (lam1 + lam2 + eps))) mu(X)^(-lam2/(..)) nu(X)^(-lam1/(..))
 * with the transport moment <mu x nu | d^2> = sum_ij a_i b_j ||x_i - y_j||^2 evaluated
 * from first and second moments in O((n + m) d) (centred, two passes).  Remark 5.2
 * uses it to initialise Algorithm 2 with gamma^0 = c* 1.  *cstar: host double.
 * Masses must be positive (UOTK_EDOMAIN otherwise).  With `comm`, the moments are
 * summed over ranks.
 */
int uotk_uot_cstar(int d, int64_t n, const double* x, const double* a,
                   int64_t m, const double* y, const double* b,
                   double eps, double lam1, double lam2, double* cstar,
                   void* comm, void* cuda_stream);

/*
 * Sinkhorn divergence of Eq. (2.12) (Rem. 2.11), the debiased UOT:
 *   sd = UOT(mu, nu) - UOT(mu, mu)/2 - UOT(nu, nu)/2 + (eps/2) (mu(X) - nu(X))^2
 * each UOT the primal value (uotk_uot_result.primal) of uotk_uot_sinkhorn with the
 * same arguments and `iters`.  *sd: host double; terms (may be NULL): host double[3] =
 * {UOT(mu,nu), UOT(mu,mu), UOT(nu,nu)}.
 */
int uotk_sinkhorn_divergence(int d, int64_t n, const double* x, const double* a,
                             int64_t m, const double* y, const double* b,
                             double eps, double lam1, double lam2, int iters,
                             double* sd, double* terms, const uotk_opts* opts,
                             void* comm, void* cuda_stream);

/*
 * lambda-scaling (Sec. 5.1.3): uotk_uot_sinkhorn solved for each entropy
 * parameter eps_list[0..n_eps-1] in turn (decreasing eps = increasing lambda = 1/eps),
 * each stage warm-started from the previous stage's gamma (the first from gamma_init,
 * or 0).  Every stage runs `iters` iterations (or fewer with opts->stop_tol).  Outputs
 * and res are those of the last stage, except res->iters = the total over all stages.
 * eps_list: host array of n_eps >= 1 positive values.
 */
int uotk_uot_sinkhorn_scaling(int d, int64_t n, const double* x, const double* a,
                              int64_t m, const double* y, const double* b,
                              const double* eps_list, int n_eps, double lam1, double lam2,
                              int iters, const double* gamma_init, double* beta, double* gamma,
                              uotk_uot_result* res, const uotk_opts* opts,
                              void* comm, void* cuda_stream);

/* Multi-GPU communicator (one process per GPU).  uotk_comm_unique_id fills 128
 * bytes on one rank; broadcast them (e.g. with torch.distributed) and call
 * uotk_comm_create on every rank with the current CUDA device set.  NCCL is
 * loaded at run time (libnccl.so.2); UOTK_ENCCL if it cannot be. */
int uotk_comm_unique_id(void* id128);
int uotk_comm_create(const void* id128, int nranks, int rank, void** comm_out);
int uotk_comm_destroy(void* comm);

/* Loopback group: nranks (1..16) communicator handles for ONE process on ONE GPU, written
 * to comms_out[0..nranks-1] (handle k = rank k).  It stands in for nranks processes (the
 * multi-rank path tested with a single device): each handle is used by one host thread,
 * all nranks threads call the same entry point concurrently with their own shards and
 * streams.  Every collective of the exchange step (all-reduce of Fourier coefficients,
 * bounding box and scalars; reduce-scatter / all-gather of the slab-distributed chain) is
 * performed by a library kernel that sums (or maxes, or copies) the nranks device buffers
 * in rank order, ordered by CUDA events and host barriers — no kernel waits on another.  A rank whose call fails aborts the group (the others fail with UOTK_ENCCL at
 * their next collective; a rank that never arrives times out after 120 s).  Results equal
 * NCCL's up to the summation order; timings are not representative.  Destroy each
 * handle with uotk_comm_destroy. */
int uotk_comm_create_loopback(int nranks, void** comms_out);

/* Thread-local description of the last error (never NULL). */
const char* uotk_last_error(void);

/* Returns UOTK_ABI_VERSION. */
int uotk_abi_version(void);

/* Releases everything the library caches between calls on the current device: the
 * Fourier-side tables D_k / circulant factors and their cuFFT plans (rebuilt on the next
 * call that needs them), the recycled device buffers, and the stream-ordered pool's
 * reserved memory.  Synchronises the device first.  Returns 0 or UOTK_ECUDA.  After it
 * the next call runs "cold" (bench.py's cold MMD^2 number). */
int uotk_release_caches(void);

/* Number of this library's kernels launched by the calling thread since the last
 * reset (bench.py's "gpu_launches"); uotk_launch_counter_reset sets it to 0. */
int64_t uotk_launch_counter(void);
void uotk_launch_counter_reset(void);

/* Live kernel timing for benchmarks.  When enabled, each launch of an instrumented
 * pass is bracketed by CUDA events recorded on its stream.  Tags: "spread", "gather",
 * "fused" (d=3 gather-update-spread), "fft" (D2Z + D_k scale + Z2D), "direct",
 * "setup".  uotk_profile_read synchronises on the recorded events and returns the
 * summed milliseconds and the number of bracketed launches of one tag. */
void uotk_profile_enable(int on);
void uotk_profile_reset(void);
int uotk_profile_read(const char* tag, double* ms, int64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* UOTK_H */
