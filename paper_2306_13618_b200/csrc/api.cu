// The C ABI (include/uotk.h): validation, host/device staging, and the drivers of the
// three operations — kernel sum (4.3), UOT Sinkhorn (Algorithm 2 / Algorithm 1) and
// MMD^2 (3.5) — over the NFFT passes (nfft.cu, fused3d.cu) or the direct kernel (direct.cu).
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "epilogue.cuh"
#include "profile.cuh"
#include "reduce.cuh"

namespace uotk {

extern thread_local std::string g_last_error;
extern thread_local int64_t g_launches;
void comm_unique_id(void* id128);
void* comm_create(const void* id128, int nranks, int rank);
void comm_destroy(void* comm);
void comm_allreduce(double* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s);
void comm_allreduce_i32(int32_t* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s);
int comm_nranks(void* comm);
bool comm_capturable(void* comm);
void comm_create_loopback(int nranks, void** out);
void comm_abort(void* comm, const std::string& why);
void ensure_pool();
cudaStream_t private_stream();  // context.cu
int64_t guard_violations();     // context.cu (UOTK_GUARD=1)

void spectrum_energy(SpectralPlan& sp, double* grid, double2* spec, double* part, int nparts, cudaStream_t s,
                     void* comm);  // nfft.cu
void box_dot(const double* g, const double* gp, const FastParams& fp, double* part, int nparts,
             cudaStream_t s);  // circgemm.cu

void apply_sinkhorn_update(const double* t, int64_t n, const EpiSinkhorn& epi, unsigned long long* dmax,
                           cudaStream_t s);  // nearfield.cu

// Fused NFFT half-step on chunked point sets (fused12d.cu / fused3d.cu).
bool chunked_available(const FastParams& fp);
void chunked_gather_spread(const PointSet& ps, const double* grid_in, double* grid_out, const FastParams& fp,
                           const EpiSinkhorn& epi, unsigned long long* dmax, cudaStream_t s);

namespace {

// AUTO: below this many source-target pairs the direct kernel wins (measured, DESIGN.md
// §10: the direct kernel evaluates ~4e11 pairs/s; a single NFFT kernel sum or MMD^2 costs
// a fixed ~0.4 ms (d <= 2), ~1 ms (d = 3 Gaussian), ~2.4 ms (d = 3 IMQ, 384^3 grid); a
// Sinkhorn iteration replayed from a graph ~35 us at C1's size).
constexpr double kDirectCrossoverPairs = 4.0e7;  // Sinkhorn
double direct_crossover_sum(int d, int kind) {   // one kernel sum / MMD^2
    if (kind == UOTK_LAP || kind == UOTK_ENERGY) return d < 3 ? 1.0e9 : 4.0e9;  // N = 256 grids + near field
    if (d < 3) return 1.5e8;
    return kind == UOTK_IMQ ? 8.0e8 : 4.0e8;
}

bool nonsmooth(int kind) { return kind == UOTK_LAP || kind == UOTK_ENERGY; }

// the near-field correction needs every partner of a target within eps_I: one rank only
void check_nearfield_ranks(int kind, const uotk_opts& o, void* comm) {
    if (nonsmooth(kind) && o.method != UOTK_DIRECT && comm_nranks(comm) > 1)
        fail(UOTK_EUNSUPPORTED, "Laplace / energy kernels (near-field correction) with a multi-rank communicator");
}

// Runs f, mapping exceptions to status codes.  With a communicator the thread's resource
// slot is the rank's (loopback groups), and a failing rank aborts a loopback group so
// that its other ranks fail at their next collective instead of waiting for it.
template <class F>
int guarded(F&& f, void* comm = nullptr) {
    SlotScope slot(comm);
    const int64_t guard0 = guard_violations();
    try {
        f();
        if (guard_violations() != guard0)
            fail(UOTK_ECUDA, "UOTK_GUARD: a kernel wrote outside a library buffer (see stderr)");
        return UOTK_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        comm_abort(comm, e.msg);
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = std::string("internal error: ") + e.what();
        comm_abort(comm, g_last_error);
        return UOTK_ECUDA;
    } catch (...) {
        g_last_error = "internal error";
        comm_abort(comm, g_last_error);
        return UOTK_ECUDA;
    }
}

uotk_opts resolve(const uotk_opts* o) {
    uotk_opts r;
    memset(&r, 0, sizeof r);
    if (o) r = *o;
    if ((r.flags & ~(UOTK_FLAG_GENERIC | UOTK_FLAG_CHUNKED | UOTK_FLAG_TRANSPORT | UOTK_FLAG_FFT |
                     UOTK_FLAG_COST_R1)) != 0)
        fail(UOTK_EINVAL, "unknown opts.flags bits");
    if (r.deterministic != 0 && r.deterministic != 1) fail(UOTK_EINVAL, "opts.deterministic must be 0 or 1");
    if ((r.flags & UOTK_FLAG_COST_R1) && (r.flags & UOTK_FLAG_TRANSPORT))
        fail(UOTK_EUNSUPPORTED, "UOTK_FLAG_TRANSPORT with the r = 1 cost");
    if ((r.flags & UOTK_FLAG_GENERIC) && (r.flags & UOTK_FLAG_CHUNKED))
        fail(UOTK_EINVAL, "opts.flags: UOTK_FLAG_GENERIC and UOTK_FLAG_CHUNKED are exclusive");
    if (r.method < 0 || r.method > 2) fail(UOTK_EINVAL, "opts.method must be AUTO, NFFT or DIRECT");
    if (r.N < 0 || r.m < 0 || r.p < 0 || r.sigma < 0 || r.eps_B < 0 || r.h < 0 || r.tol < 0 || r.tol >= 1)
        fail(UOTK_EINVAL, "negative option value");
    if (!(r.stop_tol >= 0) || r.check_every < 0 || r.reserved2 != 0)
        fail(UOTK_EINVAL, "opts.stop_tol / check_every must be >= 0 and reserved2 = 0");
    if (r.check_every == 0) r.check_every = 10;
    return r;
}

void need(bool ok, const char* msg) {
    if (!ok) fail(UOTK_EINVAL, msg);
}

void check_points_arg(int d, int64_t n, const void* p, const char* what) {
    if (n < 0) fail(UOTK_EINVAL, std::string(what) + ": negative size");
    if (n > 0 && !p) fail(UOTK_EINVAL, std::string(what) + ": null pointer");
    (void)d;
}

int pick_method(const uotk_opts& o, double pairs, void* comm, double crossover = kDirectCrossoverPairs) {
    if (o.method == UOTK_DIRECT) {
        if (comm && comm_nranks(comm) > 1) fail(UOTK_EUNSUPPORTED, "DIRECT method with a multi-rank communicator");
        return UOTK_DIRECT;
    }
    if (o.method == UOTK_NFFT) return UOTK_NFFT;
    if (comm && comm_nranks(comm) > 1) return UOTK_NFFT;
    return pairs <= crossover ? UOTK_DIRECT : UOTK_NFFT;
}

int group_code(const PointSet* ps) { return (ps && ps->chunked) ? ps->chunk_kz : 0; }

void fill_info(uotk_info* info, int method, const FastParams* fp, void* comm, const PointSet* p1 = nullptr,
               const PointSet* p2 = nullptr) {
    if (!info) return;
    memset(info, 0, sizeof *info);
    info->method_used = method;
    info->nranks = comm_nranks(comm);
    if (fp) {
        info->N = fp->N;
        info->n_grid = fp->ng;
        info->m = fp->m;
        info->h = fp->h;
        info->groups1 = group_code(p1);
        info->groups2 = group_code(p2);
    }
}

struct NfftSetup {
    FastParams fp;
    SpectralPlan sp;
};

void setup_nfft(NfftSetup& ns, int d, int kind, double param, const double* p1, int64_t n1, const double* p2,
                int64_t n2, const uotk_opts& o, void* comm, cudaStream_t s) {
    NvtxRange nvtx_("setup");
    trace_mark("setup_nfft: start");
    Geometry g = compute_geometry(d, p1, n1, p2, n2, s, comm);
    trace_mark("geometry");
    ns.fp = choose_params(d, kind, param, g, o);
    trace_mark("choose_params");
    ns.sp.fp = ns.fp;
    build_spectral_plan(ns.sp, s);
    trace_mark("spectral_plan");
}

size_t grid_elems(const FastParams& fp) {
    size_t g = 1;
    for (int t = 0; t < fp.d; ++t) g *= fp.ng;
    return g;
}

// Sinkhorn iterations are replayed from CUDA graphs (at every size: the small problems are
// launch-bound, and the large ones lose the gaps around the spectral chain's short
// kernels — C3 266 -> 261 ms per solve); UOTK_GRAPH_MAX=<points> limits it to n + m below
// that (0: never).
static int64_t graph_max_points() {
    static const int64_t v = [] {
        const char* e = getenv("UOTK_GRAPH_MAX");
        return e ? (int64_t)atoll(e) : INT64_MAX;
    }();
    return v;
}
#define kGraphMaxPoints graph_max_points()
constexpr int kGraphIters = 16;  // iterations per captured graph

// Runs iterate(0) .. iterate(iters - 1) in order on stream s.  With use_graph the first
// iteration runs eagerly (first-use initialisation: kernel attributes, cuBLAS), then
// blocks of kGraphIters identical middle iterations are captured once and replayed, and
// the remaining iterations (including the last, whose epilogue differs) run eagerly.
template <class F>
int run_iterations(int iters, F&& iterate, bool use_graph, cudaStream_t s, int check_every = 0,
                   double stop_tol = 0.0, unsigned long long* dmax = nullptr, void* comm = nullptr) {
    NvtxRange nvtx_("iterations");
    if (check_every > 0) {
        // stopping rule: after every check_every-th iteration read the two sup-norm
        // changes (non-negative doubles stored as their bit patterns) and stop if both
        // are <= stop_tol.  With a communicator the changes are maxed over ranks first, so
        // every rank takes the same decision (and issues the same collectives).
        for (int it = 0; it < iters; ++it) {
            iterate(it);
            if ((it + 1) % check_every == 0 && it + 1 < iters) {
                if (comm) comm_allreduce(reinterpret_cast<double*>(dmax), 2, 1, comm, s);
                unsigned long long h[2];
                UOTK_CUDA(cudaMemcpyAsync(h, dmax, sizeof h, cudaMemcpyDeviceToHost, s));
                UOTK_CUDA(cudaStreamSynchronize(s));
                double v[2];
                memcpy(v, h, sizeof v);
                if (v[0] <= stop_tol && v[1] <= stop_tol) return it + 1;
            }
        }
        return iters;
    }
    int it = 0;
    if (use_graph && iters >= 4) {
        iterate(it++);
        const int per = std::min(kGraphIters, iters - 2);
        const int reps = (iters - 1 - it) / per;
        if (reps >= 1) {
            cudaGraph_t g = nullptr;
            const int64_t l0 = g_launches;
            UOTK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                for (int k = 0; k < per; ++k) iterate(it + k);  // none of them is the last
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            UOTK_CUDA(cudaStreamEndCapture(s, &g));
            const int64_t per_launches = g_launches - l0;
            cudaGraphExec_t ge = nullptr;
            const cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            UOTK_CUDA(ie);
            for (int r = 0; r < reps; ++r) UOTK_CUDA(cudaGraphLaunch(ge, s));
            UOTK_CUDA(cudaGraphExecDestroy(ge));  // safe: destruction waits for nothing, launches hold refs
            g_launches += per_launches * (reps - 1);
            it += reps * per;
        }
    }
    for (; it < iters; ++it) iterate(it);
    return iters;
}

// reads the status flag (bits: 1|2 overflow in the loop, 4 bad mass, 8 non-finite
// coordinate); with a communicator the flags of all ranks are or-ed first (one max
// all-reduce of the bits spread over 4 words), so every rank fails or succeeds together
int read_flag(const DevBuf<int>& flag, cudaStream_t s, void* comm = nullptr) {
    if (comm) {
        // or over ranks, bit by bit: spread the bits into 4 words, max-reduce, fold back
        DevBuf<int32_t> bits(4, s);
        split_bits(flag.p, bits.p, s);
        comm_allreduce_i32(bits.p, 4, 1, comm, s);
        join_bits(bits.p, flag.p, s);
    }
    int h = 0;
    UOTK_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace

template struct DevBuf<int>;

// ============================================================== kernel sum
static void kernel_sum_impl(int d, int64_t n_src, const double* src, const double* alpha, int64_t n_tgt,
                            const double* tgt, int kind, double param, double* out, const uotk_opts* opts_in,
                            uotk_info* info, void* comm, cudaStream_t s) {
    NvtxRange nvtx_call("uotk_kernel_sum");
    need(d >= 1 && d <= 3, "d must be 1, 2 or 3");
    need(kind >= UOTK_GAUSS && kind <= UOTK_ENERGY, "unknown kernel kind");
    need(param > 0 && std::isfinite(param), "kernel parameter must be positive and finite");
    check_points_arg(d, n_src, src, "src");
    check_points_arg(d, n_src, alpha, "alpha");
    check_points_arg(d, n_tgt, tgt, "tgt");
    check_points_arg(d, n_tgt, out, "out");
    const uotk_opts o = resolve(opts_in);
    check_nearfield_ranks(kind, o, comm);
    ensure_pool();
    InArr S, A, T;
    S.bind(src, (size_t)n_src * d, s);
    A.bind(alpha, (size_t)n_src, s);
    T.bind(tgt, (size_t)n_tgt * d, s);
    OutArr O;
    O.bind(out, (size_t)n_tgt, s);
    const int method = pick_method(o, (double)n_src * (double)n_tgt, comm, direct_crossover_sum(d, kind));
    if (method == UOTK_DIRECT) {
        fill_info(info, method, nullptr, comm);
        // the NFFT path validates coordinates in compute_geometry; here a flag kernel does
        DevBuf<int> flag(1, s);
        flag.zero();
        check_finite(S.d, n_src * d, flag.p, 8, s);
        check_finite(T.d, n_tgt * d, flag.p, 8, s);
        if (read_flag(flag, s) & 8) fail(UOTK_EDOMAIN, "non-finite point coordinate");
        if (n_tgt > 0) {
            if (n_src == 0) UOTK_CUDA(cudaMemsetAsync(O.d, 0, n_tgt * sizeof(double), s));
            else direct_sum_epi(d, n_src, S.d, A.d, n_tgt, T.d, kind, param, EpiStore{O.d, nullptr}, nullptr, s);
        }
    } else {
        NfftSetup ns;
        setup_nfft(ns, d, kind, param, S.d, n_src, T.d, n_tgt, o, comm, s);
        PointSet PS, PT;
        DevBuf<double> w(n_src, s);
        SortedWeights sws;  // alpha in sorted order, written by the coordinate gather
        sws.w1 = A.d;
        sws.out = w.p;
        make_pointset(PS, S.d, n_src, ns.fp, s, kUseSpreadOnly, sws);
        trace_mark("pointset src");
        make_pointset(PT, T.d, n_tgt, ns.fp, s, kUseGatherOnly);
        trace_mark("pointset tgt");
        fill_info(info, method, &ns.fp, comm, &PS, &PT);
        DevBuf<double> grid(grid_elems(ns.fp), s);
        DevBuf<double2> spec(ns.sp.spec_elems, s);
        grid.zero();
        spread(PS, w.p, grid.p, ns.fp, s);
        const double* gp = fft_chain(ns.sp, grid.p, spec.p, s, comm);
        gather_epi(PT, gp, ns.fp, EpiStore{O.d, PT.perm.p}, nullptr, s);
        if (nearfield_needed(ns.fp)) {  // + sum over close pairs of (K - K_R) alpha
            NearField NS, NT;
            build_nearfield(NS, PS, ns.fp, s);
            build_nearfield(NT, PT, ns.fp, s);
            nearfield_apply(NS, w.p, NT, ns.fp, PT.perm.p, O.d, s);
        }
        trace_mark("passes enqueued");
    }
    O.flush();
    // host outputs, and host inputs staged by asynchronous copies (pinned memory), must be
    // complete before the call returns: the library keeps no caller pointer afterwards
    if (O.host || S.host || A.host || T.host) UOTK_CUDA(cudaStreamSynchronize(s));
}

// ============================================================== UOT Sinkhorn
static void uot_impl(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y, const double* b,
                     double eps, double lam1, double lam2, int iters, const double* gamma_init, double* beta_out,
                     double* gamma_out, uotk_uot_result* res, const uotk_opts* opts_in, void* comm, cudaStream_t s,
                     double* p_out = nullptr, double* q_out = nullptr) {
    NvtxRange nvtx_call("uotk_uot_sinkhorn");
    need(d >= 1 && d <= 3, "d must be 1, 2 or 3");
    // a rank's local shard may be empty (it still takes part in every collective)
    if (comm_nranks(comm) > 1) need(n >= 0 && m >= 0, "n and m must be >= 0");
    else need(n >= 1 && m >= 1, "n and m must be >= 1");
    need((x || n == 0) && (a || n == 0) && (y || m == 0) && (b || m == 0) && (beta_out || n == 0) &&
             (gamma_out || m == 0),
         "null pointer argument");
    need(eps > 0 && std::isfinite(eps), "eps must be positive and finite");
    need(lam1 > 0 && lam2 > 0 && std::isfinite(lam1) && std::isfinite(lam2), "lam1, lam2 must be positive");
    need(iters >= 0, "iters must be >= 0");
    const uotk_opts o = resolve(opts_in);
    ensure_pool();
    InArr X, A, Y, B, G0;
    X.bind(x, (size_t)n * d, s);
    A.bind(a, (size_t)n, s);
    Y.bind(y, (size_t)m * d, s);
    B.bind(b, (size_t)m, s);
    if (gamma_init) G0.bind(gamma_init, (size_t)m, s);
    OutArr BO, GO, PO, QO;
    BO.bind(beta_out, (size_t)n, s);
    GO.bind(gamma_out, (size_t)m, s);
    if (p_out) PO.bind(p_out, (size_t)n, s);
    if (q_out) QO.bind(q_out, (size_t)m, s);
    const bool want_transport = (o.flags & UOTK_FLAG_TRANSPORT) != 0;

    // the Gibbs kernel exp(-lambda d^r): Gaussian (r = 2) or Laplace with l = eps (r = 1)
    const int gk = (o.flags & UOTK_FLAG_COST_R1) ? UOTK_LAP : UOTK_GAUSS;
    check_nearfield_ranks(gk, o, comm);
    const double lam = 1.0 / eps;                 // paper lambda (Def. 2.7)
    const double c1 = lam1 / (1.0 + lam1 * lam);  // (3.3): beta = -c1 log t
    const double c2 = lam2 / (1.0 + lam2 * lam);  // (3.4): gamma = -c2 log t~

    DevBuf<int> flag(1, s);
    flag.zero();
    check_mass(A.d, n, flag.p, s);
    check_mass(B.d, m, flag.p, s);
    DevBuf<unsigned long long> dmax(2, s);
    dmax.zero();

    const int method = pick_method(o, (double)n * (double)m, comm);
    if (method == UOTK_DIRECT) {
        check_finite(X.d, n * d, flag.p, 8, s);
        check_finite(Y.d, m * d, flag.p, 8, s);
    }
    // per-point state: potentials, masses, next weights, t at x (final) and t~ at y (last)
    DevBuf<double> pot_x(n, s), pot_y(m, s), mass_x(n, s), mass_y(m, s), wx(n, s), wy(m, s), tx(n, s), ty(m, s);
    DevBuf<double> tpx;  // t' at x for the transport term
    if (want_transport) tpx.alloc(n, s);
    pot_x.zero();
    const int32_t* perm_x = nullptr;
    const int32_t* perm_y = nullptr;
    FastParams fpv;
    const FastParams* fpp = nullptr;
    NfftSetup ns;
    PointSet PX, PY;
    if (method == UOTK_DIRECT) {
        UOTK_CUDA(cudaMemcpyAsync(mass_x.p, A.d, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        UOTK_CUDA(cudaMemcpyAsync(mass_y.p, B.d, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (gamma_init) UOTK_CUDA(cudaMemcpyAsync(pot_y.p, G0.d, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
        else pot_y.zero();
    } else {
        setup_nfft(ns, d, gk, eps, X.d, n, Y.d, m, o, comm, s);
        fpv = ns.fp;
        fpp = &fpv;
        make_pointset(PX, X.d, n, ns.fp, s);
        make_pointset(PY, Y.d, m, ns.fp, s);
        perm_x = PX.perm.p;
        perm_y = PY.perm.p;
        permute_values(mass_x.p, A.d, perm_x, n, s);
        permute_values(mass_y.p, B.d, perm_y, m, s);
        if (gamma_init) permute_values(pot_y.p, G0.d, perm_y, m, s);
        else pot_y.zero();
    }
    {
        const int f0 = read_flag(flag, s, comm);
        if (f0 & 8) fail(UOTK_EDOMAIN, "non-finite point coordinate");
        if (f0 & 4) fail(UOTK_EDOMAIN, "masses must be positive and finite (KL needs mu_i > 0)");
    }

    // v = e^{lam gamma^0}: weights of the first beta-step
    scaled_mass(mass_y.p, pot_y.p, m, lam, wy.p, s);
    EpiSinkhorn ex{pot_x.p, mass_x.p, wx.p, nullptr, c1, lam, flag.p};
    EpiSinkhorn ey{pot_y.p, mass_y.p, wy.p, nullptr, c2, lam, flag.p};

    // small problems are launch-bound: replay the iteration from a CUDA graph
    const bool stop_rule = o.stop_tol > 0;
    const bool use_graph =
        comm_capturable(comm) && iters >= 4 && n + m <= kGraphMaxPoints && !profiling_enabled() && !stop_rule;
    // iterations whose sup-norm changes are recorded: the last one, and with the stopping
    // rule every check_every-th one (dmax is reset before each of them)
    auto records = [&](int it) { return it == iters - 1 || (stop_rule && (it + 1) % o.check_every == 0); };
    int done = iters;
    if (method == UOTK_DIRECT) {
        auto iterate = [&](int it) {
            const bool last = records(it);
            if (last) dmax.zero();
            direct_sum_epi(d, m, Y.d, wy.p, n, X.d, gk, eps, ex, last ? dmax.p : nullptr, s);  // (3.3)
            EpiSinkhorn e2 = ey;
            if (last) e2.t_store = ty.p;
            direct_sum_epi(d, n, X.d, wx.p, m, Y.d, gk, eps, e2, last ? dmax.p + 1 : nullptr, s);  // (3.4)
        };
        done = run_iterations(iters, iterate, use_graph, s, stop_rule ? o.check_every : 0, o.stop_tol, dmax.p, comm);
        // marginals of the recovered plan: t at x from the final gamma
        direct_sum_epi(d, m, Y.d, wy.p, n, X.d, gk, eps, EpiStore{tx.p, nullptr}, nullptr, s);
        // <pi, d^2>: t' at x with the kernel d^2 k (UOTK_GAUSS_R2) against the same weights
        if (want_transport) direct_sum_epi(d, m, Y.d, wy.p, n, X.d, UOTK_GAUSS_R2, eps, EpiStore{tpx.p, nullptr},
                                           nullptr, s);
        if (iters == 0) {
            scaled_mass(mass_x.p, pot_x.p, n, lam, wx.p, s);
            direct_sum_epi(d, n, X.d, wx.p, m, Y.d, gk, eps, EpiStore{ty.p, nullptr}, nullptr, s);
        }
    } else {
        const FastParams& fp = ns.fp;
        const size_t ge = grid_elems(fp);
        DevBuf<double> grid(ge, s), grid2;
        DevBuf<double2> spec(ns.sp.spec_elems, s);
        // the fused half-steps flush their spread with fp64 atomics: deterministic mode (and
        // the near-field corrected r = 1 kernel) runs gather, update and spread separately
        const bool nf = nearfield_needed(fp);  // r = 1: Laplace Gibbs kernel, near-field corrected
        const bool fused = chunked_available(fp) && PX.chunked && PY.chunked && !fp.deterministic && !nf;
        if (fused) {
            grid2.alloc(ge, s);
            grid2.zero();
        }
        NearField NX, NY;
        DevBuf<double> tbx, tby;  // kernel sums in sorted order (gather + near field)
        if (nf) {
            build_nearfield(NX, PX, fp, s);
            build_nearfield(NY, PY, fp, s);
            tbx.alloc(n, s);
            tby.alloc(m, s);
        }
        // t at the points of P (sorted order) from the grid g' (and, r = 1, the near field
        // of the other set Q's weights wq), then the epilogue
        auto half_step = [&](const PointSet& P, const NearField& NP, const NearField& NQ, const double* wq,
                             double* tb, int64_t np, const double* g, const EpiSinkhorn& e, unsigned long long* dm) {
            if (!nf) {
                gather_epi(P, g, fp, e, dm, s);
                return;
            }
            gather_epi(P, g, fp, EpiStore{tb, nullptr}, nullptr, s);
            nearfield_apply(NQ, wq, NP, fp, nullptr, tb, s);
            apply_sinkhorn_update(tb, np, e, dm, s);
        };
        grid.zero();
        spread(PY, wy.p, grid.p, fp, s);  // adjoint NFFT of nu (.) v at y
        auto iterate = [&](int it) {
            const bool last = records(it);
            if (last) dmax.zero();
            EpiSinkhorn e2 = ey;
            if (last) e2.t_store = ty.p;
            // the separable chain zeroes the footprint box of the next spread's target grid
            // as a side job (both grids are zero outside the box); else a full memset
            bool zd = false;
            if (fused) {
                // beta-step at x: gather t from g', update, spread mu (.) u into the other grid
                const double* g1 = fft_chain(ns.sp, grid.p, spec.p, s, comm, grid2.p, &zd);
                if (!zd) grid2.zero();
                chunked_gather_spread(PX, g1, grid2.p, fp, ex, last ? dmax.p : nullptr, s);
                const double* g2 = fft_chain(ns.sp, grid2.p, spec.p, s, comm, grid.p, &zd);
                if (!zd) grid.zero();
                chunked_gather_spread(PY, g2, grid.p, fp, e2, last ? dmax.p + 1 : nullptr, s);
            } else {
                const double* g1 = fft_chain(ns.sp, grid.p, spec.p, s, comm, grid.p, &zd);
                half_step(PX, NX, NY, wy.p, tbx.p, n, g1, ex, last ? dmax.p : nullptr);  // (3.3)
                if (!zd) grid.zero();
                spread(PX, wx.p, grid.p, fp, s);
                const double* g2 = fft_chain(ns.sp, grid.p, spec.p, s, comm, grid.p, &zd);
                half_step(PY, NY, NX, wx.p, tby.p, m, g2, e2, last ? dmax.p + 1 : nullptr);  // (3.4)
                if (!zd) grid.zero();
                spread(PY, wy.p, grid.p, fp, s);
            }
        };
        done = run_iterations(iters, iterate, use_graph, s, stop_rule ? o.check_every : 0, o.stop_tol, dmax.p, comm);
        // grid holds the spread of nu (.) v with the final v: t at x for the marginals
        if (want_transport) {
            // the same spread grid through the D_k of the kernel d^2 k (same N, n_g, h)
            DevBuf<double> gt(ge, s);
            UOTK_CUDA(cudaMemcpyAsync(gt.p, grid.p, ge * sizeof(double), cudaMemcpyDeviceToDevice, s));
            SpectralPlan sp2;
            sp2.fp = fp;
            sp2.fp.kind = UOTK_GAUSS_R2;
            build_spectral_plan(sp2, s);
            const double* g2 = fft_chain(sp2, gt.p, spec.p, s, comm);
            gather_epi(PX, g2, fp, EpiStore{tpx.p, nullptr}, nullptr, s);
        }
        const double* gx = fft_chain(ns.sp, grid.p, spec.p, s, comm);
        gather_epi(PX, gx, fp, EpiStore{tx.p, nullptr}, nullptr, s);
        if (nf) nearfield_apply(NY, wy.p, NX, fp, nullptr, tx.p, s);
        if (iters == 0) {
            scaled_mass(mass_x.p, pot_x.p, n, lam, wx.p, s);
            grid.zero();
            spread(PX, wx.p, grid.p, fp, s);
            const double* gy = fft_chain(ns.sp, grid.p, spec.p, s, comm);
            gather_epi(PY, gy, fp, EpiStore{ty.p, nullptr}, nullptr, s);
            if (nf) nearfield_apply(NX, wx.p, NY, fp, nullptr, ty.p, s);
        }
    }

    NvtxRange nvtx_obj("objectives");
    // objective terms and their global sums
    DevBuf<double> cols(5 * (size_t)std::max(n, m), s), sums(13, s);
    sums.zero();
    uot_terms(pot_x.p, mass_x.p, tx.p, n, lam, lam1, cols.p, s);
    sum_columns(cols.p, n, 5, sums.p, s);
    // column 0 now holds p (sorted order): export it
    if (p_out) {
        if (method == UOTK_DIRECT) UOTK_CUDA(cudaMemcpyAsync(PO.d, cols.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        else unpermute_values(PO.d, cols.p, perm_x, n, s);
    }
    if (want_transport) {
        // <pi, d^2> = sum_i mu_i e^{lam beta_i} t'_i: reuse cols as (w_i t'_i)
        uot_transport(pot_x.p, mass_x.p, tpx.p, n, lam, cols.p, s);
        sum_columns(cols.p, n, 1, sums.p + 12, s);
    }
    uot_terms(pot_y.p, mass_y.p, ty.p, m, lam, lam2, cols.p, s);
    sum_columns(cols.p, m, 5, sums.p + 5, s);
    if (q_out) {
        if (method == UOTK_DIRECT) UOTK_CUDA(cudaMemcpyAsync(QO.d, cols.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
        else unpermute_values(QO.d, cols.p, perm_y, m, s);
    }
    // dmax as doubles (non-negative: the bit patterns order like the values)
    UOTK_CUDA(cudaMemcpyAsync(sums.p + 10, dmax.p, 2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (comm) {
        comm_allreduce(sums.p, 10, 0, comm, s);
        comm_allreduce(sums.p + 10, 2, 1, comm, s);
        comm_allreduce(sums.p + 12, 1, 0, comm, s);
    }
    double hs[13];
    UOTK_CUDA(cudaMemcpyAsync(hs, sums.p, sizeof hs, cudaMemcpyDeviceToHost, s));
    // potentials back to caller order
    if (method == UOTK_DIRECT) {
        UOTK_CUDA(cudaMemcpyAsync(BO.d, pot_x.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        UOTK_CUDA(cudaMemcpyAsync(GO.d, pot_y.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
        unpermute_values(BO.d, pot_x.p, perm_x, n, s);
        unpermute_values(GO.d, pot_y.p, perm_y, m, s);
    }
    BO.flush();
    GO.flush();
    if (p_out) PO.flush();
    if (q_out) QO.flush();
    const int fl = read_flag(flag, s, comm);  // synchronises the stream
    if (fl & 3) fail(UOTK_EOVERFLOW, "non-positive or non-finite kernel sum / scaling in the Sinkhorn loop");

    if (res) {
        const double P = hs[0], bp = hs[1], plogp = hs[2], emb = hs[3], mx = hs[4];
        const double Q = hs[5], gq = hs[6], qlogq = hs[7], emg = hs[8], my = hs[9];
        const double tot = P;
        memset(res, 0, sizeof *res);
        // primal (2.9) / P:462 through the marginals: the <pi, d^2> terms cancel against the entropy
        res->primal = bp + gq + eps * (mx * my - tot) + lam1 * (plogp + mx - tot) + lam2 * (qlogq + my - Q);
        // dual (3.1)
        res->dual = -lam1 * emb - lam2 * emg + lam1 * mx + lam2 * my - eps * (tot - mx * my);
        res->plan_mass = tot;
        res->mass_a = mx;
        res->mass_b = my;
        res->max_dbeta = hs[10];
        res->max_dgamma = hs[11];
        res->iters = done;
        fill_info(&res->info, method, fpp, comm, &PX, &PY);
        res->transport = want_transport ? hs[12] : std::nan("");
    }
}

// ============================================================== Sinkhorn divergence (2.12)
static void sd_impl(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                    const double* b, double eps, double lam1, double lam2, int iters, double* sd, double* terms,
                    const uotk_opts* opts, void* comm, cudaStream_t s) {
    NvtxRange nvtx_call("uotk_sinkhorn_divergence");
    need(sd != nullptr, "sd output pointer is null");
    need(n >= 1 && m >= 1, "n and m must be >= 1");
    ensure_pool();
    DevBuf<double> p1(n, s), q1(m, s), p2(n, s), q2(n, s), p3(m, s), q3(m, s);  // potentials (unused)
    uotk_uot_result r1, r2, r3;
    uot_impl(d, n, x, a, m, y, b, eps, lam1, lam2, iters, nullptr, p1.p, q1.p, &r1, opts, comm, s);
    uot_impl(d, n, x, a, n, x, a, eps, lam1, lam2, iters, nullptr, p2.p, q2.p, &r2, opts, comm, s);
    uot_impl(d, m, y, b, m, y, b, eps, lam1, lam2, iters, nullptr, p3.p, q3.p, &r3, opts, comm, s);
    const double dmass = r1.mass_a - r1.mass_b;
    *sd = r1.primal - 0.5 * r2.primal - 0.5 * r3.primal + 0.5 * eps * dmass * dmass;
    if (terms) {
        terms[0] = r1.primal;
        terms[1] = r2.primal;
        terms[2] = r3.primal;
    }
}

// Graph capture is impossible on the legacy / per-thread default streams: work that
// may be replayed from CUDA graphs (small Sinkhorn problems) runs on the library's own
// non-blocking stream, ordered after and before the caller's stream by events.
template <class F>
void on_capturable_stream(cudaStream_t cs, bool graphable, F&& f) {
    const bool default_stream = (uintptr_t)cs <= 2;
    if (!(graphable && default_stream)) {
        f(cs);
        return;
    }
    cudaStream_t ps = private_stream();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    UOTK_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    UOTK_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    UOTK_CUDA(cudaEventRecord(e0, cs));
    UOTK_CUDA(cudaStreamWaitEvent(ps, e0, 0));
    auto finish = [&] {
        cudaEventRecord(e1, ps);
        cudaStreamWaitEvent(cs, e1, 0);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    };
    try {
        f(ps);
    } catch (...) {
        finish();
        throw;
    }
    finish();
}

// ============================================================== c* (Prop. 2.9)
static void cstar_impl(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                       const double* b, double eps, double lam1, double lam2, double* cstar, void* comm,
                       cudaStream_t s) {
    NvtxRange nvtx_call("uotk_uot_cstar");
    need(d >= 1 && d <= 3, "d must be 1, 2 or 3");
    if (comm_nranks(comm) > 1) need(n >= 0 && m >= 0, "n and m must be >= 0");  // empty shards take part
    else need(n >= 1 && m >= 1, "n and m must be >= 1");
    need((x || n == 0) && (a || n == 0) && (y || m == 0) && (b || m == 0) && cstar, "null pointer argument");
    need(eps > 0 && std::isfinite(eps), "eps must be positive and finite");
    need(lam1 > 0 && lam2 > 0 && std::isfinite(lam1) && std::isfinite(lam2), "lam1, lam2 must be positive");
    ensure_pool();
    InArr X, A, Y, B;
    X.bind(x, (size_t)n * d, s);
    A.bind(a, (size_t)n, s);
    Y.bind(y, (size_t)m * d, s);
    B.bind(b, (size_t)m, s);
    DevBuf<int> flag(1, s);
    flag.zero();
    check_mass(A.d, n, flag.p, s);
    check_mass(B.d, m, flag.p, s);
    check_finite(X.d, n * d, flag.p, 8, s);
    check_finite(Y.d, m * d, flag.p, 8, s);
    {
        const int f0 = read_flag(flag, s, comm);
        if (f0 & 8) fail(UOTK_EDOMAIN, "non-finite point coordinate");
        if (f0 & 4) fail(UOTK_EDOMAIN, "masses must be positive and finite");
    }
    const int nc = 2 + d;
    DevBuf<double> cols((size_t)nc * std::max(n, m), s), sums(2 * nc, s), cen(2 * d, s);
    // <mu x nu | d^2> = A B |mx - my|^2 + B sum a |x - mx|^2 + A sum b |y - my|^2 with the
    // weighted means mx, my: pass 1 the masses and first moments, pass 2 the centred
    // second moments (no cancellation between large raw moments)
    double h[2 * 5];
    auto moments = [&](const double* cx, const double* cy) {
        moment_cols(X.d, A.d, n, d, cx, cols.p, s);
        sum_columns(cols.p, n, nc, sums.p, s);
        moment_cols(Y.d, B.d, m, d, cy, cols.p, s);
        sum_columns(cols.p, m, nc, sums.p + nc, s);
        if (comm) comm_allreduce(sums.p, 2 * nc, 0, comm, s);
        UOTK_CUDA(cudaMemcpyAsync(h, sums.p, 2 * nc * sizeof(double), cudaMemcpyDeviceToHost, s));
        UOTK_CUDA(cudaStreamSynchronize(s));
    };
    moments(nullptr, nullptr);
    const double Am = h[0], Bm = h[nc];
    double mean[2 * kMaxD];
    for (int t = 0; t < d; ++t) {
        mean[t] = h[2 + t] / Am;
        mean[d + t] = h[nc + 2 + t] / Bm;
    }
    UOTK_CUDA(cudaMemcpyAsync(cen.p, mean, 2 * d * sizeof(double), cudaMemcpyHostToDevice, s));
    moments(cen.p, cen.p + d);
    double dm2 = 0.0;
    for (int t = 0; t < d; ++t) dm2 += (mean[t] - mean[d + t]) * (mean[t] - mean[d + t]);
    const double T = Am * Bm * dm2 + Bm * h[1] + Am * h[nc + 1];
    const double S = lam1 + lam2 + eps;
    *cstar = std::exp(-T / (Am * Bm * S)) * std::pow(Am, -lam2 / S) * std::pow(Bm, -lam1 / S);
}

// ============================================================== MMD^2
static void mmd2_impl(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                      const double* b, int kind, double param, double* mmd2, const uotk_opts* opts_in, uotk_info* info,
                      void* comm, cudaStream_t s) {
    NvtxRange nvtx_call("uotk_mmd2");
    need(d >= 1 && d <= 3, "d must be 1, 2 or 3");
    need(kind == UOTK_GAUSS || kind == UOTK_IMQ || kind == UOTK_LAP || kind == UOTK_ENERGY, "unknown kernel kind");
    need(param > 0 && std::isfinite(param), "kernel parameter must be positive and finite");
    need(mmd2 != nullptr, "mmd2 output pointer is null");
    check_points_arg(d, n, x, "x");
    check_points_arg(d, n, a, "a");
    check_points_arg(d, m, y, "y");
    check_points_arg(d, m, b, "b");
    const uotk_opts o = resolve(opts_in);
    check_nearfield_ranks(kind, o, comm);
    ensure_pool();
    InArr X, A, Y, B;
    X.bind(x, (size_t)n * d, s);
    A.bind(a, (size_t)n, s);
    Y.bind(y, (size_t)m * d, s);
    B.bind(b, (size_t)m, s);
    const int64_t nz = n + m;
    // z = x u y, w = (a, -b): MMD^2 = sum_i w_i (K w)_i  (3.5)
    DevBuf<double> prod(nz, s), sum(1, s);
    const int method = pick_method(o, (double)nz * (double)nz, comm, direct_crossover_sum(d, kind));
    if (nz == 0 && comm_nranks(comm) == 1) {  // with several ranks an empty shard still takes part
        fill_info(info, method, nullptr, comm);
        *mmd2 = 0.0;
        return;
    }
    if (method == UOTK_DIRECT) {
        fill_info(info, method, nullptr, comm);
        DevBuf<double> z((size_t)nz * d, s), w(nz, s);
        if (n) UOTK_CUDA(cudaMemcpyAsync(z.p, X.d, (size_t)n * d * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (m) UOTK_CUDA(cudaMemcpyAsync(z.p + (size_t)n * d, Y.d, (size_t)m * d * sizeof(double), cudaMemcpyDeviceToDevice, s));
        signed_concat(A.d, n, B.d, m, w.p, s);
        DevBuf<int> flag(1, s);
        flag.zero();
        check_finite(z.p, nz * d, flag.p, 8, s);
        if (read_flag(flag, s) & 8) fail(UOTK_EDOMAIN, "non-finite point coordinate");
        direct_sum_epi(d, nz, z.p, w.p, nz, z.p, kind, param, EpiDot{w.p, prod.p}, nullptr, s);
        sum_columns(prod.p, nz, 1, sum.p, s);
    } else {
        // spread w on the grid, FFT, and sum_k D_k |G_k|^2 (= sum_i w_i t_i of the gather
        // form exactly; no inverse FFT or interpolation needed).  With a communicator the
        // spectrum is all-reduced first, so every rank forms the same global value.  The
        // point set is x u y read in place (no concatenated copy); its weights are
        // gathered from a and -b in sorted order.
        NfftSetup ns;
        setup_nfft(ns, d, kind, param, X.d, n, Y.d, m, o, comm, s);
        PointSet PZ;
        DevBuf<double> ws(nz, s);
        SortedWeights swz;  // w = (a, -b) in sorted order, written by the coordinate gather
        swz.w1 = A.d;
        swz.w2 = B.d;
        swz.sign2 = -1.0;
        swz.out = ws.p;
        make_pointset(PZ, X.d, n, Y.d, m, ns.fp, s, kUseSpreadOnly, swz);
        fill_info(info, method, &ns.fp, comm, &PZ);
        constexpr int kParts = 296;
        DevBuf<double> grid(grid_elems(ns.fp), s), part(kParts, s);
        DevBuf<double2> spec(ns.sp.spec_elems, s);
        grid.zero();
        spread(PZ, ws.p, grid.p, ns.fp, s);
        if (ns.sp.sep_chain) {
            // Gaussian: <g, g'> with g' the separable chain's output (no FFT, no cuFFT plan);
            // with a communicator g' is global and <g_rank, g'> is summed over ranks
            const double* gp = fft_chain(ns.sp, grid.p, spec.p, s, comm);
            box_dot(grid.p, gp, ns.fp, part.p, kParts, s);
            sum_columns(part.p, kParts, 1, sum.p, s);
            if (comm) comm_allreduce(sum.p, 1, 0, comm, s);
        } else {
            spectrum_energy(ns.sp, grid.p, spec.p, part.p, kParts, s, comm);
            sum_columns(part.p, kParts, 1, sum.p, s);
        }
        if (nearfield_needed(ns.fp)) {
            // + sum_i w_i sum_{close j} (K - K_R)(z_i - z_j) w_j
            NearField NZ;
            build_nearfield(NZ, PZ, ns.fp, s);
            DevBuf<double> corr(nz, s), sum2(1, s);
            corr.zero();
            nearfield_apply(NZ, ws.p, NZ, ns.fp, nullptr, corr.p, s);
            multiply(ws.p, corr.p, nz, prod.p, s);
            sum_columns(prod.p, nz, 1, sum2.p, s);
            double h2[2];
            UOTK_CUDA(cudaMemcpyAsync(h2, sum.p, sizeof(double), cudaMemcpyDeviceToHost, s));
            UOTK_CUDA(cudaMemcpyAsync(h2 + 1, sum2.p, sizeof(double), cudaMemcpyDeviceToHost, s));
            UOTK_CUDA(cudaStreamSynchronize(s));
            *mmd2 = h2[0] + h2[1];
            return;
        }
    }
    UOTK_CUDA(cudaMemcpyAsync(mmd2, sum.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    UOTK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace uotk

// ============================================================== extern "C"
using namespace uotk;

extern "C" {

void uotk_opts_init(uotk_opts* opts) {
    if (opts) memset(opts, 0, sizeof *opts);
}

int uotk_kernel_sum(int d, int64_t n_src, const double* src, const double* alpha, int64_t n_tgt, const double* tgt,
                    int kind, double param, double* out, const uotk_opts* opts, uotk_info* info, void* comm,
                    void* cuda_stream) {
    return guarded([&] {
        kernel_sum_impl(d, n_src, src, alpha, n_tgt, tgt, kind, param, out, opts, info, comm,
                        (cudaStream_t)cuda_stream);
    }, comm);
}

int uotk_uot_sinkhorn(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y, const double* b,
                      double eps, double lam1, double lam2, int iters, const double* gamma_init, double* beta,
                      double* gamma, uotk_uot_result* res, const uotk_opts* opts, void* comm, void* cuda_stream) {
    return guarded([&] {
        cudaStream_t cs = (cudaStream_t)cuda_stream;
        const bool graphable = comm_capturable(comm) && iters >= 4 && n >= 0 && m >= 0 && n + m <= kGraphMaxPoints;
        on_capturable_stream(cs, graphable, [&](cudaStream_t st) {
            uot_impl(d, n, x, a, m, y, b, eps, lam1, lam2, iters, gamma_init, beta, gamma, res, opts, comm, st);
        });
    }, comm);
}

int uotk_mmd2(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y, const double* b,
              int kind, double param, double* mmd2, const uotk_opts* opts, uotk_info* info, void* comm,
              void* cuda_stream) {
    return guarded([&] {
        mmd2_impl(d, n, x, a, m, y, b, kind, param, mmd2, opts, info, comm, (cudaStream_t)cuda_stream);
    }, comm);
}

int uotk_uot_cstar(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y, const double* b,
                   double eps, double lam1, double lam2, double* cstar, void* comm, void* cuda_stream) {
    return guarded([&] { cstar_impl(d, n, x, a, m, y, b, eps, lam1, lam2, cstar, comm, (cudaStream_t)cuda_stream); });
}

int uotk_sinkhorn_divergence(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                             const double* b, double eps, double lam1, double lam2, int iters, double* sd,
                             double* terms, const uotk_opts* opts, void* comm, void* cuda_stream) {
    return guarded([&] {
        need(n >= 1 && m >= 1, "n and m must be >= 1");
        need(iters >= 0, "iters must be >= 0");
        cudaStream_t cs = (cudaStream_t)cuda_stream;
        const bool graphable = comm_capturable(comm) && iters >= 4 && 2 * std::max(n, m) <= kGraphMaxPoints;
        on_capturable_stream(cs, graphable, [&](cudaStream_t st) {
            sd_impl(d, n, x, a, m, y, b, eps, lam1, lam2, iters, sd, terms, opts, comm, st);
        });
    }, comm);
}

int uotk_uot_sinkhorn_ex(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                         const double* b, double eps, double lam1, double lam2, int iters, const double* gamma_init,
                         double* beta, double* gamma, double* p, double* q, uotk_uot_result* res,
                         const uotk_opts* opts, void* comm, void* cuda_stream) {
    return guarded([&] {
        cudaStream_t cs = (cudaStream_t)cuda_stream;
        const bool graphable = comm_capturable(comm) && iters >= 4 && n >= 0 && m >= 0 && n + m <= kGraphMaxPoints;
        on_capturable_stream(cs, graphable, [&](cudaStream_t st) {
            uot_impl(d, n, x, a, m, y, b, eps, lam1, lam2, iters, gamma_init, beta, gamma, res, opts, comm, st, p,
                     q);
        });
    }, comm);
}

int uotk_uot_sinkhorn_scaling(int d, int64_t n, const double* x, const double* a, int64_t m, const double* y,
                              const double* b, const double* eps_list, int n_eps, double lam1, double lam2, int iters,
                              const double* gamma_init, double* beta, double* gamma, uotk_uot_result* res,
                              const uotk_opts* opts, void* comm, void* cuda_stream) {
    return guarded([&] {
        need(eps_list != nullptr && n_eps >= 1, "eps_list must hold n_eps >= 1 values");
        for (int k = 0; k < n_eps; ++k) need(eps_list[k] > 0 && std::isfinite(eps_list[k]), "eps_list: eps > 0");
        need(n >= 1 && m >= 1 && beta && gamma, "n, m >= 1 and beta, gamma required");
        cudaStream_t cs = (cudaStream_t)cuda_stream;
        const bool graphable = comm_capturable(comm) && iters >= 4 && n + m <= kGraphMaxPoints;
        on_capturable_stream(cs, graphable, [&](cudaStream_t st) {
            // the previous stage's gamma (device, caller order) warm-starts the next stage
            DevBuf<double> g0(m, st), bt(n, st);
            const double* init = gamma_init;
            int total = 0;
            uotk_uot_result r;
            for (int k = 0; k < n_eps; ++k) {
                const bool last = k == n_eps - 1;
                double* gout = last ? gamma : g0.p;
                double* bout = last ? beta : bt.p;
                if (!last && init == g0.p) {  // gamma_in and gamma_out must not alias
                    DevBuf<double> tmp(m, st);
                    UOTK_CUDA(cudaMemcpyAsync(tmp.p, g0.p, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
                    uot_impl(d, n, x, a, m, y, b, eps_list[k], lam1, lam2, iters, tmp.p, bout, gout, &r, opts, comm,
                             st);
                } else {
                    uot_impl(d, n, x, a, m, y, b, eps_list[k], lam1, lam2, iters, init, bout, gout, &r, opts, comm,
                             st);
                }
                total += r.iters;
                init = g0.p;
            }
            r.iters = total;
            if (res) *res = r;
        });
    }, comm);
}

int uotk_comm_unique_id(void* id128) {
    return guarded([&] {
        if (!id128) fail(UOTK_EINVAL, "null id buffer");
        comm_unique_id(id128);
    });
}

int uotk_comm_create(const void* id128, int nranks, int rank, void** comm_out) {
    return guarded([&] {
        if (!id128 || !comm_out) fail(UOTK_EINVAL, "null argument");
        *comm_out = comm_create(id128, nranks, rank);
    });
}

int uotk_comm_create_loopback(int nranks, void** comms_out) {
    return guarded([&] {
        if (!comms_out) fail(UOTK_EINVAL, "null argument");
        comm_create_loopback(nranks, comms_out);
    });
}

int uotk_comm_destroy(void* comm) {
    return guarded([&] { comm_destroy(comm); });
}

const char* uotk_last_error(void) { return g_last_error.c_str(); }

int uotk_abi_version(void) { return UOTK_ABI_VERSION; }

int uotk_release_caches(void) {
    return uotk::guarded([&] {
        UOTK_CUDA(cudaDeviceSynchronize());
        uotk::release_plan_cache();
        uotk::release_fft_plans();
        uotk::block_cache_release();
        int dev = 0;
        UOTK_CUDA(cudaGetDevice(&dev));
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        cudaGetLastError();
        UOTK_CUDA(cudaDeviceSynchronize());
    });
}

int64_t uotk_launch_counter(void) { return g_launches; }

void uotk_launch_counter_reset(void) { g_launches = 0; }

}  // extern "C"
