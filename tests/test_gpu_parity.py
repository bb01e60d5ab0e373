"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (north star):
  * kernel sums: max relative error 1e-9 — per entry for positive weights, and
    max_i |ds_i| / max_i |s_i| for signed weights (reading R14);
  * UOT cost (primal), dual, plan mass: 1e-8 relative; potentials: the paper's residual
    ||dbeta||/||beta|| + ||dgamma||/||gamma|| <= 1e-8;
  * MMD^2: |d| / max(|MMD^2|, 1e-3 * sum|terms|) <= 1e-8 (reading R13).
"""

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def uk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_13618_b200 as uk
    return uk


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(got, ref, signed):
    got = np.asarray(got)
    ref = np.asarray(ref)
    if signed:
        return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


# ------------------------------------------------------------------ kernel sums
@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("signed", [False, True])
def test_kernel_sum_parity(uk, method, kind, d, signed):
    pr = W.random_sum(d, 3001, 1999, kind=kind, param=(0.0025 if kind == W.GAUSS else 0.05), seed=d, signed=signed)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got, info = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, pr.param,
                              opts={"method": method}, return_info=True)
    assert info["method"] == method
    err = rel_err(got.cpu().numpy(), ref, signed)
    assert err <= 1e-9, (err, info)


@pytest.mark.parametrize("d", [2, 3])
def test_kernel_sum_host_arrays_and_wide_gaussian(uk, d):
    """Host (numpy) inputs are staged by the library; a wide Gaussian (C1's eps=0.05)
    exercises the torus scaling h > 1 (Rem. 4.3)."""
    pr = W.random_sum(d, 2500, 1500, kind=W.GAUSS, param=0.05, seed=11)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got, info = uk.kernel_sum(pr.src, pr.alpha, pr.tgt, "gauss", 0.05, opts={"method": "nfft"}, return_info=True)
    assert isinstance(got, np.ndarray)
    assert info["h"] > 1.0
    assert rel_err(got, ref, False) <= 1e-9


def test_kernel_sum_edge_cases(uk):
    rng = np.random.default_rng(0)
    tgt = W.uniform_ball(rng, 7, 3, 0.2)
    for method in ("direct", "nfft"):
        out = uk.kernel_sum(cuda(np.zeros((0, 3))), cuda(np.zeros(0)), cuda(tgt), "gauss", 0.01,
                            opts={"method": method})
        assert torch.all(out == 0)
        out = uk.kernel_sum(cuda(tgt), cuda(np.ones(7)), cuda(np.zeros((0, 3))), "gauss", 0.01,
                            opts={"method": method})
        assert out.numel() == 0
        # single source exactly at the single target: K(0) alpha
        p = np.array([[0.01, -0.02, 0.03]])
        out = uk.kernel_sum(cuda(p), cuda(np.array([2.0])), cuda(p), "imq", 0.05, opts={"method": method})
        assert abs(out.item() - 2.0 / 0.05) <= 1e-9 * 40
        # all points coincident (zero radius cloud)
        q = np.repeat(p, 5, 0)
        out = uk.kernel_sum(cuda(q), cuda(np.ones(5)), cuda(q), "gauss", 0.01, opts={"method": method})
        assert torch.allclose(out, torch.full_like(out, 5.0), rtol=1e-9, atol=0)
    with pytest.raises(uk.UotkError) as e:
        bad = tgt.copy()
        bad[3, 1] = np.nan
        uk.kernel_sum(cuda(bad), cuda(np.ones(7)), cuda(tgt), "gauss", 0.01, opts={"method": "nfft"})
    assert e.value.code == -2


def test_kernel_sum_c5_full_size_sampled(uk):
    """C5 d=3 at n = m = 1e6 (NFFT), checked on 64 sampled targets by the oracle."""
    pr = W.c5_sum(3, 1_000_000, kind=W.GAUSS)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts={"method": "nfft"})
    idx = np.random.default_rng(1).choice(len(pr.tgt), 64, replace=False)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt[idx], pr.kind, pr.param)
    g = got.cpu().numpy()[idx]
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(g - ref)) / scale <= 1e-9


# ------------------------------------------------------------------ UOT Sinkhorn
def _pot_err(got, ref, c):
    """Element-wise potential error max_i |d_i| / (|ref_i| + c): a potential is
    -c log t (3.3)/(3.4), so a relative error rho of the kernel sum t_i moves it by c rho;
    c floors the denominator where a potential crosses zero."""
    return float(np.max(np.abs(got - ref) / (np.abs(ref) + c))) if len(ref) else 0.0


def _uot_check(res, beta, gamma, ref, eps, lam1, lam2=None, tol=1e-8):
    """UOT parity: the paper's residual ||dbeta||/||beta|| + ||dgamma||/||gamma||,
    every potential element by element (c1 = eta1/(1 + eta1/eps), c2 likewise: the scale
    of (3.3)/(3.4)), and the objective values."""
    lam2 = lam1 if lam2 is None else lam2
    resid = (np.linalg.norm(beta - ref.beta) / np.linalg.norm(ref.beta)
             + np.linalg.norm(gamma - ref.gamma) / np.linalg.norm(ref.gamma))
    assert resid <= tol, resid
    c1 = lam1 / (1.0 + lam1 / eps)
    c2 = lam2 / (1.0 + lam2 / eps)
    eb, eg = _pot_err(beta, ref.beta, c1), _pot_err(gamma, ref.gamma, c2)
    assert eb <= tol and eg <= tol, (eb, eg)
    assert abs(res.primal - ref.primal) <= tol * abs(ref.primal), (res.primal, ref.primal)
    assert abs(res.dual - ref.dual) <= tol * abs(ref.dual), (res.dual, ref.dual)
    assert abs(res.plan_mass - ref.plan_mass) <= tol * ref.plan_mass
    assert abs(res.mass_a - ref.mass_a) <= 1e-13 * ref.mass_a
    assert abs(res.mass_b - ref.mass_b) <= 1e-13 * ref.mass_b


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_c1_full(uk, method):
    """C1 exactly (configs[0]): d=2, n=m=1000, eps=0.05, lam=1, 100 iterations."""
    pr = W.c1_uot()
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": method})
    assert res.info["method"] == method
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)
    assert abs(res.max_dbeta - ref.max_dbeta) <= 1e-6 * max(ref.max_dbeta, 1e-12) + 1e-14


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_c3_like_reduced(uk, method):
    """C3 distributions and parameters (eps=0.02, lam=0.5, d=3) at reduced n, ragged sizes."""
    pr = W.c3_uot(n=1537, m=1201, iters=25)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": method})
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


@pytest.mark.parametrize("n,m", [(6000, 5003), (300, 257)])
def test_uot_c3_dense_reduced_ws_kernel(uk, n, m):
    """The headline's warp-specialised half-step (sinkhorn3d_ws_k: one-cell groups, m = 8)
    at reduced n against the oracle element by element: C3's parameters and per-cell
    density (workloads.c3_dense_uot), ragged chunks (groups of up to ~1000 points cut into
    32-point chunks with ragged tails), and a small case of ~9 chunks in 8 cells (most
    CTAs idle, every chunk partial)."""
    pr = W.c3_dense_uot(n=n, m=m, iters=10)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft"})
    assert res.info["groups"] == (16, 16), res.info  # one-cell groups on both sets: sinkhorn3d_ws_k
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)
    assert abs(res.max_dbeta - ref.max_dbeta) <= 1e-6 * ref.max_dbeta
    assert abs(res.max_dgamma - ref.max_dgamma) <= 1e-6 * ref.max_dgamma


def test_uot_unequal_penalties_gamma_init_and_zero_iters(uk):
    pr = W.c1_uot(n=300, m=250)
    g0 = np.random.default_rng(3).uniform(-0.05, 0.05, 250)
    for method in ("direct", "nfft"):
        ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, 0.7, 2.5, 12, gamma0=g0)
        beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, 0.7, lam2=2.5,
                                           iters=12, gamma_init=cuda(g0), opts={"method": method})
        _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, 0.7, 2.5)
        ref0 = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, 1.0, 1.0, 0)
        beta, gamma, res = uk.uot_sinkhorn(pr.x, pr.a, pr.y, pr.b, pr.eps, 1.0, iters=0, opts={"method": method})
        assert np.all(gamma == 0) and np.all(beta == 0)
        assert abs(res.dual - ref0.dual) <= 1e-9 * abs(ref0.dual)
        assert abs(res.primal - ref0.primal) <= 1e-9 * abs(ref0.primal)


def test_uot_bad_masses(uk):
    pr = W.c1_uot(n=50, m=40)
    a = pr.a.copy()
    a[7] = 0.0
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(cuda(pr.x), cuda(a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=3)
    assert e.value.code == -2


def test_uot_c3_full_size_sampled(uk):
    """C3 at full size (n = m = 1e6, NFFT, as bench.py runs it) for a few iterations: the
    last gamma-step identity gamma_j = -c2 log sum_i k_ij mu_i e^{lam beta_i} (3.4) checked
    by the oracle at 48 sampled j, with the returned beta."""
    pr = W.c3_uot(iters=3)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft"})
    b = beta.cpu().numpy()
    g = gamma.cpu().numpy()
    lam = 1.0 / pr.eps
    c2 = pr.lam / (1.0 + pr.lam * lam)
    idx = np.random.default_rng(2).choice(len(pr.y), 48, replace=False)
    tt = oracle.kernel_sum_direct(pr.x, pr.a * np.exp(lam * b), pr.y[idx], W.GAUSS, pr.eps)
    ref = -c2 * np.log(tt)
    assert np.max(np.abs(g[idx] - ref)) <= 1e-9 * np.max(np.abs(ref))
    assert abs(res.mass_a - pr.a.sum()) <= 1e-12 * pr.a.sum()


# ------------------------------------------------------------------ MMD^2
def _mmd_tol(x, a, y, b, kind, param):
    xx = abs(float(a @ oracle.kernel_sum_direct(x, a, x, kind, param)))
    yy = abs(float(b @ oracle.kernel_sum_direct(y, b, y, kind, param)))
    return xx + yy


@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
def test_mmd2_c2_reduced(uk, method, kind):
    pr = W.c2_mmd(n=2500, m=2100)
    param = dict(pr.kernels)[kind]
    ref = oracle.mmd2_direct(pr.x, pr.a, pr.y, pr.b, kind, param)
    got, info = uk.mmd2(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), kind, param, opts={"method": method},
                        return_info=True)
    denom = max(abs(ref), 1e-3 * _mmd_tol(pr.x, pr.a, pr.y, pr.b, kind, param))
    assert abs(got - ref) / denom <= 1e-8, (got, ref, info)


def test_mmd2_identities(uk):
    rng = np.random.default_rng(5)
    x = W.uniform_ball(rng, 400, 3, 0.2)
    a = rng.uniform(0.5, 1.5, 400)
    for method in ("direct", "nfft"):
        v = uk.mmd2(cuda(x), cuda(a), cuda(x), cuda(a), "gauss", 0.0025, opts={"method": method})
        assert abs(v) <= 1e-10 * a.sum() ** 2
        v = uk.mmd2(cuda(x[:1]), cuda(np.ones(1)), cuda(x[1:2]), cuda(np.ones(1)), "gauss", 0.0025,
                    opts={"method": method})
        r2 = float(np.sum((x[0] - x[1]) ** 2))
        assert abs(v - (2 - 2 * np.exp(-r2 / 0.0025))) <= 1e-9


# ------------------------------------------------------------------ NCCL exchange path
def test_one_rank_nccl_communicator_matches(uk):
    """The multi-GPU code path (bbox min/max, the per-sum all-reduce — of the first
    separable pass's output by default, of the truncated spectrum with UOTK_FLAG_FFT —
    and the scalar sums) through a real 1-rank NCCL communicator gives the single-GPU
    results (up to the summation order of the fp64 atomics that flush the spread)."""
    comm = uk.Comm(uk.Comm.unique_id(), 1, 0)

    def close(p, q, tol=1e-13):
        p, q = torch.as_tensor(p, dtype=torch.float64), torch.as_tensor(q, dtype=torch.float64)
        return bool(torch.max(torch.abs(p - q)) <= tol * torch.max(torch.abs(q)))

    try:
        pr = W.random_sum(3, 3001, 1999, kind=W.GAUSS, param=0.0025, seed=9)
        a = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts={"method": "nfft"})
        b = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts={"method": "nfft"},
                          comm=comm)
        assert close(a, b)
        # the spectrum all-reduce of the FFT chain (the multi-rank path) on the 1-rank comm
        nf = {"method": "nfft", "flags": uk.FLAG_FFT}
        c = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts=nf, comm=comm)
        assert close(a, c)
        u = W.c3_uot(n=1500, m=1300, iters=5)
        r1 = uk.uot_sinkhorn(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, iters=5, opts=nf)
        r2 = uk.uot_sinkhorn(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, iters=5, opts=nf, comm=comm)
        assert close(r1[0], r2[0], 1e-12) and close(r1[1], r2[1], 1e-12)
        assert close(r1[2].primal, r2[2].primal)
        # c* moments and the transport term through the communicator
        c1_ = uk.uot_cstar(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam)
        c2_ = uk.uot_cstar(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, comm=comm)
        assert abs(c1_ - c2_) <= 1e-14 * c1_
        t1 = uk.uot_sinkhorn(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, iters=5,
                             opts={"method": "nfft"}, transport=True)[2].transport
        t2 = uk.uot_sinkhorn(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, iters=5,
                             opts={"method": "nfft"}, transport=True, comm=comm)[2].transport
        assert abs(t1 - t2) <= 1e-12 * abs(t1)
        m = W.c2_mmd(n=2000, m=1800)
        v1 = uk.mmd2(cuda(m.x), cuda(m.a), cuda(m.y), cuda(m.b), "gauss", 0.0025, opts=nf)
        v2 = uk.mmd2(cuda(m.x), cuda(m.a), cuda(m.y), cuda(m.b), "gauss", 0.0025, opts=nf, comm=comm)
        assert close(v1, v2, 1e-12)
    finally:
        comm.close()


def test_one_rank_nccl_slab_chain_collectives():
    """The slab-distributed separable chain's NCCL reduce-scatter and all-gather on a real
    (1-rank) NCCL communicator: UOTK_DIST_CHAIN=2 takes the slab path even with one rank
    (the collectives are copies then), in a subprocess because the switch is read once.
    Kernel sums d = 2, 3 and a short C3-like solve must equal the communicator-free run."""
    import subprocess, sys, os, textwrap
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    code = textwrap.dedent("""
        import numpy as np, torch, paper_2306_13618_b200 as uk, workloads as W
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        comm = uk.Comm(uk.Comm.unique_id(), 1, 0)
        worst = 0.0
        for d in (2, 3):
            pr = W.random_sum(d, 3001, 1999, kind=W.GAUSS, param=0.0025, seed=40 + d)
            a = uk.kernel_sum(t(pr.src), t(pr.alpha), t(pr.tgt), "gauss", pr.param, opts={"method": "nfft"})
            b = uk.kernel_sum(t(pr.src), t(pr.alpha), t(pr.tgt), "gauss", pr.param, opts={"method": "nfft"}, comm=comm)
            worst = max(worst, float(torch.max(torch.abs(a - b)) / torch.max(torch.abs(a))))
        u = W.c3_uot(n=1500, m=1300, iters=5)
        r1 = uk.uot_sinkhorn(t(u.x), t(u.a), t(u.y), t(u.b), u.eps, u.lam, iters=5, opts={"method": "nfft"})
        r2 = uk.uot_sinkhorn(t(u.x), t(u.a), t(u.y), t(u.b), u.eps, u.lam, iters=5, opts={"method": "nfft"}, comm=comm)
        worst = max(worst, float(torch.max(torch.abs(r1[0] - r2[0])) / torch.max(torch.abs(r1[0]))))
        worst = max(worst, abs(r1[2].primal - r2[2].primal) / abs(r1[2].primal))
        comm.close()
        print("WORST", worst)
    """)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UOTK_DIST_CHAIN="2", PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.split("WORST")[-1])
    assert worst <= 1e-13, worst


# ------------------------------------------------------------------ full-size cross-checks
def test_uot_c3_full_size_nfft_vs_direct(uk):
    """C3 at full size (n = m = 1e6): the NFFT path as bench.py runs it against the GPU
    direct kernel (K6, itself oracle-validated above) for 2 iterations (1e12 pairs/sum)."""
    pr = W.c3_uot(iters=2)
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    b1, g1, r1 = uk.uot_sinkhorn(*args, iters=2, opts={"method": "nfft"})
    b2, g2, r2 = uk.uot_sinkhorn(*args, iters=2, opts={"method": "direct"})
    resid = float(torch.linalg.norm(b1 - b2) / torch.linalg.norm(b2) + torch.linalg.norm(g1 - g2) / torch.linalg.norm(g2))
    assert resid <= 1e-8, resid
    assert abs(r1.primal - r2.primal) <= 1e-8 * abs(r2.primal)
    assert abs(r1.dual - r2.dual) <= 1e-8 * abs(r2.dual)
    assert abs(r1.plan_mass - r2.plan_mass) <= 1e-8 * r2.plan_mass


@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
def test_mmd2_c2_full_size_nfft_vs_direct(uk, kind):
    """C2 at full size (n = m = 1e5, 4e10 pairs): Fourier-domain NFFT MMD^2 vs the GPU
    direct kernel, with the cancellation-aware denominator of reading R13."""
    pr = W.c2_mmd()
    param = dict(pr.kernels)[kind]
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)
    v1, info = uk.mmd2(x, a, y, b, kind, param, opts={"method": "nfft"}, return_info=True)
    v2 = uk.mmd2(x, a, y, b, kind, param, opts={"method": "direct"})
    xx = uk.mmd2(x, a, x[:0], b[:0], kind, param, opts={"method": "direct"})
    yy = uk.mmd2(y, b, y[:0], b[:0], kind, param, opts={"method": "direct"})
    denom = max(abs(v2), 1e-3 * (abs(xx) + abs(yy)))
    assert abs(v1 - v2) / denom <= 1e-8, (v1, v2, info)


# ------------------------------------------------------------------ cell-group kernels in d = 1, 2
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
@pytest.mark.parametrize("signed", [False, True])
def test_kernel_sum_cell_group_kernels(uk, d, kind, signed):
    """The cell-group (chunked) kernels forced at any density and the generic
    thread-per-point kernels, both against the oracle; ragged sizes (chunks of 32 with a
    ragged tail in every cell)."""
    pr = W.random_sum(d, 6001, 3001, kind=kind, param=(0.0025 if kind == W.GAUSS else 0.05), seed=20 + d,
                      signed=signed)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    for flags in (uk.FLAG_CHUNKED, uk.FLAG_GENERIC):
        got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, pr.param,
                            opts={"method": "nfft", "flags": flags})
        err = rel_err(got.cpu().numpy(), ref, signed)
        assert err <= 1e-9, (flags, err)


@pytest.mark.parametrize("d", [1, 2])
def test_kernel_sum_dense_cloud_auto(uk, d):
    """A dense cloud (wide Gaussian, C1's eps = 0.05) takes the cell-group kernels by
    default (hundreds of points per cell)."""
    pr = W.random_sum(d, 40_000, 2_003, kind=W.GAUSS, param=0.05, seed=31)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts={"method": "nfft"})
    assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9


@pytest.fixture(scope="module")
def c4_reduced():
    pr = W.c4_uot(n=5003, m=4001, iters=12)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    return pr, ref


@pytest.mark.parametrize("flags", ["chunked", "generic"])
@pytest.mark.parametrize("N", [0, 2048])
def test_uot_c4_like_reduced(uk, c4_reduced, flags, N):
    """C4's parameters (d = 2, eps = 0.002, lam = 2) at reduced n: the fused d = 2
    half-step (gather -> update -> spread in one launch) and the generic path, with the
    automatic bandwidth (N = 80, grid 160^2) and with the literal reading of the config's
    "oversampled grid 4096^2" (N = 2048; reading R19)."""
    pr, ref = c4_reduced
    f = uk.FLAG_CHUNKED if flags == "chunked" else uk.FLAG_GENERIC
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft", "flags": f, "N": N})
    assert res.info["n_grid"] == (4096 if N else 160)
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


def test_uot_c1_chunked_nfft(uk):
    """C1 exactly through the d = 2 fused half-step (forced; AUTO picks DIRECT at C1)."""
    pr = W.c1_uot()
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft", "flags": uk.FLAG_CHUNKED})
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


def test_uot_c4_full_size_sampled(uk):
    """C4 at full size (d = 2, n = m = 16M, eps = 0.002, lam = 2; NFFT on the cell-group
    kernels) for 3 iterations: the last gamma-step identity (3.4) checked by the oracle at
    24 sampled j with the returned beta."""
    pr = W.c4_uot(iters=3)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft"})
    b = beta.cpu().numpy()
    g = gamma.cpu().numpy()
    lam = 1.0 / pr.eps
    c2 = pr.lam / (1.0 + pr.lam * lam)
    idx = np.random.default_rng(4).choice(len(pr.y), 24, replace=False)
    tt = oracle.kernel_sum_direct(pr.x, pr.a * np.exp(lam * b), pr.y[idx], W.GAUSS, pr.eps)
    ref = -c2 * np.log(tt)
    assert np.max(np.abs(g[idx] - ref)) <= 1e-9 * np.max(np.abs(ref))
    assert abs(res.mass_a - pr.a.sum()) <= 1e-12 * pr.a.sum()


def test_uot_c4_full_size_grid4096_sampled(uk):
    """C4 at full size with the config's literal "oversampled grid 4096^2" (opts.N = 2048,
    reading R19; 134 MB grids, beyond L2): 3 iterations, then the last gamma-step identity
    (3.4) at 24 sampled j and the last beta-step identity (3.3) at 24 sampled i, each
    against the oracle with the returned potentials."""
    pr = W.c4_uot(iters=3)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts={"method": "nfft", "N": 2048})
    # ~5 points per cell at 4096^2: y-segment groups (9 cells along y, 16 x 24 footprints)
    assert res.info["n_grid"] == 4096 and res.info["groups"] == (24, 24), res.info
    b = beta.cpu().numpy()
    g = gamma.cpu().numpy()
    lam = 1.0 / pr.eps
    c = pr.lam / (1.0 + pr.lam * lam)
    rng = np.random.default_rng(8)
    jdx = rng.choice(len(pr.y), 24, replace=False)
    tt = oracle.kernel_sum_direct(pr.x, pr.a * np.exp(lam * b), pr.y[jdx], W.GAUSS, pr.eps)
    assert _pot_err(g[jdx], -c * np.log(tt), c) <= 1e-9
    # the beta-step of the last iteration saw the gamma of the previous one; the marginal
    # p_i = mu_i e^{lam beta_i} t_i (t from the final gamma) is the plan's row sum
    idx = rng.choice(len(pr.x), 24, replace=False)
    t = oracle.kernel_sum_direct(pr.y, pr.b * np.exp(lam * g), pr.x[idx], W.GAUSS, pr.eps)
    p_ref = pr.a[idx] * np.exp(lam * b[idx]) * t
    _, _, r2 = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=pr.iters,
                               opts={"method": "nfft", "N": 2048}, marginals=True)
    p = r2.p.cpu().numpy()[idx]
    assert np.max(np.abs(p - p_ref) / p_ref) <= 1e-8
    assert abs(res.mass_a - pr.a.sum()) <= 1e-12 * pr.a.sum()


@pytest.mark.parametrize("d", [1, 2])
def test_kernel_sum_c5_dense_sampled(uk, d):
    """C5 in d = 1, 2 at n = m = 1e6 (signed N(0,1) weights; cell-group kernels), checked
    on 64 sampled targets by the oracle."""
    pr = W.c5_sum(d, 1_000_000, kind=W.GAUSS)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param, opts={"method": "nfft"})
    idx = np.random.default_rng(5).choice(len(pr.tgt), 64, replace=False)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt[idx], pr.kind, pr.param)
    g = got.cpu().numpy()[idx]
    assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) <= 1e-9


@pytest.mark.parametrize("flags", ["chunked", "auto"])
def test_uot_d3_sparse_cloud(uk, flags):
    """A sparse d = 3 cloud (uniform ball, C3's eps and lam, ~1 point per cell): forced
    cell-group kernels take the z-segment groups (16 x 16 x 24 footprints) and the
    phase-locked fused half-step; AUTO may use either family — both against the oracle."""
    rng = np.random.default_rng(41)
    n, m = 3001, 2503
    x = W.uniform_ball(rng, n, 3, 0.2)
    y = W.uniform_ball(rng, m, 3, 0.2)
    a = rng.uniform(0.1, 1.0, n)
    b = rng.uniform(0.1, 1.0, m)
    ref = oracle.uot_sinkhorn_direct(x, a, y, b, 0.02, 0.5, 0.5, 8)
    opts = {"method": "nfft"}
    if flags == "chunked":
        opts["flags"] = uk.FLAG_CHUNKED
    beta, gamma, res = uk.uot_sinkhorn(cuda(x), cuda(a), cuda(y), cuda(b), 0.02, 0.5, iters=8, opts=opts)
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, 0.02, 0.5)


def test_mmd2_c2_imq_chunked_vs_generic(uk):
    """C2's IMQ MMD^2 (grid 384^3, ~4 points per cell) through the z-segment cell-group
    spread and through the generic spread: identical up to rounding, and both match the
    GPU direct sum (itself oracle-validated) with the R13 denominator."""
    pr = W.c2_mmd(n=20_000, m=18_000)
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)
    v1 = uk.mmd2(x, a, y, b, "imq", 0.05, opts={"method": "nfft", "flags": uk.FLAG_CHUNKED})
    v2 = uk.mmd2(x, a, y, b, "imq", 0.05, opts={"method": "nfft", "flags": uk.FLAG_GENERIC})
    vd = uk.mmd2(x, a, y, b, "imq", 0.05, opts={"method": "direct"})
    xx = uk.mmd2(x, a, x[:0], b[:0], "imq", 0.05, opts={"method": "direct"})
    yy = uk.mmd2(y, b, y[:0], b[:0], "imq", 0.05, opts={"method": "direct"})
    denom = max(abs(vd), 1e-3 * (abs(xx) + abs(yy)))
    assert abs(v1 - vd) / denom <= 1e-8, (v1, vd)
    assert abs(v2 - vd) / denom <= 1e-8, (v2, vd)


@pytest.mark.parametrize("d,kind", [(3, W.GAUSS), (3, W.IMQ), (2, W.IMQ), (1, W.IMQ)])
def test_kernel_sum_c5_1e7_sampled(uk, d, kind):
    """C5 at n = m = 1e7 (signed N(0,1) weights): dense d = 3 cell groups (Gauss, 140^3),
    z-segment groups (IMQ, 384^3), d = 2 / d = 1 cell groups — 32 sampled targets against
    the oracle."""
    pr = W.c5_sum(d, 10_000_000, kind=kind)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, pr.param, opts={"method": "nfft"})
    idx = np.random.default_rng(6).choice(len(pr.tgt), 32, replace=False)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt[idx], pr.kind, pr.param)
    g = got.cpu().numpy()[idx]
    assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) <= 1e-9


def test_kernel_sum_c5_1e8_d3_sampled(uk):
    """C5's largest size, n = m = 1e8 in d = 3 (Gaussian l = 0.05): 2 x 48 GB of window
    blocks on the cell-group kernels; 8 sampled targets against the oracle."""
    pr = W.c5_sum(3, 100_000_000, kind=W.GAUSS)
    src, alpha, tgt = cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt)
    got = uk.kernel_sum(src, alpha, tgt, "gauss", pr.param, opts={"method": "nfft"})
    g_all = got.cpu().numpy()
    del src, alpha, tgt, got
    torch.cuda.empty_cache()
    idx = np.random.default_rng(7).choice(len(pr.tgt), 8, replace=False)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt[idx], pr.kind, pr.param, block_bytes=1 << 31)
    assert np.max(np.abs(g_all[idx] - ref)) / np.max(np.abs(ref)) <= 1e-9


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_small_graph_replay_on_user_stream(uk, method):
    """Small problems replay captured iterations from CUDA graphs: on a caller-created
    stream (captured directly) and on the default stream (the library's own stream),
    both equal to the oracle; iteration counts that leave eager remainders."""
    pr = W.c1_uot(n=700, m=650)
    for iters in (4, 37):
        ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters)
        st = torch.cuda.Stream()
        args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            beta, gamma, res = uk.uot_sinkhorn(*args, iters=iters, opts={"method": method}, stream=st)
        st.synchronize()
        _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)
        beta2, gamma2, res2 = uk.uot_sinkhorn(*args, iters=iters, opts={"method": method})
        _uot_check(res2, beta2.cpu().numpy(), gamma2.cpu().numpy(), ref, pr.eps, pr.lam)


# ------------------------------------------------------------------ solver variants
@pytest.mark.parametrize("d", [2, 3])
def test_uot_cstar_matches_oracle(uk, d):
    """c* of Eq. (2.10): the library's centred moment formula against the oracle's
    pairwise definition of <mu x nu | d^2>; points far from the origin (shifted by 5)
    to exercise the centring."""
    rng = np.random.default_rng(50 + d)
    x = W.uniform_ball(rng, 3001, d, 0.2) + 5.0
    y = W.uniform_ball(rng, 2003, d, 0.2) + 5.05
    a = rng.uniform(0.5, 1.5, 3001)
    b = rng.uniform(0.2, 2.0, 2003)
    for (e1, e2) in ((1.0, 1.0), (0.3, 2.5)):
        ref = oracle.cstar(x, a, y, b, 0.05, e1, e2)
        got = uk.uot_cstar(cuda(x), cuda(a), cuda(y), cuda(b), 0.05, e1, e2)
        assert abs(got - ref) <= 1e-12 * ref, (got, ref)


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_gamma_init_cstar(uk, method):
    """Remark 5.2: gamma^0 = c* 1, against the oracle started from the same gamma^0."""
    pr = W.c1_uot(n=600, m=500)
    c = oracle.cstar(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, 20, gamma0=np.full(500, c))
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=20,
                                       gamma_init="cstar", opts={"method": method})
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_stopping_rule(uk, method):
    """Tolerance stopping (reading R20): same stopping iteration as the oracle (the
    tolerance sits 12-45% away from the sup-norm changes at the neighbouring checks,
    far beyond rounding), same result."""
    pr = W.c1_uot(n=300, m=250)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters=400, stop_tol=1e-9,
                                     check_every=5)
    assert ref.iters == 175
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=400,
                                       opts={"method": method, "stop_tol": 1e-9, "check_every": 5})
    assert res.iters == ref.iters
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)
    assert res.max_dbeta <= 1e-9 and res.max_dgamma <= 1e-9


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_sinkhorn_divergence_matches_oracle(uk, method):
    """Eq. (2.12) from three UOT solves, against the oracle; the tolerance is relative
    to the largest UOT term (sd itself is a cancellation of the three)."""
    pr = W.c1_uot(n=400, m=300)
    ref, terms = oracle.sinkhorn_divergence_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters=30)
    sd, got_terms = uk.sinkhorn_divergence(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=30,
                                           opts={"method": method}, return_terms=True)
    scale = max(abs(t) for t in terms)
    assert abs(sd - ref) <= 1e-8 * scale, (sd, ref)
    for g_, r_ in zip(got_terms, terms):
        assert abs(g_ - r_) <= 1e-8 * abs(r_)


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_lambda_scaling(uk, method):
    """lambda-scaling (Sec. 5.1.3): three stages eps = 0.2, 0.1, 0.05, each warm-started
    from the previous gamma, against the oracle's stage loop."""
    pr = W.c1_uot(n=500, m=450)
    eps_list = [0.2, 0.1, 0.05]
    ref = oracle.uot_sinkhorn_scaling_direct(pr.x, pr.a, pr.y, pr.b, eps_list, pr.lam, iters=15)
    beta, gamma, res = uk.uot_sinkhorn_scaling(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), eps_list, pr.lam,
                                               iters=15, opts={"method": method})
    assert res.iters == 45 == ref.iters
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, eps_list[-1], pr.lam)


# ------------------------------------------------------------------ transport term and marginals (8(f) f4)
@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_kernel_sum_gauss_r2(uk, method, d):
    """The transport-cost kernel r^2 exp(-r^2/eps) (UOTK_GAUSS_R2) against the oracle."""
    pr = W.random_sum(d, 3001, 1999, kind=W.GAUSS, param=0.02, seed=60 + d)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, 2, 0.02)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss_r2", 0.02, opts={"method": method})
    assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9


@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("d", [2, 3])
def test_uot_transport_and_marginals(uk, method, d):
    """<pi, d^2> and the plan marginals p, q (caller order) against the oracle."""
    pr = W.c1_uot(n=800, m=700, d=d) if d == 2 else W.c3_uot(n=1200, m=1000, iters=20)
    iters = 20
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters)
    p_ref, q_ref = oracle.plan_marginals(pr.x, pr.a, pr.y, pr.b, ref.beta, ref.gamma, pr.eps)
    t_ref = oracle.transport_cost(pr.x, pr.a, pr.y, pr.b, ref.beta, ref.gamma, pr.eps)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=iters,
                                       opts={"method": method}, marginals=True, transport=True)
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)
    assert rel_err(res.p.cpu().numpy(), p_ref, False) <= 1e-8
    assert rel_err(res.q.cpu().numpy(), q_ref, False) <= 1e-8
    assert abs(res.transport - t_ref) <= 1e-8 * abs(t_ref), (res.transport, t_ref)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_fft_chain_vs_separable_chain(uk, d):
    """The Gaussian's two spectral chains — cuFFT D2Z / D_k / Z2D (multi-rank path,
    UOTK_FLAG_FFT) and the box-restricted circulant GEMMs — both against the oracle."""
    pr = W.random_sum(d, 3001, 1999, kind=W.GAUSS, param=0.0025, seed=70 + d)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    for flags in (uk.FLAG_FFT, 0):
        got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param,
                            opts={"method": "nfft", "flags": flags})
        assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9, flags
    u = W.c3_uot(n=1100, m=900, iters=10) if d == 3 else W.c1_uot(n=800, m=700, d=d)
    iters = 10
    ref = oracle.uot_sinkhorn_direct(u.x, u.a, u.y, u.b, u.eps, u.lam, u.lam, iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(u.x), cuda(u.a), cuda(u.y), cuda(u.b), u.eps, u.lam, iters=iters,
                                       opts={"method": "nfft", "flags": uk.FLAG_FFT})
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, u.eps, u.lam)


@pytest.mark.parametrize("method", ["direct", "nfft"])
def test_uot_d1(uk, method):
    """UOT in d = 1 (C1's distributions and parameters on a line): the d = 1 cell-group
    half-step and the separable chain by default."""
    pr = W.c1_uot(n=2000, m=1500, d=1)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, 30)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=30,
                                       opts={"method": method})
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


# ------------------------------------------------------------------ d = 3, m = 6 cell-group kernels
M6 = {"m": 6, "sigma": 3.0}


@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
@pytest.mark.parametrize("signed", [False, True])
def test_kernel_sum_m6_cell_group_kernels(uk, kind, signed):
    """m = 6, sigma = 3 (12 taps per axis, fused3d_m6.cu): the cell-group kernels forced at
    any density and the generic kernels against the oracle (ragged chunks), and against
    each other to rounding."""
    pr = W.random_sum(3, 6001, 3001, kind=kind, param=(0.0025 if kind == W.GAUSS else 0.05), seed=41,
                      signed=signed)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    out = {}
    for flags in (uk.FLAG_CHUNKED, uk.FLAG_GENERIC):
        got, info = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, pr.param,
                                  opts=dict(M6, method="nfft", flags=flags), return_info=True)
        assert info["m"] == 6
        out[flags] = got.cpu().numpy()
        assert rel_err(out[flags], ref, signed) <= 1e-9, (flags, rel_err(out[flags], ref, signed))
    assert rel_err(out[uk.FLAG_CHUNKED], out[uk.FLAG_GENERIC], True) <= 1e-13


@pytest.mark.parametrize("flags", ["chunked", "generic"])
def test_uot_c3_like_reduced_m6(uk, flags):
    """C3 at reduced n with m = 6, sigma = 3: the m = 6 warp-specialised half-step
    (sinkhorn3d_m6_ws_k) and the generic path against the oracle."""
    pr = W.c3_uot(n=1537, m=1201, iters=25)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    f = uk.FLAG_CHUNKED if flags == "chunked" else uk.FLAG_GENERIC
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam,
                                       iters=pr.iters, opts=dict(M6, method="nfft", flags=f))
    assert res.info["m"] == 6
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


def test_uot_c3_full_size_sampled_m6(uk):
    """C3 at full size with m = 6, sigma = 3 (cell-group kernels by default at this
    density): the gamma-step identity (3.4) at 48 sampled j against the oracle, and the
    solve against the m = 8 solve (same iterations) on the objective values."""
    pr = W.c3_uot(iters=4)
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    beta, gamma, res = uk.uot_sinkhorn(*args, iters=pr.iters, opts=dict(M6, method="nfft"))
    assert res.info["m"] == 6 and res.info["n_grid"] >= 3 * res.info["N"]
    b = beta.cpu().numpy()
    g = gamma.cpu().numpy()
    lam = 1.0 / pr.eps
    c2 = pr.lam / (1.0 + pr.lam * lam)
    idx = np.random.default_rng(4).choice(len(pr.y), 48, replace=False)
    tt = oracle.kernel_sum_direct(pr.x, pr.a * np.exp(lam * b), pr.y[idx], W.GAUSS, pr.eps)
    ref = -c2 * np.log(tt)
    assert np.max(np.abs(g[idx] - ref)) <= 1e-9 * np.max(np.abs(ref))
    _, _, r8 = uk.uot_sinkhorn(*args, iters=pr.iters, opts={"method": "nfft"})
    assert abs(res.primal - r8.primal) <= 1e-9 * abs(r8.primal)
    assert abs(res.dual - r8.dual) <= 1e-9 * abs(r8.dual)


@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
def test_mmd2_c2_reduced_m6(uk, kind):
    """MMD^2 (spread + Fourier-domain sum) with the m = 6 spread kernel, forced."""
    pr = W.c2_mmd(n=2500, m=2100)
    param = dict(pr.kernels)[kind]
    ref = oracle.mmd2_direct(pr.x, pr.a, pr.y, pr.b, kind, param)
    got = uk.mmd2(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), kind, param,
                  opts=dict(M6, method="nfft", flags=uk.FLAG_CHUNKED))
    denom = max(abs(ref), 1e-3 * _mmd_tol(pr.x, pr.a, pr.y, pr.b, kind, param))
    assert abs(got - ref) / denom <= 1e-8, (got, ref)


def test_release_caches_then_cold_calls_agree(uk):
    """uotk_release_caches drops the cached tables, plans and buffers; the following calls
    (cold: tables and plans rebuilt) give the same results as the warm ones."""
    pr = W.c2_mmd(n=3001, m=2503)
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b))
    warm = [uk.mmd2(*args, kind, param, opts={"method": "nfft"}) for kind, param in pr.kernels]
    s_warm = uk.kernel_sum(args[0], args[1], args[2], "imq", 0.05, opts={"method": "nfft"})
    uk.release_caches()
    cold = [uk.mmd2(*args, kind, param, opts={"method": "nfft"}) for kind, param in pr.kernels]
    s_cold = uk.kernel_sum(args[0], args[1], args[2], "imq", 0.05, opts={"method": "nfft"})
    for w, c in zip(warm, cold):
        assert abs(w - c) <= 1e-13 * abs(w)
    assert float(torch.max(torch.abs(s_warm - s_cold))) <= 1e-13 * float(torch.max(torch.abs(s_warm)))
    uk.release_caches()


@pytest.mark.parametrize("n", [1, 31, 33, 97])
def test_kernel_sum_m6_tiny_and_ragged(uk, n):
    """m = 6 cell-group kernels (forced) at sizes below, at and just above one chunk."""
    pr = W.random_sum(3, n, n + 5, kind=W.GAUSS, param=0.02, seed=50 + n, signed=False)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param,
                        opts=dict(M6, method="nfft", flags=uk.FLAG_CHUNKED))
    assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9
    pr2 = W.c3_uot(n=n, m=n + 3, iters=5)
    ref2 = oracle.uot_sinkhorn_direct(pr2.x, pr2.a, pr2.y, pr2.b, pr2.eps, pr2.lam, pr2.lam, pr2.iters)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr2.x), cuda(pr2.a), cuda(pr2.y), cuda(pr2.b), pr2.eps, pr2.lam,
                                       iters=pr2.iters, opts=dict(M6, method="nfft", flags=uk.FLAG_CHUNKED))
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref2, pr2.eps, pr2.lam)


def test_error_paths_overflow_and_nonfinite(uk):
    """UOTK_EOVERFLOW when the Sinkhorn kernel sums underflow to 0 (far-apart clouds,
    eps tiny: exp(-0.04 / 1e-5) = 0 in fp64), and UOTK_EDOMAIN for a non-finite coordinate."""
    x = np.zeros((3, 2))
    y = np.full((4, 2), 0.2)
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(cuda(x), cuda(np.ones(3)), cuda(y), cuda(np.ones(4)), 1e-5, 1.0, iters=3,
                        opts={"method": "direct"})
    assert e.value.code == -3
    xs = W.uniform_ball(np.random.default_rng(1), 200, 3, 0.2)
    xs[17, 1] = np.nan
    with pytest.raises(uk.UotkError) as e:
        uk.kernel_sum(cuda(xs), cuda(np.ones(200)), cuda(xs), "gauss", 0.0025, opts={"method": "nfft"})
    assert e.value.code == -2


def test_auto_method_crossover(uk):
    """AUTO picks the direct kernel below the measured crossover (DESIGN.md §1 a0): a d = 3
    kernel sum of 1e4 x 1e4 pairs (1e8 < 4e8) runs direct, 3e4 x 3e4 (9e8) runs the NFFT;
    both agree with each other."""
    small = W.random_sum(3, 10_000, 10_000, kind=W.GAUSS, param=0.0025, seed=7)
    got, info = uk.kernel_sum(cuda(small.src), cuda(small.alpha), cuda(small.tgt), "gauss", small.param,
                              return_info=True)
    assert info["method"] == "direct"
    big = W.random_sum(3, 30_000, 30_000, kind=W.GAUSS, param=0.0025, seed=8)
    got_b, info_b = uk.kernel_sum(cuda(big.src), cuda(big.alpha), cuda(big.tgt), "gauss", big.param,
                                  return_info=True)
    assert info_b["method"] == "nfft"
    ref_b = uk.kernel_sum(cuda(big.src), cuda(big.alpha), cuda(big.tgt), "gauss", big.param,
                          opts={"method": "direct"})
    assert rel_err(got_b.cpu().numpy(), ref_b.cpu().numpy(), False) <= 1e-9


def test_spread_only_hybrid_groups(uk):
    """Spread-only d = 3 sets whose one-cell chunks are partly filled take hybrid groups
    (uotk_info.groups 1624: cells with >= 24 points alone, the sparser cells of a 9-cell
    z-segment on one 16 x 16 x 24 footprint, windows evaluated in the spread with the z taps
    at the point's offset): MMD^2 and a kernel sum on C2's mixtures shrunk to C2-at-1M cell
    densities (workloads.c2_dense_mmd) against the oracle, and against the generic kernels."""
    pr = W.c2_dense_mmd(n=10000)
    param = 0.0025
    v, info = uk.mmd2(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), "gauss", param, opts={"method": "nfft"},
                      return_info=True)
    assert info["groups"][0] == 1624, info
    mref = oracle.mmd2_direct(pr.x, pr.a, pr.y, pr.b, W.GAUSS, param)
    denom = max(abs(mref), 1e-3 * _mmd_tol(pr.x, pr.a, pr.y, pr.b, W.GAUSS, param))
    assert abs(v - mref) / denom <= 1e-8, (v, mref)
    gen = uk.mmd2(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), "gauss", param,
                  opts={"method": "nfft", "flags": uk.FLAG_GENERIC})
    assert abs(v - gen) <= 1e-12 * abs(gen), (v, gen)
    got, kinfo = uk.kernel_sum(cuda(pr.x), cuda(pr.a), cuda(pr.y[:2000]), "gauss", param, opts={"method": "nfft"},
                               return_info=True)
    assert kinfo["groups"][0] == 1624, kinfo
    ref = oracle.kernel_sum_direct(pr.x, pr.a, pr.y[:2000], W.GAUSS, param)
    assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9
    kgen = uk.kernel_sum(cuda(pr.x), cuda(pr.a), cuda(pr.y[:2000]), "gauss", param,
                         opts={"method": "nfft", "flags": uk.FLAG_GENERIC})
    assert rel_err(got.cpu().numpy(), kgen.cpu().numpy(), False) <= 1e-13


@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
def test_spread_only_windows_on_the_fly(uk, kind):
    """Spread-only d = 3 one-cell sets (kernel-sum sources, MMD^2's z) evaluate their window
    blocks inside the spread kernel (spread3d_fly_k): dense sources (C3 per-cell density)
    against the oracle for a kernel sum and an MMD^2, and against the precomputed-window
    spread (UOTK_SPREAD_FLY=0 in a subprocess is the A/B; here: the generic kernels)."""
    pr = W.c3_dense_uot(n=20000, m=3001)
    param = 0.02 if kind == W.GAUSS else 0.05
    got, info = uk.kernel_sum(cuda(pr.x), cuda(pr.a), cuda(pr.y), kind, param, opts={"method": "nfft"},
                              return_info=True)
    if kind == W.GAUSS:  # (the IMQ's torus scaling follows the cloud: a sparser grid, generic kernels)
        assert info["groups"][0] == 16, info
    ref = oracle.kernel_sum_direct(pr.x, pr.a, pr.y, kind, param)
    assert rel_err(got.cpu().numpy(), ref, False) <= 1e-9
    gen = uk.kernel_sum(cuda(pr.x), cuda(pr.a), cuda(pr.y), kind, param, opts={"method": "nfft", "flags": uk.FLAG_GENERIC})
    assert rel_err(got.cpu().numpy(), gen.cpu().numpy(), False) <= 1e-13
    v, minfo = uk.mmd2(cuda(pr.x), cuda(pr.a), cuda(pr.y[:2500]), cuda(pr.b[:2500]), kind, param,
                       opts={"method": "nfft"}, return_info=True)
    mref = oracle.mmd2_direct(pr.x, pr.a, pr.y[:2500], pr.b[:2500], kind, param)
    denom = max(abs(mref), 1e-3 * _mmd_tol(pr.x, pr.a, pr.y[:2500], pr.b[:2500], kind, param))
    assert abs(v - mref) / denom <= 1e-8, (v, mref, minfo)


@pytest.mark.parametrize("n,m", [(500, 450), (1201, 999)])
def test_uot_d2_y_segments(uk, n, m):
    """d = 2 clouds of a few points per cell take y-segment groups (kSegY cells along y share
    one 16 x 24 footprint; the y-windows sit at the cell's offset in the segment) in the
    warp-specialised half-step: against the oracle element by element."""
    pr = W.c1_uot(n=n, m=m)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, 12)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam, iters=12,
                                       opts={"method": "nfft"})
    assert res.info["groups"] == (24, 24), res.info
    _uot_check(res, beta.cpu().numpy(), gamma.cpu().numpy(), ref, pr.eps, pr.lam)


@pytest.mark.parametrize("kind", [W.GAUSS, W.IMQ])
def test_kernel_sum_d2_y_segments(uk, kind):
    """Stand-alone d = 2 spread and gather on y-segment groups (forced cell-group kernels)."""
    n = 3001 if kind == W.GAUSS else 30001  # ~1 point per cell (the IMQ's grid is 512^2)
    pr = W.random_sum(2, n, 2003, kind=kind, param=(0.0025 if kind == W.GAUSS else 0.05), seed=77, signed=True)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got, info = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, pr.param,
                              opts={"method": "nfft", "flags": uk.FLAG_CHUNKED}, return_info=True)
    assert info["groups"][0] == 24, info
    assert rel_err(got.cpu().numpy(), ref, True) <= 1e-9


def test_pinned_host_inputs_give_pinned_outputs(uk):
    """Host (pinned CPU tensor) inputs: the library stages the copies itself and the binding
    returns pinned CPU outputs (so the device->host copy runs at DMA speed); the values equal
    the oracle and the device-resident call's."""
    pr = W.random_sum(3, 3001, 1999, kind=W.GAUSS, param=0.0025, seed=21)
    host = [torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for v in (pr.src, pr.alpha, pr.tgt)]
    got = uk.kernel_sum(*host, "gauss", 0.0025, opts={"method": "nfft"})
    assert got.device.type == "cpu" and got.is_pinned()
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, W.GAUSS, 0.0025)
    assert rel_err(got.numpy(), ref, False) <= 1e-9
    dev = uk.kernel_sum(*(h.cuda() for h in host), "gauss", 0.0025, opts={"method": "nfft"})
    assert rel_err(got.numpy(), dev.cpu().numpy(), False) <= 1e-13
    u = W.c1_uot(n=700, m=500)
    hu = [torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for v in (u.x, u.a, u.y, u.b)]
    beta, gamma, res = uk.uot_sinkhorn(*hu, u.eps, u.lam, iters=5, opts={"method": "nfft"})
    assert beta.is_pinned() and gamma.is_pinned()
    bd, gd, _ = uk.uot_sinkhorn(*(h.cuda() for h in hu), u.eps, u.lam, iters=5, opts={"method": "nfft"})
    assert np.max(np.abs(beta.numpy() - bd.cpu().numpy())) <= 1e-12 * np.max(np.abs(bd.cpu().numpy()))
    assert np.max(np.abs(gamma.numpy() - gd.cpu().numpy())) <= 1e-12 * np.max(np.abs(gd.cpu().numpy()))
