"""Deterministic mode (uotk_opts.deterministic) and a repetition stress test of the
mbarrier / TMA-ring kernels.

* deterministic = 1: every spread pulls each grid value in the points' sorted order
  (determ.cu) and the fused half-steps run as gather + update + spread, so two calls give
  bitwise identical outputs; the results equal the oracle (same bars as
  test_gpu_parity.py) and the default (atomic) path to rounding.
* Stress: compute-sanitizer is closed on this GPU pool (profiles/r02/sanitizer.md), so the
  warp-specialised / TMA-ring kernels are run many times on small inputs and every run
  is compared with the first and with the oracle: a shared-memory race (a window slot or
  weighted-row slot reused too early) shows up as sporadic O(1) errors, far above the
  1e-13 run-to-run spread of the atomic flushes.
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


def _cases():
    rng = np.random.default_rng(3)
    sparse = W.UOTProblem("sparse-d3", W.uniform_ball(rng, 3000, 3, 0.2), rng.uniform(0.1, 1, 3000),
                          W.uniform_ball(rng, 2500, 3, 0.2), rng.uniform(0.1, 1, 2500), 0.02, 0.5, 6)
    return {
        "dense-d3 (sinkhorn3d_ws_k)": (W.c3_dense_uot(n=2000, m=1700, iters=6), {}),
        "sparse-d3 (z-segments)": (sparse, {"flags": 2}),
        "dense-d3 m6": (W.c3_dense_uot(n=2000, m=1700, iters=6), {"flags": 2, "m": 6, "sigma": 3.0}),
        "d2 (sinkhorn2d_ws_k)": (W.c1_uot(n=1500, m=1300), {"flags": 2}),
        "d1": (W.c1_uot(n=1500, m=1300, d=1), {"flags": 2}),
    }


@pytest.mark.parametrize("case", list(_cases()))
def test_uot_deterministic_bitwise(uk, case):
    pr, extra = _cases()[case]
    iters = 6
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters)
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    o = dict({"method": "nfft", "deterministic": 1}, **extra)
    b1, g1, r1 = uk.uot_sinkhorn(*args, iters=iters, opts=o)
    b2, g2, r2 = uk.uot_sinkhorn(*args, iters=iters, opts=o)
    assert torch.equal(b1, b2) and torch.equal(g1, g2)
    assert r1.primal == r2.primal and r1.dual == r2.dual
    c = pr.lam / (1 + pr.lam / pr.eps)
    for got, want in ((b1, ref.beta), (g1, ref.gamma)):
        err = float(np.max(np.abs(got.cpu().numpy() - want) / (np.abs(want) + c)))
        assert err <= 1e-8, err
    b3, g3, r3 = uk.uot_sinkhorn(*args, iters=iters, opts=dict({"method": "nfft"}, **extra))
    assert float(torch.max(torch.abs(b3 - b1))) <= 1e-12 * float(torch.max(torch.abs(b1)))
    assert abs(r3.primal - r1.primal) <= 1e-12 * abs(r1.primal)


@pytest.mark.parametrize("d,kind", [(3, W.GAUSS), (3, W.IMQ), (2, W.GAUSS), (1, W.IMQ)])
def test_kernel_sum_and_mmd_deterministic_bitwise(uk, d, kind):
    param = 0.0025 if kind == W.GAUSS else 0.05
    pr = W.random_sum(d, 4001, 3001, kind=kind, param=param, seed=80 + d, signed=True)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    o = {"method": "nfft", "deterministic": 1}
    s1 = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, param, opts=o)
    s2 = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, param, opts=o)
    assert torch.equal(s1, s2)
    assert np.max(np.abs(s1.cpu().numpy() - ref)) / np.max(np.abs(ref)) <= 1e-9
    x, y = pr.src, pr.tgt
    a, b = np.abs(pr.alpha), np.abs(pr.alpha[:len(y)])
    v1 = uk.mmd2(cuda(x), cuda(a), cuda(y), cuda(b), kind, param, opts=o)
    v2 = uk.mmd2(cuda(x), cuda(a), cuda(y), cuda(b), kind, param, opts=o)
    assert v1 == v2


@pytest.mark.parametrize("case", list(_cases()))
def test_stress_repeated_runs(uk, case):
    """40 repetitions of each half-step kernel family on one input: every run equals the
    first to 1e-12 (the atomic flush order is the only run-to-run difference)."""
    pr, extra = _cases()[case]
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    o = dict({"method": "nfft"}, **extra)
    b0, g0, _ = uk.uot_sinkhorn(*args, iters=3, opts=o)
    scale = float(torch.max(torch.abs(b0)))
    worst = 0.0
    for _ in range(40):
        b, g, _ = uk.uot_sinkhorn(*args, iters=3, opts=o)
        worst = max(worst, float(torch.max(torch.abs(b - b0))), float(torch.max(torch.abs(g - g0))))
    assert worst <= 1e-12 * scale, worst


@pytest.mark.parametrize("d,n,kind,flags", [(3, 20000, W.GAUSS, 0), (3, 3000, W.GAUSS, 2), (3, 20000, W.IMQ, 0),
                                            (2, 20000, W.IMQ, 2), (1, 20000, W.GAUSS, 2)])
def test_stress_spread_gather_rings(uk, d, n, kind, flags):
    """The stand-alone spread / gather ring kernels (kernel sums), 40 repetitions."""
    param = 0.0025 if kind == W.GAUSS else 0.05
    pr = W.random_sum(d, n, n - 9, kind=kind, param=param, seed=90 + d, radius=0.2 if n > 5000 else 0.05)
    src, al, tgt = cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt)
    o = {"method": "nfft", "flags": flags}
    s0 = uk.kernel_sum(src, al, tgt, kind, param, opts=o)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt[:200], pr.kind, pr.param)
    assert np.max(np.abs(s0.cpu().numpy()[:200] - ref) / np.abs(ref)) <= 1e-9
    worst = 0.0
    for _ in range(40):
        s = uk.kernel_sum(src, al, tgt, kind, param, opts=o)
        worst = max(worst, float(torch.max(torch.abs(s - s0) / torch.abs(s0))))
    assert worst <= 1e-12, worst


def test_stress_spread_on_the_fly_and_hybrid(uk):
    """The late round-2 spread kernels, 40 repetitions each: spread3d_fly_k on hybrid
    groups (MMD^2 on C2's mixtures at C2-at-1M cell densities, uotk_info.groups 1624) and
    on one-cell groups (kernel-sum sources at C3 density, groups 16).  Each run must equal
    the first to the atomic-flush spread, and the first must equal the oracle."""
    h = W.c2_dense_mmd(n=10000)
    args = (cuda(h.x), cuda(h.a), cuda(h.y), cuda(h.b), "gauss", 0.0025)
    v0, info = uk.mmd2(*args, opts={"method": "nfft"}, return_info=True)
    assert info["groups"][0] == 1624, info
    ref = oracle.mmd2_direct(h.x, h.a, h.y, h.b, W.GAUSS, 0.0025)
    # the energy form's cancellation scale: sum of |w_i| |w_j| K over the pairs (bounded by (sum|w|)^2)
    scale = float((np.sum(np.abs(h.a)) + np.sum(np.abs(h.b))) ** 2)
    assert abs(v0 - ref) <= 1e-12 * scale, (v0, ref)
    worst = max(abs(uk.mmd2(*args, opts={"method": "nfft"}) - v0) for _ in range(40))
    assert worst <= 1e-13 * scale, worst
    f = W.c3_dense_uot(n=20000, m=1001)
    src, al, tgt = cuda(f.x), cuda(f.a), cuda(f.y)
    s0, info = uk.kernel_sum(src, al, tgt, "gauss", 0.02, opts={"method": "nfft"}, return_info=True)
    assert info["groups"][0] == 16, info
    ref = oracle.kernel_sum_direct(f.x, f.a, f.y[:200], W.GAUSS, 0.02)
    assert np.max(np.abs(s0.cpu().numpy()[:200] - ref) / np.abs(ref)) <= 1e-9
    worst = 0.0
    for _ in range(40):
        s = uk.kernel_sum(src, al, tgt, "gauss", 0.02, opts={"method": "nfft"})
        worst = max(worst, float(torch.max(torch.abs(s - s0) / torch.abs(s0))))
    assert worst <= 1e-12, worst


def test_guard_bands_on_every_kernel_family():
    """UOTK_GUARD=1 (the memcheck substitute): every library buffer carries 64 KB guard
    bands that are checked when it is freed; scripts/sanitize_cases.py launches every
    mbarrier / TMA-ring / warp-specialised kernel family on small inputs (each checked
    against the oracle).  No band may be touched."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UOTK_GUARD="1")
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize_cases.py")], capture_output=True,
                         text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "SANITIZE_CASES_DONE" in out.stdout
    assert "GUARD VIOLATION" not in out.stderr
