"""SURVEY §8(f) f2 on the GPU: Laplace and energy kernel sums, MMD^2 with them, and the
r = 1 Sinkhorn iteration (Laplace Gibbs kernel), each against the CPU oracle.

Tolerances (reading R24): the kernels are not smooth at 0, so the NFFT path
regularises them inside eps_I = p/N and adds the exact near-field correction; the
remaining error is that of the trigonometric approximation of the regularised kernel:
measured <= 7e-13 of max|K| sum|alpha| and <= 5e-12 per entry (positive weights) at the
defaults N = 256, p = 12 in d = 1..3 (profiles/r02/f2_accuracy.jsonl; the paper's own
Laplace / energy residuals are ~1e-6, Table 4).  The bars are the north
star's:
  * kernel sums: max_i |ds_i| <= 1e-9 * max|K| * sum_j |alpha_j| (signed weights; max|K|
    over the cloud, reading R14's normalisation), per entry 1e-9 for positive weights;
  * MMD^2: |d| / max(|MMD^2|, 1e-3 * sum of |quadratic terms|) <= 1e-8 (reading R13);
  * r = 1 UOT: potentials element by element and objective values within 1e-8.
The DIRECT path must match the oracle to 1e-12 in every case.
"""

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

LAP, ENERGY = 3, 4


@pytest.fixture(scope="module")
def uk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_13618_b200 as uk
    return uk


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def kmax(kind, radius):
    return 1.0 if kind == LAP else 2.0 * radius  # |K| <= 1 (Laplace), <= the cloud diameter (energy)


@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("kind,param", [(LAP, 0.05), (LAP, 0.5), (ENERGY, 1.0)])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_kernel_sum_f2(uk, method, kind, param, d):
    pr = W.random_sum(d, 3001, 1999, kind=kind, param=param, seed=200 + d, signed=True)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, kind, param)
    got, info = uk.kernel_sum(cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), kind, param, opts={"method": method},
                              return_info=True)
    assert info["method"] == method
    err = np.max(np.abs(got.cpu().numpy() - ref)) / (kmax(kind, 0.2) * np.sum(np.abs(pr.alpha)))
    assert err <= (1e-12 if method == "direct" else 1e-9), (err, info)


@pytest.mark.parametrize("kind,param", [(LAP, 0.05), (ENERGY, 1.0)])
def test_kernel_sum_f2_chunked_ragged_and_coincident(uk, kind, param):
    """Cell-group kernels forced (ragged chunks), a cloud with coincident points (r = 0
    pairs: the near-field K(0) - Q(0) term), and a single source at the target."""
    rng = np.random.default_rng(7)
    src = W.uniform_ball(rng, 5003, 3, 0.2)
    src[100:140] = src[99]  # 41 coincident points
    tgt = np.concatenate([src[:1500], W.uniform_ball(rng, 501, 3, 0.2)])
    al = rng.uniform(0.1, 1.0, len(src))
    ref = oracle.kernel_sum_direct(src, al, tgt, kind, param)
    for flags in (2, 1):
        got = uk.kernel_sum(cuda(src), cuda(al), cuda(tgt), kind, param, opts={"method": "nfft", "flags": flags})
        err = np.max(np.abs(got.cpu().numpy() - ref)) / (kmax(kind, 0.2) * al.sum())
        assert err <= 1e-9, (flags, err)
        if kind == LAP:  # positive weights, positive kernel: per entry
            assert np.max(np.abs(got.cpu().numpy() - ref) / ref) <= 1e-9
    p = np.array([[0.01, -0.02, 0.03]])
    one = uk.kernel_sum(cuda(p), cuda(np.array([2.0])), cuda(p), kind, param, opts={"method": "nfft"})
    assert abs(one.item() - (2.0 if kind == LAP else 0.0)) <= 1e-8 * 2.0


@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("kind,param", [(LAP, 0.05), (ENERGY, 1.0)])
def test_mmd2_f2(uk, method, kind, param):
    pr = W.c2_mmd(n=2500, m=2100)
    a, b = pr.a / pr.a.sum(), pr.b / pr.b.sum()  # probability vectors (energy distance, Table 4)
    ref = oracle.mmd2_direct(pr.x, a, pr.y, b, kind, param)
    xx = abs(float(a @ oracle.kernel_sum_direct(pr.x, a, pr.x, kind, param)))
    yy = abs(float(b @ oracle.kernel_sum_direct(pr.y, b, pr.y, kind, param)))
    got = uk.mmd2(cuda(pr.x), cuda(a), cuda(pr.y), cuda(b), kind, param, opts={"method": method})
    denom = max(abs(ref), 1e-3 * (xx + yy))
    assert abs(got - ref) / denom <= (1e-12 if method == "direct" else 1e-8), (got, ref)


def test_mmd2_energy_two_dirac(uk):
    """SPEC S:200 through the library: delta_0 vs delta_1 with k^e = -r gives 2."""
    for method in ("direct", "nfft"):
        v = uk.mmd2(cuda(np.zeros((1, 1))), cuda(np.ones(1)), cuda(np.ones((1, 1))), cuda(np.ones(1)), "energy",
                    1.0, opts={"method": method})
        assert abs(v - 2.0) <= 1e-8, (method, v)


def _pot_err(got, ref, c):
    return float(np.max(np.abs(got - ref) / (np.abs(ref) + c)))


@pytest.mark.parametrize("method", ["direct", "nfft"])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("eps", [0.05, 0.2])
def test_uot_r1_laplace_gibbs(uk, method, d, eps):
    """Algorithm 2 with r = 1 (UOTK_FLAG_COST_R1): t_i = sum_j e^{-lambda ||x_i - y_j||} ...
    against the oracle's r = 1 iteration: C1's distributions and lambda = 20 (eps = 0.05,
    the paper's Table 2 parameters) and a wider kernel."""
    pr = W.c1_uot(n=1200, m=1000, d=d)
    lam, iters = 1.0, 15
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, eps, lam, lam, iters, r=1)
    beta, gamma, res = uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), eps, lam, iters=iters,
                                       opts={"method": method, "flags": uk.FLAG_COST_R1})
    c = lam / (1 + lam / eps)
    tol = 1e-12 if method == "direct" else 1e-8
    assert _pot_err(beta.cpu().numpy(), ref.beta, c) <= tol
    assert _pot_err(gamma.cpu().numpy(), ref.gamma, c) <= tol
    assert abs(res.primal - ref.primal) <= tol * abs(ref.primal)
    assert abs(res.dual - ref.dual) <= tol * abs(ref.dual)
    assert abs(res.plan_mass - ref.plan_mass) <= tol * ref.plan_mass


def test_uot_r1_unsupported_combinations(uk):
    pr = W.c1_uot(n=50, m=40)
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), 0.2, 1.0, iters=3,
                        opts={"flags": uk.FLAG_COST_R1}, transport=True)
    assert e.value.code == -8
