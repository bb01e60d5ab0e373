"""Pins of the CPU oracle against values fixed by the paper and by mathematics.

Each test is chosen so that a plausible mistake in ``oracle/`` (a dropped term, a
wrong sign or exponent, a transposed operand, a wrong kernel scaling) fails it.
None of them re-types an oracle formula; see DESIGN.md "Oracle pins".
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import closed_forms as cf
from workloads import GAUSS, IMQ, uniform_ball

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ kernel sums
@pytest.mark.parametrize("eps", [0.05, 0.002])
def test_kernel_sum_gauss_line_integral(eps):
    """Gauss-Legendre weights as alpha: sum_j K(x - y_j) w_j -> int exp(-(x-y)^2/eps) dy
    = sqrt(pi eps) (wrong kernel scaling, e.g. exp(-r^2/(2eps)) or exp(-r/eps), fails)."""
    L = 40.0 * math.sqrt(eps)
    t, w = np.polynomial.legendre.leggauss(400)
    y = (L * t)[:, None]
    s = oracle.kernel_sum_direct(y, L * w, np.array([[0.0], [0.3 * math.sqrt(eps)]]), GAUSS, eps)
    ref = cf.gauss_line_integral(eps)
    np.testing.assert_allclose(s, ref, rtol=1e-13)


def test_kernel_sum_imq_segment_integral():
    """sum_j (y_j^2 + c^2)^(-1/2) w_j -> 2 asinh(L/c) on Gauss-Legendre nodes."""
    c, L = 0.05, 0.4
    t, w = np.polynomial.legendre.leggauss(600)
    # split at 0 to resolve the peak; integrand is even
    y = (0.5 * L * (t + 1.0))[:, None]
    s = oracle.kernel_sum_direct(y, 0.5 * L * w, np.zeros((1, 1)), IMQ, c)[0]
    np.testing.assert_allclose(2.0 * s, cf.imq_segment_integral(L, c), rtol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_kernel_sum_gauss_tensor_grid(d):
    """Product point grids with product weights: the d-D Gaussian sum factorises
    into a product of 1-D sums (exact; catches per-axis distance bugs)."""
    rng = np.random.default_rng(1)
    eps = 0.03
    axes_src = [rng.uniform(-0.2, 0.2, 5) for _ in range(d)]
    axes_w = [rng.uniform(0.1, 1.0, 5) for _ in range(d)]
    tgt = rng.uniform(-0.2, 0.2, (4, d))
    mesh = np.meshgrid(*axes_src, indexing="ij")
    src = np.stack([g.ravel() for g in mesh], axis=1)
    wmesh = np.meshgrid(*axes_w, indexing="ij")
    alpha = np.prod(np.stack([g.ravel() for g in wmesh], axis=1), axis=1)
    s = oracle.kernel_sum_direct(src, alpha, tgt, GAUSS, eps)
    ref = np.ones(len(tgt))
    for t in range(d):
        ref *= oracle.kernel_sum_direct(axes_src[t][:, None], axes_w[t], tgt[:, t:t + 1], GAUSS, eps)
    np.testing.assert_allclose(s, ref, rtol=1e-14)


@pytest.mark.parametrize("kind,k0", [(GAUSS, 1.0), (IMQ, 1.0 / 0.05)])
def test_kernel_sum_single_source_at_target(kind, k0):
    """One source exactly at the target: s = K(0) alpha."""
    p = np.array([[0.1, -0.05, 0.02]])
    s = oracle.kernel_sum_direct(p, np.array([2.5]), p, kind, 0.05 if kind == IMQ else 0.02)
    np.testing.assert_allclose(s, [2.5 * k0], rtol=1e-15)


@pytest.mark.parametrize("kind", [GAUSS, IMQ])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_kernel_sum_mpmath_brute_force(kind, d):
    """50-digit brute force on tiny inputs bounds the fp64 oracle's rounding error."""
    import mpmath
    mpmath.mp.dps = 50
    rng = np.random.default_rng(d)
    src = uniform_ball(rng, 17, d, 0.2)
    tgt = uniform_ball(rng, 9, d, 0.2)
    alpha = rng.standard_normal(17)
    param = 0.02 if kind == GAUSS else 0.05
    s = oracle.kernel_sum_direct(src, alpha, tgt, kind, param)
    for i in range(len(tgt)):
        acc = mpmath.mpf(0)
        for j in range(len(src)):
            r2 = sum((mpmath.mpf(float(tgt[i, t])) - mpmath.mpf(float(src[j, t]))) ** 2 for t in range(d))
            k = mpmath.exp(-r2 / mpmath.mpf(param)) if kind == GAUSS else 1 / mpmath.sqrt(r2 + mpmath.mpf(param) ** 2)
            acc += k * mpmath.mpf(float(alpha[j]))
        scale = sum(abs(float(a)) for a in alpha) * (1.0 if kind == GAUSS else 1.0 / param)
        assert abs(float(acc) - s[i]) <= 1e-14 * scale


def test_kernel_sum_symmetry_and_rotation():
    """<w, K alpha> = <K^T w, alpha> (swapping source/target roles) and invariance
    under a rigid motion of all points (radial kernel, Eq. 4.1-4.2)."""
    rng = np.random.default_rng(3)
    x = uniform_ball(rng, 50, 3, 0.2)
    y = uniform_ball(rng, 40, 3, 0.2)
    al = rng.standard_normal(40)
    w = rng.standard_normal(50)
    for kind, param in ((GAUSS, 0.02), (IMQ, 0.05)):
        lhs = w @ oracle.kernel_sum_direct(y, al, x, kind, param)
        rhs = al @ oracle.kernel_sum_direct(x, w, y, kind, param)
        np.testing.assert_allclose(lhs, rhs, rtol=1e-12)
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        sh = np.array([0.3, -0.1, 0.05])
        s1 = oracle.kernel_sum_direct(y, al, x, kind, param)
        s2 = oracle.kernel_sum_direct(y @ Q.T + sh, al, x @ Q.T + sh, kind, param)
        np.testing.assert_allclose(s1, s2, rtol=1e-11, atol=1e-13 * np.abs(al).sum())


def test_kernel_sum_empty():
    out = oracle.kernel_sum_direct(np.zeros((0, 2)), np.zeros(0), np.ones((3, 2)), GAUSS, 0.1)
    np.testing.assert_array_equal(out, np.zeros(3))
    assert oracle.kernel_sum_direct(np.ones((3, 2)), np.ones(3), np.zeros((0, 2)), GAUSS, 0.1).shape == (0,)


# ------------------------------------------------------------------ Sinkhorn UOT
def test_sinkhorn_single_atom_golden():
    """Coincident single atoms reproduce the golden plan mass (Eq. 2.10)."""
    g = golden("sinkhorn_single_atom.json")
    eps = 1.0 / g["lambda"]
    r = oracle.uot_sinkhorn_direct(np.zeros((1, 2)), np.array([g["a"]]), np.zeros((1, 2)),
                                   np.array([g["b"]]), eps, g["eta1"], g["eta2"], iters=200)
    np.testing.assert_allclose(r.plan_mass, g["plan_mass"], rtol=1e-12)
    np.testing.assert_allclose(
        r.plan_mass, cf.single_atom_plan_mass(g["a"], g["b"], g["lambda"], g["eta1"], g["eta2"]), rtol=1e-12)


@pytest.mark.parametrize("eta1,eta2,eps", [(1.0, 1.0, 0.05), (0.7, 2.5, 0.2), (3.0, 0.4, 1.0)])
def test_sinkhorn_coincident_points_cstar(eta1, eta2, eps):
    """All points at one location: the converged plan is c* mu (x) nu with c* of
    Prop. 2.9 Eq. (2.10), for unequal eta1 != eta2 as well."""
    rng = np.random.default_rng(5)
    mu = rng.uniform(0.2, 2.0, 5)
    nu = rng.uniform(0.1, 1.5, 7)
    p0 = np.array([[0.03, -0.02]])
    r = oracle.uot_sinkhorn_direct(np.repeat(p0, 5, 0), mu, np.repeat(p0, 7, 0), nu, eps, eta1, eta2, iters=400)
    cs = cf.cstar_eq210(mu.sum(), nu.sum(), 0.0, 1.0 / eps, eta1, eta2)
    np.testing.assert_allclose(r.plan_mass, cs * mu.sum() * nu.sum(), rtol=1e-12)


def test_cstar_golden():
    g = golden("cstar_example.json")
    np.testing.assert_allclose(
        cf.cstar_eq210(g["mass_a"], g["mass_b"], 0.0, g["lambda"], g["eta1"], g["eta2"]), g["c_star"], rtol=1e-15)


@pytest.mark.parametrize("seed", [0, 1])
def test_sinkhorn_brute_force_primal(seed):
    """n, m <= 4: a generic optimiser on the primal definition finds the same
    optimum value as converged Algorithm 1 (primal and dual) and the same marginals."""
    rng = np.random.default_rng(seed)
    n, m = 3, 4
    x = uniform_ball(rng, n, 2, 0.2)
    y = uniform_ball(rng, m, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.2, 2.0, m)
    eps, eta = 0.05, 1.0
    val, pi = cf.brute_force_uot(x, mu, y, nu, eps, eta, eta)
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=3000)
    np.testing.assert_allclose(r.primal, val, rtol=1e-10)
    np.testing.assert_allclose(r.dual, val, rtol=1e-10)
    np.testing.assert_allclose(r.plan_mass, pi.sum(), rtol=1e-6)
    p, q = oracle.sinkhorn.plan_marginals(x, mu, y, nu, r.beta, r.gamma, eps)
    np.testing.assert_allclose(p, pi.sum(1), rtol=1e-5)
    np.testing.assert_allclose(q, pi.sum(0), rtol=1e-5)


def test_sinkhorn_primal_dense_vs_marginals_and_duality():
    """The marginal form of the primal equals the literal P:462 form at any iterate;
    at convergence primal == dual (strong duality, Thm 3.1)."""
    rng = np.random.default_rng(2)
    x = uniform_ball(rng, 60, 2, 0.2)
    y = uniform_ball(rng, 50, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 60)
    nu = rng.uniform(0.2, 2.0, 50)
    eps, eta = 0.05, 1.0
    for iters in (1, 3, 400):
        r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=iters)
        dense = oracle.primal_objective_dense(x, mu, y, nu, r.beta, r.gamma, eps, eta, eta)
        np.testing.assert_allclose(r.primal, dense, rtol=1e-13)
    assert abs(r.primal - r.dual) <= 1e-11 * abs(r.dual)


def test_sinkhorn_first_order_identities_and_mass_symmetry():
    """After a gamma-step q_j = nu_j e^{-gamma_j/eta2}; after a beta-step
    p_i = mu_i e^{-beta_i/eta1} (first-order conditions of (3.1)); sum p = sum q."""
    rng = np.random.default_rng(4)
    x = uniform_ball(rng, 40, 3, 0.2)
    y = uniform_ball(rng, 30, 3, 0.2)
    mu = rng.uniform(0.1, 1.0, 40)
    nu = rng.uniform(0.1, 1.0, 30)
    eps, eta1, eta2 = 0.02, 0.5, 0.8
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta1, eta2, iters=7)
    p, q = oracle.sinkhorn.plan_marginals(x, mu, y, nu, r.beta, r.gamma, eps)
    np.testing.assert_allclose(q, nu * np.exp(-r.gamma / eta2), rtol=1e-13)
    np.testing.assert_allclose(p.sum(), q.sum(), rtol=1e-13)
    # beta-step first-order identity: one more beta-step from the final gamma
    beta = oracle.sinkhorn.beta_step(x, y, nu, r.gamma, eps, eta1)
    p2, _ = oracle.sinkhorn.plan_marginals(x, mu, y, nu, beta, r.gamma, eps)
    np.testing.assert_allclose(p2, mu * np.exp(-beta / eta1), rtol=1e-13)


def test_sinkhorn_dual_monotone_and_zero_iters():
    """Alternating exact maximisation never decreases the dual; zero
    iterations returns gamma^0 = 0."""
    rng = np.random.default_rng(6)
    x = uniform_ball(rng, 30, 2, 0.2)
    y = uniform_ball(rng, 25, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 30)
    nu = rng.uniform(0.2, 2.0, 25)
    eps, eta = 0.05, 1.0
    gamma = np.zeros(25)
    beta = np.zeros(30)
    prev = oracle.dual_objective(x, mu, y, nu, beta, gamma, eps, eta, eta)
    for _ in range(10):
        beta = oracle.sinkhorn.beta_step(x, y, nu, gamma, eps, eta)
        v = oracle.dual_objective(x, mu, y, nu, beta, gamma, eps, eta, eta)
        assert v >= prev - 1e-12 * abs(prev)
        prev = v
        gamma = oracle.sinkhorn.gamma_step(x, y, mu, beta, eps, eta)
        v = oracle.dual_objective(x, mu, y, nu, beta, gamma, eps, eta, eta)
        assert v >= prev - 1e-12 * abs(prev)
        prev = v
    r0 = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=0)
    np.testing.assert_array_equal(r0.gamma, np.zeros(25))
    # dual at beta = gamma = 0 equals (1/lam)(mu(X)nu(X) - sum_ij mu_i k_ij nu_j)
    kk = np.exp(-np.sum((x[:, None] - y[None]) ** 2, 2) / eps)
    np.testing.assert_allclose(r0.dual, eps * (mu.sum() * nu.sum() - mu @ kk @ nu), rtol=1e-13)


def test_sinkhorn_balanced_limit():
    """eta -> infinity with equal total masses: the UOT plan approaches the balanced
    entropic OT plan of the textbook Sinkhorn iteration (Rem. 2.4)."""
    rng = np.random.default_rng(7)
    x = uniform_ball(rng, 12, 2, 0.2)
    y = uniform_ball(rng, 10, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 12)
    nu = rng.uniform(0.5, 1.5, 10)
    nu *= mu.sum() / nu.sum()
    eps, eta = 0.05, 1e7
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=3000)
    p, q = oracle.sinkhorn.plan_marginals(x, mu, y, nu, r.beta, r.gamma, eps)
    ref = cf.balanced_sinkhorn(x, mu, y, nu, eps, 3000)
    np.testing.assert_allclose(p, ref.sum(1), rtol=1e-5)
    np.testing.assert_allclose(q, ref.sum(0), rtol=1e-5)
    np.testing.assert_allclose(p, mu, rtol=1e-5)


def test_sinkhorn_restricted_objective_bound():
    """The converged primal is <= the objective at the best independent plan
    c* mu (x) nu of Prop. 2.9."""
    rng = np.random.default_rng(8)
    x = uniform_ball(rng, 20, 2, 0.2)
    y = uniform_ball(rng, 15, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 20)
    nu = rng.uniform(0.2, 2.0, 15)
    eps, eta = 0.05, 1.0
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=500)
    d2 = np.sum((x[:, None] - y[None]) ** 2, 2)
    mean_cost = float(mu @ d2 @ nu) / (mu.sum() * nu.sum())
    cs = cf.cstar_eq210(mu.sum(), nu.sum(), mean_cost, 1 / eps, eta, eta)
    val_cs = cf.primal_of_plan(cs * np.outer(mu, nu), d2, mu, nu, 1 / eps, eta, eta)
    assert r.primal <= val_cs + 1e-9
    # and c* is the minimiser along the ray c * mu (x) nu
    for f in (0.9, 1.1):
        assert cf.primal_of_plan(f * cs * np.outer(mu, nu), d2, mu, nu, 1 / eps, eta, eta) > val_cs


# ------------------------------------------------------------------ MMD^2
def test_mmd_two_dirac_golden():
    g = golden("mmd_two_dirac.json")
    x = np.array([[0.0, 0.0]])
    y = np.array([[g["distance"], 0.0]])
    v = oracle.mmd2_direct(x, np.array([1.0]), y, np.array([1.0]), GAUSS, g["ell"] ** 2)
    np.testing.assert_allclose(v, g["mmd2"], rtol=1e-15)


def test_mmd_identities():
    rng = np.random.default_rng(9)
    x = uniform_ball(rng, 40, 3, 0.2)
    y = uniform_ball(rng, 30, 3, 0.2)
    a = rng.uniform(0.5, 1.5, 40)
    b = rng.uniform(0.5, 1.5, 30)
    for kind, param in ((GAUSS, 0.0025), (IMQ, 0.05)):
        assert abs(oracle.mmd2_direct(x, a, x, a, kind, param)) <= 1e-12 * (a.sum() ** 2 / (param if kind else 1))
        v1 = oracle.mmd2_direct(x, a, y, b, kind, param)
        v2 = oracle.mmd2_direct(y, b, x, a, kind, param)
        v3 = oracle.mmd2_combined(x, a, y, b, kind, param)
        np.testing.assert_allclose(v1, v2, rtol=1e-12)
        np.testing.assert_allclose(v1, v3, rtol=1e-10)
        assert v1 >= 0
        kinf = 1.0 if kind == GAUSS else 1.0 / param
        assert v1 <= kinf * (a.sum() ** 2 + b.sum() ** 2)  # (2.15)
        # two atoms: (a^2 + b^2) K(0) - 2 a b K(|x-y|)
        r = 0.07
        k_r = math.exp(-r * r / param) if kind == GAUSS else 1 / math.sqrt(r * r + param * param)
        two = oracle.mmd2_direct(np.zeros((1, 3)), np.array([1.3]), np.array([[0, r, 0.0]]), np.array([0.6]), kind, param)
        np.testing.assert_allclose(two, (1.3 ** 2 + 0.6 ** 2) * kinf - 2 * 1.3 * 0.6 * k_r, rtol=1e-14)


@pytest.mark.parametrize("d,q,rtol", [(1, 24, 1e-13), (2, 16, 1e-11), (3, 12, 1e-8)])
def test_mmd_gaussian_mixture_closed_form(d, q, rtol):
    """Gauss-Hermite discretised Gaussian mixtures (C2-like, Q6 kernel e^{-r^2/l^2})
    reproduce the population MMD^2 closed form (completing the square)."""
    ex = np.zeros(d)
    ex[0] = 0.05
    mx = np.stack([ex, -ex])
    sh = np.zeros(d)
    sh[min(1, d - 1)] = 0.02
    my = mx + sh
    sigma, ell2 = 0.03, 0.05 ** 2
    px, wx = cf.gauss_hermite_mixture(mx, sigma, q, mass=1.3)
    py, wy = cf.gauss_hermite_mixture(my, sigma, q, mass=0.8)
    v = oracle.mmd2_direct(px, wx, py, wy, GAUSS, ell2)
    ref = cf.gm_population_mmd2(mx, my, sigma, ell2, 1.3, 0.8)
    np.testing.assert_allclose(v, ref, rtol=rtol)


# ------------------------------------------------------------------ c*, Sinkhorn divergence, stopping
def test_cstar_oracle_golden_coincident():
    """Eq. (2.10) with a zero transport term (all points at one location): the SPEC
    worked example mu(X)=2, nu(X)=3, eta=1, lambda=1 gives 6^(-1/3) (golden file)."""
    g = golden("cstar_example.json")
    x = np.zeros((3, 2))
    y = np.zeros((2, 2))
    mu = np.array([0.5, 1.0, 0.5]) * g["mass_a"] / 2.0
    nu = np.array([1.0, 2.0]) * g["mass_b"] / 3.0
    c = oracle.cstar(x, mu, y, nu, 1.0 / g["lambda"], g["eta1"], g["eta2"])
    np.testing.assert_allclose(c, g["c_star"], rtol=1e-14)


@pytest.mark.parametrize("eta1,eta2", [(1.0, 1.0), (0.3, 2.0)])
def test_cstar_oracle_minimises_restricted_primal(eta1, eta2):
    """c* (with the transport moment summed by the oracle) minimises the independently
    written primal of P:462 along the ray c * mu (x) nu (Prop. 2.9)."""
    rng = np.random.default_rng(12)
    x = uniform_ball(rng, 17, 3, 0.2)
    y = uniform_ball(rng, 11, 3, 0.2)
    mu = rng.uniform(0.5, 1.5, 17)
    nu = rng.uniform(0.2, 2.0, 11)
    eps = 0.05
    d2 = np.sum((x[:, None] - y[None]) ** 2, 2)
    c = oracle.cstar(x, mu, y, nu, eps, eta1, eta2)
    f = lambda cc: cf.primal_of_plan(cc * np.outer(mu, nu), d2, mu, nu, 1 / eps, eta1, eta2)  # noqa: E731
    for fac in (0.999, 1.001, 0.9, 1.1):
        assert f(fac * c) > f(c)


def test_sinkhorn_divergence_single_atoms_closed_form():
    """Eq. (2.12) for single atoms at one location: every UOT term has the closed-form
    plan mass of the coincident single-atom problem, so sd is explicit; pins the signs
    and the (eps/2)(mu(X) - nu(X))^2 term."""
    a, b, eps, eta = 2.0, 0.7, 0.3, 0.8
    lam = 1.0 / eps

    def uot_closed(m1, m2):
        pi = cf.single_atom_plan_mass(m1, m2, lam, eta, eta)
        return cf.primal_of_plan(np.array([[pi]]), np.zeros((1, 1)), np.array([m1]), np.array([m2]), lam, eta, eta)

    want = uot_closed(a, b) - 0.5 * uot_closed(a, a) - 0.5 * uot_closed(b, b) + 0.5 * eps * (a - b) ** 2
    p = np.array([[0.05, -0.1]])
    sd, _ = oracle.sinkhorn_divergence_direct(p, np.array([a]), p, np.array([b]), eps, eta, eta, iters=400)
    np.testing.assert_allclose(sd, want, rtol=1e-12, atol=1e-14)


def test_sinkhorn_divergence_identities():
    """sd(mu, mu) = 0 and sd(mu, nu) = sd(nu, mu) for eta1 = eta2 (UOT is then symmetric)."""
    rng = np.random.default_rng(13)
    x = uniform_ball(rng, 9, 2, 0.2)
    y = uniform_ball(rng, 7, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 9)
    nu = rng.uniform(0.2, 2.0, 7)
    s0, _ = oracle.sinkhorn_divergence_direct(x, mu, x, mu, 0.05, 1.0, iters=60)
    assert abs(s0) <= 1e-12 * mu.sum() ** 2
    s1, _ = oracle.sinkhorn_divergence_direct(x, mu, y, nu, 0.05, 1.0, iters=300)
    s2, _ = oracle.sinkhorn_divergence_direct(y, nu, x, mu, 0.05, 1.0, iters=300)
    np.testing.assert_allclose(s1, s2, rtol=1e-9)


def test_stopping_rule():
    """With stop_tol the oracle stops at the first multiple of check_every whose
    iteration changed both potentials by <= stop_tol, and the result equals the
    fixed-iteration run of that length."""
    rng = np.random.default_rng(14)
    x = uniform_ball(rng, 25, 2, 0.2)
    y = uniform_ball(rng, 20, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 25)
    nu = rng.uniform(0.2, 2.0, 20)
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.05, 1.0, 1.0, iters=500, stop_tol=1e-9, check_every=7)
    assert r.iters % 7 == 0 and r.iters < 500
    assert r.max_dbeta <= 1e-9 and r.max_dgamma <= 1e-9
    prev = oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.05, 1.0, 1.0, iters=r.iters - 7)
    assert prev.max_dbeta > 1e-9 or prev.max_dgamma > 1e-9
    fixed = oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.05, 1.0, 1.0, iters=r.iters)
    np.testing.assert_array_equal(fixed.beta, r.beta)


def test_lambda_scaling_converges_to_the_unique_dual_maximiser():
    """lambda-scaling (Sec. 5.1.3) warm-starts each stage; run to convergence, the last
    stage reaches the same (unique, Thm. 3.1) potentials as a cold start at the
    final eps — pins the stage ordering and the warm-start plumbing."""
    rng = np.random.default_rng(15)
    x = uniform_ball(rng, 14, 2, 0.2)
    y = uniform_ball(rng, 12, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 14)
    nu = rng.uniform(0.2, 2.0, 12)
    r = oracle.uot_sinkhorn_scaling_direct(x, mu, y, nu, [0.2, 0.1, 0.05], 1.0, iters=2000, stop_tol=1e-13,
                                           check_every=10)
    cold = oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.05, 1.0, iters=2000, stop_tol=1e-13, check_every=10)
    np.testing.assert_allclose(r.gamma, cold.gamma, atol=1e-11)
    np.testing.assert_allclose(r.primal, cold.primal, rtol=1e-11)
    single = oracle.uot_sinkhorn_scaling_direct(x, mu, y, nu, [0.05], 1.0, iters=30)
    np.testing.assert_array_equal(single.gamma, oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.05, 1.0, iters=30).gamma)


# ------------------------------------------------------------------ transport term
@pytest.mark.parametrize("eps", [0.05, 0.002])
def test_kernel_sum_gauss_r2_line_integral(eps):
    """Gauss-Legendre weights: sum_j (x-y_j)^2 exp(-(x-y_j)^2/eps) w_j ->
    int y^2 exp(-y^2/eps) dy = sqrt(pi) eps^(3/2) / 2 (the Gaussian's second moment)."""
    L = 40.0 * math.sqrt(eps)
    t, w = np.polynomial.legendre.leggauss(400)
    y = (L * t)[:, None]
    s = oracle.kernel_sum_direct(y, L * w, np.array([[0.0], [0.3 * math.sqrt(eps)]]), 2, eps)
    np.testing.assert_allclose(s, math.sqrt(math.pi) * eps ** 1.5 / 2.0, rtol=1e-12)


def test_transport_cost_entropy_identity():
    """For the recovered plan log(pi_ij / (mu_i nu_j)) = lam beta_i + lam gamma_j
    - lam d_ij^2, so <pi, d^2> = sum beta p + sum gamma q - (1/lam) sum pi log(pi/(mu nu));
    the right side is evaluated densely from an independently built plan."""
    rng = np.random.default_rng(16)
    x = uniform_ball(rng, 13, 2, 0.2)
    y = uniform_ball(rng, 11, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 13)
    nu = rng.uniform(0.2, 2.0, 11)
    eps = 0.05
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, 1.0, iters=40)
    d2 = np.sum((x[:, None] - y[None]) ** 2, 2)
    pi = np.outer(mu * np.exp(r.beta / eps), nu * np.exp(r.gamma / eps)) * np.exp(-d2 / eps)
    ent = float(np.sum(pi * np.log(pi / np.outer(mu, nu))))
    rhs = float(r.beta @ pi.sum(1) + r.gamma @ pi.sum(0)) - eps * ent
    np.testing.assert_allclose(oracle.transport_cost(x, mu, y, nu, r.beta, r.gamma, eps), rhs, rtol=1e-10)
    np.testing.assert_allclose(oracle.transport_cost(x, mu, y, nu, r.beta, r.gamma, eps), float(np.sum(pi * d2)),
                               rtol=1e-13)
