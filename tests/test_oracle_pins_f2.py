"""Pins of the oracle's Laplace and energy kernels and of the r = 1 (Laplace Gibbs kernel)
Sinkhorn iteration — SURVEY §8(f) f2 (Eq. 4.2; Table 1; Algorithm 2's
input r >= 1, and its r = 1 complexity).

As in test_oracle_pins.py, nothing here re-types an oracle formula: closed-form
integrals (a wrong scaling, exponent, norm or sign fails them), the SPEC's worked
example, 50-digit brute force, and a generic optimiser on the primal definition with
the cost d^1.
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import ENERGY, LAP
from tests import closed_forms as cf
from workloads import uniform_ball

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ Laplace kernel sums
@pytest.mark.parametrize("ell", [0.05, 0.5])
def test_laplace_segment_integral(ell):
    """Gauss-Legendre nodes on [0, L] (the cusp at 0 is a node-interval end) as sources:
    sum_j e^{-|0 - y_j|/l} w_j -> 2 l (1 - e^{-L/l}) for the two halves.  exp(-r^2/l),
    exp(-r/(2l)) or a missing abs fail."""
    L = 0.4
    t, w = np.polynomial.legendre.leggauss(300)
    y = 0.5 * L * (t + 1.0)
    src = np.concatenate([y, -y])[:, None]
    wts = np.concatenate([0.5 * L * w, 0.5 * L * w])
    s = oracle.kernel_sum_direct(src, wts, np.zeros((1, 1)), LAP, ell)[0]
    np.testing.assert_allclose(s, cf.laplace_segment_integral(L, ell), rtol=1e-13)


@pytest.mark.parametrize("ell", [0.05, 0.3])
def test_laplace_disk_and_ball_integrals(ell):
    """Polar / spherical product rules as sources, target at the centre: the 2-D and 3-D
    integrals of e^{-|y|/l} over the disk / ball (closed forms in r).  Pins the Euclidean
    norm in d = 2, 3 (an l1 or l_inf distance, or a per-axis product, fails)."""
    R = 0.4
    pts, wts = cf.polar_rule(R, 200, 64)
    s2 = oracle.kernel_sum_direct(pts, wts, np.zeros((1, 2)), LAP, ell)[0]
    np.testing.assert_allclose(s2, cf.laplace_disk_integral(R, ell), rtol=1e-12)
    pts, wts = cf.spherical_rule(R, 120, 24, 24)
    s3 = oracle.kernel_sum_direct(pts, wts, np.zeros((1, 3)), LAP, ell)[0]
    np.testing.assert_allclose(s3, cf.laplace_ball_integral(R, ell), rtol=1e-12)


# ------------------------------------------------------------------ energy kernel sums
@pytest.mark.parametrize("x0", [0.0, 0.13, -0.31])
def test_energy_segment_integral(x0):
    """k^e = -|x - y| (Table 1): Gauss-Legendre on [-L, x0] and [x0, L] (split at the kink):
    sum_j -|x0 - y_j| w_j -> -(L^2 + x0^2).  A missing sign or abs, or |.|^2, fails."""
    L = 0.4
    t, w = np.polynomial.legendre.leggauss(40)  # the integrand is linear on each piece
    a = x0 + L
    b = L - x0
    y = np.concatenate([-L + 0.5 * a * (t + 1.0), x0 + 0.5 * b * (t + 1.0)])
    wts = np.concatenate([0.5 * a * w, 0.5 * b * w])
    s = oracle.kernel_sum_direct(y[:, None], wts, np.array([[x0]]), ENERGY, 1.0)[0]
    np.testing.assert_allclose(s, cf.energy_segment_integral(L, x0), rtol=1e-14)


@pytest.mark.parametrize("kind,param,k0", [(LAP, 0.05, 1.0), (ENERGY, 1.0, 0.0)])
def test_single_source_at_target(kind, param, k0):
    p = np.array([[0.1, -0.05, 0.02]])
    s = oracle.kernel_sum_direct(p, np.array([2.5]), p, kind, param)
    np.testing.assert_allclose(s, [2.5 * k0], rtol=0, atol=1e-300)


@pytest.mark.parametrize("kind", [LAP, ENERGY])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_mpmath_brute_force(kind, d):
    """50-digit brute force on tiny inputs bounds the fp64 oracle's rounding error."""
    import mpmath
    mpmath.mp.dps = 50
    rng = np.random.default_rng(30 + d)
    src = uniform_ball(rng, 15, d, 0.2)
    tgt = uniform_ball(rng, 7, d, 0.2)
    alpha = rng.standard_normal(15)
    ell = 0.05
    s = oracle.kernel_sum_direct(src, alpha, tgt, kind, ell)
    for i in range(len(tgt)):
        acc = mpmath.mpf(0)
        for j in range(len(src)):
            r = mpmath.sqrt(sum((mpmath.mpf(float(tgt[i, t])) - mpmath.mpf(float(src[j, t]))) ** 2 for t in range(d)))
            k = mpmath.exp(-r / mpmath.mpf(ell)) if kind == LAP else -r
            acc += k * mpmath.mpf(float(alpha[j]))
        scale = sum(abs(float(a)) for a in alpha) * (1.0 if kind == LAP else 0.4)
        assert abs(float(acc) - s[i]) <= 1e-14 * scale


# ------------------------------------------------------------------ MMD^2
def test_mmd_energy_two_dirac_golden():
    """energy kernel, delta_0 vs delta_1 -> 2."""
    with open(os.path.join(GOLDEN, "mmd_energy_two_dirac.json")) as f:
        g = json.load(f)
    v = oracle.mmd2_direct(np.array([g["x"]]), np.array([1.0]), np.array([g["y"]]), np.array([1.0]), ENERGY, 1.0)
    np.testing.assert_allclose(v, g["mmd2"], rtol=1e-15)


@pytest.mark.parametrize("kind,param", [(LAP, 0.05), (ENERGY, 1.0)])
def test_mmd_identities_f2(kind, param):
    """mu = nu -> 0; symmetry; the combined form; two atoms (a^2 + b^2) k(0) - 2ab k(d);
    the energy distance of probability measures is non-negative (k^e is conditionally
    negative definite, so -k^e ... MMD^2 >= 0 for equal masses)."""
    rng = np.random.default_rng(40)
    x = uniform_ball(rng, 40, 3, 0.2)
    y = uniform_ball(rng, 30, 3, 0.2)
    a = rng.uniform(0.5, 1.5, 40)
    b = rng.uniform(0.5, 1.5, 30)
    assert abs(oracle.mmd2_direct(x, a, x, a, kind, param)) <= 1e-12 * a.sum() ** 2
    v1 = oracle.mmd2_direct(x, a, y, b, kind, param)
    np.testing.assert_allclose(v1, oracle.mmd2_direct(y, b, x, a, kind, param), rtol=1e-12)
    np.testing.assert_allclose(v1, oracle.mmd2_combined(x, a, y, b, kind, param), rtol=1e-11)
    dd = 0.17
    p0, p1 = np.zeros((1, 2)), np.array([[dd, 0.0]])
    k0, kd = (1.0, math.exp(-dd / param)) if kind == LAP else (0.0, -dd)
    np.testing.assert_allclose(oracle.mmd2_direct(p0, np.array([1.3]), p1, np.array([0.7]), kind, param),
                               (1.3 ** 2 + 0.7 ** 2) * k0 - 2 * 1.3 * 0.7 * kd, rtol=1e-14)
    ap, bp = a / a.sum(), b / b.sum()
    assert oracle.mmd2_direct(x, ap, y, bp, kind, param) > 0


# ------------------------------------------------------------------ r = 1 Sinkhorn
@pytest.mark.parametrize("seed", [0, 1])
def test_sinkhorn_r1_brute_force_primal(seed):
    """n, m <= 4, cost d^1 (Laplace Gibbs kernel e^{-lambda d}): a generic optimiser on the
    primal definition with the cost matrix d finds the value of converged
    Algorithm 1 with r = 1 (primal and dual) and its marginals.  An r = 2 iteration (or
    a kernel e^{-lambda d^2}) fails."""
    rng = np.random.default_rng(seed)
    n, m = 3, 4
    x = uniform_ball(rng, n, 2, 0.2)
    y = uniform_ball(rng, m, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.2, 2.0, m)
    eps, eta = 0.05, 1.0
    val, pi = cf.brute_force_uot(x, mu, y, nu, eps, eta, eta, r=1)
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, eta, eta, iters=3000, r=1)
    np.testing.assert_allclose(r.primal, val, rtol=1e-10)
    np.testing.assert_allclose(r.dual, val, rtol=1e-10)
    p, q = oracle.sinkhorn.plan_marginals(x, mu, y, nu, r.beta, r.gamma, eps, r=1)
    np.testing.assert_allclose(p, pi.sum(1), rtol=1e-5)
    np.testing.assert_allclose(q, pi.sum(0), rtol=1e-5)
    val2, _ = cf.brute_force_uot(x, mu, y, nu, eps, eta, eta, r=2)
    assert abs(val2 - val) > 1e-3 * abs(val)  # the two costs are distinguishable here


def test_sinkhorn_r1_primal_dense_vs_marginals():
    """The marginal form of the primal equals the literal P:462 form (cost d^1) at an
    arbitrary iterate (the <pi, d^r> term cancels for any r)."""
    rng = np.random.default_rng(5)
    x = uniform_ball(rng, 30, 2, 0.2)
    y = uniform_ball(rng, 25, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 30)
    nu = rng.uniform(0.2, 2.0, 25)
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, 0.1, 0.7, 1.3, iters=7, r=1)
    dense = oracle.primal_objective_dense(x, mu, y, nu, r.beta, r.gamma, 0.1, 0.7, 1.3, r=1)
    np.testing.assert_allclose(r.primal, dense, rtol=1e-12)


@pytest.mark.parametrize("eta1,eta2", [(1.0, 1.0), (0.3, 2.0)])
def test_cstar_r1_minimises_restricted_primal(eta1, eta2):
    """c* with r = 1 (moment <mu x nu | d^1>) minimises the independently written primal
    (cost matrix d) along the ray c mu (x) nu (Prop. 2.9)."""
    rng = np.random.default_rng(13)
    x = uniform_ball(rng, 17, 3, 0.2)
    y = uniform_ball(rng, 11, 3, 0.2)
    mu = rng.uniform(0.5, 1.5, 17)
    nu = rng.uniform(0.2, 2.0, 11)
    eps = 0.05
    dist = np.sqrt(np.sum((x[:, None] - y[None]) ** 2, 2))
    c = oracle.cstar(x, mu, y, nu, eps, eta1, eta2, r=1)
    f = lambda cc: cf.primal_of_plan(cc * np.outer(mu, nu), dist, mu, nu, 1 / eps, eta1, eta2)  # noqa: E731
    for fac in (0.999, 1.001, 0.9, 1.1):
        assert f(fac * c) > f(c)


def test_transport_cost_r1_entropy_identity():
    """<pi, d> of the Gibbs plan with r = 1 equals sum beta p + sum gamma q - eps sum pi
    log(pi/(mu nu)) (log pi_ij/(mu_i nu_j) = lambda (beta_i + gamma_j - d_ij))."""
    rng = np.random.default_rng(6)
    x = uniform_ball(rng, 20, 2, 0.2)
    y = uniform_ball(rng, 15, 2, 0.2)
    mu = rng.uniform(0.5, 1.5, 20)
    nu = rng.uniform(0.2, 2.0, 15)
    eps = 0.1
    r = oracle.uot_sinkhorn_direct(x, mu, y, nu, eps, 1.0, 1.0, iters=9, r=1)
    t = oracle.transport_cost(x, mu, y, nu, r.beta, r.gamma, eps, r=1)
    dist = np.sqrt(np.sum((x[:, None] - y[None]) ** 2, 2))
    pi = (mu * np.exp(r.beta / eps))[:, None] * np.exp(-dist / eps) * (nu * np.exp(r.gamma / eps))[None, :]
    ent = float(np.sum(pi * np.log(pi / np.outer(mu, nu))))
    np.testing.assert_allclose(t, float(r.beta @ pi.sum(1) + r.gamma @ pi.sum(0)) - eps * ent, rtol=1e-11)
