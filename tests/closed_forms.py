"""Closed forms and independent brute-force references used to PIN the oracle.

Nothing here re-types the oracle's formulas: each function is a separately derived
value (a closed-form integral, a textbook algorithm, a generic optimiser applied to
the primal definition) against which ``oracle/`` is checked.
"""

import math

import numpy as np
from scipy import optimize


# ---------------------------------------------------------------- kernels / sums
def gauss_line_integral(eps):
    """int_R exp(-y^2/eps) dy = sqrt(pi*eps)."""
    return math.sqrt(math.pi * eps)


def imq_segment_integral(L, c):
    """int_{-L}^{L} (y^2 + c^2)^(-1/2) dy = 2 asinh(L/c)."""
    return 2.0 * math.asinh(L / c)


def gauss_expectation(delta, s2, ell2, d):
    """E exp(-||Z||^2/ell2) for Z ~ N(delta, s2 I_d):
    (1 + 2 s2/ell2)^(-d/2) exp(-||delta||^2/(ell2 + 2 s2))  (completing the square)."""
    delta = np.asarray(delta, dtype=np.float64)
    return (1.0 + 2.0 * s2 / ell2) ** (-d / 2.0) * math.exp(-float(delta @ delta) / (ell2 + 2.0 * s2))


def gm_population_mmd2(means_x, means_y, sigma, ell2, mass_x=1.0, mass_y=1.0):
    """Population MMD^2 between two equal-weight isotropic Gaussian mixtures with
    total masses mass_x, mass_y, Gaussian kernel exp(-r^2/ell2).  X - X' for
    components (p, q) is N(m_p - m_q, 2 sigma^2 I)."""
    means_x = np.asarray(means_x, dtype=np.float64)
    means_y = np.asarray(means_y, dtype=np.float64)
    d = means_x.shape[1]
    s2 = 2.0 * sigma * sigma

    def cross(A, B):
        return np.mean([[gauss_expectation(p - q, s2, ell2, d) for q in B] for p in A])

    return (mass_x ** 2 * cross(means_x, means_x) - 2 * mass_x * mass_y * cross(means_x, means_y)
            + mass_y ** 2 * cross(means_y, means_y))


def gauss_hermite_mixture(means, sigma, q, mass=1.0):
    """Tensor Gauss-Hermite discretisation of an equal-weight isotropic Gaussian
    mixture: atoms and masses reproducing E f(X) for smooth f (numpy hermgauss)."""
    t, w = np.polynomial.hermite.hermgauss(q)  # int e^{-t^2} f(t) dt
    nodes1 = math.sqrt(2.0) * sigma * t
    w1 = w / math.sqrt(math.pi)
    means = np.asarray(means, dtype=np.float64)
    k, d = means.shape
    grids = np.meshgrid(*([nodes1] * d), indexing="ij")
    offs = np.stack([g.ravel() for g in grids], axis=1)
    wg = np.meshgrid(*([w1] * d), indexing="ij")
    ww = np.prod(np.stack([g.ravel() for g in wg], axis=1), axis=1)
    pts = np.concatenate([m + offs for m in means], axis=0)
    wts = np.concatenate([ww * (mass / k) for _ in means])
    return pts, wts


# ---------------------------------------------------------------- UOT
def single_atom_plan_mass(a, b, lam, eta1, eta2):
    """Coincident single atoms (d = 0): minimise over pi >= 0
    f(pi) = (1/lam)(pi log(pi/(ab)) + ab - pi) + eta1 (pi log(pi/a) + a - pi)
          + eta2 (pi log(pi/b) + b - pi);  f'(pi) = 0 gives the closed form below."""
    S = 1.0 / lam + eta1 + eta2
    return math.exp(((1.0 / lam) * math.log(a * b) + eta1 * math.log(a) + eta2 * math.log(b)) / S)


def cstar_eq210(mass_a, mass_b, mean_cost, lam, eta1, eta2):
    """Prop. 2.9, Eq. (2.10): optimal c for plans c * mu (x) nu;
    mean_cost = <mu (x) nu | d^r> / (mu(X) nu(X))."""
    S = eta1 + eta2 + 1.0 / lam
    return math.exp(-mean_cost / S) * mass_a ** (-eta2 / S) * mass_b ** (-eta1 / S)


def primal_of_plan(pi, d2, mu, nu, lam, eta1, eta2):
    """The discrete primal objective of P:462 for an arbitrary non-negative plan,
    written independently of the oracle (generalised KL)."""
    def kl(p, r):
        p = np.asarray(p, dtype=np.float64)
        m = p > 0
        return float(np.sum(p[m] * np.log(p[m] / r[m]))) + float(np.sum(r)) - float(np.sum(p))

    munu = np.outer(mu, nu)
    return (float(np.sum(d2 * pi)) + kl(pi.ravel(), munu.ravel()) / lam
            + eta1 * kl(pi.sum(axis=1), mu) + eta2 * kl(pi.sum(axis=0), nu))


def brute_force_uot(x, mu, y, nu, eps, eta1, eta2, r=2):
    """Minimise the primal (2.9)/ with cost d^r over all plans pi in R_+^{n x m}
    with a generic quasi-Newton optimiser on log pi.  Tiny n, m only."""
    lam = 1.0 / eps
    x = np.asarray(x, dtype=np.float64).reshape(len(mu), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(nu), -1)
    d2 = np.sum((x[:, None, :] - y[None, :, :]) ** 2, axis=2)
    if r == 1:
        d2 = np.sqrt(d2)  # the cost matrix d^r (named d2 below)
    n, m = d2.shape

    def f(z):
        pi = np.exp(z.reshape(n, m))
        val = primal_of_plan(pi, d2, mu, nu, lam, eta1, eta2)
        # gradient wrt log pi: pi * dP/dpi
        p, q = pi.sum(1), pi.sum(0)
        g = d2 + np.log(pi / np.outer(mu, nu)) / lam + eta1 * np.log(p / mu)[:, None] + eta2 * np.log(q / nu)[None, :]
        return val, (pi * g).ravel()

    z0 = np.log(np.outer(mu, nu) * 0.5).ravel()
    res = optimize.minimize(f, z0, jac=True, method="L-BFGS-B",
                            options={"maxiter": 20000, "ftol": 1e-16, "gtol": 1e-13})
    pi = np.exp(res.x.reshape(n, m))
    return res.fun, pi


def balanced_sinkhorn(x, a, y, b, eps, iters):
    """Textbook balanced entropic OT (Cuturi 2013): u = a/(K v), v = b/(K^T u),
    K = exp(-C/eps), C = squared distances.  Returns the plan."""
    x = np.asarray(x, dtype=np.float64).reshape(len(a), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(b), -1)
    C = np.sum((x[:, None, :] - y[None, :, :]) ** 2, axis=2)
    K = np.exp(-C / eps)
    v = np.ones(len(b))
    for _ in range(iters):
        u = a / (K @ v)
        v = b / (K.T @ u)
    return u[:, None] * K * v[None, :]


# ---------------------------------------------------------------- Laplace / energy kernels (NEXT-f2)
def laplace_segment_integral(L, ell):
    """int_{-L}^{L} exp(-|y|/l) dy = 2 l (1 - e^{-L/l})."""
    return 2.0 * ell * (1.0 - math.exp(-L / ell))


def laplace_disk_integral(R, ell):
    """int_{|y| <= R} exp(-|y|/l) dy over the disk in R^2 = 2 pi l^2 (1 - e^{-R/l}(1 + R/l))."""
    u = R / ell
    return 2.0 * math.pi * ell ** 2 * (1.0 - math.exp(-u) * (1.0 + u))


def laplace_ball_integral(R, ell):
    """int_{|y| <= R} exp(-|y|/l) dy over the ball in R^3 = 4 pi l^3 (2 - e^{-R/l}(u^2 + 2u + 2)), u = R/l."""
    u = R / ell
    return 4.0 * math.pi * ell ** 3 * (2.0 - math.exp(-u) * (u * u + 2.0 * u + 2.0))


def energy_segment_integral(L, x):
    """int_{-L}^{L} -|x - y| dy = -(L^2 + x^2) for |x| <= L."""
    return -(L * L + x * x)


def polar_rule(R, nr, nt):
    """Product quadrature on the disk of radius R: Gauss-Legendre in r on [0, R] (weight r),
    the trapezoidal rule in the angle (exact for trigonometric polynomials)."""
    t, w = np.polynomial.legendre.leggauss(nr)
    r = 0.5 * R * (t + 1.0)
    wr = 0.5 * R * w * r
    th = 2.0 * math.pi * np.arange(nt) / nt
    pts = np.stack([np.outer(r, np.cos(th)).ravel(), np.outer(r, np.sin(th)).ravel()], axis=1)
    wts = np.outer(wr, np.full(nt, 2.0 * math.pi / nt)).ravel()
    return pts, wts


def spherical_rule(R, nr, nc, nphi):
    """Product quadrature on the ball of radius R: Gauss-Legendre in r (weight r^2) and in
    cos(theta), the trapezoidal rule in phi."""
    t, w = np.polynomial.legendre.leggauss(nr)
    r = 0.5 * R * (t + 1.0)
    wr = 0.5 * R * w * r * r
    c, wc = np.polynomial.legendre.leggauss(nc)
    s = np.sqrt(1.0 - c * c)
    ph = 2.0 * math.pi * np.arange(nphi) / nphi
    R_, C_, P_ = np.meshgrid(r, c, ph, indexing="ij")
    S_ = np.sqrt(1.0 - C_ * C_)
    pts = np.stack([(R_ * S_ * np.cos(P_)).ravel(), (R_ * S_ * np.sin(P_)).ravel(), (R_ * C_).ravel()], axis=1)
    W = np.einsum("i,j,k->ijk", wr, wc, np.full(nphi, 2.0 * math.pi / nphi)).ravel()
    del s
    return pts, W
