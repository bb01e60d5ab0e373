"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no kernels, no sums, no Sinkhorn):
it only draws points and masses.  Both sides of every parity test consume the
arrays it returns.  Recipes:

* Random generator: ``numpy.random.default_rng(seed)`` (PCG64); draw order is
  points x, points y, masses a, masses b (for mixtures: component means first).
* "uniform in ball of radius R": a normalised Gaussian direction times R*U^(1/d).
* Gaussian mixture: equal component weights, isotropic N(mean, sigma^2 I);
  "clipped to radius R" = reject and redraw any sample with ||x|| > R.

The five configurations are BASELINE.json ``configs[0..4]`` (C1..C5).  They stand
in for the paper's Sec. 5.1.1 workload (U[0,1]^d points, U[0,1] weights)
already placed in the fast-summation ball; no public dataset is involved.
"""

from dataclasses import dataclass, field

import numpy as np

GAUSS = 0
IMQ = 1
GAUSS_R2 = 2


def uniform_ball(rng, n, d, radius):
    """n points uniform in the d-ball of the given radius."""
    g = rng.standard_normal((n, d))
    nrm = np.linalg.norm(g, axis=1, keepdims=True)
    nrm[nrm == 0] = 1.0
    r = radius * rng.random(n) ** (1.0 / d)
    return g / nrm * r[:, None]


def gaussian_mixture(rng, n, means, sigma, clip=None):
    """n points from an equal-weight isotropic Gaussian mixture, optional rejection clip."""
    means = np.asarray(means, dtype=np.float64)
    k, d = means.shape
    out = np.empty((n, d))
    filled = 0
    while filled < n:
        need = n - filled
        comp = rng.integers(0, k, need)
        pts = means[comp] + sigma * rng.standard_normal((need, d))
        if clip is not None:
            pts = pts[np.linalg.norm(pts, axis=1) <= clip]
        out[filled:filled + len(pts)] = pts
        filled += len(pts)
    return out


@dataclass
class UOTProblem:
    name: str
    x: np.ndarray
    a: np.ndarray
    y: np.ndarray
    b: np.ndarray
    eps: float
    lam: float
    iters: int
    meta: dict = field(default_factory=dict)

    @property
    def d(self):
        return self.x.shape[1]


@dataclass
class MMDProblem:
    name: str
    x: np.ndarray
    a: np.ndarray
    y: np.ndarray
    b: np.ndarray
    kernels: tuple  # ((kind, param), ...)
    meta: dict = field(default_factory=dict)

    @property
    def d(self):
        return self.x.shape[1]


@dataclass
class SumProblem:
    name: str
    src: np.ndarray
    alpha: np.ndarray
    tgt: np.ndarray
    kind: int
    param: float
    meta: dict = field(default_factory=dict)


def c1_uot(n=1000, m=None, seed=0, d=2):
    """C1: UOT d=2, n=m=1000, uniform ball R=0.2, a~U(0.5,1.5), b~U(0.2,2.0),
    Gaussian exp(-r^2/eps) eps=0.05, KL penalty lam=1.0, 100 iterations, seed 0."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x = uniform_ball(rng, n, d, 0.2)
    y = uniform_ball(rng, m, d, 0.2)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.2, 2.0, m)
    return UOTProblem("C1", x, a, y, b, eps=0.05, lam=1.0, iters=100)


def c2_mmd(n=100_000, m=None, seed=0):
    """C2: MMD^2 d=3, n=m=1e5; mu = 2-component GM (means +-0.05 e1, sigma=0.03),
    nu = the same shifted by 0.02 e2; weights U(0.5,1.5); Gaussian sigma=0.05
    (param eps = sigma^2 = 0.0025, reading R6) and IMQ c = 0.05."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    mx = np.array([[0.05, 0.0, 0.0], [-0.05, 0.0, 0.0]])
    my = mx + np.array([0.0, 0.02, 0.0])
    x = gaussian_mixture(rng, n, mx, 0.03)
    y = gaussian_mixture(rng, m, my, 0.03)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.5, 1.5, m)
    return MMDProblem("C2", x, a, y, b, kernels=((GAUSS, 0.05 ** 2), (IMQ, 0.05)),
                      meta={"means_x": mx, "means_y": my, "sigma": 0.03})


def c2_dense_mmd(n=10_000, m=None, seed=0, shrink=0.2):
    """C2's mixtures (means +-0.05 e1, sigma 0.03, nu shifted by 0.02 e2, weights
    U(0.5,1.5)) shrunk by ``shrink`` about the origin, so that a reduced n fills the grid
    cells (the Gaussian's h is floored by its width) about as unevenly as C2 at 1M: dense
    cells next to sparse ones, the mix the hybrid spread groups serve (tests only)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    mx = shrink * np.array([[0.05, 0.0, 0.0], [-0.05, 0.0, 0.0]])
    my = mx + shrink * np.array([0.0, 0.02, 0.0])
    x = gaussian_mixture(rng, n, mx, 0.03 * shrink)
    y = gaussian_mixture(rng, m, my, 0.03 * shrink)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.5, 1.5, m)
    return MMDProblem("C2-dense", x, a, y, b, kernels=((GAUSS, 0.05 ** 2), (IMQ, 0.05)),
                      meta={"shrink": shrink})


def c3_uot(n=1_000_000, m=None, seed=0, iters=200):
    """C3: UOT d=3, n=m=1M from 8-component Gaussian mixtures clipped to radius 0.2
    (reading R15: means uniform in the ball of radius 0.12, sigma = 0.025),
    masses U(0.1,1.0), Gaussian eps=0.02, lam=0.5, 200 iterations."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    mx = uniform_ball(rng, 8, 3, 0.12)
    my = uniform_ball(rng, 8, 3, 0.12)
    x = gaussian_mixture(rng, n, mx, 0.025, clip=0.2)
    y = gaussian_mixture(rng, m, my, 0.025, clip=0.2)
    a = rng.uniform(0.1, 1.0, n)
    b = rng.uniform(0.1, 1.0, m)
    return UOTProblem("C3", x, a, y, b, eps=0.02, lam=0.5, iters=iters)


def c3_dense_uot(n=6000, m=None, seed=0, iters=10):
    """C3's parameters (d=3, eps=0.02, lam=0.5, masses U(0.1,1.0)) and C3's per-cell
    density at reduced n: the mixture geometry of ``c3_uot`` shrunk by s = (n/1e6)^(1/3)
    (means in the ball of radius 0.12 s, sigma 0.025 s, clip 0.2 s), so the points fill
    the grid cells as densely as at 1M and the NFFT path forms one-cell groups — the
    layout the headline's warp-specialised half-step runs on (tests only)."""
    m = n if m is None else m
    s = (max(n, m) / 1e6) ** (1.0 / 3.0)
    rng = np.random.default_rng(seed)
    mx = uniform_ball(rng, 8, 3, 0.12 * s)
    my = uniform_ball(rng, 8, 3, 0.12 * s)
    x = gaussian_mixture(rng, n, mx, 0.025 * s, clip=0.2 * s)
    y = gaussian_mixture(rng, m, my, 0.025 * s, clip=0.2 * s)
    a = rng.uniform(0.1, 1.0, n)
    b = rng.uniform(0.1, 1.0, m)
    return UOTProblem("C3-dense", x, a, y, b, eps=0.02, lam=0.5, iters=iters, meta={"shrink": s})


def c4_uot(n=16_000_000, m=None, seed=0, iters=50):
    """C4: UOT d=2, n=m=16M uniform ball R=0.2, eps=0.002, lam=2.0, 50 iterations;
    masses a~U(0.5,1.5), b~U(0.2,2.0) (reading R16)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x = uniform_ball(rng, n, 2, 0.2)
    y = uniform_ball(rng, m, 2, 0.2)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.2, 2.0, m)
    return UOTProblem("C4", x, a, y, b, eps=0.002, lam=2.0, iters=iters)


def c5_sum(d, n, m=None, kind=GAUSS, seed=0):
    """C5: kernel sum, uniform ball R=0.2, weights N(0,1); Gaussian l=0.05
    (param 0.0025) or IMQ c=0.05 (reading R7)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    src = uniform_ball(rng, n, d, 0.2)
    tgt = uniform_ball(rng, m, d, 0.2)
    alpha = rng.standard_normal(n)
    param = 0.05 ** 2 if kind == GAUSS else 0.05
    return SumProblem(f"C5-d{d}-n{n}", src, alpha, tgt, kind, param)


def random_sum(d, n_src, n_tgt, kind=GAUSS, param=None, seed=0, radius=0.2, signed=False):
    """Small generic kernel-sum instance (tests)."""
    rng = np.random.default_rng(seed)
    src = uniform_ball(rng, n_src, d, radius)
    tgt = uniform_ball(rng, n_tgt, d, radius)
    alpha = rng.standard_normal(n_src) if signed else rng.uniform(0.1, 1.0, n_src)
    if param is None:
        param = 0.02 if kind == GAUSS else 0.05
    return SumProblem(f"rand-d{d}", src, alpha, tgt, kind, param)
