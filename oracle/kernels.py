"""Radial kernels of the paper, fp64 (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Paper Eq. (4.2):  K^Gauss(y) = exp(-||y||^2 / l^2),  K^IMQ(y) = 1/sqrt(||y||^2 + c^2),
K^Lap(y) = exp(-||y|| / l),  K^abs(y) = ||y||.
Table 1 uses the same forms, and writes the energy kernel with a minus sign,
k^e(x, x~) = -||x - x~||, which is the form used here (MMD^2 with k^e is the energy
distance).  The configs (BASELINE.json) write the Gaussian as
exp(-||x-y||^2 / eps), i.e. ``param = eps = l^2``; the IMQ ``param`` is c; the Laplace
``param`` is l; the energy kernel has no parameter (``param`` is ignored).
"""

import numpy as np

GAUSS = 0
IMQ = 1
GAUSS_R2 = 2
LAP = 3
ENERGY = 4


def gauss(r2, eps):
    """exp(-r^2/eps) from the squared distance r2 (Eq. 4.2, with l^2 = eps)."""
    return np.exp(-np.asarray(r2, dtype=np.float64) / eps)


def imq(r2, c):
    """(r^2 + c^2)^(-1/2) from the squared distance r2 (Eq. 4.2)."""
    return 1.0 / np.sqrt(np.asarray(r2, dtype=np.float64) + c * c)


def gauss_r2(r2, eps):
    """r^2 exp(-r^2/eps): the transport-cost kernel d^2 k of the Gibbs plan."""
    r2 = np.asarray(r2, dtype=np.float64)
    return r2 * np.exp(-r2 / eps)


def laplace(r2, ell):
    """exp(-r/l) from the squared distance r2 (Eq. 4.2; Table 1)."""
    return np.exp(-np.sqrt(np.asarray(r2, dtype=np.float64)) / ell)


def energy(r2):
    """k^e = -r from the squared distance r2 (Table 1: k^e(x, x~) = -||x - x~||)."""
    return -np.sqrt(np.asarray(r2, dtype=np.float64))


def kernel_fn(kind, param):
    """Return K as a function of the squared distance."""
    if kind == GAUSS:
        return lambda r2: gauss(r2, param)
    if kind == IMQ:
        return lambda r2: imq(r2, param)
    if kind == GAUSS_R2:
        return lambda r2: gauss_r2(r2, param)
    if kind == LAP:
        return lambda r2: laplace(r2, param)
    if kind == ENERGY:
        return lambda r2: energy(r2)
    raise ValueError(f"unknown kernel kind {kind!r}")
