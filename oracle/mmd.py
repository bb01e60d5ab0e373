"""Discrete MMD^2, Eq. (3.5) — TEST INFRASTRUCTURE ONLY.

    MMD_k^2(mu, nu) = sum_{i,j} mu_i mu_j k(x_i, x_j) - 2 sum_{i,j} mu_i nu_j k(x_i, x~_j)
                      + sum_{i,j} nu_i nu_j k(x~_i, x~_j)

including the diagonal i = j terms, as printed (a V-statistic; reading R8).
"""

import numpy as np

from .direct import kernel_sum_direct


def mmd2_direct(x, a, y, b, kind, param):
    """The three double sums of (3.5), each by a direct kernel sum (4.3)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    xx = float(np.sum(a * kernel_sum_direct(x, a, x, kind, param)))
    xy = float(np.sum(a * kernel_sum_direct(y, b, x, kind, param)))
    yy = float(np.sum(b * kernel_sum_direct(y, b, y, kind, param)))
    return xx - 2.0 * xy + yy


def mmd2_combined(x, a, y, b, kind, param):
    """(3.5) as one quadratic form over z = x u y with signed weights w = (a, -b).

    sum_{i,j in z} w_i w_j k(z_i, z_j) expands to exactly the three sums of (3.5).
    """
    x = np.asarray(x, dtype=np.float64).reshape(len(a), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(b), -1)
    z = np.concatenate([x, y], axis=0)
    w = np.concatenate([np.asarray(a, dtype=np.float64), -np.asarray(b, dtype=np.float64)])
    return float(np.sum(w * kernel_sum_direct(z, w, z, kind, param)))
