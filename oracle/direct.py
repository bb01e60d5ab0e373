"""Direct kernel sum, Eq. (4.3) — TEST INFRASTRUCTURE ONLY.

    s(x_i) = sum_j K(x_i - x~_j) alpha~_j ,   i = 1..n

computed by its plain definition: for each target, all pairwise differences are
formed explicitly (no ||x||^2 + ||y||^2 - 2 x.y expansion, which loses digits),
the kernel is applied, and the row is summed with numpy's pairwise summation.
Targets are processed in blocks only to bound memory; nothing is reordered.
"""

import numpy as np

from .kernels import kernel_fn


def _as_points(p):
    p = np.asarray(p, dtype=np.float64)
    if p.ndim == 1:
        p = p[:, None]
    return p


def kernel_sum_direct(src, alpha, tgt, kind, param, block_bytes=1 << 27):
    """Return s with s_i = sum_j K(||tgt_i - src_j||) alpha_j (Eq. 4.3).

    src: (n_src, d), alpha: (n_src,), tgt: (n_tgt, d); kind 0 = Gauss, 1 = IMQ.
    """
    src = _as_points(src)
    tgt = _as_points(tgt)
    alpha = np.asarray(alpha, dtype=np.float64)
    n_src, d = src.shape
    n_tgt = tgt.shape[0]
    assert tgt.shape[1] == d and alpha.shape == (n_src,)
    K = kernel_fn(kind, param)
    out = np.empty(n_tgt, dtype=np.float64)
    if n_tgt == 0:
        return out
    if n_src == 0:
        out[:] = 0.0
        return out
    bt = max(1, int(block_bytes // (8 * n_src * max(d, 1))))
    for i0 in range(0, n_tgt, bt):
        i1 = min(n_tgt, i0 + bt)
        diff = tgt[i0:i1, None, :] - src[None, :, :]  # (bt, n_src, d)
        r2 = np.sum(diff * diff, axis=2)
        out[i0:i1] = np.sum(K(r2) * alpha[None, :], axis=1)
    return out
