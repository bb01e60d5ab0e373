"""Time the Gaussian spectral step (tag "fft": the separable DMMA chain) inside kernel sums
of the C3 / C4 geometries (diagnostic)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
cases = [("C3", W.c3_uot(n=200_000, iters=1), {}), ("C4 auto", W.c4_uot(n=200_000, iters=1), {}),
         ("C4 N=2048", W.c4_uot(n=200_000, iters=1), {"N": 2048})]
for name, pr, o in cases:
    args = (t(pr.y), t(pr.b), t(pr.x), "gauss", pr.eps)
    for _ in range(3):
        uk.kernel_sum(*args, opts=dict(o, method="nfft"))
    uk.profile_reset()
    uk.profile_enable(True)
    for _ in range(10):
        _, info = uk.kernel_sum(*args, opts=dict(o, method="nfft"), return_info=True)
    torch.cuda.synchronize()
    prof = uk.profile_read()
    uk.profile_enable(False)
    ms, cnt = prof["fft"]
    print(f"{name}: n_grid {info['n_grid']} chain {1e3 * ms / max(cnt, 1):.1f} us per kernel sum", flush=True)
