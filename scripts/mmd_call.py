"""MMD^2 at n = m = 1M (C2 distributions, Gaussian): warm whole-call time, median of 30
host-timed calls (the call returns a host scalar, so it synchronises) — diagnostics."""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

pr = W.c2_mmd(n=1_000_000)
x, a, y, b = (torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b))
for _ in range(5):
    v = uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
torch.cuda.synchronize()
ts = []
for _ in range(30):
    t0 = time.perf_counter()
    v = uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
    ts.append(1e3 * (time.perf_counter() - t0))
print(f"mmd2 call median {statistics.median(ts):.3f} ms (min {min(ts):.3f}) value {v!r}", flush=True)
