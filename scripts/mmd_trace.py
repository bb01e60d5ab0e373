"""Phase timeline of one MMD^2 call at n = m = 1M (C2 distributions, Gaussian), for the
call-overhead analysis: run with UOTK_TRACE=1 (host time between marks) or =2 (device
synchronised at each mark)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

pr = W.c2_mmd(n=int(os.environ.get("MMD_N", "1000000")))
x, a, y, b = (torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b))
for _ in range(3):
    uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
torch.cuda.synchronize()
print("---- timed call", file=sys.stderr, flush=True)
t0 = time.perf_counter()
v = uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
print(f"call {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
uk.profile_enable(True)
uk.profile_reset()
for _ in range(5):
    uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
print({k: (round(ms / 5, 4), c // 5) for k, (ms, c) in uk.profile_read().items()}, file=sys.stderr)
