"""C1 (d = 2, n = m = 1000, 100 iterations, AUTO -> direct) solved a few times, for an
ncu launch list of the direct half-step kernel."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

pr = W.c1_uot()
x, a, y, b = (torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b))
for _ in range(3):
    uk.uot_sinkhorn(x, a, y, b, pr.eps, pr.lam, iters=pr.iters)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    uk.uot_sinkhorn(x, a, y, b, pr.eps, pr.lam, iters=pr.iters)
e.record()
torch.cuda.synchronize()
print(f"C1 solve {s.elapsed_time(e) / 10:.3f} ms", flush=True)
