"""Where the end-to-end (pinned host buffers) C3 solve spends its time beyond the
device-resident one: raw H2D / D2H copy times of the same bytes, and the two solves —
diagnostics for DESIGN §10."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402


def ev_time(fn, reps=3):
    s = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), out


pr = W.c3_uot()
host = [torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for v in (pr.x, pr.a, pr.y, pr.b)]
dev = [h.cuda() for h in host]
outp = [torch.empty(len(pr.a), dtype=torch.float64, pin_memory=True), torch.empty(len(pr.b), dtype=torch.float64,
                                                                                   pin_memory=True)]
outd = [torch.empty(len(pr.a), dtype=torch.float64, device="cuda"), torch.empty(len(pr.b), dtype=torch.float64,
                                                                               device="cuda")]
print("h2d 64 MB pinned ms", ev_time(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(dev, host)]))
print("d2h 16 MB pinned ms", ev_time(lambda: [h.copy_(d, non_blocking=True) for d, h in zip(outd, outp)]))
kw = dict(iters=pr.iters, opts={"method": "nfft"})
uk.uot_sinkhorn(*dev, pr.eps, pr.lam, **kw)
print("solve device ms", ev_time(lambda: uk.uot_sinkhorn(*dev, pr.eps, pr.lam, **kw)))
uk.uot_sinkhorn(*host, pr.eps, pr.lam, **kw)
print("solve host ms", ev_time(lambda: uk.uot_sinkhorn(*host, pr.eps, pr.lam, **kw)))
t0 = time.perf_counter()
uk.uot_sinkhorn(*host, pr.eps, pr.lam, **kw)
print("solve host wall ms", 1e3 * (time.perf_counter() - t0))
