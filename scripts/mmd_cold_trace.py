"""Host phase timeline of a COLD MMD^2 call at n = m = 1M (after uotk_release_caches):
run with UOTK_TRACE=1."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

pr = W.c2_mmd(n=1_000_000)
x, a, y, b = (torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b))
for _ in range(3):
    uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
for _ in range(3):
    uk.release_caches()
    torch.cuda.synchronize()
    print("---- cold call", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
    print(f"cold call {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
