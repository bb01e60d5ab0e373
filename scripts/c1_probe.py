"""C1 (configs[0]) whole-solve timing with the AUTO method (direct kernel), median of 20 (diagnostic)."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

pr = W.c1_uot()
args = [torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b)]
st = torch.cuda.current_stream()
for _ in range(5):
    uk.uot_sinkhorn(*args, pr.eps, pr.lam, iters=pr.iters)
per = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _, _, res = uk.uot_sinkhorn(*args, pr.eps, pr.lam, iters=pr.iters)
    e1.record(st)
    torch.cuda.synchronize()
    per.append(e0.elapsed_time(e1))
ms = statistics.median(per)
print(f"wpt={os.environ.get('UOTK_DIRECT_WPT', 'auto')} method={res.info['method']} {ms:.3f} ms/solve "
      f"{pr.iters / ms * 1e3:.0f} it/s primal {res.primal:.12g}")
