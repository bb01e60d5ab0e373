"""A/B probe (diagnostics): device time per launch of the MMD^2 spread at 1M (C2
distributions) and of the C3 fused half-step (20-iteration solve), from the library's
per-tag CUDA-event profile.  Run under different env switches / UOTK_LIB_PATH builds."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "mmd,c3"
out = {}
if "mmd" in which:
    pr = W.c2_mmd(n=1_000_000)
    x, a, y, b = (torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b))
    for _ in range(3):
        uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
    torch.cuda.synchronize()
    uk.profile_enable(True)
    uk.profile_reset()
    for _ in range(10):
        v = uk.mmd2(x, a, y, b, "gauss", 0.0025, opts={"method": "nfft"})
    p = uk.profile_read()
    out["mmd_spread_ms"] = round(p["spread"][0] / p["spread"][1], 4)
    out["mmd2"] = v
    uk.profile_enable(False)
if "c3" in which:
    pr = W.c3_uot(iters=20)
    args = [torch.from_numpy(v).cuda() for v in (pr.x, pr.a, pr.y, pr.b)]
    uk.uot_sinkhorn(*args, pr.eps, pr.lam, iters=20, opts={"method": "nfft"})
    torch.cuda.synchronize()
    uk.profile_enable(True)
    uk.profile_reset()
    _, _, res = uk.uot_sinkhorn(*args, pr.eps, pr.lam, iters=20, opts={"method": "nfft"})
    p = uk.profile_read()
    out["c3_fused_ms"] = round(p["fused"][0] / p["fused"][1], 4)
    out["c3_primal"] = res.primal
    uk.profile_enable(False)
if "c5" in which:
    for kind, param in ((W.GAUSS, None), (W.IMQ, None)):
        pr = W.c5_sum(3, 1_000_000, kind=kind)
        args = [torch.from_numpy(v).cuda() for v in (pr.src, pr.alpha, pr.tgt)]
        for _ in range(3):
            uk.kernel_sum(*args, kind, pr.param, opts={"method": "nfft"})
        torch.cuda.synchronize()
        uk.profile_enable(True)
        uk.profile_reset()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(5):
            r, info = uk.kernel_sum(*args, kind, pr.param, opts={"method": "nfft"}, return_info=True)
        ev1.record()
        torch.cuda.synchronize()
        p = uk.profile_read()
        out[f"c5_{kind}_spread_ms"] = round(p["spread"][0] / p["spread"][1], 4)
        out[f"c5_{kind}_call_ms"] = round(ev0.elapsed_time(ev1) / 5, 4)
        out[f"c5_{kind}_groups"] = info["groups"]
        out[f"c5_{kind}_sum0"] = float(r[0])
        uk.profile_enable(False)
print(os.environ.get("UOTK_COST", "default"), out, flush=True)
