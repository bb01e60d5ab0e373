"""Full-size cross-check of the NFFT path against the GPU direct kernel (K6, itself
oracle-validated in tests/test_gpu_parity.py) on complete solves (SURVEY §8(d) parity
(iii)): C3 with all 200 iterations (2 x 1e12 pairs per iteration on the direct side,
~11 min on one B200), with the paper's window (m = 8, sigma = 2) and with m = 6,
sigma = 3, and C2's MMD^2 (Gaussian and IMQ).  Writes one JSON object.

    python scripts/crosscheck_full.py [--iters 200] > profiles/r01/crosscheck_full.json
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=200)
    a = p.parse_args()
    out = {"what": "NFFT vs GPU DIRECT on full-size solves (DESIGN.md §4, SURVEY 8(d) parity iii)"}
    pr = W.c3_uot(iters=a.iters)
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    t0 = time.time()
    b2, g2, r2 = uk.uot_sinkhorn(*args, iters=a.iters, opts={"method": "direct"})
    torch.cuda.synchronize()
    t_direct = time.time() - t0
    # the paper's window (m = 8, sigma = 2, the default) and the m = 6, sigma = 3 window
    for key, o in (("C3", {}), ("C3_m6_sigma3", {"m": 6, "sigma": 3.0})):
        t0 = time.time()
        b1, g1, r1 = uk.uot_sinkhorn(*args, iters=a.iters, opts=dict(o, method="nfft"))
        torch.cuda.synchronize()
        t_nfft = time.time() - t0
        resid = float(torch.linalg.norm(b1 - b2) / torch.linalg.norm(b2)
                      + torch.linalg.norm(g1 - g2) / torch.linalg.norm(g2))
        out[key] = {
            "n": len(pr.x), "m": len(pr.y), "iters": a.iters, "window": r1.info,
            "residual_beta_gamma": resid,
            "primal_nfft": r1.primal, "primal_direct": r2.primal,
            "primal_rel_diff": abs(r1.primal - r2.primal) / abs(r2.primal),
            "dual_rel_diff": abs(r1.dual - r2.dual) / abs(r2.dual),
            "plan_mass_rel_diff": abs(r1.plan_mass - r2.plan_mass) / r2.plan_mass,
            "max_abs_dbeta": float(torch.max(torch.abs(b1 - b2))),
            "seconds_nfft": t_nfft, "seconds_direct": t_direct,
            "pass_1e-8": resid <= 1e-8 and abs(r1.primal - r2.primal) <= 1e-8 * abs(r2.primal),
        }
        print(json.dumps(out[key]), file=sys.stderr, flush=True)
    m = W.c2_mmd()
    x, aa, y, b = cuda(m.x), cuda(m.a), cuda(m.y), cuda(m.b)
    out["C2"] = {}
    for kind, param in m.kernels:
        v1 = uk.mmd2(x, aa, y, b, kind, param, opts={"method": "nfft"})
        v2 = uk.mmd2(x, aa, y, b, kind, param, opts={"method": "direct"})
        xx = uk.mmd2(x, aa, x[:0], b[:0], kind, param, opts={"method": "direct"})
        yy = uk.mmd2(y, b, y[:0], b[:0], kind, param, opts={"method": "direct"})
        denom = max(abs(v2), 1e-3 * (abs(xx) + abs(yy)))
        out["C2"]["gauss" if kind == W.GAUSS else "imq"] = {
            "mmd2_nfft": v1, "mmd2_direct": v2, "rel_diff_R13": abs(v1 - v2) / denom,
            "pass_1e-8": abs(v1 - v2) / denom <= 1e-8}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
