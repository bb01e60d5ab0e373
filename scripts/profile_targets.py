"""One invocation of each hot kernel family, for ncu captures (profiles/r01/ncu_*.md).

    ncu --set full --clock-control none --import-source on -k regex:'<kernel>' -c 1 \\
        -o gpurun_out/<name> python scripts/profile_targets.py <target>

targets:
  sum3d    kernel sum d=3 (C5 recipe, n = m = 4e6, Gaussian l = 0.05): chunked3d_k spread
           (mode 1) and gather (mode 2), cuFFT D2Z / scale_spectrum_k / Z2D on 140^3
  c4       two C4 iterations (d = 2, n = m = 16M): chunked2d_k fused half-steps, 160^2 FFTs
  c3       two C3 iterations (d = 3, n = m = 1M): sinkhorn3d_ws_k, 96^3 FFTs
  c3m6     the same with m = 6, sigma = 3: sinkhorn3d_m6_ws_k, 144^3 grid
  mmd      MMD^2 at n = m = 1M (C2 distributions, Gaussian l = 0.05), the bench's MMD leg
  mmdimq   the same with the inverse multiquadric (c = 0.05)
  c3sum    one kernel sum on C3's points (x -> y, Gaussian eps = 0.02): stand-alone spread and
           gather kernels on a dense cloud (env M=6 selects m = 6, sigma = 3)
  direct   direct kernel sum d = 3, n = m = 2e5 (direct_k, FP64 exp)
  sum3dimq kernel sum d=3, n = m = 1e6, IMQ c = 0.05 (N = 192, grid 384^3)
  c1       five C1 solves (d = 2, 1000 + 1000 points, DIRECT: direct_warp_k)
  sum1d    kernel sum d = 1, n = m = 1e7 (chunked1d_k)
Each target runs its call twice (the first call warms plans and caches); the second runs
inside the NVTX range "prof" (ncu --nvtx --nvtx-include "prof/").
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main(target):
    if target == "sum3d":
        pr = W.c5_sum(3, 4_000_000, kind=W.GAUSS)
        args = (cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param)
        call = lambda: uk.kernel_sum(*args, opts={"method": "nfft"})  # noqa: E731
    elif target == "sum3dimq":
        pr = W.c5_sum(3, 1_000_000, kind=W.IMQ)
        args = (cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "imq", pr.param)
        call = lambda: uk.kernel_sum(*args, opts={"method": "nfft"})  # noqa: E731
    elif target == "c1":
        pr = W.c1_uot()
        args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
        call = lambda: uk.uot_sinkhorn(*args, iters=pr.iters, opts={"method": "direct"})  # noqa: E731
    elif target == "sum1d":
        pr = W.c5_sum(1, 10_000_000, kind=W.GAUSS)
        args = (cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param)
        call = lambda: uk.kernel_sum(*args, opts={"method": "nfft"})  # noqa: E731
    elif target == "direct":
        pr = W.c5_sum(3, 200_000, kind=W.GAUSS)
        args = (cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt), "gauss", pr.param)
        call = lambda: uk.kernel_sum(*args, opts={"method": "direct"})  # noqa: E731
    elif target in ("mmd", "mmdimq"):
        pr = W.c2_mmd(n=1_000_000)
        kk = pr.kernels[0] if target == "mmd" else pr.kernels[1]
        args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), kk[0], kk[1])
        call = lambda: uk.mmd2(*args, opts={"method": "nfft"})  # noqa: E731
    elif target == "c3sum":
        pr = W.c3_uot(iters=2)
        args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), "gauss", pr.eps)
        o = {"method": "nfft"}
        if os.environ.get("M") == "6":
            o.update(m=6, sigma=3.0)
        call = lambda: uk.kernel_sum(*args, opts=o)  # noqa: E731
    elif target in ("c3", "c4", "c3m6"):
        pr = W.c4_uot(iters=2) if target == "c4" else W.c3_uot(iters=2)
        args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
        o = {"method": "nfft"}
        if target == "c3m6":
            o.update(m=6, sigma=3.0)
        call = lambda: uk.uot_sinkhorn(*args, iters=2, opts=o)  # noqa: E731
    else:
        raise SystemExit(f"unknown target {target}")
    call()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")  # ncu --nvtx --nvtx-include "prof/" captures this call only
    call()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"{target}: ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "sum3d")
