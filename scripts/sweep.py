"""Timing sweep over the non-headline configs (BASELINE.json configs C1, C2, C4, C5):
per call device time (CUDA events on the calling stream) and the per-kernel-tag
breakdown of the library's profiling hooks.  Prints one JSON object per case.

    python scripts/sweep.py [--cases c1,c2,c4,c5] [--c5-max 1e7] [--c4-iters 5]

Diagnostics only: bench.py is the contract; this script shows where the other
configurations spend their time.
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


def spin_up(seconds=0.3):
    """Keep the GPU busy briefly so that the SM clock has left its idle state (the
    library's host synchronisations between short calls otherwise let it drop)."""
    a = torch.randn(2048, 2048, device="cuda")
    t0 = time.time()
    while time.time() - t0 < seconds:
        a = (a @ a).clamp_(-1, 1)
    torch.cuda.synchronize()


def timed(fn, reps=3):
    """Median device time per call over `reps` unprofiled calls (each bracketed by CUDA
    events on the current stream); then one profiled call for the per-tag kernel times
    (profiling brackets every launch with events and disables the CUDA-graph replay)."""
    fn()
    fn()  # a second warm-up: the first calls grow the memory pool and build plans
    spin_up()
    torch.cuda.synchronize()
    uk.reset_launch_counter()
    times, walls = [], []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - w0) * 1e3)
        times.append(s.elapsed_time(e))
    launches = uk.launch_counter() / reps
    timed.wall_ms = float(np.median(walls))
    timed.all_ms = [round(t, 3) for t in times]
    ms = float(np.median(times))
    uk.profile_enable(True)
    uk.profile_reset()
    fn()
    torch.cuda.synchronize()
    prof = {k: round(v[0], 4) for k, v in uk.profile_read().items() if v[1]}
    uk.profile_enable(False)
    return ms, prof, launches, out


def emit(**kw):
    kw["wall_ms"] = round(getattr(timed, "wall_ms", 0.0), 3)
    kw["all_ms"] = getattr(timed, "all_ms", None)
    print(json.dumps(kw), flush=True)


def case_c1():
    pr = W.c1_uot()
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    for method in ("direct", "nfft"):
        ms, prof, nl, out = timed(lambda: uk.uot_sinkhorn(*args, iters=pr.iters, opts={"method": method}))
        emit(case="C1", method=method, ms_per_call=ms, iters_per_s=pr.iters / ms * 1e3, prof=prof, launches=nl,
             info=out[2].info)


def case_c2():
    pr = W.c2_mmd()
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)
    for kind, param in pr.kernels:
        for method in ("nfft", "direct"):
            ms, prof, nl, out = timed(lambda: uk.mmd2(x, a, y, b, kind, param, opts={"method": method},
                                                      return_info=True), reps=3)
            emit(case="C2", kind=kind, method=method, ms_per_call=ms, evals_per_s=1e3 / ms, prof=prof, launches=nl,
                 info=out[1], mmd2=out[0])


def case_c4(iters):
    t0 = time.time()
    pr = W.c4_uot(iters=iters)
    gen = time.time() - t0
    args = (cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b), pr.eps, pr.lam)
    ms, prof, nl, out = timed(lambda: uk.uot_sinkhorn(*args, iters=iters, opts={"method": "nfft"}), reps=1)
    ms0, prof0, _, _ = timed(lambda: uk.uot_sinkhorn(*args, iters=0, opts={"method": "nfft"}), reps=1)
    per_it = (ms - ms0) / iters
    emit(case="C4", iters=iters, ms_per_call=ms, ms_zero_iter_call=ms0, ms_per_iter=per_it,
         iters_per_s=1e3 / per_it, prof=prof, launches=nl, info=out[2].info, gen_s=gen)


def case_c5(max_n, dims=(1, 2, 3), min_n=10_000):
    for d in dims:
        for kind in (W.GAUSS, W.IMQ):
            n = min_n
            while n <= max_n:
                pr = W.c5_sum(d, n, kind=kind)
                s, al, t = cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt)
                methods = ["nfft"] + (["direct"] if n <= 1_000_000 else [])
                for method in methods:
                    ms, prof, nl, out = timed(lambda: uk.kernel_sum(s, al, t, kind, pr.param,
                                                                    opts={"method": method}, return_info=True),
                                              reps=3 if method == "nfft" else 1)
                    emit(case="C5", d=d, kind=kind, n=n, method=method, ms_per_call=ms, prof=prof, launches=nl,
                         info=out[1], pts_per_s=2 * n / ms * 1e3)
                del s, al, t, pr
                torch.cuda.empty_cache()
                n *= 10


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cases", default="c1,c2,c4,c5")
    p.add_argument("--c5-max", type=float, default=1e7)
    p.add_argument("--c4-iters", type=int, default=5)
    p.add_argument("--c5-dims", default="1,2,3")
    p.add_argument("--c5-min", type=float, default=1e4)
    a = p.parse_args()
    cases = a.cases.split(",")
    if "c1" in cases:
        case_c1()
    if "c2" in cases:
        case_c2()
    if "c5" in cases:
        case_c5(int(a.c5_max), tuple(int(x) for x in a.c5_dims.split(",")), int(a.c5_min))
    if "c4" in cases:
        case_c4(a.c4_iters)


if __name__ == "__main__":
    main()
