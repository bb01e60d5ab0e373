"""Accuracy of the Laplace / energy fast sums (reading R24): max error relative to
max|K| * sum|alpha| against the oracle, and per-entry relative error with positive
weights, over d = 1..3, kernel widths and (N, p).  Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


for d in (1, 2, 3):
    for kind, param in ((3, 0.05), (3, 0.2), (3, 0.5), (4, 1.0)):
        for N, p in ((0, 0), (128, 12), (256, 10), (256, 12), (256, 14)):
            if d == 3 and N == 0:
                pass
            pr = W.random_sum(d, 6000, 3000, kind=kind, param=param, seed=d, signed=False)
            ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, kind, param)
            opts = {"method": "nfft"}
            if N:
                opts.update(N=N, p=p)
            got, info = uk.kernel_sum(t(pr.src), t(pr.alpha), t(pr.tgt), kind, param, opts=opts, return_info=True)
            g = got.cpu().numpy()
            kmax = 1.0 if kind == 3 else 0.4
            e_abs = float(np.max(np.abs(g - ref)) / (kmax * pr.alpha.sum()))
            e_rel = float(np.max(np.abs(g - ref) / np.abs(ref)))
            print(json.dumps({"d": d, "kind": kind, "param": param, "N": info["N"], "p": p or 12, "h": info["h"],
                              "err_abs_norm": e_abs, "err_rel_entry": e_rel}), flush=True)
