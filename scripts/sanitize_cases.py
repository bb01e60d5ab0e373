"""Small cases that launch every mbarrier / TMA-ring / warp-specialised kernel of
libuotk.so once or twice, for compute-sanitizer (racecheck, synccheck, memcheck — one
tool per gpurun call):

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py

Each case is checked against the CPU oracle as well (a sanitizer run must also be a
correct run).  Sizes are tiny: the tools instrument every shared-memory access.
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2306_13618_b200 as uk  # noqa: E402
import workloads as W  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def uot(name, pr, opts, iters=2, expect_groups=None):
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters)
    beta, gamma, res = uk.uot_sinkhorn(t(pr.x), t(pr.a), t(pr.y), t(pr.b), pr.eps, pr.lam, iters=iters,
                                       opts=dict({"method": "nfft"}, **opts))
    torch.cuda.synchronize()
    err = float(np.max(np.abs(beta.cpu().numpy() - ref.beta)) / np.max(np.abs(ref.beta)))
    assert err < 1e-8, (name, err)
    if expect_groups is not None:
        assert res.info["groups"] == expect_groups, (name, res.info)
    print(f"{name}: ok (groups {res.info['groups']}, err {err:.1e})", flush=True)


def ksum(name, d, n, kind, param, opts, radius=0.2, expect=None):
    pr = W.random_sum(d, n, n - 7, kind=kind, param=param, seed=n, radius=radius)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    got, info = uk.kernel_sum(t(pr.src), t(pr.alpha), t(pr.tgt), kind, param, opts=dict(opts, method="nfft"),
                              return_info=True)
    err = float(np.max(np.abs(got.cpu().numpy() - ref) / np.abs(ref)))
    assert err < 1e-9, (name, err)
    if expect is not None:
        assert info["groups"] == expect, (name, info)
    print(f"{name}: ok (groups {info['groups']}, err {err:.1e})", flush=True)


def main():
    torch.cuda.set_device(0)
    CH = {"flags": uk.FLAG_CHUNKED}
    # d = 3 half-steps: warp-specialised (one-cell groups, C3 density), phase-locked z-segment
    uot("sinkhorn3d_ws_k", W.c3_dense_uot(n=900, m=700), {}, expect_groups=(16, 16))
    rng = np.random.default_rng(3)
    sparse = W.UOTProblem("sparse", W.uniform_ball(rng, 3000, 3, 0.2), rng.uniform(0.1, 1, 3000),
                          W.uniform_ball(rng, 2500, 3, 0.2), rng.uniform(0.1, 1, 2500), 0.02, 0.5, 2)
    uot("chunked3d_k<0,24>", sparse, CH, expect_groups=(24, 24))
    # m = 6 half-step and stand-alone kernels
    uot("sinkhorn3d_m6_ws_k", W.c3_dense_uot(n=900, m=700), dict(CH, m=6, sigma=3.0))
    # d = 2 and d = 1 half-steps
    uot("sinkhorn2d_ws_k", W.c1_uot(n=800, m=600), CH)
    uot("fused d=1", W.c1_uot(n=800, m=600, d=1), CH)
    # stand-alone spread / gather rings (kernel sums): one-cell, 9-cell and 25-cell segments
    ksum("spread3d_k/gather3d_k, z-segments", 3, 1200, W.GAUSS, 0.02, CH, radius=0.05)
    ksum("spread3d_k/gather3d_k, one-cell groups", 3, 600, W.GAUSS, 0.0025, CH)
    ksum("spread3d_k<40> (IMQ, sparse spread-only)", 3, 20000, W.IMQ, 0.05, {})
    ksum("m6 spread/gather", 3, 700, W.GAUSS, 0.02, dict(CH, m=6, sigma=3.0), radius=0.05)
    ksum("chunked2d", 2, 900, W.IMQ, 0.05, CH)
    ksum("chunked1d", 1, 900, W.GAUSS, 0.0025, CH)
    # MMD^2 (spread + pruned transform + energy) and the direct kernels
    m = W.c2_mmd(n=700, m=600)
    v = uk.mmd2(t(m.x), t(m.a), t(m.y), t(m.b), "gauss", 0.0025, opts={"method": "nfft", "flags": uk.FLAG_CHUNKED})
    ref = oracle.mmd2_direct(m.x, m.a, m.y, m.b, W.GAUSS, 0.0025)
    print(f"mmd2: {v:.6e} vs {ref:.6e}", flush=True)
    # late round 2: spread3d_fly_k (windows evaluated in the spread) on one-cell and on
    # hybrid groups (dense cells alone, sparse cells in 9-cell z-segments)
    h = W.c2_dense_mmd(n=10000)
    v, info = uk.mmd2(t(h.x), t(h.a), t(h.y), t(h.b), "gauss", 0.0025, opts={"method": "nfft"}, return_info=True)
    assert info["groups"][0] == 1624, info
    ref = oracle.mmd2_direct(h.x, h.a, h.y, h.b, W.GAUSS, 0.0025)
    assert abs(v - ref) <= 1e-8 * max(abs(ref), 1e-12), (v, ref)
    print(f"spread3d_fly_k<hybrid> (mmd2): {v:.6e} vs {ref:.6e}", flush=True)
    f = W.c3_dense_uot(n=20000, m=1001)
    got, info = uk.kernel_sum(t(f.x), t(f.a), t(f.y), "gauss", 0.02, opts={"method": "nfft"}, return_info=True)
    assert info["groups"][0] == 16, info
    ref = oracle.kernel_sum_direct(f.x, f.a, f.y, W.GAUSS, 0.02)
    err = float(np.max(np.abs(got.cpu().numpy() - ref) / np.abs(ref)))
    assert err < 1e-9, err
    print(f"spread3d_fly_k<one-cell> (kernel sum): ok (err {err:.1e})", flush=True)
    uot("direct", W.c1_uot(n=300, m=200), {"method": "direct"})
    uot("deterministic (pull spread)", W.c3_dense_uot(n=900, m=700), {"deterministic": 1})
    print("SANITIZE_CASES_DONE", flush=True)


if __name__ == "__main__":
    main()
