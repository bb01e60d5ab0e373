"""Benchmark of the hot path: UOT Sinkhorn iterations/s (and MMD^2 evals/s) at n=m=1M, d=3, fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C3|C1]

A "step" is one full uot_sinkhorn call on the C3 workload (BASELINE.json configs[2]:
d=3, n=m=1M, 8-component Gaussian mixtures clipped to radius 0.2, masses U(0.1,1),
eps=0.02, lam=0.5, 200 iterations): point scaling, sorting, kernel coefficients and
200 x (two NFFT kernel sums + Sinkhorn updates), then the objective values — every
row of SURVEY.md §8(a).  value = iterations/s of the whole job (all ranks), inputs
resident in HBM.  e2e = the same metric through the C ABI with pinned HOST buffers
(H2D of the inputs and D2H of beta, gamma and the objectives inside the timed region).

Multi-GPU (torchrun, one rank per GPU): the points are sharded over ranks (contiguous
blocks), every rank spreads its shard and the oversampled Fourier coefficients are
summed with NCCL inside libuotk.so (one all-reduce per kernel sum) — strong scaling.

--impl reference times the CPU fp64 oracle (oracle/, Algorithm 1 with direct sums) on a
bounded sample of the same workload on the host cores and extrapolates to its
iterations/s (the paper's code is not available).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
# FP64 FMA pipe: 148 SMs x 64 DFMA/clk/SM x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS_NOMINAL = 148 * 64 * 2 * 1.965e9 / 1e12
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="C3", choices=["C3", "C1", "C4"])
    p.add_argument("--iters", type=int, default=None, help="override the config's iteration count")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-mmd", action="store_true")
    p.add_argument("--no-c4", action="store_true", help="skip the C4 (d=2, 16M points) side leg")
    p.add_argument("--no-c1", action="store_true", help="skip the C1 (d=2, 1000 points) side leg")
    p.add_argument("--no-m6", action="store_true", help="skip the C3 leg with the m = 6, sigma = 3 window")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ncu", action="store_true", help="short run for ncu launch lists (no side legs)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_problem(name, iters):
    if name == "C3":
        pr = W.c3_uot()
    elif name == "C4":
        pr = W.c4_uot()
    else:
        pr = W.c1_uot()
    if iters is not None:
        pr.iters = iters
    return pr


def shard(arr, world, rank):
    from paper_2306_13618_b200.dist import shard as _shard
    return _shard(arr, world, rank)


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [v for v in sm if v > 300] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- reference arm / cpu baseline
def oracle_sample(pr, n_targets, seed=0):
    """Time the oracle's direct kernel sum (Algorithm 1's mat-vec, Eq. 3.3) for a
    sample of targets against ALL sources; extrapolate to one Sinkhorn iteration
    (two kernel sums over n + m targets — direct cost is linear in the targets)."""
    import oracle
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(pr.x), n_targets, replace=False)
    w = pr.b * np.ones(len(pr.b))
    t0 = time.perf_counter()
    oracle.kernel_sum_direct(pr.y, w, pr.x[idx], W.GAUSS, pr.eps)
    dt = time.perf_counter() - t0
    per_iter = dt * (len(pr.x) + len(pr.y)) / n_targets
    return dt, per_iter


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    pr = make_problem(args.workload, args.iters)
    n_t = 200 if args.workload == "C3" else 1000
    times = []
    for _ in range(args.warmup):
        oracle_sample(pr, min(n_t, 50))
    for _ in range(args.steps):
        dt, per_iter = oracle_sample(pr, n_t)
        times.append(per_iter)
    per_iter = statistics.median(times)
    value = 1.0 / per_iter
    sample = (f"oracle direct kernel sum (numpy fp64) of {n_t} sampled targets x {len(pr.y)} sources per step, "
              f"extrapolated x{(len(pr.x) + len(pr.y)) / n_t:.0f} to one iteration (2 kernel sums)")
    line = {
        "impl": "reference", "metric": "UOT Sinkhorn iterations/s", "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_iter * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(pr),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(pr, extra=None):
    cfg = {"workload": f"{pr.name}: UOT Sinkhorn d={pr.d} n={len(pr.x)} m={len(pr.y)} eps={pr.eps} "
                       f"lam={pr.lam} iters={pr.iters}", "n": len(pr.x), "m": len(pr.y), "d": pr.d,
           "eps": pr.eps, "lam": pr.lam, "iters": pr.iters}
    if extra:
        cfg.update(extra)
    return cfg


# ---------------------------------------------------------------------- our arm
def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2306_13618_b200 as uk

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = uk.Comm.from_torch_distributed()

    def barrier():
        if world > 1:
            dist.barrier()

    pr = make_problem(args.workload, args.iters)
    x, a, y, b = (shard(v, world, rank) for v in (pr.x, pr.a, pr.y, pr.b))
    xd, ad, yd, bd = (torch.from_numpy(v).to(dev) for v in (x, a, y, b))
    opts = {"method": "nfft"}
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def step():
        return uk.uot_sinkhorn(xd, ad, yd, bd, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

    for _ in range(args.warmup):
        beta, gamma, res = step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    uk.reset_launch_counter()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            beta, gamma, res = step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = uk.launch_counter()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    ms_per_step = total_ms / args.steps
    value = pr.iters * args.steps / (total_ms / 1e3)

    out = {}
    if not args.ncu:
        out["roofline"] = roofline_leg(uk, step, pr, res, world)
        if not args.no_e2e:
            out["e2e"] = e2e_leg(uk, pr, x, a, y, b, comm, barrier, world, dev)
        if not args.no_mmd:
            out["mmd2"] = mmd_leg(uk, world, rank, comm, dev, barrier)
        if not args.no_m6 and args.workload == "C3":
            out["c3_m6"] = c3_m6_leg(uk, pr, xd, ad, yd, bd, comm, barrier, world, dev, res)
        if not args.no_c4 and args.workload == "C3":
            out["c4"] = c4_leg(uk, world, rank, comm, dev, barrier)
        if not args.no_c1 and args.workload == "C3" and world == 1:
            out["c1"] = c1_leg(uk, dev)
    if rank == 0:
        line = {
            "metric": "UOT Sinkhorn iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gaussian mixtures, BASELINE.json configs[2])",
            "config": workload_config(pr, {"method": res.info["method"], "N": res.info["N"],
                                           "n_grid": res.info["n_grid"], "window_m": res.info["m"],
                                           "h": res.info["h"], "parallelism": f"points sharded x{world}",
                                           "l2": "flushed between steps (256 MB write outside the events)"}),
            "gpu_launches": launches,
            "step_ms": [round(v, 3) for v in step_ms],
            "clocks": clk.summary(),
            "result": {"primal": res.primal, "dual": res.dual, "plan_mass": res.plan_mass,
                       "max_dbeta": res.max_dbeta, "max_dgamma": res.max_dgamma},
        }
        line.update({k: v for k, v in out.items() if v is not None})
        if not args.ncu and not args.no_cpu_baseline and world == 1:
            dt, per_iter = oracle_sample(pr, 200 if args.workload == "C3" else 1000)
            line["cpu_baseline"] = {
                "value": 1.0 / per_iter, "unit": "iterations/s", "cores": 1, "kind": "oracle",
                "sample": f"oracle direct kernel sum of 200 sampled targets x {len(pr.y)} sources "
                          f"({dt:.1f} s), extrapolated linearly to one iteration (2 sums over n+m targets)"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            j = json.load(f)
        return float(j["tflops"]), (f"measured FP64 peak, max of DMMA {j.get('dmma_tflops')} and DFMA "
                                    f"{j.get('dfma_tflops')} TFLOP/s microbenchmarks (profiles/fp64_peak.json)")
    except (OSError, ValueError, KeyError):
        return FP64_PEAK_TFLOPS_NOMINAL, "nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"


def roofline_leg(uk, step, pr, res, world):
    """Average duration of the dominant kernel measured live with CUDA events on its
    stream over one profiled step; algorithmic FLOPs per launch = points x (2m)^d x 2
    (one FMA per window tap) per spread or gather pass."""
    import torch
    uk.profile_reset()
    uk.profile_enable(True)
    step()
    torch.cuda.synchronize()
    prof = uk.profile_read()
    uk.profile_enable(False)
    uk.profile_reset()
    taps = (2 * res.info["m"]) ** pr.d
    n_local = len(pr.x) // world
    kern = max(("fused", "spread", "gather"), key=lambda k: prof[k][0])
    ms, cnt = prof[kern]
    passes = 2 if kern == "fused" else 1
    flops = n_local * taps * 2 * passes
    avg_ms = ms / max(cnt, 1)
    achieved = flops / (avg_ms / 1e3) / 1e12
    peak, peak_src = fp64_peak()
    total = sum(v[0] for v in prof.values())
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            traffic = json.load(f).get(kern)
    except (OSError, ValueError):
        pass
    if pr.d <= 2:  # d <= 2 cell-group kernels stream precomputed windows: HBM-bound
        nb = n_local * (pr.d * 2 * res.info["m"] * 8 + 32)
        gbs = nb / (avg_ms / 1e3) / 1e9
        return {"bound": "hbm", "kernel": kern, "achieved": gbs, "peak": hbm_peak(), "unit": "GB/s",
                "frac": gbs / hbm_peak(), "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "avg_launch_ms": avg_ms, "launches_per_step": cnt, "share_of_step": ms / total if total else None,
                "per_tag_ms": {k: round(v[0], 3) for k, v in prof.items()}}
    return {"bound": "alu", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src + " (FP64 FMA pipe)",
            "avg_launch_ms": avg_ms, "launches_per_step": cnt, "share_of_step": ms / total if total else None,
            "per_tag_ms": {k: round(v[0], 3) for k, v in prof.items()}}


def e2e_leg(uk, pr, x, a, y, b, comm, barrier, world, dev):
    import torch
    hx, ha, hy, hb = (torch.from_numpy(v).pin_memory() for v in (x, a, y, b))
    opts = {"method": "nfft"}
    stream = torch.cuda.current_stream()
    uk.uot_sinkhorn(hx, ha, hy, hb, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm, stream=stream)
    steps = 2
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        beta, gamma, res = uk.uot_sinkhorn(hx, ha, hy, hb, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm,
                                           stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    h2d = sum(v.numel() * 8 for v in (hx, ha, hy, hb))
    d2h = (len(a) + len(b)) * 8 + 8 * 7
    return {"value": pr.iters * steps / (ms / 1e3), "unit": "iterations/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "path": "uotk_uot_sinkhorn with pinned host buffers (library stages copies)"}


def mmd_leg(uk, world, rank, comm, dev, barrier):
    """MMD^2 evals/s at n=m=1M, d=3 (C2 distributions at the metric's size, Gaussian l=0.05)."""
    import torch
    pr = W.c2_mmd(n=1_000_000)
    x, a, y, b = (torch.from_numpy(shard(v, world, rank)).to(dev) for v in (pr.x, pr.a, pr.y, pr.b))
    kind, param = pr.kernels[0]
    opts = {"method": "nfft"}
    uk.release_caches()  # start from the library state a fresh process has (no C3 buffers cached)
    for _ in range(3):
        v = uk.mmd2(x, a, y, b, kind, param, opts=opts, comm=comm)
    steps = 10
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        v = uk.mmd2(x, a, y, b, kind, param, opts=opts, comm=comm)  # returns a host scalar (synchronises)
    dt = time.perf_counter() - t0
    # cold: every cache released first, so the call also rebuilds the
    # Fourier tables, the cuFFT plans and its device buffers
    cold = []
    for _ in range(5):
        uk.release_caches()
        barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        uk.mmd2(x, a, y, b, kind, param, opts=opts, comm=comm)
        cold.append(time.perf_counter() - t1)
    cold_s = statistics.median(cold)
    # C2's second kernel, the inverse multiquadric (c = 0.05: grid 384^3, pruned transform)
    kind2, param2 = pr.kernels[1]
    for _ in range(2):
        v2 = uk.mmd2(x, a, y, b, kind2, param2, opts=opts, comm=comm)
    barrier()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(steps):
        v2 = uk.mmd2(x, a, y, b, kind2, param2, opts=opts, comm=comm)
    dt2 = time.perf_counter() - t2
    return {"metric": "MMD^2 evals/s", "value": steps / dt, "unit": "evals/s", "mmd2": v,
            "imq": {"value": steps / dt2, "unit": "evals/s", "mmd2": v2,
                    "config": "same points, inverse multiquadric (r^2 + 0.05^2)^(-1/2)"},
            "config": "C2 distributions at n=m=1M, d=3, Gaussian exp(-r^2/0.0025), full call incl. sort and "
                      "window blocks (warm: Fourier tables and plans cached)",
            "cold": {"value": 1.0 / cold_s, "unit": "evals/s", "ms_per_eval": cold_s * 1e3,
                     "what": "uotk_release_caches() before each call: tables, cuFFT plans, buffers rebuilt"}}


def c3_m6_leg(uk, pr, xd, ad, yd, bd, comm, barrier, world, dev, res8):
    """C3 with the window m = 6, sigma = 3 (opts; the headline uses the paper's m = 8,
    sigma = 2): Kaiser-Bessel error bound 4e-12 against 4e-14, 12^3 instead of 16^3 taps per
    point (fused3d_m6.cu).  Whole solves (median of 3, setup included, inputs in HBM), the
    fused kernel against the FP64 roofline with algorithmic flops 2 x 12^3 x 2 per point, and
    the objective values against the m = 8 solve of the headline."""
    import torch
    opts = {"method": "nfft", "m": 6, "sigma": 3.0}
    stream = torch.cuda.current_stream()

    def solve():
        return uk.uot_sinkhorn(xd, ad, yd, bd, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

    for _ in range(2):
        solve()
    barrier()
    torch.cuda.synchronize()
    per = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, res = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
    barrier()
    ms = statistics.median(per)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    uk.profile_reset()
    uk.profile_enable(True)
    solve()
    torch.cuda.synchronize()
    prof = uk.profile_read()
    uk.profile_enable(False)
    uk.profile_reset()
    fms, fcnt = prof["fused"]
    roof = None
    if fcnt:
        avg = fms / fcnt
        flops = len(pr.x) // world * 12 ** 3 * 2 * 2
        achieved = flops / (avg / 1e3) / 1e12
        peak, peak_src = fp64_peak()
        roof = {"bound": "alu", "kernel": "sinkhorn3d_m6_ws_k", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "avg_launch_ms": avg, "launches_per_solve": fcnt,
                "share_of_solve": fms / sum(v[0] for v in prof.values()), "peak_source": peak_src}
    return {"metric": "UOT Sinkhorn iterations/s", "value": pr.iters / (ms / 1e3), "unit": "iterations/s",
            "ms_per_solve": ms, "solve_ms": [round(v, 2) for v in per],
            "config": "C3 as the headline with opts m=6, sigma=3 (N and h unchanged, grid "
                      f"{res.info['n_grid']}^3); median of 3 whole solves incl. setup",
            "primal": res.primal, "primal_rel_diff_vs_m8": abs(res.primal - res8.primal) / abs(res8.primal),
            "dual_rel_diff_vs_m8": abs(res.dual - res8.dual) / abs(res8.dual), "roofline": roof}


def c4_leg(uk, world, rank, comm, dev, barrier):
    """C4 (BASELINE.json configs[3]): UOT d=2, n=m=16M uniform in the ball of radius 0.2,
    eps=0.002, lam=2, 50 iterations — whole solves (setup included), device-timed, inputs
    resident in HBM; and the d=2 fused half-step kernel against the HBM roofline
    (algorithmic bytes per point: 2 x 16 window values + mass + potential read, potential
    and next weight written = 288 B)."""
    import torch
    pr = W.c4_uot()
    x, a, y, b = (torch.from_numpy(shard(v, world, rank)).to(dev) for v in (pr.x, pr.a, pr.y, pr.b))
    opts = {"method": "nfft"}
    stream = torch.cuda.current_stream()

    def solve():
        return uk.uot_sinkhorn(x, a, y, b, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

    for _ in range(2):
        solve()
    steps = 3
    barrier()
    torch.cuda.synchronize()
    per = []
    for _ in range(steps):  # median of whole solves: robust to one-off host stalls
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, res = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
    barrier()
    ms = statistics.median(per) * steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    uk.profile_reset()
    uk.profile_enable(True)
    solve()
    torch.cuda.synchronize()
    prof = uk.profile_read()
    uk.profile_enable(False)
    uk.profile_reset()
    fms, fcnt = prof["fused"]
    roof = None
    if fcnt:
        avg = fms / fcnt
        per_launch_bytes = (len(x) + len(y)) / 2 * 288  # one half-step visits one point set
        achieved = per_launch_bytes / (avg / 1e3) / 1e9
        peak = hbm_peak()
        traffic = None
        try:
            with open(TRAFFIC_FILE) as f:
                traffic = json.load(f).get("fused2d")
        except (OSError, ValueError):
            pass
        roof = {"bound": "hbm", "kernel": "sinkhorn2d_ws_k (fused d=2 half-step)", "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "avg_launch_ms": avg,
                "launches_per_solve": fcnt, "share_of_solve": fms / sum(v[0] for v in prof.values())}
    return {"metric": "UOT Sinkhorn iterations/s", "value": pr.iters * steps / (ms / 1e3), "unit": "iterations/s",
            "ms_per_solve": ms / steps, "solve_ms": [round(v, 2) for v in per],
            "config": f"C4: UOT d=2 n=m={len(pr.x)} eps={pr.eps} lam={pr.lam} "
            f"iters={pr.iters} (median of 3 whole solves incl. setup, inputs in HBM)",
            "n_grid": res.info["n_grid"], "N": res.info["N"], "plan_mass": res.plan_mass, "roofline": roof}


def c1_leg(uk, dev):
    """C1 (BASELINE.json configs[0]): UOT d=2, n=m=1000, eps=0.05, lam=1, 100 iterations —
    whole solves, device-timed (median of 5), with the AUTO choice (the direct kernel at
    1e6 pairs per sum) and with the NFFT path; both replay the iteration from CUDA graphs."""
    import torch
    pr = W.c1_uot()
    args = [torch.from_numpy(v).to(dev) for v in (pr.x, pr.a, pr.y, pr.b)]
    stream = torch.cuda.current_stream()
    out = {"metric": "UOT Sinkhorn iterations/s", "unit": "iterations/s",
           "config": f"C1: UOT d=2 n=m={len(pr.x)} eps={pr.eps} lam={pr.lam} iters={pr.iters} (whole solves)"}
    for method in ("auto", "nfft"):
        def solve():
            return uk.uot_sinkhorn(*args, pr.eps, pr.lam, iters=pr.iters, opts={"method": method})
        for _ in range(3):
            solve()
        torch.cuda.synchronize()
        per = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, _, res = solve()
            e1.record(stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
        ms = statistics.median(per)
        out[method] = {"value": pr.iters / (ms / 1e3), "ms_per_solve": ms, "method_used": res.info["method"]}
    return out


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6550.7


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    main_ours(args)


if __name__ == "__main__":
    main()
