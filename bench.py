"""Benchmark of the hot path: UOT Sinkhorn iterations/s (and MMD^2 evals/s) at n=m=1M, d=3, fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C3|C1|C4]

A "step" is one full uot_sinkhorn call on the C3 workload (BASELINE.json configs[2]:
d=3, n=m=1M, 8-component Gaussian mixtures clipped to radius 0.2, masses U(0.1,1),
eps=0.02, lam=0.5, 200 iterations): point scaling, sorting, kernel coefficients and
200 x (two NFFT kernel sums + Sinkhorn updates), then the objective values — every
row of SURVEY.md §8(a).  value = iterations/s of the whole job (all ranks), inputs
resident in HBM.  e2e = the same metric through the C ABI with pinned HOST buffers
(H2D of the inputs and D2H of beta, gamma and the objectives inside the timed region).

Side legs (one JSON line; each with its own roofline and CPU-oracle baseline):
  mmd2  MMD^2 evals/s at n=m=1M (the metric's second half), warm / cold / IMQ
  c2    configs[1]: MMD^2 at n=m=1e5, Gaussian and IMQ
  c3_m6 C3 with the opt-in m=6, sigma=3 window
  c4    configs[3]: d=2, n=m=16M, automatic grid (160^2) and the literal 4096^2 grid
  c1    configs[0]: d=2, n=m=1000, AUTO (direct kernel) and NFFT
  c5    configs[4]: kernel sums d=1..3, n=m=1e6 / 1e7, Gaussian and IMQ

Multi-GPU (torchrun, one rank per GPU): the points are sorted by a coarse global cell
order and sharded in contiguous blocks (spatially compact shards), every rank spreads
its shard and the truncated Fourier coefficients are summed with NCCL inside
libuotk.so (one all-reduce per kernel sum) — strong scaling (total n fixed).

CPU baseline (rank 0 at N=1; --impl reference): the CPU fp64 oracle (oracle/, the direct
sums of Algorithm 1 / Eq. 3.5) run as it stands, in one process per host core on a
bounded sample of targets against ALL sources of the leg's workload; the pair rate is
converted to the leg's metric (direct cost is exactly linear in the targets).  The
CPU baselines run BEFORE the GPU is initialised (the worker processes are forked).
"""

import argparse
import json
import os
import statistics
import subprocess
import threading
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
# algorithmic FP64 flops per direct kernel pair: d differences, d products,
# d-1 additions, ~20 for exp (range reduction + degree-11 polynomial) or 8 for rsqrt+Newton
# (IMQ), and the multiply-add with the weight
DIRECT_FLOPS_PER_PAIR = {(d, k): 3 * d + 1 + (20 if k == W.GAUSS else 8) for d in (1, 2, 3) for k in (0, 1)}

# The paper's CPU timings (Intel i7-7700, Julia + NFFT3.jl) — context only
PAPER_CONTEXT = {
    "hardware": "Intel Core i7-7700 (4 cores / 8 threads), 15 GB RAM; Julia + NFFT3.jl (P:675, P:693-695)",
    "note": "different workload (U[0,1]^d points, l=1/2, c=1, unstated iteration counts): context, not a target",
    "table2_uot_nfft_s": {"d3_n1e6": 419.27, "d3_n1e5": 202.17, "d2_n1e6": 77.24, "d2_n1e3": 0.72},
    "table5_mmd_nfft_s": {"gauss_d3_n1e6": 34.96, "gauss_d3_n1e5": 17.20, "imq_d3_n1e6": 32.63,
                          "imq_d3_n1e5": 28.10},
}


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
    p.add_argument("--no-c2", action="store_true")
    p.add_argument("--no-c4", action="store_true", help="skip the C4 (d=2, 16M points) side leg")
    p.add_argument("--no-c1", action="store_true", help="skip the C1 (d=2, 1000 points) side leg")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 kernel-sum legs")
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


def cell_order(*point_sets, cells=64):
    """Permutations sorting each point set by a coarse global cell order (lexicographic on a
    cells^d grid over the common bounding box): contiguous blocks of the sorted sets are
    spatially compact shards."""
    allp = np.vstack(point_sets)
    lo, hi = allp.min(0), allp.max(0)
    scale = cells / np.maximum(hi - lo, 1e-300)
    out = []
    for p in point_sets:
        c = np.minimum(((p - lo) * scale).astype(np.int64), cells - 1)
        key = np.zeros(len(p), dtype=np.int64)
        for t in range(p.shape[1]):
            key = key * cells + c[:, t]
        out.append(np.argsort(key, kind="stable"))
    return out


def shard(arr, world, rank):
    from paper_2306_13618_b200.dist import shard as _shard
    return _shard(arr, world, rank)


def shard_problem(pr, world, rank):
    """x, a, y, b of this rank (cell-ordered contiguous blocks when world > 1)."""
    x, a, y, b = pr.x, pr.a, pr.y, pr.b
    if world > 1:
        ox, oy = cell_order(x, y)
        x, a, y, b = x[ox], a[ox], y[oy], b[oy]
    return tuple(shard(v, world, rank) for v in (x, a, y, b))


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        # nvidia-smi is started and has produced its first sample BEFORE the caller's timed
        # region begins (its start-up — NVML initialisation, a process spawn — otherwise
        # lands in the first timed step); samples are taken every 200 ms throughout, and
        # summary() keeps those from start() on
        self.lines, self.t_start = [], None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def reader():
            for ln in self.proc.stdout:
                if ln.strip():
                    self.lines.append((time.perf_counter(), ln))

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
            time.sleep(0.01)
        return self

    def start(self):
        self.t_start = time.perf_counter()

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)  # one more sample after the timed region's last kernels
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)
        t = self.t_start or 0.0
        timed = [ln for ts, ln in self.lines if ts >= t]
        self.lines = timed or [ln for _, ln in self.lines[-1:]]

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


# ---------------------------------------------------------------------- CPU oracle (all host cores)
_G = {}


def _oracle_chunk(idx):
    import oracle
    g = _G
    t0 = time.perf_counter()
    oracle.kernel_sum_direct(g["src"], g["w"], g["tgt"][idx], g["kind"], g["param"])
    return time.perf_counter() - t0


def oracle_pair_rate(src, w, tgt, kind, param, per_core=None, budget_s=4.0, seed=0):
    """Pairs/s of the oracle's direct kernel sum (Eq. 4.3 / the mat-vec of Algorithm 1 and
    of (3.5)) on all host cores: one forked process per core, each summing over ALL
    sources for its own sampled targets.  The sample is sized from a one-target probe so
    the whole measurement takes about `budget_s` seconds of wall time.  Returns
    (pairs_per_s, cores, n_targets, wall_s)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    # each worker holds the oracle's block temporaries (>= 128 MB, or one target's n_src x d
    # differences): cap the workers at half the available memory
    try:
        import psutil
        avail = psutil.virtual_memory().available
        per_proc = 3.0 * max(1 << 27, 8 * len(src) * np.asarray(src).reshape(len(src), -1).shape[1])
        cores = max(1, min(cores, int(0.5 * avail / per_proc)))
    except Exception:  # noqa: BLE001
        pass
    _G.update(src=src, w=w, tgt=tgt, kind=kind, param=param)
    rng = np.random.default_rng(seed)
    probe = rng.choice(len(tgt), min(4, len(tgt)), replace=False)
    t_probe = _oracle_chunk(probe) / len(probe)
    if per_core is None:
        per_core = int(max(1, min(2000, budget_s / max(t_probe, 1e-9))))
    n_t = min(len(tgt), per_core * cores)
    idx = rng.choice(len(tgt), n_t, replace=False)
    chunks = [c for c in np.array_split(idx, cores) if len(c)]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(chunks)) as pool:
        t0 = time.perf_counter()
        pool.map(_oracle_chunk, chunks)
        wall = time.perf_counter() - t0
    return n_t * len(src) / wall, len(chunks), n_t, wall


def cpu_baseline(rate, pairs_per_unit, unit, what, cores, n_t, n_src, wall):
    return {"value": rate / pairs_per_unit, "unit": unit, "cores": cores, "kind": "oracle",
            "sample": f"{what}: oracle direct kernel sum (numpy fp64, one process per core) of {n_t} sampled "
                      f"targets x {n_src} sources in {wall:.1f} s wall = {rate:.3g} pairs/s, extrapolated linearly "
                      f"to {pairs_per_unit:.3g} pairs per {unit.split('/')[0][:-1]}"}


def run_cpu_baselines(args, pr):
    """All CPU-oracle baselines of the line (before the GPU is touched)."""
    out = {}
    n, m = len(pr.x), len(pr.y)
    rate, cores, n_t, wall = oracle_pair_rate(pr.y, pr.b, pr.x, W.GAUSS, pr.eps)
    out["main"] = cpu_baseline(rate, 2.0 * n * m, "iterations/s", f"{pr.name} beta-step sum", cores, n_t, m, wall)
    if args.ncu:
        return out
    if not args.no_mmd:
        mp_ = W.c2_mmd(n=1_000_000)
        z = np.vstack([mp_.x, mp_.y])
        wz = np.concatenate([mp_.a, -mp_.b])
        rate, cores, n_t, wall = oracle_pair_rate(z, wz, z, W.GAUSS, 0.0025)
        out["mmd2"] = cpu_baseline(rate, float(len(z)) ** 2, "evals/s", "MMD^2 1M (z = x u y, Gaussian)", cores, n_t,
                                   len(z), wall)
    if not args.no_c2:
        c2 = W.c2_mmd()
        z = np.vstack([c2.x, c2.y])
        wz = np.concatenate([c2.a, -c2.b])
        for kind, param in c2.kernels:
            rate, cores, n_t, wall = oracle_pair_rate(z, wz, z, kind, param, budget_s=3.0)
            out[f"c2_{kind}"] = cpu_baseline(rate, float(len(z)) ** 2, "evals/s", f"C2 MMD^2 kind {kind}", cores, n_t,
                                             len(z), wall)
    if not args.no_c4:
        c4 = W.c4_uot()
        rate, cores, n_t, wall = oracle_pair_rate(c4.y, c4.b, c4.x, W.GAUSS, c4.eps, budget_s=3.0)
        out["c4"] = cpu_baseline(rate, 2.0 * len(c4.x) * len(c4.y), "iterations/s", "C4 beta-step sum", cores, n_t,
                                 len(c4.y), wall)
    if not args.no_c1:
        import oracle
        c1 = W.c1_uot()
        t0 = time.perf_counter()
        oracle.uot_sinkhorn_direct(c1.x, c1.a, c1.y, c1.b, c1.eps, c1.lam, c1.lam, c1.iters)
        dt = time.perf_counter() - t0
        out["c1"] = {"value": c1.iters / dt, "unit": "iterations/s", "cores": 1, "kind": "oracle",
                     "sample": f"the full C1 solve (oracle.uot_sinkhorn_direct, {c1.iters} iterations, 2e8 pair "
                               f"evaluations) in {dt:.2f} s on one core — not extrapolated"}
    if not args.no_c5:
        # the oracle's pair rate per (d, kernel) on the 1e6-point C5 sets (all sources), applied
        # to every C5 size of that (d, kernel): direct cost is n_src x n_tgt pairs
        for d, kind in sorted({(d, k) for d, _, k in C5_CASES}):
            c5 = W.c5_sum(d, 1_000_000, kind=kind)
            rate, cores, n_t, wall = oracle_pair_rate(c5.src, c5.alpha, c5.tgt, kind, c5.param, budget_s=2.0)
            for dd, n5, kk in C5_CASES:
                if (dd, kk) == (d, kind):
                    out[f"c5_{d}_{n5}_{kind}"] = cpu_baseline(rate, float(n5) * n5, "sums/s",
                                                              f"C5 d={d} n=1e6 sample, kind {kind}", cores, n_t,
                                                              len(c5.src), wall)
    return out


def run_reference(args):
    """--impl reference: the CPU oracle on all host cores, the headline's metric and config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    pr = make_problem(args.workload, args.iters)
    per = []
    for _ in range(args.warmup):
        oracle_pair_rate(pr.y, pr.b, pr.x, W.GAUSS, pr.eps, per_core=2)
    for _ in range(args.steps):
        rate, cores, n_t, wall = oracle_pair_rate(pr.y, pr.b, pr.x, W.GAUSS, pr.eps, budget_s=6.0)
        per.append((rate, cores, n_t, wall))
    rate = statistics.median(r[0] for r in per)
    _, cores, n_t, wall = per[-1]
    value = rate / (2.0 * len(pr.x) * len(pr.y))
    cb = cpu_baseline(rate, 2.0 * len(pr.x) * len(pr.y), "iterations/s", f"{pr.name} beta-step sum", cores, n_t,
                      len(pr.y), wall)
    line = {
        "impl": "reference", "metric": "UOT Sinkhorn iterations/s", "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(pr), "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)


def workload_config(pr, extra=None):
    cfg = {"workload": f"{pr.name}: UOT Sinkhorn d={pr.d} n={len(pr.x)} m={len(pr.y)} eps={pr.eps} "
                       f"lam={pr.lam} iters={pr.iters}", "n": len(pr.x), "m": len(pr.y), "d": pr.d,
           "eps": pr.eps, "lam": pr.lam, "iters": pr.iters}
    if extra:
        cfg.update(extra)
    return cfg


# ---------------------------------------------------------------------- rooflines
def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            j = json.load(f)
        return float(j["tflops"]), (f"measured FP64 peak, max of DMMA {j.get('dmma_tflops')} and DFMA "
                                    f"{j.get('dfma_tflops')} TFLOP/s microbenchmarks (profiles/fp64_peak.json)")
    except (OSError, ValueError, KeyError):
        return FP64_PEAK_TFLOPS_NOMINAL, "nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6550.7


def traffic_of(key):
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f).get(key)
    except (OSError, ValueError):
        return None


def profiled(uk, fn):
    """Run fn once with live per-launch CUDA-event timing; {tag: (ms, launches)}."""
    import torch
    uk.profile_reset()
    uk.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    prof = uk.profile_read()
    uk.profile_enable(False)
    uk.profile_reset()
    return prof


def pass_roofline(prof, d, m, n_spread, n_gather, kind_name="", fused=False, traffic_key=None):
    """Roofline of the dominant NFFT pass of a profiled call.  d = 3: FP64 datapath, algorithmic
    flops = points x (2m)^3 taps x 2 per spread or gather (window values precomputed);
    d <= 2: HBM, algorithmic bytes = points x (d x 2m window values + weight or result) x 8."""
    tags = ("fused",) if fused else ("spread", "gather")
    kern = max(tags, key=lambda k: prof[k][0])
    ms, cnt = prof[kern]
    if not cnt:
        return None
    avg = ms / cnt
    total = sum(v[0] for v in prof.values())
    npts = {"spread": n_spread, "gather": n_gather, "fused": n_spread}[kern]
    passes = 2 if kern == "fused" else 1
    base = {"kernel": f"{kern}{kind_name}", "avg_launch_ms": avg, "launches": cnt,
            "share_of_call": ms / total if total else None, "traffic": traffic_of(traffic_key) if traffic_key else None,
            "per_tag_ms": {k: round(v[0], 4) for k, v in prof.items() if v[1]}}
    if d == 3:
        flops = npts * (2 * m) ** 3 * 2 * passes
        peak, src = fp64_peak()
        ach = flops / (avg / 1e3) / 1e12
        return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": src, "per_unit": f"{(2 * m) ** 3 * 2 * passes} flop per point", **base}
    bpp = (d * 2 * m + 1) * 8 * passes + (16 if kern == "fused" else 0)
    gbs = npts * bpp / (avg / 1e3) / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": hbm_peak(), "unit": "GB/s", "frac": gbs / hbm_peak(),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs", "per_unit": f"{bpp} B per point", **base}


def direct_roofline(prof, d, kind, pairs_per_launch):
    ms, cnt = prof["direct"]
    if not cnt:
        return None
    avg = ms / cnt
    fl = DIRECT_FLOPS_PER_PAIR[(d, kind)]
    ach = pairs_per_launch * fl / (avg / 1e3) / 1e12
    peak, src = fp64_peak()
    return {"bound": "alu", "kernel": "direct", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "peak_source": src, "per_unit": f"{fl} flop per pair", "avg_launch_ms": avg,
            "launches": cnt, "share_of_call": ms / sum(v[0] for v in prof.values())}


# ---------------------------------------------------------------------- our arm
C5_CASES = [(3, 1_000_000, W.GAUSS), (3, 1_000_000, W.IMQ), (3, 10_000_000, W.GAUSS), (3, 10_000_000, W.IMQ),
            (2, 10_000_000, W.GAUSS), (1, 10_000_000, W.GAUSS)]


def main_ours(args):
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    pr = make_problem(args.workload, args.iters)
    # CPU baselines first (rank 0 at N=1 only): forked oracle workers, GPU not yet initialised
    cpu = {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baselines(args, pr)

    import torch
    import torch.distributed as dist

    import paper_2306_13618_b200 as uk

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    # UOTK_BENCH_COMM=1: the NCCL communicator path also at one rank (a check of the
    # multi-GPU code path on a one-GPU box; with UOTK_DIST_CHAIN=2 including the slab chain)
    if world > 1 or os.environ.get("UOTK_BENCH_COMM") == "1":
        os.environ.setdefault("UOTK_COMM_VERBOSE", "1")  # one stderr line per rank: rank / nranks / device
        dist.init_process_group("nccl", device_id=dev)
        comm = uk.Comm.from_torch_distributed()

    def barrier():
        if world > 1:
            dist.barrier()

    x, a, y, b = shard_problem(pr, world, rank)
    xd, ad, yd, bd = (torch.from_numpy(v).to(dev) for v in (x, a, y, b))
    opts = {"method": "nfft"}
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def step():
        return uk.uot_sinkhorn(xd, ad, yd, bd, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

    # the clock sampler runs from before the warm-up (its start-up is not in the timed
    # region, and the GPU does not idle between the warm-up and the timed steps); its
    # summary keeps the samples taken from clk.start() on
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.warmup):
            beta, gamma, res = step()
        torch.cuda.synchronize()

        # ---- timed region: K steps, L2 flushed between steps (outside the events)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        uk.reset_launch_counter()
        barrier()
        torch.cuda.synchronize()
        clk.start()
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
        prof = profiled(uk, step)
        out["roofline"] = pass_roofline(prof, pr.d, res.info["m"], len(x), len(y), fused=True,
                                        traffic_key="fused" if pr.d == 3 else "fused2d")
        if not args.no_e2e:
            out["e2e"] = e2e_leg(uk, pr, x, a, y, b, comm, barrier, world, dev)
        if not args.no_mmd:
            out["mmd2"] = mmd_leg(uk, world, rank, comm, dev, barrier, cpu.get("mmd2"))
        if not args.no_c2:
            out["c2"] = c2_leg(uk, world, rank, comm, dev, barrier, cpu)
        if not args.no_m6 and args.workload == "C3":
            out["c3_m6"] = c3_m6_leg(uk, pr, xd, ad, yd, bd, comm, barrier, world, dev, res)
        if not args.no_c4 and args.workload == "C3":
            out["c4"] = c4_leg(uk, world, rank, comm, dev, barrier, cpu.get("c4"))
        if not args.no_c1 and args.workload == "C3" and world == 1:
            out["c1"] = c1_leg(uk, dev, cpu.get("c1"))
        if not args.no_c5 and args.workload == "C3":
            out["c5"] = c5_legs(uk, world, rank, comm, dev, barrier, cpu)
    if rank == 0:
        line = {
            "metric": "UOT Sinkhorn iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gaussian mixtures, BASELINE.json configs[2])",
            "config": workload_config(pr, {"method": res.info["method"], "N": res.info["N"],
                                           "n_grid": res.info["n_grid"], "window_m": res.info["m"],
                                           "h": res.info["h"], "groups": res.info["groups"],
                                           "parallelism": f"points sharded x{world} (cell-ordered blocks)",
                                           "comm": {"nranks": res.info["nranks"],
                                                    "backend": "nccl" if comm is not None else None},
                                           "l2": "flushed between steps (256 MB write outside the events)"}),
            "gpu_launches": launches,
            "step_ms": [round(v, 3) for v in step_ms],
            "clocks": clk.summary(),
            "result": {"primal": res.primal, "dual": res.dual, "plan_mass": res.plan_mass,
                       "max_dbeta": res.max_dbeta, "max_dgamma": res.max_dgamma},
        }
        line.update({k: v for k, v in out.items() if v is not None})
        if "main" in cpu:
            line["cpu_baseline"] = cpu["main"]
        line["paper_context"] = PAPER_CONTEXT
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist.is_initialized():
        dist.destroy_process_group()


def e2e_leg(uk, pr, x, a, y, b, comm, barrier, world, dev):
    import torch
    hx, ha, hy, hb = (torch.from_numpy(v).pin_memory() for v in (x, a, y, b))
    opts = {"method": "nfft"}
    stream = torch.cuda.current_stream()
    steps = 2
    # warm-up in the timed loop's own pattern (each call's outputs alive while the next one
    # allocates), so the pinned host allocator already holds the output blocks it recycles
    for _ in range(steps):
        beta, gamma, res = uk.uot_sinkhorn(hx, ha, hy, hb, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm,
                                           stream=stream)
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


def _timed_calls(fn, steps, barrier):
    """Wall time of `steps` calls that each return a host value (so each synchronises)."""
    import torch
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        v = fn()
    return (time.perf_counter() - t0) / steps, v


def _mmd_roofline(uk, fn, n_z, traffic_key=None):
    """MMD^2 (Fourier-domain form: spread + pruned forward FFT + sum_k D_k |G_k|^2): the
    spread kernel against the FP64 roofline, and its share of the whole call."""
    prof = profiled(uk, fn)
    return pass_roofline(prof, 3, 8, n_z, 0, traffic_key=traffic_key)


def mmd_leg(uk, world, rank, comm, dev, barrier, cpu=None):
    """MMD^2 evals/s at n=m=1M, d=3 (C2 distributions at the metric's size, Gaussian l=0.05)."""
    import torch
    pr = W.c2_mmd(n=1_000_000)
    x, a, y, b = (torch.from_numpy(v).to(dev) for v in shard_problem(pr, world, rank))
    kind, param = pr.kernels[0]
    opts = {"method": "nfft"}
    uk.release_caches()  # start from the library state a fresh process has (no C3 buffers cached)

    def call():
        return uk.mmd2(x, a, y, b, kind, param, opts=opts, comm=comm)

    for _ in range(3):
        call()
    dt, v = _timed_calls(call, 10, barrier)
    roof = _mmd_roofline(uk, call, len(x) + len(y), traffic_key="mmd_spread")
    if roof:
        roof["call_ms"] = dt * 1e3
    # cold: every cache released first, so the call also rebuilds the
    # Fourier tables, the cuFFT plans and its device buffers
    cold = []
    for _ in range(5):
        uk.release_caches()
        barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        call()
        cold.append(time.perf_counter() - t1)
    cold_s = statistics.median(cold)
    # C2's second kernel, the inverse multiquadric (c = 0.05: grid 384^3, pruned transform)
    kind2, param2 = pr.kernels[1]

    def call2():
        return uk.mmd2(x, a, y, b, kind2, param2, opts=opts, comm=comm)

    for _ in range(2):
        call2()
    dt2, v2 = _timed_calls(call2, 10, barrier)
    out = {"metric": "MMD^2 evals/s", "value": 1.0 / dt, "unit": "evals/s", "ms_per_eval": dt * 1e3, "mmd2": v,
           "roofline": roof,
           "imq": {"value": 1.0 / dt2, "unit": "evals/s", "mmd2": v2,
                   "config": "same points, inverse multiquadric (r^2 + 0.05^2)^(-1/2)"},
           "config": "C2 distributions at n=m=1M, d=3, Gaussian exp(-r^2/0.0025), full call incl. sort and "
                     "window blocks (warm: Fourier tables and plans cached)",
           "cold": {"value": 1.0 / cold_s, "unit": "evals/s", "ms_per_eval": cold_s * 1e3,
                    "what": "uotk_release_caches() before each call: tables, cuFFT plans, buffers rebuilt"}}
    if cpu:
        out["cpu_baseline"] = cpu
    return out


def c2_leg(uk, world, rank, comm, dev, barrier, cpu):
    """configs[1]: MMD^2 d=3, n=m=1e5 (2-component mixtures), Gaussian l=0.05 and IMQ c=0.05."""
    pr = W.c2_mmd()
    import torch
    x, a, y, b = (torch.from_numpy(v).to(dev) for v in shard_problem(pr, world, rank))
    out = {"metric": "MMD^2 evals/s", "unit": "evals/s",
           "config": "C2: MMD^2 d=3 n=m=1e5, mixtures +-0.05 e1 (sigma 0.03), nu shifted 0.02 e2; full calls"}
    for kind, param in pr.kernels:
        def call():
            return uk.mmd2(x, a, y, b, kind, param, opts={"method": "nfft"}, comm=comm)
        for _ in range(3):
            call()
        dt, v = _timed_calls(call, 20, barrier)
        roof = _mmd_roofline(uk, call, len(x) + len(y))
        if roof:
            roof["call_ms"] = dt * 1e3
        leg = {"value": 1.0 / dt, "ms_per_eval": dt * 1e3, "mmd2": v, "roofline": roof}
        if f"c2_{kind}" in cpu:
            leg["cpu_baseline"] = cpu[f"c2_{kind}"]
        out["gauss" if kind == W.GAUSS else "imq"] = leg
    return out


def _solves(uk, solve, barrier, world, dev, reps=3):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(2):
        solve()
    barrier()
    torch.cuda.synchronize()
    per = []
    for _ in range(reps):  # median of whole solves: robust to one-off host stalls
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
    return ms, per, res


def c3_m6_leg(uk, pr, xd, ad, yd, bd, comm, barrier, world, dev, res8):
    """C3 with the window m = 6, sigma = 3 (opts; the headline uses the paper's m = 8,
    sigma = 2): Kaiser-Bessel error bound 4e-12 against 4e-14, 12^3 instead of 16^3 taps per
    point (fused3d_m6.cu).  Whole solves (median of 3, setup included, inputs in HBM), the
    fused kernel against the FP64 roofline with algorithmic flops 2 x 12^3 x 2 per point, and
    the objective values against the m = 8 solve of the headline."""
    opts = {"method": "nfft", "m": 6, "sigma": 3.0}

    def solve():
        return uk.uot_sinkhorn(xd, ad, yd, bd, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

    ms, per, res = _solves(uk, solve, barrier, world, dev)
    roof = pass_roofline(profiled(uk, solve), 3, 6, len(xd), len(yd), fused=True, traffic_key="fused_m6")
    return {"metric": "UOT Sinkhorn iterations/s", "value": pr.iters / (ms / 1e3), "unit": "iterations/s",
            "ms_per_solve": ms, "solve_ms": [round(v, 2) for v in per],
            "config": "C3 as the headline with opts m=6, sigma=3 (N and h unchanged, grid "
                      f"{res.info['n_grid']}^3); median of 3 whole solves incl. setup",
            "primal": res.primal, "primal_rel_diff_vs_m8": abs(res.primal - res8.primal) / abs(res8.primal),
            "dual_rel_diff_vs_m8": abs(res.dual - res8.dual) / abs(res8.dual), "roofline": roof}


def c4_leg(uk, world, rank, comm, dev, barrier, cpu=None):
    """C4 (BASELINE.json configs[3]): UOT d=2, n=m=16M uniform in the ball of radius 0.2,
    eps=0.002, lam=2, 50 iterations — whole solves (setup included), device-timed, inputs
    resident in HBM; with the automatic bandwidth (N=80, grid 160^2, reading R19) and with
    the config's literal "oversampled grid 4096^2" (opts N=2048).  The d=2 fused half-step
    against the HBM roofline (algorithmic bytes per point: 2 x 16 window values + mass +
    potential read, potential and next weight written = 288 B)."""
    import torch
    pr = W.c4_uot()
    x, a, y, b = (torch.from_numpy(v).to(dev) for v in shard_problem(pr, world, rank))
    out = {"metric": "UOT Sinkhorn iterations/s", "unit": "iterations/s",
           "config": f"C4: UOT d=2 n=m={len(pr.x)} eps={pr.eps} lam={pr.lam} iters={pr.iters} "
                     "(median of 3 whole solves incl. setup, inputs in HBM)"}
    for name, N in (("auto", 0), ("grid4096", 2048)):
        opts = {"method": "nfft", "N": N}

        def solve():
            return uk.uot_sinkhorn(x, a, y, b, pr.eps, pr.lam, iters=pr.iters, opts=opts, comm=comm)

        ms, per, res = _solves(uk, solve, barrier, world, dev)
        prof = profiled(uk, solve)
        fms, fcnt = prof["fused"]
        roof = None
        if fcnt:
            avg = fms / fcnt
            per_launch_bytes = (len(x) + len(y)) / 2 * 288  # one half-step visits one point set
            achieved = per_launch_bytes / (avg / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": "sinkhorn2d_ws_k (fused d=2 half-step)", "achieved": achieved,
                    "peak": hbm_peak(), "unit": "GB/s", "frac": achieved / hbm_peak(), "per_unit": "288 B per point",
                    "traffic": traffic_of("fused2d"), "avg_launch_ms": avg, "launches_per_solve": fcnt,
                    "share_of_solve": fms / sum(v[0] for v in prof.values()),
                    "per_tag_ms": {k: round(v[0], 3) for k, v in prof.items() if v[1]}}
        out[name] = {"value": pr.iters / (ms / 1e3), "ms_per_solve": ms, "solve_ms": [round(v, 2) for v in per],
                     "n_grid": res.info["n_grid"], "N": res.info["N"], "plan_mass": res.plan_mass,
                     "primal": res.primal, "roofline": roof}
    out["value"] = out["auto"]["value"]
    out["primal_rel_diff_grid4096_vs_auto"] = abs(out["grid4096"]["primal"] - out["auto"]["primal"]) / abs(
        out["auto"]["primal"])
    if cpu:
        out["cpu_baseline"] = cpu
    return out


def c1_leg(uk, dev, cpu=None):
    """C1 (BASELINE.json configs[0]): UOT d=2, n=m=1000, eps=0.05, lam=1, 100 iterations —
    whole solves, device-timed (median of 5), with the AUTO choice (the direct kernel at
    1e6 pairs per sum) and with the NFFT path; both replay the iteration from CUDA graphs.
    Roofline of the direct kernel: FP64 flops per pair (DIRECT_FLOPS_PER_PAIR) over its
    live launch time (a launch-latency-bound size: 1e6 pairs per launch)."""
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
        prof = profiled(uk, solve)
        if res.info["method"] == "direct":
            roof = direct_roofline(prof, 2, W.GAUSS, len(pr.x) * len(pr.y))
        else:
            roof = pass_roofline(prof, 2, 8, len(pr.x), len(pr.y), fused=True)
        out[method] = {"value": pr.iters / (ms / 1e3), "ms_per_solve": ms, "method_used": res.info["method"],
                       "roofline": roof}
    out["value"] = out["auto"]["value"]
    if cpu:
        out["cpu_baseline"] = cpu
    return out


def c5_legs(uk, world, rank, comm, dev, barrier, cpu):
    """configs[4]: kernel sums (NFFT) at n=m=1e6 and 1e7, uniform ball R=0.2, N(0,1)
    weights, Gaussian l=0.05 / IMQ c=0.05 (reading R7): whole calls (setup included),
    median of 5, and the dominant pass against its roofline."""
    import torch
    out = []
    for d, n, kind in C5_CASES:
        pr = W.c5_sum(d, n, kind=kind)
        src, alpha, tgt = (torch.from_numpy(shard(v, world, rank)).to(dev) for v in (pr.src, pr.alpha, pr.tgt))
        stream = torch.cuda.current_stream()

        def call():
            return uk.kernel_sum(src, alpha, tgt, kind, pr.param, opts={"method": "nfft"}, comm=comm,
                                 return_info=True)

        for _ in range(2):
            call()
        barrier()
        torch.cuda.synchronize()
        per = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, info = call()
            e1.record(stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
        ms = statistics.median(per)
        roof = pass_roofline(profiled(uk, call), d, 8, len(src), len(tgt))
        leg = {"workload": f"C5 d={d} n=m={n} {'gauss' if kind == W.GAUSS else 'imq'}", "metric": "kernel sums/s",
               "value": 1e3 / ms, "unit": "sums/s", "ms_per_sum": ms, "N": info["N"], "n_grid": info["n_grid"],
               "groups": info["groups"], "roofline": roof}
        key = f"c5_{d}_{n}_{kind}"
        if key in cpu:
            leg["cpu_baseline"] = cpu[key]
        out.append(leg)
        del src, alpha, tgt
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    main_ours(args)


if __name__ == "__main__":
    main()
