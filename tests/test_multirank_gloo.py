"""World-size-2 gloo tests (CPU) of the multi-rank path's host logic.

The CUDA kernels need a GPU, so these tests check what the sharded path relies on:
* the contiguous point sharding covers every point exactly once;
* the exchange step is correct: with sources sharded, the kernel sums at each rank's
  targets equal the sum over ranks of the local partial sums (the all-reduce the library
  performs on the Fourier coefficients is this sum, by linearity of (4.6) in alpha);
* global MMD^2 / objective scalars are sums of per-rank partial sums;
* timings are combined as the max over ranks;
* a 128-byte NCCL-style unique id broadcast reaches every rank intact.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2306_13618_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        pr = W.random_sum(3, 401, 333, kind=W.GAUSS, param=0.02, seed=4, signed=True)
        # sources and targets sharded
        src, al = D.shard(pr.src, world, rank), D.shard(pr.alpha, world, rank)
        tgt_all = pr.tgt
        partial = oracle.kernel_sum_direct(src, al, tgt_all, pr.kind, pr.param)
        import torch
        t = torch.from_numpy(partial.copy())
        dist.all_reduce(t)  # the exchange step: sum of per-rank contributions
        lo, hi = D.shard_bounds(len(tgt_all), world, rank)
        full = oracle.kernel_sum_direct(pr.src, pr.alpha, tgt_all[lo:hi], pr.kind, pr.param)
        res["sum_err"] = float(np.max(np.abs(t.numpy()[lo:hi] - full)) / np.max(np.abs(full)))
        # MMD^2 from per-rank partial quadratic forms: sum_i in shard w_i (K w)_i
        mp_ = W.c2_mmd(n=300, m=260)
        z = np.concatenate([mp_.x, mp_.y])
        w = np.concatenate([mp_.a, -mp_.b])
        zs, ws = D.shard(z, world, rank), D.shard(w, world, rank)
        s_local = oracle.kernel_sum_direct(zs, ws, z, W.GAUSS, 0.0025)
        tt = torch.from_numpy(s_local.copy())
        dist.all_reduce(tt)
        lo, hi = D.shard_bounds(len(z), world, rank)
        part = float(ws @ tt.numpy()[lo:hi])
        res["mmd2"] = D.sum_over_ranks([part])[0]
        res["mmd2_ref"] = oracle.mmd2_direct(mp_.x, mp_.a, mp_.y, mp_.b, W.GAUSS, 0.0025)
        res["tmax"] = D.max_over_ranks(10.0 + rank)
        uid = D.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        res["uid_ok"] = uid == bytes(range(128))
        cover = D.sum_over_ranks([float(np.sum(D.shard(np.arange(1001.0), world, rank)))])[0]
        res["cover"] = cover
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = out[r]
        assert res["sum_err"] <= 1e-13
        assert abs(res["mmd2"] - res["mmd2_ref"]) <= 1e-10 * abs(res["mmd2_ref"])
        assert res["tmax"] == 10.0 + world - 1
        assert res["uid_ok"]
        assert res["cover"] == float(np.sum(np.arange(1001.0)))


def test_shard_bounds_cover():
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            got = [D.shard_bounds(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_bounds(10, 2, 2)
