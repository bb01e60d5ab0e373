"""Host-side multi-rank helpers (one process per GPU).

The data-path exchange (the per-kernel-sum all-reduce of the oversampled Fourier
coefficients) runs inside libuotk.so over NCCL; this module only holds the plumbing
around it: how points are sharded, how the NCCL unique id reaches every rank, and how
per-rank timings are combined (max over ranks).  Every function works with any
torch.distributed backend, so the logic is tested with `gloo` on CPU.
"""

import numpy as np


def shard_bounds(n, world, rank):
    """Contiguous block [lo, hi) of n items owned by `rank` (sizes differ by at most 1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return n * rank // world, n * (rank + 1) // world


def shard(arr, world, rank):
    lo, hi = shard_bounds(len(arr), world, rank)
    return np.ascontiguousarray(arr[lo:hi])


def broadcast_bytes(payload, src=0):
    """Broadcast a bytes object from `src` over the default process group."""
    import torch.distributed as dist
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (multi-GPU timings are reported as the max)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def sum_over_ranks(values, device=None):
    """Elementwise sum of a list of floats over all ranks."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]
