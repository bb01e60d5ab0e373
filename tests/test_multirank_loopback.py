"""The library's multi-rank path executed with P = 2, 4, 8 ranks on ONE GPU.

A loopback communicator group (``uotk_comm_create_loopback``) stands in for P processes:
P host threads call the same entry point concurrently, each with its own shard, rank
handle and CUDA stream; every exchange of the path (global bounding box, the all-reduce
of each kernel sum's truncated Fourier coefficients — linearity of (4.6) in alpha~,
P:590-592 — the stopping rule's sup-norms, the objective scalars, the error flags) runs
through the library's collective layer exactly as with NCCL, the reduction being an
in-library kernel over the P device buffers.  Results are checked against the CPU
oracle on the concatenated shards, element by element (bars as in test_gpu_parity.py).
"""

import threading

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def uk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_13618_b200 as uk
    return uk


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def shard_bounds(n, P, empty_rank=None):
    """Contiguous shard [lo, hi) per rank; rank `empty_rank` gets none."""
    ranks = [r for r in range(P) if r != empty_rank]
    cuts = np.linspace(0, n, len(ranks) + 1).round().astype(int)
    out = {r: (0, 0) for r in range(P)}
    for k, r in enumerate(ranks):
        out[r] = (int(cuts[k]), int(cuts[k + 1]))
    return [out[r] for r in range(P)]


def run_ranks(uk, P, fn):
    """fn(rank, comm, stream) on P threads of one loopback group; returns the P results
    (re-raises the first exception; UotkError codes are collected in .codes)."""
    comms = uk.Comm.loopback(P)
    results, errors = [None] * P, [None] * P

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                results[r] = fn(r, comms[r], st)
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in comms:
        c.close()
    if any(e is not None for e in errors):
        err = next(e for e in errors if e is not None)
        err.all_errors = errors
        raise err
    return results


def _np(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


# ------------------------------------------------------------------ kernel sums
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("d,kind,flags", [(3, W.GAUSS, 0), (3, W.GAUSS, 8), (3, W.IMQ, 0), (2, W.IMQ, 0),
                                          (2, W.GAUSS, 0), (1, W.GAUSS, 8)])
def test_kernel_sum_sharded(uk, P, d, kind, flags):
    """Sources and targets sharded over P ranks: each rank obtains, at its own targets,
    the sum over ALL ranks' sources.  Gaussian on the separable chain (slab-distributed:
    reduce-scatter of the first pass's column / plane blocks, 1/P of the next pass per
    rank, all-gather) and on the cuFFT chain (flags 8: truncated-spectrum all-reduce);
    IMQ on the pruned d = 3 chain and the full d = 2 chain."""
    param = 0.0025 if kind == W.GAUSS else 0.05
    pr = W.random_sum(d, 4001, 3001, kind=kind, param=param, seed=100 + d + P, signed=True)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    sb, tb = shard_bounds(4001, P), shard_bounds(3001, P)
    src, alpha, tgt = cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt)

    def fn(r, comm, st):
        (s0, s1), (t0, t1) = sb[r], tb[r]
        out, info = uk.kernel_sum(src[s0:s1], alpha[s0:s1], tgt[t0:t1], kind, param,
                                  opts={"method": "nfft", "flags": flags}, comm=comm, stream=st, return_info=True)
        return _np(out), info

    res = run_ranks(uk, P, fn)
    got = np.concatenate([o for o, _ in res])
    assert all(info["nranks"] == P for _, info in res)
    assert len({info["h"] for _, info in res}) == 1 and len({info["N"] for _, info in res}) == 1
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-9


@pytest.mark.parametrize("P", [3, 8])
@pytest.mark.parametrize("d", [2, 3])
def test_kernel_sum_sharded_small_box(uk, P, d):
    """A wide Gaussian (small grid, footprint box of a few cells): the slab split of the
    separable chain leaves some ranks with no column / plane block (w < P * ceil(w/P) or
    w < P); they still take part in every collective.  P = 3 gives ragged blocks."""
    pr = W.random_sum(d, 2001, 1501, kind=W.GAUSS, param=0.08, seed=300 + d + P, signed=True)
    ref = oracle.kernel_sum_direct(pr.src, pr.alpha, pr.tgt, pr.kind, pr.param)
    sb, tb = shard_bounds(2001, P), shard_bounds(1501, P)
    src, alpha, tgt = cuda(pr.src), cuda(pr.alpha), cuda(pr.tgt)

    def fn(r, comm, st):
        (s0, s1), (t0, t1) = sb[r], tb[r]
        return _np(uk.kernel_sum(src[s0:s1], alpha[s0:s1], tgt[t0:t1], W.GAUSS, 0.08,
                                 opts={"method": "nfft"}, comm=comm, stream=st))

    got = np.concatenate(run_ranks(uk, P, fn))
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-9


# ------------------------------------------------------------------ UOT Sinkhorn
def _pot_err(got, ref, c):
    return float(np.max(np.abs(got - ref) / (np.abs(ref) + c)))


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("case", ["c3", "c3-fft", "c1-d2"])
def test_uot_sharded(uk, P, case):
    """UOT Sinkhorn with x and y sharded over P ranks (every half-step's kernel sum
    exchanges its coefficients): the concatenated potentials element by element and the
    global objective values (identical on every rank) against the oracle."""
    if case.startswith("c3"):
        pr = W.c3_dense_uot(n=4003, m=3001, iters=8)
    else:
        pr = W.c1_uot(n=1500, m=1201)
    iters = 8
    flags = 8 if case.endswith("fft") else 0
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters)
    xb, yb = shard_bounds(len(pr.x), P), shard_bounds(len(pr.y), P)
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)

    def fn(r, comm, st):
        (x0, x1), (y0, y1) = xb[r], yb[r]
        be, ga, res = uk.uot_sinkhorn(x[x0:x1], a[x0:x1], y[y0:y1], b[y0:y1], pr.eps, pr.lam, iters=iters,
                                      opts={"method": "nfft", "flags": flags}, comm=comm, stream=st)
        return _np(be), _np(ga), res

    out = run_ranks(uk, P, fn)
    beta = np.concatenate([o[0] for o in out])
    gamma = np.concatenate([o[1] for o in out])
    c = pr.lam / (1.0 + pr.lam / pr.eps)
    assert _pot_err(beta, ref.beta, c) <= 1e-8
    assert _pot_err(gamma, ref.gamma, c) <= 1e-8
    for _, _, res in out:
        assert res.info["nranks"] == P
        assert abs(res.primal - ref.primal) <= 1e-8 * abs(ref.primal)
        assert abs(res.dual - ref.dual) <= 1e-8 * abs(ref.dual)
        assert abs(res.plan_mass - ref.plan_mass) <= 1e-8 * ref.plan_mass
        assert abs(res.mass_a - ref.mass_a) <= 1e-13 * ref.mass_a
    assert len({res.primal for _, _, res in out}) == 1  # bitwise identical on all ranks


def test_uot_sharded_empty_shard_and_stopping_rule(uk):
    """One rank holds no points at all (it still takes part in every collective), and
    the tolerance stopping rule decides on the sup-norm changes maxed over ranks: all
    ranks stop at the oracle's iteration."""
    P = 4
    pr = W.c1_uot(n=300, m=250)
    ref = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, iters=400, stop_tol=1e-9,
                                     check_every=5)
    xb, yb = shard_bounds(300, P, empty_rank=2), shard_bounds(250, P, empty_rank=2)
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)

    def fn(r, comm, st):
        (x0, x1), (y0, y1) = xb[r], yb[r]
        be, ga, res = uk.uot_sinkhorn(x[x0:x1], a[x0:x1], y[y0:y1], b[y0:y1], pr.eps, pr.lam, iters=400,
                                      opts={"method": "nfft", "stop_tol": 1e-9, "check_every": 5}, comm=comm,
                                      stream=st)
        return _np(be), _np(ga), res

    out = run_ranks(uk, P, fn)
    assert [o[2].iters for o in out] == [ref.iters] * P
    beta = np.concatenate([o[0] for o in out])
    gamma = np.concatenate([o[1] for o in out])
    c = pr.lam / (1.0 + pr.lam / pr.eps)
    assert _pot_err(beta, ref.beta, c) <= 1e-8 and _pot_err(gamma, ref.gamma, c) <= 1e-8


def test_errors_are_global(uk):
    """A non-positive mass on ONE rank's shard: every rank returns UOTK_EDOMAIN (the flag
    is or-ed over ranks before the decision), nobody hangs."""
    P = 3
    pr = W.c1_uot(n=300, m=250)
    a_bad = pr.a.copy()
    a_bad[250] = 0.0  # in the last rank's shard
    xb, yb = shard_bounds(300, P), shard_bounds(250, P)
    x, a, y, b = cuda(pr.x), cuda(a_bad), cuda(pr.y), cuda(pr.b)
    codes = []

    def fn(r, comm, st):
        (x0, x1), (y0, y1) = xb[r], yb[r]
        try:
            uk.uot_sinkhorn(x[x0:x1], a[x0:x1], y[y0:y1], b[y0:y1], pr.eps, pr.lam, iters=5,
                            opts={"method": "nfft"}, comm=comm, stream=st)
            codes.append(0)
        except uk.UotkError as e:
            codes.append(e.code)

    run_ranks(uk, P, fn)
    assert codes == [-2] * P


# ------------------------------------------------------------------ MMD^2
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("kind,flags", [(W.GAUSS, 0), (W.IMQ, 0), (W.GAUSS, 8)])
def test_mmd2_sharded(uk, P, kind, flags):
    """MMD^2 with both measures sharded (one rank's shard empty for P = 4): the ranks'
    Fourier coefficients are summed before the energy sum_k D_k |G_k|^2; every rank
    returns the same global value, equal to the oracle's."""
    pr = W.c2_mmd(n=3001, m=2503)
    param = dict(pr.kernels)[kind]
    ref = oracle.mmd2_direct(pr.x, pr.a, pr.y, pr.b, kind, param)
    xx = abs(float(pr.a @ oracle.kernel_sum_direct(pr.x, pr.a, pr.x, kind, param)))
    yy = abs(float(pr.b @ oracle.kernel_sum_direct(pr.y, pr.b, pr.y, kind, param)))
    denom = max(abs(ref), 1e-3 * (xx + yy))
    empty = 1 if P == 4 else None
    xb, yb = shard_bounds(3001, P, empty), shard_bounds(2503, P, empty)
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)

    def fn(r, comm, st):
        (x0, x1), (y0, y1) = xb[r], yb[r]
        return uk.mmd2(x[x0:x1], a[x0:x1], y[y0:y1], b[y0:y1], kind, param,
                       opts={"method": "nfft", "flags": flags}, comm=comm, stream=st)

    vals = run_ranks(uk, P, fn)
    assert len(set(vals)) == 1
    assert abs(vals[0] - ref) / denom <= 1e-8, (vals[0], ref)


def test_cstar_sharded(uk):
    """c* (Eq. 2.10): the moments are summed over ranks."""
    P = 4
    pr = W.c1_uot(n=3001, m=2003)
    ref = oracle.cstar(pr.x, pr.a, pr.y, pr.b, pr.eps, 0.3, 2.5)
    xb, yb = shard_bounds(3001, P), shard_bounds(2003, P, empty_rank=3)
    x, a, y, b = cuda(pr.x), cuda(pr.a), cuda(pr.y), cuda(pr.b)

    def fn(r, comm, st):
        (x0, x1), (y0, y1) = xb[r], yb[r]
        return uk.uot_cstar(x[x0:x1], a[x0:x1], y[y0:y1], b[y0:y1], pr.eps, 0.3, 2.5, comm=comm, stream=st)

    vals = run_ranks(uk, P, fn)
    assert all(abs(v - ref) <= 1e-12 * ref for v in vals)
