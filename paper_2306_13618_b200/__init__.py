"""B200-native fast radial-kernel sums for unbalanced OT and MMD (arXiv 2306.13618).

Python surface of the C ABI in ``include/uotk.h``: three operations with the same
names as the C entry points, marshalling arguments only.

* :func:`kernel_sum`   — s_i = sum_j k(||tgt_i - src_j||) alpha_j       (Eq. 4.3)
* :func:`uot_sinkhorn` — entropic UOT by Sinkhorn, Algorithm 2
* :func:`mmd2`         — MMD^2 of Eq. (3.5)

Arrays may be torch tensors (CUDA or CPU) or numpy arrays, float64 and contiguous;
points are row-major (n, d).  Outputs are allocated like the inputs (CUDA tensors for
CUDA inputs, host arrays otherwise — the library then stages the copies itself).
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import UotkError, UotkOpts, UotkInfo, UotkUotResult  # noqa: F401

GAUSS = 0
IMQ = 1
GAUSS_R2 = 2  # k(r) = r^2 exp(-r^2/param): kernel sums only (transport-cost kernel)
LAP = 3       # k(r) = exp(-r/param)
ENERGY = 4    # k(r) = -r (Table 1's energy kernel; param ignored)
AUTO, NFFT, DIRECT = 0, 1, 2
FLAG_GENERIC, FLAG_CHUNKED = 1, 2  # opts["flags"]: kernel family of the NFFT passes (uotk.h)
_KIND = {"gauss": GAUSS, "gaussian": GAUSS, "imq": IMQ, "gauss_r2": GAUSS_R2, "laplace": LAP, "lap": LAP,
         "energy": ENERGY, GAUSS: GAUSS, IMQ: IMQ, GAUSS_R2: GAUSS_R2, LAP: LAP, ENERGY: ENERGY}
FLAG_TRANSPORT = 4
FLAG_FFT = 8  # always the cuFFT spectral chain (the multi-rank path), never the separable GEMMs
FLAG_COST_R1 = 16  # uot: cost d^1, the Laplace Gibbs kernel exp(-|x-y|/eps) (Algorithm 2, r = 1)
_METHOD = {"auto": AUTO, "nfft": NFFT, "direct": DIRECT, AUTO: AUTO, NFFT: NFFT, DIRECT: DIRECT}

__all__ = ["kernel_sum", "uot_sinkhorn", "uot_sinkhorn_scaling", "mmd2", "uot_cstar", "sinkhorn_divergence", "release_caches", "Comm", "UOTResult", "GAUSS",
           "IMQ", "UotkError",
           "launch_counter", "reset_launch_counter", "library_path"]


def library_path():
    return _native.LIB_PATH


def _torch():
    try:
        import torch
        return torch
    except ImportError:  # pragma: no cover
        return None


class _Arr:
    """Pointer view of a caller array (torch tensor or numpy array), float64, contiguous."""

    def __init__(self, a, name, ncols=None):
        self.obj = a
        torch = _torch()
        if torch is not None and isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise TypeError(f"{name}: expected float64, got {a.dtype}")
            if not a.is_contiguous():
                raise ValueError(f"{name}: tensor must be contiguous")
            self.is_torch = True
            self.is_cuda = a.is_cuda
            self.ptr = a.data_ptr() if a.numel() else None
            self.shape = tuple(a.shape)
        else:
            a = np.asarray(a)
            if a.dtype != np.float64:
                raise TypeError(f"{name}: expected float64, got {a.dtype}")
            if not a.flags.c_contiguous:
                raise ValueError(f"{name}: array must be C-contiguous")
            self.obj = a
            self.is_torch = False
            self.is_cuda = False
            self.ptr = a.ctypes.data if a.size else None
            self.shape = a.shape
        if ncols is not None:
            if len(self.shape) == 1 and ncols == 1:
                self.shape = (self.shape[0], 1)
            if len(self.shape) != 2 or self.shape[1] != ncols:
                raise ValueError(f"{name}: expected shape (n, {ncols}), got {self.shape}")

    @property
    def n(self):
        return self.shape[0]


def _dim(points, name):
    shp = points.shape if hasattr(points, "shape") else np.asarray(points).shape
    if len(shp) == 1:
        return 1
    if len(shp) != 2:
        raise ValueError(f"{name}: expected an (n, d) array")
    return shp[1]


def _like(ref, n):
    """Allocate an output of n doubles like `ref` (CUDA tensor, CPU tensor or numpy); a
    pinned CPU tensor gets a pinned output, so the library's device->host copy of it runs
    at full DMA speed instead of through the driver's pageable bounce buffer."""
    torch = _torch()
    if ref.is_torch:
        pin = ref.obj.device.type == "cpu" and ref.obj.is_pinned()
        return torch.empty(n, dtype=torch.float64, device=ref.obj.device, pin_memory=pin)
    return np.empty(n, dtype=np.float64)


def _stream(stream, arrays):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    torch = _torch()
    if torch is not None and any(a.is_cuda for a in arrays):
        return torch.cuda.current_stream().cuda_stream
    return 0


def _opts(opts):
    o = UotkOpts()
    _native.load().uotk_opts_init(ctypes.byref(o))
    if opts:
        for k, v in opts.items():
            if k == "method":
                v = _METHOD[v]
            setattr(o, k, v)
    return o


def _comm_ptr(comm):
    return None if comm is None else comm.handle


def _info_dict(info):
    return {"method": {1: "nfft", 2: "direct"}.get(info.method_used, "?"), "N": info.N,
            "n_grid": info.n_grid, "m": info.m, "h": info.h, "groups": (info.groups1, info.groups2),
            "nranks": info.nranks}


def kernel_sum(src, alpha, tgt, kind="gauss", param=None, opts=None, comm=None, stream=None, out=None,
               return_info=False):
    """s_i = sum_j k(||tgt_i - src_j||) alpha_j  (Eq. 4.3).  kind 'gauss': exp(-r^2/param);
    'imq': (r^2 + param^2)^(-1/2).  opts: dict of uotk_opts fields (method='auto'|'nfft'|'direct')."""
    lib = _native.load()
    d = _dim(src, "src")
    S, A, T = _Arr(src, "src", d), _Arr(alpha, "alpha"), _Arr(tgt, "tgt", d)
    if A.shape != (S.n,):
        raise ValueError("alpha must have shape (n_src,)")
    if out is None:
        out = _like(T, T.n)
    O = _Arr(out, "out")
    info = UotkInfo()
    o = _opts(opts)
    code = lib.uotk_kernel_sum(d, S.n, S.ptr, A.ptr, T.n, T.ptr, _KIND[kind], float(param), O.ptr,
                               ctypes.byref(o), ctypes.byref(info), _comm_ptr(comm),
                               _stream(stream, [S, A, T, O]))
    _native.check(code)
    return (O.obj, _info_dict(info)) if return_info else O.obj


@dataclass
class UOTResult:
    primal: float
    dual: float
    plan_mass: float
    mass_a: float
    mass_b: float
    max_dbeta: float
    max_dgamma: float
    iters: int
    info: dict
    transport: float = float("nan")  # <pi, d^2> (uot_sinkhorn(..., transport=True))
    p: object = None                 # plan marginals (uot_sinkhorn(..., marginals=True))
    q: object = None

    @property
    def uot_cost(self):
        """UOT_{2;eta;lambda} value: the primal (2.9) at the final iterate (reading R3)."""
        return self.primal


def uot_sinkhorn(x, a, y, b, eps, lam, lam2=None, iters=100, gamma_init=None, opts=None, comm=None, stream=None,
                 marginals=False, transport=False):
    """Entropic UOT (Def. 2.7) by Algorithm 2: Gaussian Gibbs kernel exp(-|x-y|^2/eps),
    eps = 1/lambda_paper, marginal penalties lam (= eta_1) and lam2 (= eta_2, default lam).
    Returns (beta, gamma, UOTResult)."""
    lib = _native.load()
    d = _dim(x, "x")
    X, A, Y, B = _Arr(x, "x", d), _Arr(a, "a"), _Arr(y, "y", d), _Arr(b, "b")
    if A.shape != (X.n,) or B.shape != (Y.n,):
        raise ValueError("masses must match the point counts")
    if isinstance(gamma_init, str):
        if gamma_init != "cstar":
            raise ValueError("gamma_init: an array, None or 'cstar'")
        # Remark 5.2: gamma^0 = c* 1 with c* of Eq. (2.10)
        c = uot_cstar(x, a, y, b, eps, lam, lam2, comm=comm, stream=stream)
        gamma_init = _like(Y, Y.n)
        gamma_init[:] = c
    G0 = _Arr(gamma_init, "gamma_init") if gamma_init is not None else None
    beta = _like(X, X.n)
    gamma = _like(Y, Y.n)
    BO, GO = _Arr(beta, "beta"), _Arr(gamma, "gamma")
    res = UotkUotResult()
    o = _opts(opts)
    lam2 = lam if lam2 is None else lam2
    if marginals or transport:
        if transport:
            o.flags |= FLAG_TRANSPORT
        PO = _Arr(_like(X, X.n), "p") if marginals else None
        QO = _Arr(_like(Y, Y.n), "q") if marginals else None
        code = lib.uotk_uot_sinkhorn_ex(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, float(eps), float(lam), float(lam2),
                                        int(iters), G0.ptr if G0 else None, BO.ptr, GO.ptr,
                                        PO.ptr if PO else None, QO.ptr if QO else None, ctypes.byref(res),
                                        ctypes.byref(o), _comm_ptr(comm), _stream(stream, [X, A, Y, B, BO, GO]))
    else:
        PO = QO = None
        code = lib.uotk_uot_sinkhorn(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, float(eps), float(lam), float(lam2),
                                     int(iters), G0.ptr if G0 else None, BO.ptr, GO.ptr, ctypes.byref(res),
                                     ctypes.byref(o), _comm_ptr(comm), _stream(stream, [X, A, Y, B, BO, GO]))
    _native.check(code)
    r = UOTResult(res.primal, res.dual, res.plan_mass, res.mass_a, res.mass_b, res.max_dbeta, res.max_dgamma,
                  res.iters, _info_dict(res.info), res.transport, PO.obj if PO else None, QO.obj if QO else None)
    return BO.obj, GO.obj, r


def uot_sinkhorn_scaling(x, a, y, b, eps_list, lam, lam2=None, iters=100, gamma_init=None, opts=None, comm=None,
                         stream=None):
    """lambda-scaling (Sec. 5.1.3): uot_sinkhorn for each eps in eps_list (decreasing),
    each stage warm-started from the previous gamma.  Returns (beta, gamma, UOTResult) of
    the last stage; UOTResult.iters is the total over the stages."""
    lib = _native.load()
    d = _dim(x, "x")
    X, A, Y, B = _Arr(x, "x", d), _Arr(a, "a"), _Arr(y, "y", d), _Arr(b, "b")
    if A.shape != (X.n,) or B.shape != (Y.n,):
        raise ValueError("masses must match the point counts")
    G0 = _Arr(gamma_init, "gamma_init") if gamma_init is not None else None
    eps_arr = np.ascontiguousarray(np.asarray(eps_list, dtype=np.float64))
    beta = _like(X, X.n)
    gamma = _like(Y, Y.n)
    BO, GO = _Arr(beta, "beta"), _Arr(gamma, "gamma")
    res = UotkUotResult()
    o = _opts(opts)
    lam2 = lam if lam2 is None else lam2
    code = lib.uotk_uot_sinkhorn_scaling(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, eps_arr.ctypes.data, len(eps_arr),
                                         float(lam), float(lam2), int(iters), G0.ptr if G0 else None, BO.ptr, GO.ptr,
                                         ctypes.byref(res), ctypes.byref(o), _comm_ptr(comm),
                                         _stream(stream, [X, A, Y, B, BO, GO]))
    _native.check(code)
    r = UOTResult(res.primal, res.dual, res.plan_mass, res.mass_a, res.mass_b, res.max_dbeta, res.max_dgamma,
                  res.iters, _info_dict(res.info), res.transport)
    return BO.obj, GO.obj, r


def uot_cstar(x, a, y, b, eps, lam, lam2=None, comm=None, stream=None):
    """The constant c* of Prop. 2.9 / Eq. (2.10) for r = 2 (host float)."""
    lib = _native.load()
    d = _dim(x, "x")
    X, A, Y, B = _Arr(x, "x", d), _Arr(a, "a"), _Arr(y, "y", d), _Arr(b, "b")
    if A.shape != (X.n,) or B.shape != (Y.n,):
        raise ValueError("masses must match the point counts")
    out = ctypes.c_double(0.0)
    lam2 = lam if lam2 is None else lam2
    code = lib.uotk_uot_cstar(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, float(eps), float(lam), float(lam2),
                              ctypes.byref(out), _comm_ptr(comm), _stream(stream, [X, A, Y, B]))
    _native.check(code)
    return out.value


def sinkhorn_divergence(x, a, y, b, eps, lam, lam2=None, iters=100, opts=None, comm=None, stream=None,
                        return_terms=False):
    """Debiased UOT of Eq. (2.12): UOT(mu,nu) - UOT(mu,mu)/2 - UOT(nu,nu)/2 + eps/2 (mu(X)-nu(X))^2."""
    lib = _native.load()
    d = _dim(x, "x")
    X, A, Y, B = _Arr(x, "x", d), _Arr(a, "a"), _Arr(y, "y", d), _Arr(b, "b")
    if A.shape != (X.n,) or B.shape != (Y.n,):
        raise ValueError("masses must match the point counts")
    sd = ctypes.c_double(0.0)
    terms = (ctypes.c_double * 3)()
    o = _opts(opts)
    lam2 = lam if lam2 is None else lam2
    code = lib.uotk_sinkhorn_divergence(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, float(eps), float(lam),
                                        float(lam2), int(iters), ctypes.byref(sd), terms, ctypes.byref(o),
                                        _comm_ptr(comm), _stream(stream, [X, A, Y, B]))
    _native.check(code)
    return (sd.value, tuple(terms)) if return_terms else sd.value


def mmd2(x, a, y, b, kind="gauss", param=None, opts=None, comm=None, stream=None, return_info=False):
    """MMD^2 of Eq. (3.5) (V-statistic) between sum_i a_i delta_{x_i} and sum_j b_j delta_{y_j}."""
    lib = _native.load()
    d = _dim(x, "x")
    X, A, Y, B = _Arr(x, "x", d), _Arr(a, "a"), _Arr(y, "y", d), _Arr(b, "b")
    if A.shape != (X.n,) or B.shape != (Y.n,):
        raise ValueError("weights must match the point counts")
    val = ctypes.c_double(0.0)
    info = UotkInfo()
    o = _opts(opts)
    code = lib.uotk_mmd2(d, X.n, X.ptr, A.ptr, Y.n, Y.ptr, B.ptr, _KIND[kind], float(param), ctypes.byref(val),
                         ctypes.byref(o), ctypes.byref(info), _comm_ptr(comm), _stream(stream, [X, A, Y, B]))
    _native.check(code)
    return (val.value, _info_dict(info)) if return_info else val.value


class Comm:
    """Multi-GPU communicator (NCCL inside libuotk.so).  Create collectively on all ranks:
    ``Comm.from_torch_distributed()`` broadcasts the NCCL unique id over the default
    torch.distributed process group."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        lib = _native.load()
        buf = ctypes.create_string_buffer(unique_id, 128)
        h = ctypes.c_void_p()
        _native.check(lib.uotk_comm_create(buf, nranks, rank, ctypes.byref(h)))
        self.handle = h.value
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _native.check(_native.load().uotk_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def loopback(cls, nranks: int):
        """nranks rank handles of one loopback group (uotk_comm_create_loopback): the
        multi-rank path in one process on one GPU, one host thread per rank."""
        lib = _native.load()
        hs = (ctypes.c_void_p * nranks)()
        _native.check(lib.uotk_comm_create_loopback(nranks, hs))
        out = []
        for k in range(nranks):
            c = cls.__new__(cls)
            c.handle, c.nranks, c.rank = hs[k], nranks, k
            out.append(c)
        return out

    @classmethod
    def from_torch_distributed(cls):
        import torch.distributed as dist

        from .dist import broadcast_bytes
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = broadcast_bytes(cls.unique_id() if rank == 0 else None)
        return cls(uid, world, rank)

    def close(self):
        if self.handle:
            _native.check(_native.load().uotk_comm_destroy(self.handle))
            self.handle = None


def release_caches():
    """Drop the library's cached Fourier tables, cuFFT plans and device buffers (the next
    call runs cold; see uotk_release_caches in include/uotk.h)."""
    _native.check(_native.load().uotk_release_caches())


def launch_counter():
    """Kernels this library launched on the calling thread since the last reset."""
    return _native.load().uotk_launch_counter()


def reset_launch_counter():
    _native.load().uotk_launch_counter_reset()


PROFILE_TAGS = ("spread", "gather", "fused", "fft", "direct", "setup")


def profile_enable(on=True):
    """Bracket every instrumented launch with CUDA events on its stream (see uotk.h)."""
    _native.load().uotk_profile_enable(1 if on else 0)


def profile_reset():
    _native.load().uotk_profile_reset()


def profile_read():
    """{tag: (total_ms, launches)} of the bracketed launches since the last reset."""
    lib = _native.load()
    out = {}
    for tag in PROFILE_TAGS:
        ms, cnt = ctypes.c_double(), ctypes.c_int64()
        _native.check(lib.uotk_profile_read(tag.encode(), ctypes.byref(ms), ctypes.byref(cnt)))
        out[tag] = (ms.value, cnt.value)
    return out
