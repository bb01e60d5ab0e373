"""ctypes binding of include/uotk.h (argument marshalling only — every step runs in libuotk.so).

The shared library is built in-tree by ``paper_2306_13618_b200.build`` and loaded from
this package's directory.  There is no fallback: if the library is missing, every call
raises.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UOTK_LIB_PATH") or os.path.join(HERE, "libuotk.so")  # override: A/B builds

UOTK_OK = 0
STATUS = {
    -1: "UOTK_EINVAL", -2: "UOTK_EDOMAIN", -3: "UOTK_EOVERFLOW", -4: "UOTK_ENOMEM",
    -5: "UOTK_ECUDA", -6: "UOTK_ECUFFT", -7: "UOTK_ENCCL", -8: "UOTK_EUNSUPPORTED",
}

# every symbol include/uotk.h declares (tests check the library exports all of them)
EXPORTED = (
    "uotk_opts_init", "uotk_kernel_sum", "uotk_uot_sinkhorn", "uotk_mmd2",
    "uotk_uot_cstar", "uotk_sinkhorn_divergence", "uotk_uot_sinkhorn_scaling", "uotk_uot_sinkhorn_ex",
    "uotk_comm_unique_id", "uotk_comm_create", "uotk_comm_create_loopback", "uotk_comm_destroy",
    "uotk_last_error", "uotk_abi_version", "uotk_launch_counter", "uotk_launch_counter_reset",
    "uotk_profile_enable", "uotk_profile_reset", "uotk_profile_read", "uotk_release_caches",
)


class UotkOpts(ctypes.Structure):
    _fields_ = [
        ("method", ctypes.c_int32), ("N", ctypes.c_int32), ("sigma", ctypes.c_double),
        ("m", ctypes.c_int32), ("p", ctypes.c_int32), ("eps_B", ctypes.c_double),
        ("h", ctypes.c_double), ("tol", ctypes.c_double), ("flags", ctypes.c_int32),
        ("deterministic", ctypes.c_int32), ("stop_tol", ctypes.c_double), ("check_every", ctypes.c_int32),
        ("reserved2", ctypes.c_int32),
    ]


class UotkInfo(ctypes.Structure):
    _fields_ = [
        ("method_used", ctypes.c_int32), ("N", ctypes.c_int32), ("n_grid", ctypes.c_int32),
        ("m", ctypes.c_int32), ("h", ctypes.c_double), ("groups1", ctypes.c_int32),
        ("groups2", ctypes.c_int32), ("nranks", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class UotkUotResult(ctypes.Structure):
    _fields_ = [
        ("primal", ctypes.c_double), ("dual", ctypes.c_double), ("plan_mass", ctypes.c_double),
        ("mass_a", ctypes.c_double), ("mass_b", ctypes.c_double), ("max_dbeta", ctypes.c_double),
        ("max_dgamma", ctypes.c_double), ("iters", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("info", UotkInfo), ("transport", ctypes.c_double),
    ]


class UotkError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
D = ctypes.c_double
INT = ctypes.c_int


def load():
    """Load libuotk.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2306_13618_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    lib.uotk_opts_init.argtypes = [ctypes.POINTER(UotkOpts)]
    lib.uotk_opts_init.restype = None
    lib.uotk_kernel_sum.argtypes = [INT, I64, P, P, I64, P, INT, D, P, ctypes.POINTER(UotkOpts),
                                    ctypes.POINTER(UotkInfo), P, P]
    lib.uotk_kernel_sum.restype = INT
    lib.uotk_uot_sinkhorn.argtypes = [INT, I64, P, P, I64, P, P, D, D, D, INT, P, P, P,
                                      ctypes.POINTER(UotkUotResult), ctypes.POINTER(UotkOpts), P, P]
    lib.uotk_uot_sinkhorn.restype = INT
    lib.uotk_mmd2.argtypes = [INT, I64, P, P, I64, P, P, INT, D, ctypes.POINTER(D),
                              ctypes.POINTER(UotkOpts), ctypes.POINTER(UotkInfo), P, P]
    lib.uotk_mmd2.restype = INT
    lib.uotk_uot_cstar.argtypes = [INT, I64, P, P, I64, P, P, D, D, D, ctypes.POINTER(D), P, P]
    lib.uotk_uot_cstar.restype = INT
    lib.uotk_sinkhorn_divergence.argtypes = [INT, I64, P, P, I64, P, P, D, D, D, INT, ctypes.POINTER(D), P,
                                             ctypes.POINTER(UotkOpts), P, P]
    lib.uotk_sinkhorn_divergence.restype = INT
    lib.uotk_uot_sinkhorn_ex.argtypes = [INT, I64, P, P, I64, P, P, D, D, D, INT, P, P, P, P, P,
                                         ctypes.POINTER(UotkUotResult), ctypes.POINTER(UotkOpts), P, P]
    lib.uotk_uot_sinkhorn_ex.restype = INT
    lib.uotk_uot_sinkhorn_scaling.argtypes = [INT, I64, P, P, I64, P, P, P, INT, D, D, INT, P, P, P,
                                              ctypes.POINTER(UotkUotResult), ctypes.POINTER(UotkOpts), P, P]
    lib.uotk_uot_sinkhorn_scaling.restype = INT
    lib.uotk_comm_unique_id.argtypes = [P]
    lib.uotk_comm_unique_id.restype = INT
    lib.uotk_comm_create.argtypes = [P, INT, INT, ctypes.POINTER(P)]
    lib.uotk_comm_create.restype = INT
    lib.uotk_comm_create_loopback.argtypes = [INT, ctypes.POINTER(P)]
    lib.uotk_comm_create_loopback.restype = INT
    lib.uotk_comm_destroy.argtypes = [P]
    lib.uotk_comm_destroy.restype = INT
    lib.uotk_last_error.argtypes = []
    lib.uotk_last_error.restype = ctypes.c_char_p
    lib.uotk_abi_version.argtypes = []
    lib.uotk_abi_version.restype = INT
    lib.uotk_launch_counter.argtypes = []
    lib.uotk_launch_counter.restype = I64
    lib.uotk_launch_counter_reset.argtypes = []
    lib.uotk_launch_counter_reset.restype = None
    lib.uotk_profile_enable.argtypes = [INT]
    lib.uotk_profile_enable.restype = None
    lib.uotk_profile_reset.argtypes = []
    lib.uotk_profile_reset.restype = None
    if getattr(lib, "uotk_release_caches", None) is not None:  # absent from older A/B builds
        lib.uotk_release_caches.argtypes = []
        lib.uotk_release_caches.restype = ctypes.c_int
    lib.uotk_profile_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(D), ctypes.POINTER(I64)]
    lib.uotk_profile_read.restype = INT
    _lib = lib
    return lib


def check(code):
    if code != UOTK_OK:
        raise UotkError(code, load().uotk_last_error().decode(errors="replace"))
