"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/uotk.h declares, the ctypes structs match the C layout, and argument
validation fails with the documented status codes before touching the device."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uotk.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2306_13618_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _native.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(uotk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_list():
    from paper_2306_13618_b200 import _native
    assert declared_functions() == sorted(_native.EXPORTED)


def test_library_exports_every_declared_symbol(lib):
    from paper_2306_13618_b200 import _native
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (uotk_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)


def test_abi_version(lib):
    assert lib.uotk_abi_version() == 3


def test_struct_layout_matches_c(tmp_path):
    """Compile a tiny C program against uotk.h and compare sizeof/offsetof with ctypes."""
    from paper_2306_13618_b200 import _native
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "uotk.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(uotk_opts), sizeof(uotk_info),"
        " sizeof(uotk_uot_result), offsetof(uotk_opts, tol), offsetof(uotk_uot_result, info),"
        " offsetof(uotk_uot_result, iters)); return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals == [ctypes.sizeof(_native.UotkOpts), ctypes.sizeof(_native.UotkInfo),
                    ctypes.sizeof(_native.UotkUotResult), _native.UotkOpts.tol.offset,
                    _native.UotkUotResult.info.offset, _native.UotkUotResult.iters.offset]


def test_invalid_arguments_rejected_without_gpu(lib):
    import paper_2306_13618_b200 as uk
    from paper_2306_13618_b200 import _native
    x = np.zeros((4, 4))
    with pytest.raises(uk.UotkError) as e:
        uk.kernel_sum(x, np.ones(4), x, "gauss", 0.1)  # d = 4
    assert e.value.code == -1
    x = np.zeros((4, 2))
    with pytest.raises(uk.UotkError) as e:
        uk.kernel_sum(x, np.ones(4), x, "gauss", -1.0)
    assert e.value.code == -1
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(x, np.ones(4), x, np.ones(4), eps=0.0, lam=1.0, iters=3)
    assert e.value.code == -1
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(x, np.ones(4), x, np.ones(4), eps=0.1, lam=1.0, iters=-1)
    assert e.value.code == -1
    with pytest.raises(uk.UotkError) as e:
        uk.mmd2(x, np.ones(4), x, np.ones(4), "imq", 0.0)
    assert e.value.code == -1
    for bad in (32, uk.FLAG_GENERIC | uk.FLAG_CHUNKED):
        with pytest.raises(uk.UotkError) as e:
            uk.kernel_sum(x, np.ones(4), x, "gauss", 0.1, opts={"flags": bad})
        assert e.value.code == -1
        assert "flags" in _native.load().uotk_last_error().decode()


def test_dtype_and_shape_checks():
    import paper_2306_13618_b200 as uk
    with pytest.raises(TypeError):
        uk.kernel_sum(np.zeros((3, 2), np.float32), np.ones(3), np.zeros((3, 2)), "gauss", 0.1)
    with pytest.raises(ValueError):
        uk.kernel_sum(np.zeros((3, 2)), np.ones(4), np.zeros((3, 2)), "gauss", 0.1)


def test_solver_variant_argument_errors():
    import paper_2306_13618_b200 as uk
    x = np.zeros((4, 2))
    with pytest.raises(uk.UotkError) as e:
        uk.uot_cstar(x, np.ones(4), x, np.ones(4), 0.0, 1.0)
    assert e.value.code == -1
    with pytest.raises(uk.UotkError) as e:
        uk.uot_sinkhorn(x, np.ones(4), x, np.ones(4), 0.1, 1.0, iters=3, opts={"stop_tol": -1.0})
    assert e.value.code == -1
    with pytest.raises(uk.UotkError) as e:
        uk.sinkhorn_divergence(x[:0], np.ones(0), x, np.ones(4), 0.1, 1.0)
    assert e.value.code == -1
