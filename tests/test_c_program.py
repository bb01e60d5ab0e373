"""The C ABI from a plain C program (tests/c/uotk_c_client.c): it links libuotk.so,
includes only include/uotk.h, and calls uotk_kernel_sum, uotk_uot_sinkhorn and uotk_mmd2
on host buffers.  CPU: it compiles, links and passes its argument-validation self test.
GPU: its results equal the CPU oracle's on the same (Python-written) inputs."""

import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2306_13618_b200")


def build_client(tmp_path):
    from paper_2306_13618_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    exe = tmp_path / "uotk_c_client"
    subprocess.run(["gcc", "-O2", "-std=c99", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "uotk_c_client.c"), "-L", PKG, "-luotk",
                    "-Wl,-rpath," + PKG, "-o", str(exe)], check=True)
    return exe


def test_c_client_builds_and_validates_arguments(tmp_path):
    exe = build_client(tmp_path)
    out = subprocess.run([str(exe), "--selftest"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "selftest ok" in out.stdout


@pytest.mark.gpu
def test_c_client_matches_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    import workloads as W
    exe = build_client(tmp_path)
    pr = W.c3_uot(n=2003, m=1501, iters=10)
    kind, param = W.GAUSS, 0.0025
    d = tmp_path / "case"
    d.mkdir()
    for name, arr in (("x", pr.x), ("a", pr.a), ("y", pr.y), ("b", pr.b)):
        np.ascontiguousarray(arr, dtype="<f8").tofile(d / f"{name}.bin")
    (d / "meta.txt").write_text(f"3 {len(pr.x)} {len(pr.y)} {pr.eps!r} {pr.lam!r} {pr.iters} {kind} {param!r}\n")
    out = subprocess.run([str(exe), str(d)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    s = np.fromfile(d / "sum.bin", dtype="<f8")
    ref = oracle.kernel_sum_direct(pr.x, pr.a, pr.y, kind, param)
    assert np.max(np.abs(s - ref) / np.abs(ref)) <= 1e-9
    r = oracle.uot_sinkhorn_direct(pr.x, pr.a, pr.y, pr.b, pr.eps, pr.lam, pr.lam, pr.iters)
    beta = np.fromfile(d / "beta.bin", dtype="<f8")
    gamma = np.fromfile(d / "gamma.bin", dtype="<f8")
    c = pr.lam / (1 + pr.lam / pr.eps)
    assert np.max(np.abs(beta - r.beta) / (np.abs(r.beta) + c)) <= 1e-8
    assert np.max(np.abs(gamma - r.gamma) / (np.abs(r.gamma) + c)) <= 1e-8
    primal, dual, mass, mmd2, iters, _ = (float(v) for v in (d / "scalars.txt").read_text().split())
    assert abs(primal - r.primal) <= 1e-8 * abs(r.primal) and abs(dual - r.dual) <= 1e-8 * abs(r.dual)
    mref = oracle.mmd2_direct(pr.x, pr.a, pr.y, pr.b, kind, param)
    xx = float(pr.a @ oracle.kernel_sum_direct(pr.x, pr.a, pr.x, kind, param))
    yy = float(pr.b @ oracle.kernel_sum_direct(pr.y, pr.b, pr.y, kind, param))
    assert abs(mmd2 - mref) / max(abs(mref), 1e-3 * (xx + yy)) <= 1e-8
