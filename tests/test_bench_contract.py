"""bench.py's JSON contract: the reference arm (the CPU oracle, no GPU needed) and a short
run of our arm (GPU) each print one JSON line with the keys the driver reads."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["metric"] == "UOT Sinkhorn iterations/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "workload" in line["config"]


@pytest.mark.gpu
def test_our_arm_json_line_short_run():
    """A short run of our arm (5 iterations, side legs off) on the GPU: the JSON line carries
    value, e2e, roofline (with the measured FP64 peak), clocks, gpu_launches and the MMD leg."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3", "--iters",
                          "5", "--no-c4", "--no-c1", "--no-m6", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.strip()][-1])
    assert line["value"] > 0 and line["unit"] == "iterations/s" and line["dtype"] == "f64"
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    roof = line["roofline"]
    assert roof["bound"] == "alu" and 0 < roof["frac"] <= 1.0 and roof["peak"] > 30
    assert line["gpu_launches"] > 0
    assert "sm_mhz" in line["clocks"]
    assert line["mmd2"]["value"] > 0
