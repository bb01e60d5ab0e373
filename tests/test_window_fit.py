"""Host-side check of the piecewise-polynomial Kaiser-Bessel window (csrc/window_fit.h)
that the window-block precomputation evaluates: compiled with g++ against the header and
compared with the window's closed form evaluated in 30-digit arithmetic (mpmath), no GPU."""

import os
import subprocess

import pytest

mp = pytest.importorskip("mpmath")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2306_13618_b200", "csrc")

PROG = r"""
#include <cstdio>
#include <cstdlib>
#include "window_fit.h"
int main(int argc, char** argv) {
    const int m = atoi(argv[1]);
    const double b = atof(argv[2]);
    const uotk::KBHorner h = uotk::kb_horner_fit(b, m);
    for (int a = 0; a < 2 * m; ++a)
        for (int i = 1; i < 40; ++i) {
            const double f = i / 40.0, t = f - 0.5;
            double v = h.c[a][uotk::kHornerDeg];
            for (int j = uotk::kHornerDeg - 1; j >= 0; --j) v = __builtin_fma(v, t, h.c[a][j]);
            printf("%d %.17g %.17g\n", a, f, v);
        }
}
"""


def phi(v, m, b):
    """KB window normalised to phi(0) = 1 (window.cuh): sinh(b s)/s * m/sinh(b m), s = sqrt(m^2 - v^2)."""
    s2 = m * m - v * v
    if s2 <= 0:
        return mp.mpf(0)
    s = mp.sqrt(s2)
    return mp.sinh(b * s) / s * m / mp.sinh(b * m)


@pytest.mark.parametrize("m,sigma", [(8, 2.0), (6, 3.0), (8, 2.0833333333333335)])
def test_horner_window_matches_closed_form(tmp_path, m, sigma):
    src = tmp_path / "fit.cpp"
    src.write_text(PROG)
    exe = tmp_path / "fit"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    b = mp.pi * (2 - mp.mpf(1) / sigma)
    out = subprocess.run([str(exe), str(m), repr(float(b))], capture_output=True, text=True, check=True).stdout
    mp.mp.dps = 30
    worst = 0.0
    rows = [ln.split() for ln in out.strip().splitlines()]
    assert len(rows) == 2 * m * 39
    for a, f, v in rows:
        a, f, v = int(a), mp.mpf(f), float(v)
        worst = max(worst, abs(v - float(phi(f + m - 1 - a, m, mp.mpf(float(b))))))
    assert worst <= 4e-16, worst
