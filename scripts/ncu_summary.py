"""Summarise an ncu report: key throughput metrics, stall reasons, hot SASS opcodes.
usage: python scripts/ncu_summary.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
keys = ["gpu__time_duration.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for row in raw[2:]:
    name = row[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    print("==", name[:110])
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"   {k} = {row[i]} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(row[i]), h.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
