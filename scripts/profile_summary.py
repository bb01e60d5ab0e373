"""Summaries committed under profiles/ from ncu outputs brought back in gpurun_out/.

  python scripts/profile_summary.py full  <report.ncu-rep> <kernel-regex> <out.md> [traffic.json tag]
  python scripts/profile_summary.py list  <launches.csv> <out.md>

`full` writes the key metrics of one `ncu --set full` capture (and, with a tag, records
dram read+write bytes per launch into profiles/ncu_traffic.json for bench.py);
`list` aggregates a `--metrics gpu__time_duration.sum` launch list into per-kernel
totals and shares (cold-cache, serialised: compare shares, not absolute times).
"""

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe busy (% of active)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe busy (% of active)"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "tensor FP64 ops (% of peak, elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth achieved"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread instructions"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread instructions"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread instructions"),
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def full(rep, pat, out, tag=None):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    rx = re.compile(pat)
    lines = [f"# ncu --set full: `{os.path.basename(rep)}` (kernels matching `{pat}`)\n"]
    traffic = []
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")]
        if not rx.search(name):
            continue
        lines.append(f"## {name[:160]}\n")
        lines.append("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {label} (`{k}`) | {row[i]} {units[i]} |")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(row[i]), h.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        lines.append("\nwarp stalls per issued instruction: " +
                     ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]) + "\n")
        try:
            fl = sum(float(row[hdr.index(k)].replace(",", "")) * w for k, w in (
                ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 2),
                ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 1),
                ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 1)))
            dur = float(row[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            dur *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}[units[hdr.index("gpu__time_duration.sum")]]
            lines.append(f"scalar FP64 (2 DFMA + DADD + DMUL, DMMA excluded): {fl / dur / 1e12:.2f} TFLOP/s\n")
        except (ValueError, KeyError, IndexError):
            pass
        rd = to_bytes(row[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(row[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        traffic.append(rd + wr)
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if tag and traffic:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[tag] = sum(traffic) / len(traffic)
        d[f"{tag}_source"] = os.path.relpath(out, ROOT)
        json.dump(d, open(path, "w"), indent=1)
    print(f"wrote {out}")


def launch_list(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki])[:90]
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# ncu launch list: `{os.path.basename(path)}`\n",
             "Cold-cache, serialised per-launch times (`gpu__time_duration.sum`, `--clock-control none`);",
             "compare shares, not absolute values.\n",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{name}` | {cnt[name]} | {v:.1f} | {100 * v / total:.1f}% |")
    lines.append(f"| **all** | {sum(cnt.values())} | {total:.1f} | 100% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"wrote {out}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
    else:
        launch_list(sys.argv[2], sys.argv[3])
