"""Per-opcode and per-region warp-stall samples of one kernel in an ncu report (needs -lineinfo
and --import-source).  usage: python scripts/ncu_sass_hot.py report.ncu-rep [window]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
hdr = rows[h]
si, wi, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
seq = []
for r in rows[h + 1:]:
    if len(r) <= wi:
        break
    try:
        seq.append((int(r[wi]), int(r[ei]), r[si].strip()))
    except ValueError:
        break
tot = sum(x[0] for x in seq)
ops = collections.Counter()
for v, e, s in seq:
    tok = s.split()
    op = tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "")
    ops[op.split(".")[0]] += v
print("total samples", tot, "instructions", len(seq))
print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(14)))
regions = []
for i in range(0, len(seq), win):
    chunk = seq[i:i + win]
    regions.append((sum(x[0] for x in chunk), i, collections.Counter(x[2].split()[0].split(".")[0] for x in chunk).most_common(4)))
for v, i, c in sorted(regions, reverse=True)[:10]:
    print(f"  [{i:5d}..{i + win:5d}) {100 * v / tot:5.1f}%  {c}")

# segments between barriers (BAR.SYNC), with DFMA counts
bars = [i for i, x in enumerate(seq) if "BAR.SYNC" in x[2]]
prev = 0
print("segments between BAR.SYNC:")
for b in bars + [len(seq)]:
    part = seq[prev:b]
    s = sum(x[0] for x in part)
    nd = sum(1 for x in part if x[2].startswith("DFMA") or x[2].startswith("@") and "DFMA" in x[2])
    ex = sum(x[1] for x in part if "DFMA" in x[2])
    print(f"  [{prev:5d}..{b:5d})  {100 * s / max(tot, 1):5.1f}%  static DFMA {nd:4d}  executed DFMA {ex}")
    prev = b
