"""Warp-stall samples of one kernel in an ncu report (--set full, --import-source), summed over
windows of consecutive SASS instructions: share of samples, top stall reasons, DMMA count and
opcodes per window.  usage: python scripts/ncu_stall_regions.py report.ncu-rep [window]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; win = int(sys.argv[2]) if len(sys.argv) > 2 else 48
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
hdr = rows[h]
# newer ncu: one section per profiled launch ("Kernel Name" row, header row, instructions);
# keep the first launch's instructions only
end = next((i for i in range(h + 1, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
rows = rows[:end]
si = hdr.index("Source"); wi = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
ins = []
for r in rows[h+1:]:
    if len(r) <= max(stall_cols + [wi]): continue
    try: ins.append((r[si].strip(), int(r[wi] or 0), [int(r[i] or 0) for i in stall_cols], int(r[hdr.index("Instructions Executed")] or 0)))
    except ValueError: pass
tot = sum(x[1] for x in ins)
print("total samples", tot, "instructions", len(ins))
for w0 in range(0, len(ins), win):
    seg = ins[w0:w0+win]
    s = sum(x[1] for x in seg)
    if s < 0.01 * tot: continue
    agg = [sum(x[2][k] for x in seg) for k in range(len(stall_cols))]
    top = sorted(zip(agg, [hdr[i][6:] for i in stall_cols]), reverse=True)[:4]
    ops = collections.Counter(x[0].split()[0] if not x[0].startswith('@') else x[0].split()[1] for x in seg)
    dmma = sum(1 for x in seg if 'DMMA' in x[0])
    print(f"[{w0:5d}..{w0+win:5d}) {100*s/tot:5.1f}%  " + ", ".join(f"{n} {100*a/max(s,1):.0f}%" for a, n in top) + f" | DMMA {dmma} | " + " ".join(f"{k}:{v}" for k, v in ops.most_common(5)))
