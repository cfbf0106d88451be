"""Per-opcode / per-region instruction histogram of one kernel from an ncu report
(`ncu -i REP --page source --csv --print-source sass`).  Usage: python tools/sass_hist.py REP [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}
ops = collections.Counter(); tot = 0; seq = []
for r in rows[2:]:
    if len(r) < len(h): continue
    n = int(r[idx["Instructions Executed"]] or 0)
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    ops[op.split(".")[0]] += n; tot += n
    seq.append((r[idx["Address"]], src, n, int(r[idx["# Samples"]] or 0)))
print(f"total warp instructions executed: {tot}")
for op, n in ops.most_common(top): print(f"{op:14s} {n:12d} {100*n/tot:6.2f}%")
if "--hot" in sys.argv:
    for a, s, n, smp in seq:
        if n > tot * 0.0015: print(f"{a[-5:]} {n:10d} {smp:6d}  {s}")
