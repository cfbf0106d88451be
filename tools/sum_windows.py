"""Summarise tools/time_windows.py logs: trajectory-average pass time over the first 400
iterations and the steady (200, 400] window, per variant block ('=== name')."""
import re
import sys

cur = None
res = {}
for l in open(sys.argv[1]):
    if l.startswith("==="):
        cur = l.strip("= \n")
        res.setdefault(cur, [])
        tot = 0.0
        continue
    m = re.search(r"first pass \+ 1 iter: ([\d.]+)", l)
    if m:
        tot = 2 * float(m.group(1))
        first = float(m.group(1))
        continue
    m = re.search(r"iters \(\s*(\d+),\s*(\d+)\]: pass\s+([\d.]+)", l)
    if m:
        a, b, t = int(m.group(1)), int(m.group(2)), float(m.group(3))
        tot += (b - a) * t
        if b == 400:
            res[cur].append((round(tot / 401, 2), t, first))
for k, v in res.items():
    print(f"{k:10s} avg/steady/first: {v}")
