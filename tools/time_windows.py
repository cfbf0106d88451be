"""Fused-pass device time per window of the Lloyd trajectory (deterministic, so
runs with max_iters T1 < T2 share their first T1 passes).
Usage: python tools/time_windows.py cfg3 [path]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg1": (10_000, 5, 4), "cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "cfg4": (2_000_000, 25, 512), "k64": (2_000_000, 25, 64), "k128": (2_000_000, 25, 128)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
path = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
eng.set_kernel_path(path)
c0 = x[:k].astype(np.float64)
eng.lloyd(c0, 3, 0.0, want_labels=False)
prev = None
for T in (1, 2, 3, 5, 10, 20, 50, 100, 200, 400):
    eng.reset_stats()
    eng.set_profiling(True)
    _, _, _, it, conv = eng.lloyd(c0, T, 0.0, want_labels=False)
    st = eng.stats()
    cur = (T, st["pass_ms_total"], st["pass_timed"], st["changed"], st["rechecked"])
    if prev:
        dt = (cur[1] - prev[1]) / max(1, cur[2] - prev[2])
        print(f"{name} iters ({prev[0]:3d},{T:3d}]: pass {dt*1e3:8.1f} us  {n*(4*m+4)/(dt*1e-3)/1e9:6.0f} GB/s  "
              f"changed/iter {(cur[3]-prev[3])/max(1,T-prev[0]):9.0f}  rechecked/iter {(cur[4]-prev[4])/max(1,T-prev[0]):7.0f}",
              flush=True)
    else:
        print(f"{name} first pass + 1 iter: {cur[1]/max(1,cur[2])*1e3:.1f} us/pass", flush=True)
    prev = cur
