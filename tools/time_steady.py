"""Steady-state pass time: warm the first-K trajectory to iteration `warm`, then time one resident
km_lloyd call of `iters` iterations from those centres (device time of the launches / passes).
Usage: python tools/time_steady.py cfg3 [warm] [iters]   (KM_TC_DBG / KM_LIB_VARIANT for experiments)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg3": (2_000_000, 25, 16), "k64": (2_000_000, 25, 64), "k128": (2_000_000, 25, 128),
       "cfg5": (64_000_000, 25, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 400
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
c, _, _, it0, _ = eng.lloyd(x[:k].astype(np.float64), warm, 0.0, want_labels=False)
res = []
for rep in range(3):
    eng.reset_stats()
    eng.set_profiling(True)
    eng.lloyd(c, iters, 0.0, want_labels=False)
    st = eng.stats()
    res.append(st["pass_ms_total"] / max(1, st["pass_timed"]) * 1e3)
print(f"{name} dbg={os.environ.get('KM_TC_DBG', '0')} variant={os.environ.get('KM_LIB_VARIANT', '-')}: "
      f"{min(res):.1f} us/pass (from iteration {it0}, {iters} iterations, first pass + sums included)", flush=True)
