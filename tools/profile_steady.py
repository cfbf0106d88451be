"""Steady-state resident Lloyd launch for ncu: run `warm` iterations from the first-K
start (one launch), then `iters` more from those centres (the launch to profile:
ncu -k regex:lloyd_pass_tc -s 1 -c 1).  Usage: python tools/profile_steady.py cfg3 400 50"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg1": (10_000, 5, 4), "cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "cfg4": (2_000_000, 25, 512),
       "k64": (2_000_000, 25, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 400
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
c_mid, _, _, it0, _ = eng.lloyd(x[:k].astype(np.float64), warm, 0.0, want_labels=False)
eng.reset_stats()
c, cnt, _, it, conv = eng.lloyd(c_mid, iters, 0.0, want_labels=False)
st = eng.stats()
print(f"warm {it0} iterations, profiled launch: {it} iterations (converged={conv}), passes={st['passes']}, "
      f"rechecked={st['rechecked']}, changed={st['changed']}, launches={st['kernel_launches']}")
