"""Repeat one BASELINE golden run many times on one engine (each km_lloyd call restarts from C0, so
every repetition must reproduce the reference bit for bit) — hunts timing-dependent races.
Usage: python tools/stress_golden.py cfg5_3 [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = dict(np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / f"bench_{name}.npz"))
x = generate_synthetic_array(int(g["n"]), int(g["m"]), int(g["k"]), seed=int(g["seed"]), dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
bad = 0
for r in range(reps):
    centers, counts, labels, iters, conv = eng.lloyd(g["c0"], int(g["max_iters"]), float(g["tol"]), want_labels=False)
    ok = iters == int(g["iterations"]) and np.array_equal(counts, g["counts"])
    if not ok:
        bad += 1
        d = counts - g["counts"]
        print(f"rep {r}: MISMATCH iterations {iters}, count diffs at {np.nonzero(d)[0][:8]} = {d[np.nonzero(d)[0][:8]]}", flush=True)
print(f"{name}: {reps - bad}/{reps} repetitions match the reference", flush=True)
