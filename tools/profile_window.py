"""The bench's timed call for ncu: one km_lloyd(C0, max_iters=T) from the first-K start (launches:
begin, labels-only tensor-core pass, cluster sums, resident tensor-core loop, publish).  Profile the
resident loop with `ncu -k regex:lloyd_pass_tc -s 1 -c 1`, the sums with `-k regex:cluster_sums -c 1`.
Usage: python tools/profile_window.py cfg3 [T]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "k64": (2_000_000, 25, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
_, _, _, it, conv = eng.lloyd(x[:k].astype(np.float64), T, 0.0, want_labels=False)
print(f"{name}: km_lloyd from C0, {it} iterations, converged={conv}, stats={eng.stats()}")
