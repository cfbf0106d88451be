"""Kernel-level timing of the first pass of a run: km_lloyd(max_iters=1) repeated, with CUDA
events around the call (used with ncu --metrics gpu__time_duration for per-kernel times)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

n, m, k = 2_000_000, 25, 16
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    eng.lloyd(x[:k].astype(np.float64), 1, 0.0, want_labels=False)
