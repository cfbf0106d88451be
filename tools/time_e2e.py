"""Break the bench's end-to-end fit (pinned H2D load + km_lloyd + int64 label D2H) into phases."""
import sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

n, m, k = 2_000_000, 25, 16
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
pinned = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = x
hx = pinned.numpy()
c0 = x[:k].astype(np.float64)
eng = _native.NativeEngine(0)
for rep in range(3):
    t0 = time.perf_counter()
    eng.load(hx)
    t1 = time.perf_counter()
    c, cnt, lab, it, conv = eng.lloyd(c0, 1000, 0.0, want_labels=False)
    t2 = time.perf_counter()
    c, cnt, lab, it, conv = eng.lloyd(c0, 1000, 0.0, want_labels=True)
    t3 = time.perf_counter()
    print(f"rep {rep}: load {1e3*(t1-t0):7.2f} ms  lloyd(no labels) {1e3*(t2-t1):7.2f} ms  lloyd(+labels) {1e3*(t3-t2):7.2f} ms  it={it}")
