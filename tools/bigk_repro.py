import sys, numpy as np
sys.path.insert(0, '.')
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
n, m, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
x = generate_synthetic_array(n, m, 64, seed=1, dtype=np.float32)
eng = _native.NativeEngine(0); eng.load(x); eng.set_kernel_path(2)
try:
    labels, counts = eng.assign(x[:k].astype(np.float64)); print("assign ok", counts.sum())
except Exception as e: print("assign failed:", e); sys.exit(1)
try:
    c, cnt, lab, it, conv = eng.lloyd(x[:k].astype(np.float64), 3, 0.0); print("lloyd ok", it)
except Exception as e: print("lloyd failed:", e)
