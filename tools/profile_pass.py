"""Run a few device-resident Lloyd iterations at a BASELINE config (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

cfg = {"cfg3": (2_000_000, 25, 16), "cfg4": (2_000_000, 25, 512), "cfg2": (100_000, 10, 8),
       "cfg1": (10_000, 5, 4)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
path = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, m, k = cfg
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
eng = _native.NativeEngine(0)
eng.load(x)
eng.set_kernel_path(path)
c, cnt, lab, it, conv = eng.lloyd(x[:k].astype(np.float64), iters, 0.0)
print("iterations", it, "path", eng.kernel_path(), eng.stats())
