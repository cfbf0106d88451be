import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
n = int(sys.argv[1]); T = int(sys.argv[2])
x = generate_synthetic_array(n, 25, 16, seed=0, dtype=np.float32)
e = _native.NativeEngine(0); e.load(x)
try:
    c, cnt, l, it, conv = e.lloyd(x[:16].astype(np.float64), T, 0.0, want_labels=False)
    print(n, T, "ok", it, conv, e.stats()["repairs"], flush=True)
except Exception as ex:
    print(n, T, "FAIL", ex, flush=True)
