"""Average fused-pass device time (CUDA events inside km_lloyd) per BASELINE config.
Usage: [KM_LIB_VARIANT=w1] python tools/time_pass.py cfg3 [iters] [path]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg1": (10_000, 5, 4), "cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "cfg4": (2_000_000, 25, 512),
       "cfg5s": (8_000_000, 25, 64)}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg3"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
path = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for name in names:
    n, m, k = CFG[name]
    x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
    eng = _native.NativeEngine(0)
    eng.load(x)
    eng.set_kernel_path(path)
    c0 = x[:k].astype(np.float64)
    eng.lloyd(c0, 3, 0.0, want_labels=False)
    eng.reset_stats()
    eng.set_profiling(True)
    import time
    t0 = time.perf_counter()
    _, _, _, it, _ = eng.lloyd(c0, iters, 0.0, want_labels=False)
    el = time.perf_counter() - t0
    st = eng.stats()
    pass_ms = st["pass_ms_total"] / max(1, st["pass_timed"])
    gbs = n * (4 * m + 4) / (pass_ms * 1e-3) / 1e9
    print(f"{name}: path={eng.kernel_path()} pass {pass_ms*1e3:8.1f} us  ({gbs:6.0f} GB/s alg, {gbs/6534.1:.3f} of HBM)  "
          f"step {el/it*1e3:8.1f} us  rechecked/iter {st['rechecked']/max(1,st['passes']):.0f}", flush=True)
    eng.close()
