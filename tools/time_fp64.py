"""The fp64 input path: RegimeKMeans / km_load_points_f64 with data that is NOT fp32-representable
(datasets.generate_synthetic returns such float64 coordinates) keeps the points in fp64.  The
tensor-core pass streams their fp32 shadow for the certified filter and reads the exact fp64 rows
only for the recheck and the Δ of changed points (KM_NO_FP32_SHADOW=1: the SIMT fp64 pass instead).
Device time per Lloyd iteration at the cfg3 shape, from the first-K start (CUDA events around each
call), next to the fp32 path.  "GB/s of points" counts the caller's bytes (8 B per fp64 coordinate).
Usage: python tools/time_fp64.py [n m k]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

n, m, k = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (2_000_000, 25, 16)
x64 = generate_synthetic_array(n, m, k, seed=0)  # float64, not fp32-representable
s = torch.cuda.current_stream()
for name, x in (("fp32", x64.astype(np.float32)), ("fp64", x64)):
    eng = _native.NativeEngine(0)
    eng.set_stream(s.cuda_stream)
    eng.load(x)
    info = eng.points_info()
    c0 = x[:k].astype(np.float64)
    eng.lloyd(c0, 3, 0.0, want_labels=False)
    for T in (20, 100):
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            _, _, _, it, _ = eng.lloyd(c0, T, 0.0, want_labels=False)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / it)
        print(f"{name} points ({info['point_bytes']} B/coordinate, kernel path {eng.kernel_path()}): "
              f"{statistics.median(ts):.1f} us per iteration over {T} iterations "
              f"({n * m * info['point_bytes'] / statistics.median(ts) / 1e3:.0f} GB/s of points)", flush=True)
    eng.close()
