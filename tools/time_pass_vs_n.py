"""Resident pass time vs n (m = 25, k = 16): for each n, start from the centres of iteration
it_conv/3 and time km_lloyd calls of 10 and 60 iterations (CUDA events); (t60 − t10) / 50 is the
per-pass time without the call's fixed costs.  The intercept of time(n) = a + b·n is the fixed
per-pass cost (tail, grid barrier, pipeline drain / refill), the slope the streaming cost.
Usage: python tools/time_pass_vs_n.py"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

s = torch.cuda.current_stream()
res = []
for n in (500_000, 1_000_000, 2_000_000, 4_000_000, 8_000_000):
    x = generate_synthetic_array(n, 25, 16, seed=0, dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    eng = _native.NativeEngine(0)
    eng.set_stream(s.cuda_stream)
    eng.attach_device_f32(xd.data_ptr(), n, 25)
    c0 = x[:16].astype(np.float64)
    _, _, _, it_conv, _ = eng.lloyd(c0, 2000, 0.0, want_labels=False)
    cw, _, _, _, _ = eng.lloyd(c0, max(1, it_conv // 3), 0.0, want_labels=False)

    def t(T):
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            _, _, _, it, _ = eng.lloyd(cw, T, 0.0, want_labels=False)
            b.record(s)
            torch.cuda.synchronize()
            assert it == T
            ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts)

    per = (t(60) - t(10)) / 50
    res.append((n, per))
    print(f"n={n:>9}: {per:6.1f} us per pass (iterations {it_conv // 3}..{it_conv // 3 + 60} of {it_conv})", flush=True)
    eng.close()
ns = np.array([r[0] for r in res], float)
ts = np.array([r[1] for r in res])
b, a = np.polyfit(ns, ts, 1)
print(f"fit: {a:.1f} us + {b * 1e6:.2f} us per 1M rows (stream at 6458 GB/s: {104e6 / 6458e3:.2f} us per 1M rows)", flush=True)
