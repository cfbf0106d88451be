"""Device time of whole km_lloyd calls (CUDA events on the engine stream around the call, as the
bench), for max_iters T = 1, 2, 3, 5, 10, 20 from the first-K start.  Usage: python tools/time_call.py cfg3"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg1": (10_000, 5, 4), "cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "cfg4": (2_000_000, 25, 512),
       "k64": (2_000_000, 25, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
xd = torch.from_numpy(x).cuda()
s = torch.cuda.current_stream()
eng = _native.NativeEngine(0)
eng.set_stream(s.cuda_stream)
eng.attach_device_f32(xd.data_ptr(), n, m)
c0 = x[:k].astype(np.float64)
eng.lloyd(c0, 3, 0.0, want_labels=False)
for T in (1, 2, 3, 5, 10, 20, 50):
    ts = []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        eng.lloyd(c0, T, 0.0, want_labels=False)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    med = statistics.median(ts)
    print(f"{name} km_lloyd max_iters={T:3d}: {med:8.1f} us per call, {med / T:7.1f} us per iteration", flush=True)
