"""Device time of the update step (km_update: cluster sums + finish) at a BASELINE shape, CUDA
events on the engine stream; the labels are the first-K assignment.  Usage: python tools/time_sums.py cfg3"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

CFG = {"cfg2": (100_000, 10, 8), "cfg3": (2_000_000, 25, 16), "k64": (2_000_000, 25, 64), "k128": (2_000_000, 25, 128)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n, m, k = CFG[name]
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
s = torch.cuda.current_stream()
eng = _native.NativeEngine(0)
eng.set_stream(s.cuda_stream)
eng.load(x)
labels, _ = eng.assign(x[:k].astype(np.float64))
ts = []
for _ in range(30):
    lab = labels.copy()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    eng.update(lab, k)
    b.record(s)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
med = statistics.median(ts[5:])
print(f"{name} km_update (H2D 4n label bytes + sums + finish): {med:.1f} us; n*(4m+4) = {n*(4*m+4)/1e6:.0f} MB")
