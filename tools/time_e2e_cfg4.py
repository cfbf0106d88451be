import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
n, m, k = 2_000_000, 25, 512
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
pinned = torch.empty((n, m), dtype=torch.float32, pin_memory=True); pinned.numpy()[:] = x; hx = pinned.numpy()
c0 = x[:k].astype(np.float64)
eng = _native.NativeEngine(0)
for rep in range(3):
    t0 = time.perf_counter(); eng.load(hx); t1 = time.perf_counter()
    c, cnt, l, it, conv = eng.lloyd(c0, 1000, 0.0, want_labels=True); t2 = time.perf_counter()
    st = eng.stats()
    print(f"load {1e3*(t1-t0):.1f} ms, lloyd {1e3*(t2-t1):.1f} ms ({it} its, {1e3*(t2-t1)/it:.2f} ms/it) repairs={st['repairs']} syncs={st['host_syncs']} launches={st['kernel_launches']}", flush=True)
    eng.reset_stats()
