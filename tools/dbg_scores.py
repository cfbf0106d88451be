import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
for (n,m,k) in [(200000,25,16),(4096,25,16),(4096,10,8)]:
    x = generate_synthetic_array(n, m, k, seed=11, dtype=np.float32)
    c = x[:k].astype(np.float64) + 0.37
    eng = _native.NativeEngine(0); eng.load(x)
    got = eng.debug_filter_scores(c)
    cf = c.astype(np.float32).astype(np.float64); xd = x.astype(np.float64)
    want = (cf*cf).sum(1)[None,:] - 2*xd@cf.T
    err = np.abs(got-want)
    bad = np.argwhere(err > 1e-2)
    print(n,m,k,"max err", err.max(), "nbad", len(bad), "first bad", bad[:5], got[bad[:3,0], bad[:3,1]] if len(bad) else "", want[bad[:3,0], bad[:3,1]] if len(bad) else "")
    rows = np.unique(bad[:,0]) if len(bad) else []
    print(" bad rows mod 128:", np.unique(np.asarray(rows) % 128)[:20], "count rows", len(rows), "tiles", np.unique(np.asarray(rows)//128)[:10])
