"""Time the device seeding at the headline shape: diameter (capped and uncapped) + maximin."""
import sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import KmeansConfig, diameter, init_centers
from paper_1402_3788_b200.datasets import generate_synthetic_array
from paper_1402_3788_b200.model import Dataset

n, m, k = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2_000_000, 25, 16)
x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
ds = Dataset(x)
ds.device_engine()
for cap in (2_000_000, 2_000_000_000, None):
    t0 = time.perf_counter()
    d = diameter(ds, pair_cap=cap)
    t1 = time.perf_counter()
    c = init_centers(ds, KmeansConfig(k=k), d)
    t2 = time.perf_counter()
    print(f"n={n} m={m} k={k} pair_cap={cap}: diameter {d.d:.6f} ({d.i},{d.j}) in {t1-t0:.3f} s; "
          f"maximin {k} centres in {1e3*(t2-t1):.1f} ms", flush=True)
