"""One BASELINE golden run in a fresh process (new CUDA context every time): the points are cached
as .npy under /tmp (scratch on the GPU box).  Usage: python tools/stress_fresh.py cfg5_3"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_3"
g = dict(np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / f"bench_{name}.npz"))
cache = Path(f"/tmp/km_points_{name}.npy")
if cache.exists():
    x = np.load(cache, mmap_mode="r")
else:
    x = generate_synthetic_array(int(g["n"]), int(g["m"]), int(g["k"]), seed=int(g["seed"]), dtype=np.float32)
    np.save(cache, x)
eng = _native.NativeEngine(0)
eng.load(np.ascontiguousarray(x))
c, n, l, it, conv = eng.lloyd(g["c0"], int(g["max_iters"]), float(g["tol"]))
st = eng.stats()
ok_n = np.array_equal(n, g["counts"])
ok_l = hashlib.sha256(l.astype(np.int64).tobytes()).hexdigest() == g["labels_sha256"].item().decode()
own = np.bincount(l, minlength=n.size)
print(f"{name}: it={it} counts_ok={ok_n} labels_ok={ok_l} counts==bincount(labels)={np.array_equal(own, n)} "
      f"rechecked={st['rechecked']} changed={st['changed']}", flush=True)
