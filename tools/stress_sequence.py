"""The tests/test_gpu_bench_configs.py sequence in one process (a fresh engine per golden, closed
after), repeated — hunts state- or timing-dependent failures.  Usage: python tools/stress_sequence.py [rounds]"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array

G = Path(__file__).resolve().parent.parent / "tests" / "golden"
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cache = {}
fails = 0
for rnd in range(rounds):
    for name in ["cfg2", "cfg3", "cfg3_20", "cfg4_20", "cfg5_3"]:
        g = dict(np.load(G / f"bench_{name}.npz"))
        key = (int(g["n"]), int(g["m"]), int(g["k"]), int(g["seed"]))
        if key not in cache:
            cache.clear()
            cache[key] = generate_synthetic_array(key[0], key[1], key[2], seed=key[3], dtype=np.float32)
        x = cache[key]
        eng = _native.NativeEngine(0)
        eng.load(x)
        c, n, l, it, conv = eng.lloyd(g["c0"], int(g["max_iters"]), float(g["tol"]))
        st = eng.stats()
        eng.close()
        ok = it == int(g["iterations"]) and np.array_equal(n, g["counts"])
        if "labels_sha256" in g:
            ok = ok and hashlib.sha256(l.astype(np.int64).tobytes()).hexdigest() == g["labels_sha256"].item().decode()
        elif "labels" in g:
            ok = ok and np.array_equal(l, g["labels"].astype(np.int64))
        if not ok:
            fails += 1
            d = n - g["counts"]
            nz = np.nonzero(d)[0]
            print(f"round {rnd} {name}: MISMATCH it={it} rechecked={st['rechecked']} count diffs {list(zip(nz[:6], d[nz[:6]]))}", flush=True)
print(f"{rounds} rounds, {fails} mismatches", flush=True)
