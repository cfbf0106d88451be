# cluster-sums: grouped form (W=4) vs per-row form (W=16), device time in the km_lloyd trace ([3])
mkdir -p gpurun_out
cat > /tmp/sums_ab.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
for name, (n, m, k, f64) in {"cfg2": (100_000, 10, 8, False), "cfg3": (2_000_000, 25, 16, False), "k64": (2_000_000, 25, 64, False),
                             "k128": (2_000_000, 25, 128, False), "cfg3_f64": (2_000_000, 25, 16, True)}.items():
    x = generate_synthetic_array(n, m, k, seed=0, dtype=None if f64 else np.float32)
    e = _native.NativeEngine(0); e.load(x)
    for _ in range(6):
        e.lloyd(x[:k].astype(np.float64), 1, 0.0, want_labels=False)
    print(name, file=sys.stderr, flush=True)
    e.close()
PY
for w in 4 16; do echo "KM_SUMS_W=$w"; KM_SUMS_W=$w KM_CALL_TRACE=1 timeout 300 python /tmp/sums_ab.py 2>&1 | grep -v "^$" | awk '/trace/{n++; if (n%6==0) print} !/trace/{print}'; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
