"""Synthetic workload generator — same draws as the reference's
datasets.generate_synthetic (/root/reference/pkg/src/kmeans_regimes/datasets.py:73-97):
``default_rng(seed)``, blob centres U[-10, 10]^m, near-equal blob sizes,
N(0, 1)·spread jitter, one global permutation.  Identical parameters give
identical bytes, so the bench, the parity tests and the reference all see the
same points.  ``dtype=np.float32`` returns the fp32 cast the B200 path streams
(the reference receives its exact float64 upcast)."""

import numpy as np

from .exceptions import ContractViolationError
from .validation import check_positive_int


def generate_synthetic_array(n, m, k_true, seed, spread=1.0, dtype=np.float64):
    n = check_positive_int(n, name="n")
    m = check_positive_int(m, name="m")
    k_true = check_positive_int(k_true, name="k_true")
    if k_true > n:
        raise ContractViolationError(f"k_true={k_true} exceeds sample count n={n}")
    if not spread >= 0.0:
        raise ContractViolationError(f"spread must be >= 0, got {spread}")
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-10.0, 10.0, size=(k_true, m))
    base, extra = divmod(n, k_true)
    parts = []
    for c in range(k_true):
        size = base + (1 if c < extra else 0)
        parts.append(centers[c] + spread * rng.standard_normal((size, m)))
    coords = np.concatenate(parts, axis=0)[rng.permutation(n)]
    return np.ascontiguousarray(coords.astype(dtype, copy=False))


def generate_synthetic(n, m, k_true, seed, spread=1.0):
    from .model import Dataset

    return Dataset(generate_synthetic_array(n, m, k_true, seed, spread), copy=False)
