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


def generate_synthetic_shard(n, m, k_true, seed, lo, hi, spread=1.0, dtype=np.float32, chunk_rows=1 << 18):
    """Rows [lo, hi) of ``generate_synthetic_array(n, m, k_true, seed, spread, dtype)`` — the same
    bytes — without materialising the other n − (hi − lo) rows: the row-sharded bench gives every
    rank its contiguous shard of ONE dataset (partition.plan_chunks rule) at 64M points, where the
    full float64 array (12.8 GB) per rank would not fit 8 ranks on one host.

    Two passes over the generator stream: the first only advances it past the blob draws to the
    final permutation; the second regenerates the blob rows in chunks (the same sequence of
    standard normals, so the same values) and keeps the ones the permutation sends into [lo, hi)."""
    n = check_positive_int(n, name="n")
    m = check_positive_int(m, name="m")
    k_true = check_positive_int(k_true, name="k_true")
    if not 0 <= lo <= hi <= n:
        raise ContractViolationError(f"shard [{lo}, {hi}) outside [0, {n})")
    base, extra = divmod(n, k_true)
    sizes = [base + (1 if c < extra else 0) for c in range(k_true)]

    def draws(rng):  # (blob, first concatenated row, normals) in stream order
        row = 0
        for c, size in enumerate(sizes):
            for a in range(0, size, chunk_rows):
                b = min(size, a + chunk_rows)
                yield c, row + a, rng.standard_normal((b - a, m))
            row += size

    rng = np.random.default_rng(seed)
    centers = rng.uniform(-10.0, 10.0, size=(k_true, m))
    for _ in draws(rng):
        pass
    src = rng.permutation(n)[lo:hi]             # concatenated row of each output row
    order = np.argsort(src, kind="stable")
    src_sorted = src[order]
    out = np.empty((hi - lo, m), dtype=dtype)
    rng = np.random.default_rng(seed)
    rng.uniform(-10.0, 10.0, size=(k_true, m))
    for c, r0, z in draws(rng):
        a = np.searchsorted(src_sorted, r0)
        b = np.searchsorted(src_sorted, r0 + z.shape[0])
        if a < b:
            rows = (centers[c] + spread * z[src_sorted[a:b] - r0]).astype(dtype, copy=False)
            out[order[a:b]] = rows
    return out
