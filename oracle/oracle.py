"""ctypes wrapper of the C oracle (oracle/kmeans_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline and --impl reference legs) as the checker / CPU
baseline.  The product package (paper_1402_3788_b200/) never imports this.

Every function restates the reference (/root/reference/pkg/src/kmeans_regimes)
with the same fp64 rounding sequence; see the file:line map at the top of
kmeans_oracle.c.  Pinned against the reference's own outputs in
tests/golden/ (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libkmeans_oracle.so"
DEFAULT_BLOCK = 65536  # model.py:24

_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        import sys

        sys.path.insert(0, str(HERE.parent))
        from paper_1402_3788_b200 import build as _build

        _build.build_oracle()
    lib = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.c_void_p
    I = ctypes.c_int64
    lib.ko_assign_block.argtypes = [P, I, P, I, P, I, I]
    lib.ko_assign_parallel.argtypes = [P, I, I, P, I, P, P, ctypes.c_int]
    lib.ko_update_parallel.argtypes = [P, I, I, P, I, I, P, P, ctypes.c_int]
    lib.ko_update_parallel.restype = I
    lib.ko_converged.argtypes = [P, P, I, I, ctypes.c_double]
    lib.ko_converged.restype = ctypes.c_int
    lib.ko_squared_distance.argtypes = [P, P, I]
    lib.ko_squared_distance.restype = ctypes.c_double
    lib.ko_wcss.argtypes = [P, I, I, P, P, I]
    lib.ko_wcss.restype = ctypes.c_double
    lib.ko_self_distances.argtypes = [P, I, P, P, I, I, P]
    lib.ko_iterate.argtypes = [P, I, I, P, I, I, ctypes.c_double, I, ctypes.c_int, P, P, P,
                               ctypes.POINTER(ctypes.c_int)]
    lib.ko_iterate.restype = I
    lib.ko_cluster_sums_block.argtypes = [P, I, P, I, I, I, P, P]
    lib.ko_cluster_sums_block.restype = I
    _lib = lib
    return lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def assign(coords, centers, n_workers=1):
    """engine.assign_step / partition.assign_parallel → (labels int64, counts int64)."""
    lib = _load()
    coords = _f64(coords)
    centers = _f64(centers)
    n, m = coords.shape
    k = centers.shape[0]
    labels = np.empty(n, dtype=np.int64)
    counts = np.zeros(k, dtype=np.int64)
    lib.ko_assign_parallel(_ptr(coords), n, m, _ptr(centers), k, _ptr(labels), _ptr(counts), int(n_workers))
    return labels, counts


def update(coords, labels, k, block=DEFAULT_BLOCK, n_workers=1):
    """engine.update_step → (centers, counts, labels-after-repair)."""
    lib = _load()
    coords = _f64(coords)
    n, m = coords.shape
    labels = np.array(labels, dtype=np.int64, copy=True)
    centers = np.empty((k, m), dtype=np.float64)
    counts = np.zeros(k, dtype=np.int64)
    bad = lib.ko_update_parallel(_ptr(coords), n, m, _ptr(labels), k, block, _ptr(centers), _ptr(counts),
                                 int(n_workers))
    if bad >= 0:
        raise ValueError(f"label out of range [0, {k}) at sample {bad}")
    return centers, counts, labels


def converged(prev, nxt, tol):
    lib = _load()
    prev = _f64(prev)
    nxt = _f64(nxt)
    k, m = prev.shape
    return bool(lib.ko_converged(_ptr(prev), _ptr(nxt), k, m, float(tol)))


def wcss(coords, centers, labels, block=DEFAULT_BLOCK):
    lib = _load()
    coords = _f64(coords)
    centers = _f64(centers)
    labels = np.ascontiguousarray(labels, dtype=np.int64)
    n, m = coords.shape
    return float(lib.ko_wcss(_ptr(coords), n, m, _ptr(centers), _ptr(labels), block))


def self_distances(coords, centers, labels):
    lib = _load()
    coords = _f64(coords)
    centers = _f64(centers)
    labels = np.ascontiguousarray(labels, dtype=np.int64)
    n, m = coords.shape
    out = np.empty(n, dtype=np.float64)
    lib.ko_self_distances(_ptr(coords), m, _ptr(centers), _ptr(labels), 0, n, _ptr(out))
    return out


def lloyd(coords, c0, max_iters=1000, tol=0.0, block=DEFAULT_BLOCK, n_workers=1):
    """engine.iterate from explicit initial centres → dict like tests/oracles.oracle_lloyd."""
    lib = _load()
    coords = _f64(coords)
    c0 = _f64(c0)
    n, m = coords.shape
    k = c0.shape[0]
    centers = np.empty((k, m), dtype=np.float64)
    counts = np.zeros(k, dtype=np.int64)
    labels = np.empty(n, dtype=np.int64)
    conv = ctypes.c_int(0)
    iters = lib.ko_iterate(_ptr(coords), n, m, _ptr(c0), k, int(max_iters), float(tol), block, int(n_workers),
                           _ptr(centers), _ptr(counts), _ptr(labels), ctypes.byref(conv))
    return {"labels": labels, "centers": centers, "counts": counts, "iterations": int(iters),
            "converged": bool(conv.value)}


def cpu_count():
    return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# Seeding, restated in numpy: elementwise fp64 operations in the
# reference's feature order (numpy never fuses a multiply-add), so every squared
# distance is bit-identical to the numba kernels.
# ---------------------------------------------------------------------------
class DegenerateData(Exception):
    """engine.py:162-168 / :190-193 (DegenerateDataError)."""


def scan_rows(n, pair_cap=None):
    """engine.scan_rows (engine.py:124-138)."""
    import math

    if n < 2:
        return np.empty(0, dtype=np.int64)
    total = n * (n - 1) // 2
    if pair_cap is None or total <= pair_cap:
        return np.arange(n - 1, dtype=np.int64)
    stride = max(2, math.ceil(total / pair_cap))
    return np.arange(0, n - 1, stride, dtype=np.int64)


def diameter(coords, pair_cap=None):
    """engine.diameter + _kernels.max_pair_rows (engine.py:141-154, _kernels.py:49-81):
    rows ascending, j > i ascending, d² = Σ_f (x_if − x_jf)² left to right, strict '>'
    (the first maximum in scan order = smallest (i, j)).  Returns (d, i, j)."""
    x = _f64(coords)
    n, m = x.shape
    best, bi, bj = -1.0, -1, -1
    for i in scan_rows(n, pair_cap):
        rest = x[i + 1:]
        d2 = np.zeros(rest.shape[0])
        for f in range(m):
            d = x[i, f] - rest[:, f]
            d2 += d * d
        if d2.size:
            jj = int(np.argmax(d2))
            if d2[jj] > best:
                best, bi, bj = float(d2[jj]), int(i), int(i + 1 + jj)
    return float(np.sqrt(best)), bi, bj


def max_pair_rows(coords, rows):
    """_kernels.max_pair_rows (_kernels.py:48-81) over an explicit ascending row list (the
    MAX_PAIR device job, device.py:204-216): (d2, i, j), (-1.0, -1, -1) when no pair."""
    x = _f64(coords)
    best, bi, bj = -1.0, -1, -1
    for i in np.asarray(rows, dtype=np.int64):
        rest = x[i + 1:]
        d2 = np.zeros(rest.shape[0])
        for f in range(x.shape[1]):
            d = x[i, f] - rest[:, f]
            d2 += d * d
        if d2.size:
            jj = int(np.argmax(d2))
            if d2[jj] > best:
                best, bi, bj = float(d2[jj]), int(i), int(i + 1 + jj)
    return best, bi, bj


def block_sums(coords, start, stop, block, labels=None, k=1):
    """HostReferenceDevice._execute sum jobs (device.py:218-239): per-block sequential fp64 sums
    (_kernels.cluster_sums_block, _kernels.py:97-113; coord_sums_block = every label 0).
    Returns (sums, counts, bad) with bad = the first out-of-range sample or -1."""
    lib = _load()
    x = _f64(coords)
    n, m = x.shape
    lab = np.zeros(n, dtype=np.int64) if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
    kk = 1 if labels is None else int(k)
    bounds = [(s, min(s + block, stop)) for s in range(start, stop, block)]
    sums = np.zeros((len(bounds), kk, m))
    counts = np.zeros((len(bounds), kk), dtype=np.int64)
    for b, (s, e) in enumerate(bounds):
        bad = lib.ko_cluster_sums_block(_ptr(x), m, _ptr(lab), kk, s, e, _ptr(sums[b]), _ptr(counts[b]))
        if bad >= 0:
            return None, None, int(bad)
    if labels is None:
        return sums[:, 0, :], None, -1
    return sums, counts, -1


def _lower_min_d2(x, c, min_d2):
    """_kernels.update_min_d2 (_kernels.py:144-155)."""
    d2 = np.zeros(x.shape[0])
    for f in range(x.shape[1]):
        d = x[:, f] - x[c, f]
        d2 += d * d
    np.minimum(min_d2, d2, out=min_d2)


def init_centers(coords, k, init="maximin", seed=0, diam=None):
    """engine.init_centers (engine.py:171-215) → (k, m) initial centres."""
    x = _f64(coords)
    n = x.shape[0]
    if diam is None:
        diam = diameter(x)
    d, i0, j0 = diam
    min_d2 = np.full(n, np.inf)
    chosen = []

    def append(idx):
        chosen.append(int(idx))
        _lower_min_d2(x, int(idx), min_d2)

    def farthest():
        idx = int(np.argmax(min_d2))
        if min_d2[idx] == 0.0:
            raise DegenerateData("dataset has fewer distinct points than requested centers")
        return idx

    if init == "maximin":
        append(i0)
        if k >= 2:
            if d == 0.0:
                raise DegenerateData("dataset has fewer distinct points than requested centers")
            append(j0)
        while len(chosen) < k:
            append(farthest())
    else:
        rng = np.random.default_rng(seed)
        thr2 = (d / (2.0 * k)) ** 2
        draws, limit = 0, 10 * n
        while len(chosen) < k:
            accepted = False
            while draws < limit:
                cand = int(rng.integers(n))
                draws += 1
                if not chosen or min_d2[cand] > thr2:
                    append(cand)
                    accepted = True
                    break
            if not accepted:
                append(farthest())
    return x[np.asarray(chosen, dtype=np.int64)].copy()
