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
