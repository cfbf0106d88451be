"""Shared fixtures.  `-m gpu` tests need a B200 and the built CUDA engine;
`-m "not gpu"` tests run on CPU (oracle vs golden vectors, host logic, C ABI
exports, gloo multi-process host logic)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA engine")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build the in-tree native libraries once per session if stale."""
    from paper_1402_3788_b200 import build

    build.build_all()
    return True


@pytest.fixture
def rng():
    return np.random.default_rng(20260821)


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_indexed(name):
    """Split a fixture with keys '<field>_<idx>' into {idx: {field: value}}."""
    raw = np.load(GOLDEN / f"{name}.npz")
    out = {}
    for key in raw.files:
        field, idx = key.rsplit("_", 1)
        out.setdefault(int(idx), {})[field] = raw[key]
    return out


def random_coords(rng, n, m, kind=None):
    """Same generator families as the reference test suite (pkg/tests/conftest.py:16-35)."""
    kind = kind if kind is not None else rng.integers(3)
    if kind == 0:
        coords = rng.standard_normal((n, m)) * rng.uniform(0.5, 3.0)
    elif kind == 1:
        coords = rng.uniform(-50.0, 50.0, size=(n, m))
    else:
        blobs = int(rng.integers(2, 6))
        centers = rng.uniform(-20.0, 20.0, size=(blobs, m))
        which = rng.integers(blobs, size=n)
        coords = centers[which] + rng.standard_normal((n, m))
    if n > 16 and rng.random() < 0.3:
        dup = rng.integers(1, 5)
        src = rng.integers(n, size=dup)
        dst = rng.integers(n, size=dup)
        coords[dst] = coords[src]
    return np.ascontiguousarray(coords, dtype=np.float64)


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
