"""Tensor-core pass (path 2) under adversarial inputs, each against the C oracle
(the reference restatement, `oracle/kmeans_oracle.c`).

* magnitudes past the filter's certified range (|x| > 2^50: `exact_only`, every
  real centre re-evaluated in fp64) with k not a multiple of 16, so padded
  centres exist and must never become candidates;
* caller-supplied centres far outside the data range (predict-style
  `km_assign`, and as C0 of a fit) with k = 15 (one padded slot);
* lattice ties and duplicated centres at >= 1M points: every tied point fails
  the certificate and the recheck must return the lowest index, as the
  reference's strict '<' (`_kernels.py:36-43`);
* large common offsets (|x| ~ 1e3, spread ~1e-2): the fp16 hi/lo scores lose
  most of their bits to cancellation, the bound must still hold.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CENTER_RTOL = 1e-12


def rel_err(a, b, floor=1.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


@pytest.fixture(scope="module")
def native():
    from paper_1402_3788_b200 import _native

    return _native


def fit(native, x, c0, iters, path=2):
    eng = native.NativeEngine(0)
    eng.load(x)
    eng.set_kernel_path(path)
    centers, counts, labels, it, conv = eng.lloyd(c0, iters, 0.0)
    st = eng.stats()
    used = eng.kernel_path()
    eng.close()
    return dict(centers=centers, counts=counts, labels=labels, iterations=it, converged=conv, stats=st, path=used)


def check_vs_oracle(want, got, name, floor=1.0):
    assert got["iterations"] == want["iterations"], name
    assert got["converged"] == want["converged"], name
    assert np.array_equal(got["labels"], want["labels"]), name
    assert np.array_equal(got["counts"], want["counts"]), name
    assert rel_err(got["centers"], want["centers"], floor) <= CENTER_RTOL, name


@pytest.mark.parametrize("k", [40, 15, 1, 3])
def test_tc_exact_only_padded_centres(native, k):
    """|x| > 2^50: the filter threshold is +inf, so every centre is a candidate — but only the k
    real ones (the KP − k padded slots must never be read or win)."""
    from oracle import oracle

    rng = np.random.default_rng(100 + k)
    x = (rng.standard_normal((40_000, 13)) * 2.0 ** 55).astype(np.float32)
    c0 = x[:k].astype(np.float64)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=5, n_workers=8)
    got = fit(native, x, c0, 5)
    assert got["path"] == 2
    assert got["labels"].max() < k and got["labels"].min() >= 0
    assert got["iterations"] == want["iterations"] and np.array_equal(got["labels"], want["labels"])
    assert np.array_equal(got["counts"], want["counts"])
    assert rel_err(got["centers"] / 2.0 ** 55, want["centers"] / 2.0 ** 55) <= 1e-9


@pytest.mark.parametrize("scale", [100.0, 1e4, 1e-3])
def test_tc_assign_centres_outside_data_range(native, scale):
    """predict()-style assignment with centres `scale`× the data range and k = 15: the fp16 operand
    scale must cover the centres too, or real scores overflow past the +65504 padding score."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    k = 15
    x = generate_synthetic_array(60_000, 25, 8, seed=3, dtype=np.float32)
    rng = np.random.default_rng(7)
    c = rng.standard_normal((k, 25)) * np.abs(x).max() * scale
    eng = native.NativeEngine(0)
    eng.load(x)
    eng.set_kernel_path(2)
    labels, counts = eng.assign(c)
    assert eng.kernel_path() == 2
    eng.close()
    want_l, want_c = oracle.assign(x.astype(np.float64), c, n_workers=8)
    assert labels.max() < k
    assert np.array_equal(labels, want_l)
    assert np.array_equal(counts, want_c)
    # and as C0 of a fit
    want = oracle.lloyd(x.astype(np.float64), c, max_iters=6, n_workers=8)
    check_vs_oracle(want, fit(native, x, c, 6), f"fit from C0 x{scale}")


def test_tc_lattice_ties_duplicated_centres_1m(native):
    """1M integer-lattice points, duplicated centres: exact ties everywhere (lowest index wins)."""
    from oracle import oracle

    rng = np.random.default_rng(21)
    x = rng.integers(-3, 4, size=(1_000_000, 6)).astype(np.float32)
    k = 24
    c0 = x[:k].astype(np.float64).copy()
    c0[12:] = c0[:12]  # every centre has a twin with a higher index
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=6, n_workers=8)
    got = fit(native, x, c0, 6)
    assert got["path"] == 2
    check_vs_oracle(want, got, "lattice ties 1M")
    assert got["stats"]["rechecked"] > 0


def test_tc_large_offset_cancellation(native):
    """Common offset 1e3 with 1e-2 spread: S = ‖c‖² − 2x·c cancels ~10 of its bits."""
    from oracle import oracle

    rng = np.random.default_rng(5)
    base = rng.uniform(-1, 1, size=(6, 17)) * 0.05
    which = rng.integers(6, size=300_000)
    x = (1000.0 + base[which] + rng.standard_normal((300_000, 17)) * 0.01).astype(np.float32)
    c0 = x[:16].astype(np.float64)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=8, n_workers=8)
    got = fit(native, x, c0, 8)
    assert got["path"] == 2
    check_vs_oracle(want, got, "offset 1e3")
