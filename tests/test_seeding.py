"""Seeding phase: the dataset diameter and the maximin /
random-far initial centres, then the full default fit (RegimeKMeans / run_b200
without explicit centres).

CPU tests pin the numpy restatement (oracle/oracle.py) to vectors produced by
the real reference (oracle/make_golden.py → tests/golden/seeding.npz).  GPU
tests check the device (km_diameter, km_seed_*) against both: diameter value
and pair bit-exact, initial centres bit-exact, the fit's labels/iterations/
counts exact and centres within 1e-12 relative.
"""

import numpy as np
import pytest

from conftest import golden


def cases():
    g = golden("seeding")
    per = {}
    for key, v in g.items():
        if key == "count":
            continue
        field, idx = key.rsplit("_", 1)
        per.setdefault(int(idx), {})[field] = v
    for t in sorted(per):
        yield t, per[t]


def test_oracle_seeding_matches_reference():
    from oracle import oracle

    for t, c in cases():
        cap = None if int(c["cap"]) < 0 else int(c["cap"])
        d, i, j = oracle.diameter(c["coords"], cap)
        assert (d, i, j) == (float(c["d"]), int(c["i"]), int(c["j"])), t
        init = bytes(c["init"]).decode()
        if bool(c["degenerate"]):
            with pytest.raises(oracle.DegenerateData):
                oracle.init_centers(c["coords"], int(c["k"]), init, int(c["seed"]), (d, i, j))
        else:
            c0 = oracle.init_centers(c["coords"], int(c["k"]), init, int(c["seed"]), (d, i, j))
            assert np.array_equal(c0, c["c0"]), t


def test_scan_rows_rule():
    from oracle import oracle
    from paper_1402_3788_b200.engine import scan_rows

    for n in (0, 1, 2, 3, 10, 1001):
        for cap in (None, 1, 2, 7, 100, 10**9):
            assert np.array_equal(scan_rows(n, cap), oracle.scan_rows(n, cap))


@pytest.mark.gpu
def test_device_seeding_and_fit_vs_reference():
    from paper_1402_3788_b200 import KmeansConfig, RegimeKMeans, diameter, init_centers
    from paper_1402_3788_b200.exceptions import DegenerateDataError
    from paper_1402_3788_b200.model import Dataset

    for t, c in cases():
        cap = None if int(c["cap"]) < 0 else int(c["cap"])
        init = bytes(c["init"]).decode()
        k = int(c["k"])
        ds = Dataset(c["coords"])
        diam = diameter(ds, pair_cap=cap)
        assert (diam.d, diam.i, diam.j) == (float(c["d"]), int(c["i"]), int(c["j"])), t
        cfg = KmeansConfig(k=k, init=init, seed=int(c["seed"]), diameter_pair_cap=cap)
        if bool(c["degenerate"]):
            with pytest.raises(DegenerateDataError):
                init_centers(ds, cfg, diam)
            continue
        assert np.array_equal(init_centers(ds, cfg, diam).centers, c["c0"]), t
        est = RegimeKMeans(k, init=init, random_state=int(c["seed"]), diameter_pair_cap=cap).fit(c["coords"])
        assert est.n_iter_ == int(c["iterations"]) and est.converged_ == bool(c["converged"]), t
        assert np.array_equal(est.labels_, c["labels"]), t
        rel = np.max(np.abs(est.cluster_centers_ - c["centers"]) / np.maximum(np.abs(c["centers"]), 1.0))
        assert rel <= 1e-12, (t, rel)
        assert abs(est.inertia_ - float(c["inertia"])) <= 1e-9 * max(1.0, abs(float(c["inertia"]))), t
        assert est.diameter_pair_ == (int(c["i"]), int(c["j"]))
        assert np.allclose(est.global_centroid_, c["centroid"], rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,cap", [(20_000, 25, None), (50_000, 10, 5_000_000), (3_001, 70, None),
                                     (12_345, 3, 1_000)])
def test_device_diameter_vs_oracle(n, m, cap):
    from oracle import oracle
    from paper_1402_3788_b200 import diameter
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, 8, seed=n % 13, dtype=np.float32)
    want = oracle.diameter(x.astype(np.float64), cap)
    got = diameter(x, pair_cap=cap)
    assert (got.d, got.i, got.j) == want


@pytest.mark.gpu
def test_device_diameter_ties_and_duplicates():
    from oracle import oracle
    from paper_1402_3788_b200 import diameter

    # a square with equal diagonals: ties resolve to the smallest (i, j)
    sq = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]] * 3)
    got = diameter(sq)
    assert (got.d, got.i, got.j) == oracle.diameter(sq) == (np.sqrt(2.0), 0, 3)
    # fp64-only data (not fp32-representable) takes the exact path
    x = np.random.default_rng(1).standard_normal((700, 4)) * 1e3 + 1e-7
    got = diameter(x)
    assert (got.d, got.i, got.j) == oracle.diameter(x)
