"""Pin the C oracle (oracle/kmeans_oracle.c) against vectors produced by the
REAL reference (oracle/make_golden.py).  Bit-exact: same fp64 rounding
sequence, no tolerances — the reference's own test style (test_kernels.py)."""

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_indexed
from oracle import oracle

LLOYD_CASES = ["blob4", "synth_10k_5_4", "synth_20k_25_16", "synth_30k_10_8", "maxiter1", "maxiter5", "k1",
               "dup_center_repair", "all_dup_repair", "tol_pos"]


def _check_lloyd(g, res):
    assert res["iterations"] == int(g["iterations"])
    assert res["converged"] == bool(g["converged"])
    assert np.array_equal(res["labels"], g["labels"].astype(np.int64))
    assert np.array_equal(res["centers"], g["centers"])
    assert np.array_equal(res["counts"], g["counts"])


@pytest.mark.parametrize("name", LLOYD_CASES)
@pytest.mark.parametrize("workers", [1, 3])
def test_lloyd_matches_reference(name, workers):
    g = golden(name)
    res = oracle.lloyd(g["coords"].astype(np.float64), g["c0"], int(g["max_iters"]), float(g["tol"]),
                       n_workers=workers)
    _check_lloyd(g, res)


def test_random_fp64_instances():
    cases = golden_indexed("random_fp64")
    assert len(cases) >= 30
    for idx, g in cases.items():
        res = oracle.lloyd(g["coords"], g["c0"])
        _check_lloyd(g, res)


def test_update_step_vectors():
    for idx, g in golden_indexed("update_random").items():
        centers, counts, labels = oracle.update(g["coords"], g["labels_in"], int(g["k"]))
        assert np.array_equal(labels, g["labels_out"]), idx
        assert np.array_equal(counts, g["counts"]), idx
        occ = g["counts"] > 0
        assert np.array_equal(centers[occ], g["centers"][occ]), idx


def test_repair_known_answer():
    g = golden("update_repair")
    centers, counts, labels = oracle.update(g["coords"], g["labels_in"], int(g["k"]))
    assert labels.tolist() == [0, 0, 1]
    assert counts.tolist() == [2, 1]
    assert np.array_equal(centers[1], [8.0, 0.0])
    assert np.array_equal(labels, g["labels_out"])


def test_assign_vectors_and_wcss():
    for idx, g in golden_indexed("assign_random").items():
        labels, counts = oracle.assign(g["coords"], g["centers"])
        assert np.array_equal(labels, g["labels"]), idx
        assert np.array_equal(counts, g["counts"]), idx
        assert oracle.wcss(g["coords"], g["centers"], labels) == float(g["wcss"]), idx


def test_tie_goes_to_lower_center():
    g = golden("assign_tie")
    labels, _ = oracle.assign(g["coords"], g["centers"])
    assert labels.tolist() == [0] == g["labels"].tolist()


def test_converged_cases():
    for idx, g in golden_indexed("converged_cases").items():
        assert oracle.converged(g["prev"], g["next"], float(g["tol"])) == bool(g["out"]), idx


def test_worker_count_invariance():
    g = golden("synth_30k_10_8")
    x = g["coords"].astype(np.float64)
    base = oracle.lloyd(x, g["c0"], max_iters=7)
    for w in (2, 5, 8):
        other = oracle.lloyd(x, g["c0"], max_iters=7, n_workers=w)
        assert np.array_equal(other["centers"], base["centers"])
        assert np.array_equal(other["labels"], base["labels"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3_20"])
def test_oracle_matches_reference_bench_configs(name):
    """The C restatement against the REAL reference at benchmark sizes (many 65,536-row
    accumulation blocks: the multi-block fold, model.py:163-173)."""
    import hashlib

    from paper_1402_3788_b200.datasets import generate_synthetic_array

    g = dict(np.load(GOLDEN / f"bench_{name}.npz"))
    x = generate_synthetic_array(int(g["n"]), int(g["m"]), int(g["k"]), seed=int(g["seed"]), dtype=np.float32)
    assert hashlib.sha256(x.tobytes()).hexdigest() == g["coords_sha256"].item().decode()
    want = oracle.lloyd(x.astype(np.float64), g["c0"], max_iters=int(g["max_iters"]), n_workers=8)
    assert want["iterations"] == int(g["iterations"]) and want["converged"] == bool(g["converged"])
    assert np.array_equal(want["labels"], g["labels"].astype(np.int64))
    assert np.array_equal(want["counts"], g["counts"])
    assert np.array_equal(want["centers"], g["centers"])  # same sequential fp64 arithmetic: bit-identical
