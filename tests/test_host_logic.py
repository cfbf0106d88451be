"""Host-side contracts that need no GPU: config validation, containers,
validation helpers, exception hierarchy (mirrors the reference's
test_model.py / test_engine.py contract tests)."""

import numpy as np
import pytest

from paper_1402_3788_b200 import (
    Assignment, ClusterModel, ContractViolationError, Dataset, KmeansConfig, block_bounds, distance, fold_blocks,
)
from paper_1402_3788_b200 import exceptions as ex
from paper_1402_3788_b200.datasets import generate_synthetic_array
from paper_1402_3788_b200.validation import check_labels


class TestConfig:
    def test_defaults(self):
        c = KmeansConfig(k=3)
        assert (c.max_iters, c.tol, c.init, c.accum_block) == (1000, 0.0, "maximin", 65536)

    @pytest.mark.parametrize("kw", [dict(k=0), dict(k=2, max_iters=0), dict(k=2, tol=-1.0),
                                    dict(k=2, tol=float("nan")), dict(k=2, init="kmeans++"),
                                    dict(k=2, metric="cosine"), dict(k=2, accum_block=0),
                                    dict(k=2, diameter_pair_cap=0)])
    def test_rejects(self, kw):
        with pytest.raises(ContractViolationError):
            KmeansConfig(**kw)

    def test_k_larger_than_n(self):
        with pytest.raises(ContractViolationError):
            KmeansConfig(k=3).validate_for(Dataset([[0.0], [1.0]]))


class TestDataset:
    def test_float64_coercion_and_readonly(self):
        ds = Dataset([[1, 2], [3, 4]])
        assert ds.coords.dtype == np.float64 and not ds.coords.flags.writeable
        with pytest.raises(AttributeError):
            ds.coords = None

    def test_float32_kept(self):
        ds = Dataset(np.zeros((3, 2), dtype=np.float32))
        assert ds.coords.dtype == np.float32

    def test_one_dimensional(self):
        assert Dataset([1.0, 2.0, 3.0]).coords.shape == (3, 1)

    @pytest.mark.parametrize("bad", [[], [[np.nan, 1.0]], [[np.inf]], np.zeros((2, 2, 2))])
    def test_rejects(self, bad):
        with pytest.raises(ContractViolationError):
            Dataset(bad)

    def test_copy_isolates(self):
        src = np.zeros((2, 2))
        ds = Dataset(src)
        src[0, 0] = 5
        assert ds.coords[0, 0] == 0


class TestContainers:
    def test_model_counts(self):
        m = ClusterModel(np.zeros((3, 2)))
        assert m.counts.tolist() == [0, 0, 0] and m.counts.dtype == np.int64
        with pytest.raises(ContractViolationError):
            ClusterModel(np.zeros((3, 2)), [1, 2])
        with pytest.raises(ContractViolationError):
            ClusterModel(np.zeros((2, 2)), [1, -1])

    def test_assignment(self):
        a = Assignment([0, 1, 1])
        assert a.labels.dtype == np.int64 and a.n == 3
        with pytest.raises(ContractViolationError):
            Assignment(np.zeros((2, 2)))

    def test_labels_check(self):
        with pytest.raises(ContractViolationError):
            check_labels([0, 5], n=2, k=2)
        with pytest.raises(ContractViolationError):
            check_labels([0], n=2, k=2)

    def test_blocks(self):
        assert block_bounds(10, 4) == [(0, 4), (4, 8), (8, 10)]
        p = np.arange(12, dtype=np.float64).reshape(3, 4)
        assert np.array_equal(fold_blocks(p), p.sum(axis=0))

    def test_distance(self):
        assert distance([0, 0], [3, 4]) == 5.0
        with pytest.raises(ContractViolationError):
            distance([0, 0], [1, 2, 3])


def test_exception_hierarchy():
    assert issubclass(ex.ContractViolationError, ValueError)
    for name in ("EmptyClusterError", "DeviceLostError", "DeviceUnavailableError", "CapacityExceededError",
                 "ValidationFailureError", "OutputMismatchError"):
        assert issubclass(getattr(ex, name), ex.ClusteringError)
    e = ex.ParseError("x", row=3, column=2)
    assert (e.row, e.column) == (3, 2)


def test_generator_matches_golden_bytes():
    from conftest import golden

    g = golden("synth_10k_5_4")
    x = generate_synthetic_array(10_000, 5, 4, seed=0, dtype=np.float32)
    assert np.array_equal(x, g["coords"])


def test_estimator_is_a_sklearn_estimator():
    """RegimeKMeans(ClusterMixin, BaseEstimator) as the reference's (estimator.py:19): clone /
    get_params / set_params by constructor introspection, NotFittedError before fit
    (check_is_fitted, estimator.py:177,185) — no device needed for any of these."""
    from sklearn.base import BaseEstimator, ClusterMixin, clone
    from sklearn.exceptions import NotFittedError

    from paper_1402_3788_b200 import RegimeKMeans

    est = RegimeKMeans(5, max_iter=7, tol=1e-3, diameter_pair_cap=100)
    assert isinstance(est, BaseEstimator) and isinstance(est, ClusterMixin)
    p = est.get_params()
    assert p["n_clusters"] == 5 and p["max_iter"] == 7 and p["tol"] == 1e-3 and p["diameter_pair_cap"] == 100
    c = clone(est)
    assert c is not est and c.get_params() == p
    c.set_params(n_clusters=3)
    assert c.n_clusters == 3 and est.n_clusters == 5
    import numpy as np

    with pytest.raises(NotFittedError):
        est.predict(np.zeros((3, 2)))
    with pytest.raises(NotFittedError):
        est.transform(np.zeros((3, 2)))


@pytest.mark.parametrize("n,m,k,lo,hi", [(10007, 5, 4, 0, 10007), (10007, 5, 4, 123, 5000), (50000, 25, 16, 25000, 50000),
                                         (3000, 3, 7, 2999, 3000), (3000, 3, 7, 10, 10)])
def test_synthetic_shard_is_a_slice_of_the_full_dataset(n, m, k, lo, hi):
    """bench.py's row shards of ONE dataset (the 64M strong-scaling config) are the same bytes as
    rows [lo, hi) of the reference generator's array (datasets.py:73-97)."""
    from paper_1402_3788_b200.datasets import generate_synthetic_shard

    full = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
    assert np.array_equal(generate_synthetic_shard(n, m, k, 0, lo, hi, chunk_rows=777), full[lo:hi])
