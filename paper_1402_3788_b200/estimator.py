"""scikit-learn-style estimator over the B200 engine — the reference's
``RegimeKMeans`` (estimator.py:81-192) with every numeric step on the device.

Same constructor, attributes and methods.  ``regime`` / ``n_workers`` /
``auto_prefer`` / ``device`` are accepted for compatibility: the run is the
device-resident Lloyd loop (``regime_used_ == "gpu"``).  There is no CPU
fallback: a missing or lost device raises.
"""

from __future__ import annotations

import numpy as np
from sklearn.base import BaseEstimator, ClusterMixin
from sklearn.utils.validation import check_is_fitted

from .engine import KmeansConfig, run_b200
from .exceptions import ContractViolationError
from .model import DEFAULT_BLOCK, ClusterModel, Dataset, wcss
from .validation import check_coordinates


class RegimeKMeans(ClusterMixin, BaseEstimator):
    """K-means with the reference's seeding (diameter + maximin / random-far) and
    Lloyd iteration, bit-compatible labels and iteration counts.

    A scikit-learn estimator like the reference's (estimator.py:19): ``get_params`` /
    ``set_params`` / ``clone`` come from ``BaseEstimator`` (constructor introspection),
    ``fit_predict`` from ``ClusterMixin``, and an unfitted ``predict`` / ``transform``
    raises sklearn's ``NotFittedError`` (``check_is_fitted``, estimator.py:177,185)."""

    def __init__(self, n_clusters=8, *, regime="auto", n_workers=None, device="b200", init="maximin",
                 max_iter=1000, tol=0.0, random_state=0, auto_prefer="gpu", accum_block=DEFAULT_BLOCK,
                 diameter_pair_cap=None, track_wcss=False):
        self.n_clusters = n_clusters
        self.regime = regime
        self.n_workers = n_workers
        self.device = device
        self.init = init
        self.max_iter = max_iter
        self.tol = tol
        self.random_state = random_state
        self.auto_prefer = auto_prefer
        self.accum_block = accum_block
        self.diameter_pair_cap = diameter_pair_cap
        self.track_wcss = track_wcss

    def _config(self):
        return KmeansConfig(k=self.n_clusters, max_iters=self.max_iter, tol=self.tol,
                            seed=self.random_state if self.random_state is not None else 0, init=self.init,
                            accum_block=self.accum_block, diameter_pair_cap=self.diameter_pair_cap,
                            track_wcss=self.track_wcss)

    def _device_index(self):
        return self.device if isinstance(self.device, int) else 0

    def fit(self, X, y=None):
        """Seed and cluster X on the device (estimator.py:122-164)."""
        dataset = X if isinstance(X, Dataset) else Dataset(X)
        config = self._config()
        config.validate_for(dataset)
        result = run_b200(dataset, config, device=self._device_index())
        self.cluster_centers_ = result.model.centers
        self.labels_ = result.assignment.labels
        self.inertia_ = wcss(dataset, result.model, result.assignment, block=config.accum_block)
        self.n_iter_ = result.iterations
        self.converged_ = result.converged
        self.diameter_ = result.diameter.d
        self.diameter_pair_ = (result.diameter.i, result.diameter.j)
        self.global_centroid_ = result.global_centroid
        self.regime_used_ = "gpu"
        self.n_features_in_ = dataset.m
        self.wcss_history_ = result.wcss_history
        self.fallback_reason_ = result.fallback_reason
        return self

    def _check_input(self, X):
        arr = check_coordinates(X, name="X")
        if arr.shape[1] != self.n_features_in_:
            raise ContractViolationError(
                f"X has {arr.shape[1]} features, but this estimator was fitted with {self.n_features_in_}")
        return arr

    def predict(self, X):
        """Nearest-centre label per sample, ties toward the lower index (estimator.py:175-181)."""
        check_is_fitted(self, "cluster_centers_")
        arr = self._check_input(X)
        ds = Dataset(arr)
        labels, _ = ds.device_engine(self._device_index()).assign(self.cluster_centers_)
        return labels

    def transform(self, X):
        """Distance from each sample to each centre, shape (n, k) (estimator.py:183-189)."""
        check_is_fitted(self, "cluster_centers_")
        arr = self._check_input(X)
        return Dataset(arr).device_engine(self._device_index()).center_distances(self.cluster_centers_)

    def fit_transform(self, X, y=None):
        return self.fit(X).transform(X)
