"""The Lloyd hot path with the reference's entry points and result layout.

Mirrors /root/reference/pkg/src/kmeans_regimes/engine.py:
  KmeansConfig (:52-107), KmeansResult (:110-121), DiameterResult (:43-49),
  assign_step (:218-230), update_step (:281-294), converged (:297-310),
  iterate (:320-343), and adds run_b200 — the device-resident loop that
  replaces run_single / run_multi / run_gpu (:346-370, partition.py:264-305,
  device.py:365-382) for the iteration phase.

Every numeric step runs in the CUDA engine (libkmeans_b200.so via _native);
nothing here computes distances or sums on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

import math

from .exceptions import ContractViolationError, DegenerateDataError, InsufficientDataError
from .model import DEFAULT_BLOCK, SUPPORTED_METRICS, Assignment, ClusterModel, Dataset, wcss
from .validation import check_coordinates, check_labels

INIT_STRATEGIES = ("maximin", "random-far")


@dataclass(frozen=True)
class DiameterResult:
    d: float
    i: int
    j: int


@dataclass(frozen=True)
class KmeansConfig:
    """Clustering parameters (engine.py:52-107), same fields and validation.

    ``accum_block`` is accepted for compatibility; the B200 engine's sums are
    exact integers, so results do not depend on it.
    """

    k: int
    max_iters: int = 1000
    tol: float = 0.0
    seed: int = 0
    init: str = "maximin"
    metric: str = "euclidean"
    accum_block: int = DEFAULT_BLOCK
    diameter_pair_cap: Optional[int] = None
    balanced_rows: bool = False
    track_wcss: bool = False

    def __post_init__(self):
        if self.k < 1:
            raise ContractViolationError(f"k must be >= 1, got {self.k}")
        if self.max_iters < 1:
            raise ContractViolationError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.tol >= 0.0:
            raise ContractViolationError(f"tol must be >= 0, got {self.tol}")
        if self.init not in INIT_STRATEGIES:
            raise ContractViolationError(f"init must be one of {INIT_STRATEGIES}, got {self.init!r}")
        if self.metric not in SUPPORTED_METRICS:
            raise ContractViolationError(f"metric must be one of {SUPPORTED_METRICS}, got {self.metric!r}")
        if self.accum_block < 1:
            raise ContractViolationError(f"accum_block must be >= 1, got {self.accum_block}")
        if self.diameter_pair_cap is not None and self.diameter_pair_cap < 1:
            raise ContractViolationError(f"diameter_pair_cap must be >= 1, got {self.diameter_pair_cap}")

    def validate_for(self, dataset):
        if self.k > dataset.n:
            raise ContractViolationError(f"k={self.k} exceeds sample count n={dataset.n}")


@dataclass
class KmeansResult:
    """Everything a clustering run produces (engine.py:110-121)."""

    model: ClusterModel
    assignment: Assignment
    iterations: int
    converged: bool
    diameter: Optional[DiameterResult]
    global_centroid: Optional[np.ndarray]
    wcss_history: Optional[list] = None
    fallback_reason: Optional[str] = None


def _dataset(d) -> Dataset:
    return d if isinstance(d, Dataset) else Dataset(d)


def assign_step(dataset, model):
    """Nearest centre per sample, ties → lower index; sets model.counts to the
    label histogram (engine.py:218-230)."""
    dataset = _dataset(dataset)
    if model.m != dataset.m:
        raise ContractViolationError(
            f"center dimension {model.m} does not match dataset dimension {dataset.m}")
    labels, counts = dataset.device_engine().assign(model.centers)
    model.counts[:] = counts
    return Assignment(labels)


def update_step(dataset, assignment, k, *, block=DEFAULT_BLOCK):
    """Centres of gravity with empty-cluster repair; the repair relabels
    ``assignment.labels`` IN PLACE (engine.py:249-294)."""
    dataset = _dataset(dataset)
    check_labels(assignment.labels, n=dataset.n, k=k, name="labels")
    if assignment.labels.dtype != np.int64 or not assignment.labels.flags.c_contiguous:
        assignment.labels = np.ascontiguousarray(assignment.labels, dtype=np.int64)
    centers, counts = dataset.device_engine().update(assignment.labels, int(k))
    return ClusterModel(centers, counts)


_default_engine = None


def _any_engine():
    global _default_engine
    if _default_engine is None:
        from ._native import NativeEngine

        _default_engine = NativeEngine(0)
    return _default_engine


def converged(prev, next_model, tol):
    """max_c ‖prev_c − next_c‖ ≤ tol, exactly for tol = 0 (engine.py:297-310)."""
    if prev.k != next_model.k or prev.m != next_model.m:
        raise ContractViolationError(
            f"cannot compare models of shape ({prev.k}, {prev.m}) and ({next_model.k}, {next_model.m})")
    if not tol >= 0.0:
        raise ContractViolationError(f"tol must be >= 0, got {tol}")
    return _any_engine().converged(prev.centers, next_model.centers, tol)


def iterate(dataset, config, model, assign_fn, update_fn):
    """The reference's loop seam (engine.py:320-343), verbatim semantics.

    With ``assign_step``/``update_step`` closures every step runs on the
    device; ``run_b200`` runs the same loop entirely on the device.
    """
    assignment = assign_fn(model)
    history = [] if config.track_wcss else None
    done = False
    iterations = 0
    for _ in range(config.max_iters):
        new_model = update_fn(assignment)
        iterations += 1
        if history is not None:
            history.append(wcss(dataset, new_model, assignment, block=config.accum_block))
        if converged(model, new_model, config.tol):
            model = new_model
            done = True
            break
        model = new_model
        assignment = assign_fn(model)
    return model, assignment, iterations, done, history


def global_centroid_of(dataset, *, block=DEFAULT_BLOCK):
    """Centre of gravity of the whole dataset (engine.py:313-317), on the device."""
    from .model import centroid_of

    return centroid_of(_dataset(dataset), block=block)


def scan_rows(n, pair_cap=None):
    """Row indices the diameter scan visits (engine.py:124-138), as a pure function of (n, cap)."""
    if n < 2:
        return np.empty(0, dtype=np.int64)
    total = n * (n - 1) // 2
    if pair_cap is None or total <= pair_cap:
        return np.arange(n - 1, dtype=np.int64)
    stride = max(2, math.ceil(total / pair_cap))
    return np.arange(0, n - 1, stride, dtype=np.int64)


def diameter(dataset, *, pair_cap=None, device=0):
    """Largest pairwise distance (engine.py:141-154) on the device: exact fp64 value of the
    reference recurrence, ties → smallest (i, j), rows per ``scan_rows``."""
    dataset = _dataset(dataset)
    if dataset.n < 2:
        raise InsufficientDataError(f"diameter needs at least 2 samples, got {dataset.n}")
    d, i, j = dataset.device_engine(device).diameter(pair_cap)
    return DiameterResult(float(d), int(i), int(j))


def init_centers(dataset, config, diam, global_centroid=None, *, device=0):
    """The k initial centres (engine.py:171-215): maximin (diameter pair, then the sample
    farthest from the chosen ones, lowest index on ties) or random-far (seeded uniform draws
    kept when farther than D/(2k), maximin fallback after 10n rejected draws).  The per-sample
    minimum distances live on the device (exact fp64 recurrence); only the draw logic runs here.
    """
    dataset = _dataset(dataset)
    config.validate_for(dataset)
    eng = dataset.device_engine(device)
    n, k = dataset.n, config.k
    eng.seed_reset()
    chosen = []
    far = [0.0, -1]  # (max min_d2, its first index) after the last addition

    def append(index):
        chosen.append(int(index))
        far[0], far[1] = eng.seed_add(int(index))

    def farthest_unchosen():
        if far[0] == 0.0:
            raise DegenerateDataError("dataset has fewer distinct points than requested centers")
        return far[1]

    if config.init == "maximin":
        append(diam.i)
        if k >= 2:
            if diam.d == 0.0:
                raise DegenerateDataError("dataset has fewer distinct points than requested centers")
            append(diam.j)
        while len(chosen) < k:
            append(farthest_unchosen())
    else:
        rng = np.random.default_rng(config.seed)
        thr2 = (diam.d / (2.0 * k)) ** 2
        draws = 0
        limit = 10 * n
        while len(chosen) < k:
            accepted = False
            while draws < limit:
                cand = int(rng.integers(n))
                draws += 1
                if not chosen or eng.seed_min_d2(cand) > thr2:
                    append(cand)
                    accepted = True
                    break
            if not accepted:
                append(farthest_unchosen())
    centers = dataset.coords[np.asarray(chosen, dtype=np.int64)].astype(np.float64)
    return ClusterModel(centers, np.zeros(k, dtype=np.int64))


def run_b200(dataset, config, *, init_centers=None, device=0, want_labels=True):
    """Cluster with the device-resident Lloyd loop.

    ``init_centers`` (k × m) is the explicit initial model (the reference has
    no array init — engine.py:86-89 — so this is the parity harness's entry
    point; a default ``fit()`` needs the seeding phase).
    Returns a KmeansResult with the reference layout.  Semantics of
    ``iterations``/``converged``/returned labels follow engine.iterate exactly.
    """
    dataset = _dataset(dataset)
    config.validate_for(dataset)
    diam = centroid = None
    if init_centers is None:  # the reference's seeding phase (run_single, engine.py:358-362), on the device
        diam = diameter(dataset, pair_cap=config.diameter_pair_cap, device=device)
        centroid = global_centroid_of(dataset, block=config.accum_block)
        init_centers = globals()["init_centers"](dataset, config, diam, centroid, device=device).centers
    c0 = check_coordinates(init_centers, name="init_centers")
    if c0.shape != (config.k, dataset.m):
        raise ContractViolationError(f"init_centers must have shape ({config.k}, {dataset.m}), got {c0.shape}")
    eng = dataset.device_engine(device)
    if config.track_wcss:
        # the per-update objective needs the host between updates: step-wise loop
        model, assignment, iterations, done, history = iterate(
            dataset, config, ClusterModel(c0.copy()),
            lambda mdl: assign_step(dataset, mdl),
            lambda a: update_step(dataset, a, config.k),
        )
        return KmeansResult(model, assignment, iterations, done, diam, centroid, history)
    centers, counts, labels, iters, conv = eng.lloyd(c0, config.max_iters, config.tol, want_labels=want_labels)
    return KmeansResult(ClusterModel(centers, counts), Assignment(labels if labels is not None else np.empty(0)),
                        iters, conv, diam, centroid, None)
