"""The reference's offload-device protocol on B200.

Mirrors ``kmeans_regimes.device`` (device.py:63-261): the three job kinds
(MAX_PAIR / COORD_SUM / CLUSTER_SUM), ``DeviceJob`` / ``DeviceResult``, the job
constructors with their range checks, the ticketing ``Device`` base class
(``submit`` → ticket, ``collect`` exactly once, ``outstanding``) and a
``get_device`` registry.  ``B200Device._execute`` runs each job through the
C ABI (``km_max_pair_rows``, ``km_block_sums``) on points kept resident per
coordinate buffer, so a caller of the reference's ``Device`` seam (the
``run_gpu`` offload regime, a bridge runner) reaches the B200 kernels.

Compatibility only: the Lloyd hot path itself goes through ``run_b200`` /
``km_lloyd`` (assignment and update fused on the device), not through jobs.
Result semantics follow ``HostReferenceDevice`` (device.py:204-239): MAX_PAIR
returns the exact fp64 d² of the lexicographically first maximising pair;
sum jobs return per-block partials with the block index leading.  Block
sums are exact fixed-point sums rounded once to fp64, so they agree with the
reference's sequential fp64 block sums to ~1e-15 relative (the reference's
own real-device rule accepts ≈1e-13, frontend/README.md:43-44).
"""

from __future__ import annotations

import itertools
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .exceptions import (
    CapacityExceededError,
    ContractViolationError,
    DeviceUnavailableError,
    DoubleCollectError,
    UnknownTicketError,
    ValidationFailureError,
)
from .model import DEFAULT_BLOCK

MAX_PAIR = "max-pair-distance"
COORD_SUM = "coordinate-sum"
CLUSTER_SUM = "cluster-sum"

JOB_KINDS = (MAX_PAIR, COORD_SUM, CLUSTER_SUM)


@dataclass
class PartialMax:
    """One job's largest-distance pair (partition.py:56-66)."""

    d2: float
    i: int
    j: int

    @property
    def d(self):
        return float(np.sqrt(self.d2))


@dataclass
class PartialSums:
    """Per-block sums of a contiguous span of blocks (partition.py:69-81): (blocks, k, m) with
    counts (blocks, k) for cluster sums, (blocks, m) with counts None for coordinate sums."""

    first_block: int
    sums: np.ndarray
    counts: Optional[np.ndarray] = None


@dataclass
class DeviceJob:
    """One unit of device work over a read-only slice of the dataset (device.py:67-98)."""

    kind: str
    n: int
    m: int
    coords: Optional[np.ndarray] = None
    coords_t: Optional[np.ndarray] = None
    rows: Optional[np.ndarray] = None
    labels: Optional[np.ndarray] = None
    start: int = 0
    stop: int = 0
    block: int = DEFAULT_BLOCK
    k: int = 0

    def nbytes(self):
        """Bytes of buffer the device must hold to run this job."""
        return sum(b.nbytes for b in (self.coords, self.coords_t, self.rows, self.labels) if b is not None)


@dataclass
class DeviceResult:
    """Result of one device job, mirroring the host partial shapes (device.py:101-112)."""

    kind: str
    pair: Optional[PartialMax] = None
    partial: Optional[PartialSums] = None


def max_pair_job(coords_t, rows, n):
    """device.py:115-120."""
    m = coords_t.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size and (rows.min() < 0 or rows.max() >= n):
        raise ContractViolationError(f"scan rows must lie in [0, {n})")
    return DeviceJob(MAX_PAIR, n, m, coords_t=coords_t, rows=rows)


def coord_sum_job(coords, start, stop, block=DEFAULT_BLOCK):
    """device.py:123-126."""
    n, m = coords.shape
    _check_range(start, stop, n, block)
    return DeviceJob(COORD_SUM, n, m, coords=coords, start=start, stop=stop, block=block)


def cluster_sum_job(coords, labels, k, start, stop, block=DEFAULT_BLOCK):
    """device.py:129-136."""
    n, m = coords.shape
    _check_range(start, stop, n, block)
    if k < 1:
        raise ContractViolationError(f"k must be >= 1, got {k}")
    return DeviceJob(CLUSTER_SUM, n, m, coords=coords, labels=labels, start=start, stop=stop, block=block, k=k)


def _check_range(start, stop, n, block):
    """device.py:139-150."""
    if not 0 <= start <= stop <= n:
        raise ContractViolationError(f"job range [{start}, {stop}) must lie within [0, {n}]")
    if block < 1:
        raise ContractViolationError(f"block size must be >= 1, got {block}")
    if start % block != 0:
        raise ContractViolationError(
            f"job range must start on an accumulation-block boundary (start={start}, block={block})")


class Device:
    """Ticket bookkeeping and capacity checks around ``_execute`` (device.py:153-201).

    ``submit`` validates the job against the device's buffer capability and
    hands out a unique ticket; ``collect`` delivers each result exactly once.
    Both are safe to call from concurrent workers.
    """

    name = "abstract"

    def __init__(self, max_buffer_bytes=16 << 30, preferred_block=DEFAULT_BLOCK):
        self.max_buffer_bytes = max_buffer_bytes
        self.preferred_block = preferred_block
        self._lock = threading.Lock()
        self._tickets = itertools.count(1)
        self._pending = {}
        self._collected = set()

    def submit(self, job):
        if job.kind not in JOB_KINDS:
            raise ContractViolationError(f"unknown job kind {job.kind!r}")
        if job.nbytes() > self.max_buffer_bytes:
            raise CapacityExceededError(
                f"job needs {job.nbytes()} bytes, device holds {self.max_buffer_bytes}; split the range")
        result = self._execute(job)
        with self._lock:
            ticket = next(self._tickets)
            self._pending[ticket] = result
        return ticket

    def collect(self, ticket):
        with self._lock:
            if ticket in self._pending:
                self._collected.add(ticket)
                return self._pending.pop(ticket)
            if ticket in self._collected:
                raise DoubleCollectError(f"ticket {ticket} was already collected")
        raise UnknownTicketError(f"ticket {ticket} was never issued by this device")

    def outstanding(self):
        """Number of submitted-but-uncollected tickets (0 after a clean run)."""
        with self._lock:
            return len(self._pending)

    def _execute(self, job):
        raise NotImplementedError


class B200Device(Device):
    """Jobs on one B200 through the C ABI.  The coordinates of a job are uploaded once per
    buffer (keyed by its address, shape and dtype — the bridge keeps one copy per digest,
    bridge.py:103-119; the reference's datasets are read-only, model.py:34-47) and stay
    resident for the following jobs.  One engine, one CUDA stream; jobs are serialised."""

    name = "b200"

    def __init__(self, device=0, **kwargs):
        super().__init__(**kwargs)
        from . import _native

        self._engine = _native.NativeEngine(device)
        self._key = None
        self._exec_lock = threading.Lock()

    def _resident(self, job):
        if job.kind == MAX_PAIR:
            buf = job.coords_t
            key = ("t", buf.__array_interface__["data"][0], buf.shape, buf.dtype.str, buf.strides)
            if key != self._key:
                self._engine.load(np.ascontiguousarray(buf.T))
        else:
            buf = job.coords
            key = ("r", buf.__array_interface__["data"][0], buf.shape, buf.dtype.str, buf.strides)
            if key != self._key:
                self._engine.load(buf)
        self._key = key
        return self._engine

    def _execute(self, job):
        with self._exec_lock:
            eng = self._resident(job)
            if job.kind == MAX_PAIR:
                d2, i, j = eng.max_pair_rows(job.rows)
                return DeviceResult(MAX_PAIR, pair=PartialMax(d2, int(i), int(j)) if d2 >= 0.0 else None)
            first_block = job.start // job.block
            if job.kind == COORD_SUM:
                sums, _ = eng.block_sums(job.start, job.stop, job.block)
                return DeviceResult(COORD_SUM, partial=PartialSums(first_block, sums))
            try:
                sums, counts = eng.block_sums(job.start, job.stop, job.block, labels=job.labels, k=job.k)
            except ValidationFailureError as exc:  # device.py:233-238 message form
                raise ValidationFailureError(str(exc).replace(" on device", "")) from exc
            return DeviceResult(CLUSTER_SUM, partial=PartialSums(first_block, sums, counts))


def get_device(name, **kwargs):
    """Device registry (device.py:242-261).  "b200" (alias "gpu") is the B200 device; there is
    no host device in this package (no CPU fallback) — the reference's HostReferenceDevice is
    the reference."""
    if name in ("b200", "gpu"):
        return B200Device(**kwargs)
    raise DeviceUnavailableError(f"no device named {name!r}")
