"""The reference's offload-device protocol (device.py:63-261) — host side.

CPU tests: the oracle's MAX_PAIR / sum-job restatement bit-exact against vectors from the
real reference's HostReferenceDevice (oracle/make_golden_device.py → tests/golden/
device_jobs.npz), the ticket bookkeeping of ``Device`` (submit / collect exactly once /
outstanding / capacity, device.py:153-201) on a stub device, the job constructors' range
checks (device.py:115-150) and the registry (device.py:242-261).  The B200 execution of
the same jobs is tests/test_gpu_device.py."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle
from paper_1402_3788_b200 import device as dev
from paper_1402_3788_b200.exceptions import (
    CapacityExceededError, ContractViolationError, DeviceUnavailableError, DoubleCollectError,
    UnknownTicketError,
)

G = dict(np.load(GOLDEN / "device_jobs.npz"))
CASES = sorted({k.split("_")[0] for k in G})


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", ["contig", "bal"])
def test_oracle_max_pair_rows_matches_reference(case, mode):
    x = G[f"{case}_x"]
    pairs = G[f"{case}_{mode}_pairs"]
    for pi in range(pairs.shape[0]):
        d2, i, j = oracle.max_pair_rows(x, G[f"{case}_{mode}_rows{pi}"])
        assert (d2, i, j) == (pairs[pi, 0], int(pairs[pi, 1]), int(pairs[pi, 2]))


@pytest.mark.parametrize("case", CASES)
def test_oracle_block_sums_match_reference(case):
    x, labels = G[f"{case}_x"], G[f"{case}_labels"]
    n, m, k, block, _ = (int(v) for v in G[f"{case}_meta"])
    s = int(G[f"{case}_span"][0])
    for ji, (a, b) in enumerate(((0, s), (s, n))):
        sums, _, bad = oracle.block_sums(x, a, b, block)
        assert bad == -1 and np.array_equal(sums, G[f"{case}_coord{ji}"])
        sums, counts, bad = oracle.block_sums(x, a, b, block, labels=labels, k=k)
        assert bad == -1
        assert np.array_equal(sums, G[f"{case}_clus{ji}"])
        assert np.array_equal(counts, G[f"{case}_clus{ji}_counts"])


def test_oracle_block_sums_reports_first_bad_label():
    x = np.arange(40.0).reshape(20, 2)
    labels = np.zeros(20, dtype=np.int64)
    labels[[7, 13]] = [5, -1]
    assert oracle.block_sums(x, 0, 20, 4, labels=labels, k=3)[2] == 7


class _StubDevice(dev.Device):
    name = "stub"

    def _execute(self, job):
        return dev.DeviceResult(job.kind)


def test_ticketing_exactly_once():
    d = _StubDevice()
    x = np.zeros((10, 2))
    t1 = d.submit(dev.coord_sum_job(x, 0, 10, 5))
    t2 = d.submit(dev.coord_sum_job(x, 5, 10, 5))
    assert t1 != t2 and d.outstanding() == 2
    assert d.collect(t2).kind == dev.COORD_SUM
    with pytest.raises(DoubleCollectError):
        d.collect(t2)
    with pytest.raises(UnknownTicketError):
        d.collect(12345)
    d.collect(t1)
    assert d.outstanding() == 0


def test_capacity_and_kind_checks():
    d = _StubDevice(max_buffer_bytes=64)
    with pytest.raises(CapacityExceededError):
        d.submit(dev.coord_sum_job(np.zeros((10, 2)), 0, 10, 5))
    with pytest.raises(ContractViolationError):
        d.submit(dev.DeviceJob("bogus", 1, 1))


def test_job_constructor_checks():
    x = np.zeros((10, 2))
    with pytest.raises(ContractViolationError):
        dev.coord_sum_job(x, 3, 10, 5)           # not on a block boundary
    with pytest.raises(ContractViolationError):
        dev.coord_sum_job(x, 0, 11, 5)           # past n
    with pytest.raises(ContractViolationError):
        dev.cluster_sum_job(x, np.zeros(10, dtype=np.int64), 0, 0, 10, 5)  # k < 1
    with pytest.raises(ContractViolationError):
        dev.max_pair_job(np.zeros((2, 10)), [0, 10], 10)  # row out of range
    j = dev.cluster_sum_job(x, np.zeros(10, dtype=np.int64), 3, 5, 10, 5)
    assert j.nbytes() == x.nbytes + 80


def test_registry():
    with pytest.raises(DeviceUnavailableError):
        dev.get_device("reference")  # no host device: no CPU fallback in this package
