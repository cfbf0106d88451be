"""B200Device: the reference's device jobs on the GPU through the C ABI
(km_max_pair_rows, km_block_sums) vs the real reference's HostReferenceDevice outputs
(tests/golden/device_jobs.npz) and the C oracle.  MAX_PAIR: bit-exact (d², i, j).  Sum
jobs: counts exact, sums exact fixed point rounded once (≤ 1e-12 of the block's Σ|x|)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

pytestmark = pytest.mark.gpu

G = dict(np.load(GOLDEN / "device_jobs.npz"))
CASES = sorted({k.split("_")[0] for k in G})


@pytest.fixture(scope="module")
def device():
    from paper_1402_3788_b200.device import get_device

    return get_device("b200")


def _scale(x, labels, k, a, b, block):
    """Per (block, cluster, feature) Σ|x| — the error scale of a sum."""
    ax = np.abs(x)
    out = []
    for s in range(a, b, block):
        e = min(s + block, b)
        lab = labels[s:e] if labels is not None else np.zeros(e - s, dtype=np.int64)
        out.append(np.stack([ax[s:e][lab == c].sum(axis=0) for c in range(k)]))
    return np.array(out)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", ["contig", "bal"])
def test_max_pair_jobs_match_reference(device, case, mode):
    from paper_1402_3788_b200 import device as d

    x = G[f"{case}_x"]
    n = x.shape[0]
    xt = np.ascontiguousarray(x.T)
    pairs = G[f"{case}_{mode}_pairs"]
    best = None
    for pi in range(pairs.shape[0]):
        r = device.collect(device.submit(d.max_pair_job(xt, G[f"{case}_{mode}_rows{pi}"], n)))
        want = pairs[pi]
        if want[1] < 0:
            assert r.pair is None
            continue
        assert (r.pair.d2, r.pair.i, r.pair.j) == (want[0], int(want[1]), int(want[2]))
        if best is None or r.pair.d2 > best.d2:  # partition.merge_max: strict '>' keeps the first
            best = r.pair
    meta = G[f"{case}_meta"]
    cap = None if meta[4] < 0 else int(meta[4])
    dd, i, j = oracle.diameter(x, cap)
    assert (best.i, best.j) == (i, j) and np.sqrt(best.d2) == dd


@pytest.mark.parametrize("case", CASES)
def test_sum_jobs_match_reference(device, case):
    from paper_1402_3788_b200 import device as d

    x, labels = G[f"{case}_x"], G[f"{case}_labels"]
    n, m, k, block, _ = (int(v) for v in G[f"{case}_meta"])
    s = int(G[f"{case}_span"][0])
    for ji, (a, b) in enumerate(((0, s), (s, n))):
        r = device.collect(device.submit(d.coord_sum_job(x, a, b, block)))
        assert r.partial.first_block == a // block and r.partial.counts is None
        want = G[f"{case}_coord{ji}"]
        assert r.partial.sums.shape == want.shape
        tol = 1e-12 * np.maximum(_scale(x, None, 1, a, b, block)[:, 0, :], 1e-300)
        assert np.all(np.abs(r.partial.sums - want) <= tol)
        r = device.collect(device.submit(d.cluster_sum_job(x, labels, k, a, b, block)))
        assert np.array_equal(r.partial.counts, G[f"{case}_clus{ji}_counts"])
        want = G[f"{case}_clus{ji}"]
        tol = 1e-12 * np.maximum(_scale(x, labels, k, a, b, block), 1e-300)
        assert np.all(np.abs(r.partial.sums - want) <= tol)
    assert device.outstanding() == 0


def test_bad_label_raises_validation_failure(device):
    from paper_1402_3788_b200 import device as d
    from paper_1402_3788_b200.exceptions import ValidationFailureError

    x = np.random.default_rng(1).standard_normal((5000, 6))
    labels = np.zeros(5000, dtype=np.int64)
    labels[[3100, 4000]] = [9, -2]
    with pytest.raises(ValidationFailureError, match="at sample 3100"):
        device.submit(d.cluster_sum_job(x, labels, 4, 0, 5000, 1000))
    assert device.outstanding() == 0


def test_large_range_many_blocks(device):
    """cfg3-sized coordinate sum over many blocks vs the oracle (fp32 data, 31 blocks)."""
    from paper_1402_3788_b200 import device as d
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(2_000_000, 25, 16, seed=0, dtype=np.float32)
    labels = np.random.default_rng(2).integers(0, 16, size=x.shape[0]).astype(np.int64)
    r = device.collect(device.submit(d.cluster_sum_job(x, labels, 16, 0, x.shape[0], 65536)))
    sums, counts, bad = oracle.block_sums(x.astype(np.float64), 0, x.shape[0], 65536, labels=labels, k=16)
    assert bad == -1 and np.array_equal(r.partial.counts, counts)
    # sequential fp64 sums over 65536-sample blocks: error ≤ (block − 1)·u·Σ|x| (typically far less)
    tol = 1e-11 * np.maximum(_scale(x.astype(np.float64), labels, 16, 0, x.shape[0], 65536), 1e-300)
    assert np.all(np.abs(r.partial.sums - sums) <= tol)
