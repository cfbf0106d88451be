"""Generate tests/golden/device_jobs.npz by running the REAL reference's device protocol.

TEST INFRASTRUCTURE ONLY.  Usage (build container; /root/reference is not on the GPU box,
so the vectors are committed):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden_device.py

Cases: MAX_PAIR / COORD_SUM / CLUSTER_SUM jobs through the reference's own
``HostReferenceDevice`` (device.py:204-239) — submit → collect — on seeded data, with the
scan rows split the way the offload regime splits them (``partition._split_rows`` contiguous
and balanced, partition.py:122-143) and sum ranges on block boundaries (``_block_spans``).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "device_jobs.npz"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF_SRC))

from kmeans_regimes import device as rdev  # noqa: E402
from kmeans_regimes.engine import scan_rows  # noqa: E402
from kmeans_regimes.partition import _split_rows  # noqa: E402


def main():
    rng = np.random.default_rng(20260)
    dev = rdev.HostReferenceDevice()
    out = {}
    cases = [(3000, 7, 5, 512, None), (2500, 25, 16, 1000, 400_000), (1201, 3, 4, 300, None)]
    for ci, (n, m, k, block, cap) in enumerate(cases):
        x = rng.standard_normal((n, m)) * rng.uniform(0.5, 20.0)
        if ci == 1:
            x = x.astype(np.float32).astype(np.float64)  # fp32-representable (fp32 resident path)
        x[n // 3] = x[n // 5]  # a duplicate row: equal-distance ties in the pair scan
        labels = rng.integers(0, k, size=n).astype(np.int64)
        out[f"c{ci}_x"] = x
        out[f"c{ci}_labels"] = labels
        out[f"c{ci}_meta"] = np.array([n, m, k, block, -1 if cap is None else cap], dtype=np.int64)
        xt = np.ascontiguousarray(x.T)
        rows = scan_rows(n, cap)
        for mode, balanced in (("contig", False), ("bal", True)):
            parts = _split_rows(rows, 3, balanced)
            res = []
            for pi, part in enumerate(parts):
                r = dev.collect(dev.submit(rdev.max_pair_job(xt, part, n)))
                pair = r.pair
                out[f"c{ci}_{mode}_rows{pi}"] = np.asarray(part, dtype=np.int64)
                res.append([-1.0, -1, -1] if pair is None else [pair.d2, pair.i, pair.j])
            out[f"c{ci}_{mode}_pairs"] = np.array(res, dtype=np.float64)
        # sum jobs over block-aligned spans (two jobs: [0, s) and [s, n))
        s = block * ((n // block) // 2)
        for ji, (a, b) in enumerate(((0, s), (s, n))):
            r = dev.collect(dev.submit(rdev.coord_sum_job(x, a, b, block)))
            out[f"c{ci}_coord{ji}"] = r.partial.sums
            out[f"c{ci}_coord{ji}_first"] = np.array([r.partial.first_block])
            r = dev.collect(dev.submit(rdev.cluster_sum_job(x, labels, k, a, b, block)))
            out[f"c{ci}_clus{ji}"] = r.partial.sums
            out[f"c{ci}_clus{ji}_counts"] = r.partial.counts
        out[f"c{ci}_span"] = np.array([s], dtype=np.int64)
    assert dev.outstanding() == 0
    OUT.parent.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({len(out)} arrays)")


if __name__ == "__main__":
    main()
