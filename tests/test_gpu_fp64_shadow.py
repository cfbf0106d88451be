"""fp64 points that are not fp32-representable (km_load_points_f64 keeps them in fp64): the
tensor-core pass streams their fp32 shadow (round to nearest) for the certified filter, and the
exact fp64 rows feed the recheck, the Δ of changed points and the cluster sums.  The labels must
still be exactly the reference's (`_kernels.py:22-45` on the fp64 coordinates), so the cases below
put the decision below fp32 resolution:

* points within 1e-12 (relative) of the bisector of two centres: their fp32 shadows are ties
  the filter cannot certify; only the fp64 recheck of the exact row gets them right;
* a 2M × 25 × 16 run (the cfg3 shape) with fp64 coordinates, to convergence;
* the A/B switch (KM_NO_FP32_SHADOW, the SIMT fp64 pass) must give the same bits.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CENTER_RTOL = 1e-12


def rel_err(a, b, floor=1.0):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def fit(x, c0, iters):
    from paper_1402_3788_b200 import _native

    eng = _native.NativeEngine(0)
    eng.load(x)
    info = eng.points_info()
    centers, counts, labels, it, conv = eng.lloyd(c0, iters, 0.0)
    out = dict(centers=centers, counts=counts, labels=labels, iterations=it, converged=conv,
               path=eng.kernel_path(), point_bytes=info["point_bytes"], stats=eng.stats())
    eng.close()
    return out


def check(want, got, name):
    assert got["iterations"] == want["iterations"], name
    assert got["converged"] == want["converged"], name
    assert np.array_equal(got["labels"], want["labels"]), name
    assert np.array_equal(got["counts"], want["counts"]), name
    assert rel_err(got["centers"], want["centers"]) <= CENTER_RTOL, name


def test_fp64_bisector_points_below_fp32_resolution():
    from oracle import oracle

    rng = np.random.default_rng(11)
    m, k = 12, 16
    c = rng.standard_normal((k, m))
    n = 200_000
    a = rng.integers(k, size=n)
    b = (a + 1 + rng.integers(k - 1, size=n)) % k
    mid = 0.5 * (c[a] + c[b])
    # ±1e-12·|c| along (c_b − c_a): the nearest centre flips with the sign, fp32 cannot see it
    eps = rng.choice([-1.0, 1.0], size=(n, 1)) * 1e-12
    x = mid + eps * (c[b] - c[a])
    x[: n // 2] += rng.standard_normal((n // 2, m)) * 0.3  # and ordinary points
    want_l, want_c = oracle.assign(x, c, n_workers=8)
    from paper_1402_3788_b200 import _native

    eng = _native.NativeEngine(0)
    eng.load(x)
    assert eng.points_info()["point_bytes"] == 8
    labels, counts = eng.assign(c)
    assert eng.kernel_path() == 2
    eng.close()
    assert np.array_equal(labels, want_l) and np.array_equal(counts, want_c)
    # and as a fit (the bisector points keep flipping as the centres move)
    want = oracle.lloyd(x, c, max_iters=6, n_workers=8)
    got = fit(x, c, 6)
    assert got["path"] == 2 and got["point_bytes"] == 8
    check(want, got, "bisector fit")
    assert got["stats"]["rechecked"] > 0


def test_fp64_cfg3_shape_to_convergence():
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(2_000_000, 25, 16, seed=0)  # float64, not fp32-representable
    assert x.dtype == np.float64 and not np.array_equal(x.astype(np.float32).astype(np.float64), x)
    c0 = x[:16].copy()
    got = fit(x, c0, 1000)
    assert got["path"] == 2 and got["point_bytes"] == 8
    want = oracle.lloyd(x, c0, max_iters=1000, n_workers=16)
    check(want, got, "cfg3 fp64")


_AB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
x = generate_synthetic_array(300_000, 25, 40, seed=5)
e = _native.NativeEngine(0); e.load(x)
c, n, l, it, conv = e.lloyd(x[:40].copy(), 25, 0.0)
np.savez({out!r}, c=c, n=n, l=l, it=it, conv=conv, path=e.kernel_path())
"""


def test_fp64_shadow_matches_simt_fp64_pass(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for name, env in (("tc", {}), ("simt", {"KM_NO_FP32_SHADOW": "1"})):
        out = str(tmp_path / f"{name}.npz")
        subprocess.run([sys.executable, "-c", _AB.format(root=root, out=out)], check=True, timeout=600,
                       env={**os.environ, **env})
        res[name] = np.load(out)
    assert int(res["tc"]["path"]) == 2 and int(res["simt"]["path"]) != 2
    for key in ("c", "n", "l", "it", "conv"):
        assert np.array_equal(res["tc"][key], res["simt"][key]), key
