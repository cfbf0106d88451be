"""tcgen05 fused pass: the certified error bound of the 3xTF32 tensor-core
filter holds on real hardware, and the tensor-core and SIMT kernels return
bit-identical results (both must equal the reference)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def native():
    from paper_1402_3788_b200 import _native

    return _native


def exact_scores(x, c):
    """‖c~‖² − 2 x·c~ in fp64 with c~ = fl32(c) (what the filter approximates), plus per-point ‖x‖."""
    cf = c.astype(np.float32).astype(np.float64)
    xd = x.astype(np.float64)
    return (cf * cf).sum(1)[None, :] - 2.0 * xd @ cf.T


@pytest.mark.parametrize("n,m,k", [(200_000, 25, 16), (100_000, 10, 8), (50_000, 5, 4), (60_000, 31, 64),
                                   (30_000, 23, 40), (10_000, 1, 3)])
def test_filter_error_within_certified_bound(n, m, k):
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, k, seed=11, dtype=np.float32)
    c = x[:k].astype(np.float64) + 0.37  # centres not on data points
    eng = native().NativeEngine(0)
    eng.load(x)
    assert eng.kernel_path() in (1, 2)
    got = eng.debug_filter_scores(c)
    eng.close()
    want = exact_scores(x, c)
    nx = np.sqrt((x.astype(np.float64) ** 2).sum(1))
    cmax = np.sqrt((c.astype(np.float32).astype(np.float64) ** 2).sum(1)).max()
    scale = (nx + cmax) ** 2
    mp = 7 if m <= 7 else 15 if m <= 15 else 23 if m <= 23 else 31
    ks = (mp + 1 + 7) // 8
    coef = max((m + 8 + 12 * ks) * 2.0 ** -23, 2.0 ** -18)
    ratio = np.abs(got - want) / scale[:, None]
    worst = float(ratio.max())
    print(f"n={n} m={m} k={k}: max |S_tc - S| / (|x|+C)^2 = {worst:.3e}, certified coef = {coef:.3e}, "
          f"margin {coef / max(worst, 1e-30):.1f}x")
    assert worst <= coef / 4, "tensor-core filter error too close to (or above) its certified bound"


@pytest.mark.parametrize("name", ["synth_10k_5_4", "synth_20k_25_16", "synth_30k_10_8"])
def test_tensorcore_and_simt_agree(name):
    g = golden(name)
    out = {}
    for path in (1, 2):
        eng = native().NativeEngine(0)
        eng.load(g["coords"])
        eng.set_kernel_path(path)
        out[path] = eng.lloyd(g["c0"], int(g["max_iters"]), float(g["tol"]))
        assert eng.kernel_path() == path
        eng.close()
    a, b = out[1], out[2]
    assert a[3] == b[3] == int(g["iterations"])
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[2], g["labels"].astype(np.int64))
    assert np.array_equal(a[0], b[0])  # same exact integer sums → bit-identical centres
    assert np.array_equal(a[1], b[1])


def test_headline_shape_uses_tensor_cores():
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(4096, 25, 16, seed=0, dtype=np.float32)
    eng = native().NativeEngine(0)
    eng.load(x)
    eng.lloyd(x[:16].astype(np.float64), 2, 0.0)
    assert eng.kernel_path() == 2
    eng.close()


def test_filter_scores_full_size_no_races():
    """Every tensor-core score of a 2M-point pass (≈15.6k tiles through the TMA / transform /
    MMA / epilogue rings) is within the certified bound: a ring race shows up as rows scored
    with another point's coordinates."""
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    n, m, k = 2_000_000, 25, 16
    x = generate_synthetic_array(n, m, k, seed=5, dtype=np.float32)
    c = x[:k].astype(np.float64) + 0.25
    eng = native().NativeEngine(0)
    eng.load(x)
    got = eng.debug_filter_scores(c)
    eng.close()
    want = exact_scores(x, c)
    nx = np.sqrt((x.astype(np.float64) ** 2).sum(1))
    cmax = np.sqrt((c.astype(np.float32).astype(np.float64) ** 2).sum(1)).max()
    ratio = np.abs(got - want) / ((nx + cmax) ** 2)[:, None]
    assert float(ratio.max()) <= max((m + 8 + 48) * 2.0 ** -23, 2.0 ** -18) / 4


def _coef(m):
    mp = 7 if m <= 7 else 15 if m <= 15 else 23 if m <= 23 else 31
    ks = (mp + 1 + 7) // 8
    return max((m + 8 + 12 * ks) * 2.0 ** -23, 2.0 ** -18)


@pytest.mark.parametrize("log_ratio", [-8, -12, -16, -18, -20, -22, -24, -26, -30])
@pytest.mark.parametrize("signs", ["same", "alternating"])
def test_filter_bound_adversarial_alignment(log_ratio, signs):
    """Adversarial inputs for the tensor core's internal adder: in every MMA k-step one large
    product next to 24 small ones (ratio 2^log_ratio), all of one sign (maximal truncation
    loss if the adder drops bits below the largest product) or alternating (cancellation).
    The certified coefficient must cover the worst case for every ratio — i.e. the bound does not
    rely on the error averaging out, whatever alignment width the hardware adder keeps."""
    n, m, k = 4096, 25, 16
    rng = np.random.default_rng(abs(log_ratio) * 7 + (signs == "same"))
    r = 2.0 ** (log_ratio / 2)  # per-operand ratio: small products = r² × the large one
    big = rng.uniform(1.0, 2.0, size=n)
    x = np.empty((n, m))
    x[:, 0] = big
    x[:, 1:] = r * rng.uniform(1.0, 2.0, size=(n, m - 1))
    c = np.empty((k, m))
    c[:, 0] = -rng.uniform(1.0, 2.0, size=k)
    c[:, 1:] = -r * rng.uniform(1.0, 2.0, size=(k, m - 1))
    if signs == "alternating":
        x[:, 1::2] *= -1.0
    x = x.astype(np.float32)
    # the big feature first in a point, but also rotated into other k-step positions
    for i in range(1, 8):
        x[i * 512:(i + 1) * 512] = np.roll(x[i * 512:(i + 1) * 512], 3 * i, axis=1)
    eng = native().NativeEngine(0)
    eng.load(x)
    got = eng.debug_filter_scores(c)
    eng.close()
    want = exact_scores(x, c)
    nx = np.sqrt((x.astype(np.float64) ** 2).sum(1))
    cmax = np.sqrt((c.astype(np.float32).astype(np.float64) ** 2).sum(1)).max()
    worst = float((np.abs(got - want) / ((nx + cmax) ** 2)[:, None]).max())
    print(f"ratio 2^{log_ratio} {signs}: worst {worst:.3e} (certified {_coef(m):.3e})")
    assert worst <= _coef(m) / 4
