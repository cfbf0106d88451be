"""CUDA path vs the reference (golden vectors) and vs the C oracle, through
the C ABI (paper_1402_3788_b200._native → libkmeans_b200.so).

Bar (BASELINE.json north_star): labels and iteration counts bit-exact;
centroids within 1e-5 relative.  The engine decides labels with the
reference's exact fp64 recurrence whenever its certified fp32 filter is not
conclusive, so on the same centres its labels are bit-identical; its centres
come from exact fixed-point sums and agree with the reference's sequential
fp64 sums to ~1e-15, so we hold them to CENTER_RTOL = 1e-12 (far inside the
north-star 1e-5).
"""

import numpy as np
import pytest

from conftest import golden, golden_indexed, random_coords

pytestmark = pytest.mark.gpu

CENTER_RTOL = 1e-12  # north_star allows 1e-5


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


@pytest.fixture(scope="module")
def native():
    from paper_1402_3788_b200 import _native

    return _native


def run(native, coords, c0, max_iters=1000, tol=0.0):
    eng = native.NativeEngine(0)
    eng.load(coords)
    centers, counts, labels, iters, conv = eng.lloyd(c0, max_iters, tol)
    stats = eng.stats()
    eng.close()
    return dict(centers=centers, counts=counts, labels=labels, iterations=iters, converged=conv, stats=stats)


def check(g, res, name=""):
    assert res["iterations"] == int(g["iterations"]), name
    assert res["converged"] == bool(g["converged"]), name
    assert np.array_equal(res["labels"], g["labels"].astype(np.int64)), name
    assert np.array_equal(res["counts"], g["counts"]), name
    assert rel_err(res["centers"], g["centers"]) <= CENTER_RTOL, (name, rel_err(res["centers"], g["centers"]))


@pytest.mark.parametrize("name", ["blob4", "synth_10k_5_4", "synth_20k_25_16", "synth_30k_10_8", "maxiter1",
                                  "maxiter5", "k1", "dup_center_repair", "all_dup_repair", "tol_pos"])
def test_lloyd_golden(native, name):
    g = golden(name)
    coords = g["coords"]  # float32 fixtures are fp32-representable bench-family data
    res = run(native, coords, g["c0"], int(g["max_iters"]), float(g["tol"]))
    check(g, res, name)


def test_lloyd_golden_fp64_inputs(native):
    for idx, g in golden_indexed("random_fp64").items():
        check(g, run(native, g["coords"], g["c0"]), f"random_fp64[{idx}]")


def test_assign_step_golden():
    from paper_1402_3788_b200 import ClusterModel, Dataset, assign_step

    for idx, g in golden_indexed("assign_random").items():
        model = ClusterModel(g["centers"].copy())
        a = assign_step(Dataset(g["coords"]), model)
        assert np.array_equal(a.labels, g["labels"]), idx
        assert np.array_equal(model.counts, g["counts"]), idx


def test_tie_lowest_index():
    from paper_1402_3788_b200 import ClusterModel, Dataset, assign_step

    g = golden("assign_tie")
    assert assign_step(Dataset(g["coords"]), ClusterModel(g["centers"].copy())).labels.tolist() == [0]


def test_update_step_golden():
    from paper_1402_3788_b200 import Assignment, Dataset, update_step

    for idx, g in golden_indexed("update_random").items():
        a = Assignment(g["labels_in"].copy())
        model = update_step(Dataset(g["coords"]), a, int(g["k"]))
        assert np.array_equal(a.labels, g["labels_out"]), idx  # in-place relabel (engine.py:258,272)
        assert np.array_equal(model.counts, g["counts"]), idx
        assert rel_err(model.centers, g["centers"]) <= CENTER_RTOL, idx


def test_repair_known_answer():
    from paper_1402_3788_b200 import Assignment, Dataset, update_step

    g = golden("update_repair")
    a = Assignment([0, 0, 0])
    model = update_step(Dataset(g["coords"]), a, 2)
    assert a.labels.tolist() == [0, 0, 1]
    assert model.counts.tolist() == [2, 1]
    assert np.array_equal(model.centers[1], [8.0, 0.0])


def test_converged_golden():
    from paper_1402_3788_b200 import ClusterModel, converged

    for idx, g in golden_indexed("converged_cases").items():
        assert converged(ClusterModel(g["prev"]), ClusterModel(g["next"]), float(g["tol"])) == bool(g["out"]), idx


def test_wcss_and_transform_golden():
    from paper_1402_3788_b200 import Assignment, ClusterModel, Dataset, wcss
    from paper_1402_3788_b200.model import Dataset as DS

    for idx, g in golden_indexed("assign_random").items():
        ds = Dataset(g["coords"])
        w = wcss(ds, ClusterModel(g["centers"].copy()), Assignment(g["labels"]))
        assert abs(w - float(g["wcss"])) <= 1e-12 * max(1.0, abs(float(g["wcss"]))), idx
        dist = DS(g["coords"]).device_engine().center_distances(g["centers"])
        assert np.array_equal(dist, g["dist"]), idx  # same fp64 recurrence + IEEE sqrt


def test_iterate_seam_with_device_steps():
    """engine.iterate with the device step closures == the device-resident loop."""
    from paper_1402_3788_b200 import ClusterModel, Dataset, KmeansConfig, assign_step, iterate, update_step

    g = golden("synth_10k_5_4")
    ds = Dataset(g["coords"])
    cfg = KmeansConfig(k=4)
    model, assignment, iters, done, _ = iterate(ds, cfg, ClusterModel(g["c0"].copy()),
                                                lambda mdl: assign_step(ds, mdl),
                                                lambda a: update_step(ds, a, 4))
    assert iters == int(g["iterations"]) and done == bool(g["converged"])
    assert np.array_equal(assignment.labels, g["labels"].astype(np.int64))
    assert rel_err(model.centers, g["centers"]) <= CENTER_RTOL


# --- vs the C oracle on seeded inputs ------------------------------------------------------------


@pytest.mark.parametrize("n,m,k,iters", [(100_000, 10, 8, 1000), (200_000, 25, 16, 40), (50_000, 25, 64, 15),
                                         (20_000, 7, 33, 25), (4_099, 3, 5, 1000), (1_000, 70, 6, 30),
                                         (30_000, 25, 512, 4), (400_000, 25, 64, 6), (400_000, 25, 128, 4)])
def test_vs_oracle_seeded(native, n, m, k, iters):
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, k, seed=n + m + k, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=iters, n_workers=8)
    got = run(native, x, c0, iters)
    check(want, got, f"{n}x{m}x{k}")


def test_random_instances_vs_oracle(native):
    from oracle import oracle

    rng = np.random.default_rng(4242)
    for t in range(60):
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(1, 40))
        x = random_coords(rng, n, m)
        if t % 2:
            x = x.astype(np.float32).astype(np.float64)  # fp32-representable → fp32 resident path
        k = int(rng.integers(1, min(12, n) + 1))
        c0 = x[rng.choice(n, size=k, replace=False)].copy()
        want = oracle.lloyd(x, c0, max_iters=50)
        check(want, run(native, x, c0, 50), f"instance {t} n={n} m={m} k={k}")


def test_extreme_magnitudes_use_exact_path(native):
    from oracle import oracle

    rng = np.random.default_rng(3)
    for scale in (1e30, 1e-30, 1e-200):
        x = rng.standard_normal((500, 4)) * scale
        c0 = x[:5].copy()
        want = oracle.lloyd(x, c0, max_iters=20)
        got = run(native, x, c0, 20)
        assert got["iterations"] == want["iterations"]
        assert np.array_equal(got["labels"], want["labels"])
        assert rel_err(got["centers"] / scale, want["centers"] / scale) <= 1e-9


def test_deterministic_bits(native):
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(300_000, 25, 16, seed=1, dtype=np.float32)
    a = run(native, x, x[:16].astype(np.float64), 30)
    b = run(native, x, x[:16].astype(np.float64), 30)
    assert np.array_equal(a["centers"], b["centers"]) and np.array_equal(a["labels"], b["labels"])


# --- full BASELINE sizes: size-independent properties ------------------------------------------


@pytest.mark.parametrize("n,m,k,iters", [(2_000_000, 25, 16, 12), (2_000_000, 25, 64, 5), (2_000_000, 25, 128, 4),
                                         (2_000_000, 25, 512, 2)])
def test_full_size_properties(native, n, m, k, iters):
    """At BASELINE sizes: (1) the labels are the reference argmin for the
    returned centres (checked with the oracle on a 20k-row sample),
    (2) counts = histogram of labels, (3) the centres equal the fp64 means of
    the points per label (np.bincount), (4) counts sum to n."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    eng = native.NativeEngine(0)
    eng.load(x)
    centers, counts, labels, it, conv = eng.lloyd(c0, iters, 0.0)
    assert it == iters and not conv
    # exhausted ⇒ labels = A(C_T), counts = bincount(labels)
    assert counts.sum() == n
    assert np.array_equal(np.bincount(labels, minlength=k), counts)
    rows = np.random.default_rng(0).choice(n, size=20_000, replace=False)
    ref_labels, _ = oracle.assign(x[rows].astype(np.float64), centers)
    assert np.array_equal(labels[rows], ref_labels)
    # one more update on the device vs fp64 means of the pre-repair labels
    # (repaired clusters take a sample's coordinates; donor centres are not
    # recomputed — engine.py:265-276)
    lab = labels.copy()
    c_next, cnt_next = eng.update(lab, k)
    xd = x.astype(np.float64)
    before = np.bincount(labels, minlength=k)
    occ = before > 0
    for f in range(m):
        s = np.bincount(labels, weights=xd[:, f], minlength=k)
        assert rel_err(c_next[occ, f], s[occ] / before[occ]) <= 1e-12
    for c in np.flatnonzero(~occ):  # repaired: centre = the relabelled sample
        assert np.array_equal(c_next[c], xd[np.flatnonzero(lab == c)[0]])
    eng.close()


# --- register-blocked large-K SIMT pass (lloyd_pass_blocked_kernel) ------------------------------


def run_path(native, x, c0, iters, path):
    eng = native.NativeEngine(0)
    eng.load(x)
    eng.set_kernel_path(path)
    centers, counts, labels, it, conv = eng.lloyd(c0, iters, 0.0)
    st = eng.stats()
    eng.close()
    return dict(centers=centers, counts=counts, labels=labels, iterations=it, converged=conv, stats=st)


@pytest.mark.parametrize("n,m,k,iters", [(20_000, 7, 33, 20), (30_000, 16, 200, 6), (25_000, 25, 512, 4),
                                         (9_999, 32, 100, 10), (12_000, 26, 40, 12), (15_000, 25, 1000, 3),
                                         (1_025, 25, 300, 5)])
def test_blocked_pass_vs_oracle_and_unblocked(native, n, m, k, iters):
    """Large-K SIMT pass (fp32, k ≥ 32, m ≤ 32; k = 1000 exceeds the shared-memory accumulators and
    takes the global-atomics variant; n = 1025 leaves a ragged last tile): labels, counts and
    centres equal the C oracle and are bit-identical to the one-point-per-thread kernel (path 3)."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, min(k, n // 2), seed=k + m, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    blk = run_path(native, x, c0, iters, 1)
    ref = run_path(native, x, c0, iters, 3)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=iters, n_workers=8)
    check(want, blk, f"blocked {n}x{m}x{k}")
    assert np.array_equal(blk["labels"], ref["labels"])
    assert np.array_equal(blk["centers"], ref["centers"])
    assert np.array_equal(blk["counts"], ref["counts"])


def test_blocked_pass_ties_and_exact_only(native):
    """Blocked pass edge cases: duplicated centres and points equidistant from several centres (every
    such point fails the certificate; the warp-cooperative recheck must return the lowest index, as
    the reference's strict '<'), and magnitudes past the filter's certified range (exact_only: every
    centre re-evaluated in fp64)."""
    from oracle import oracle

    rng = np.random.default_rng(11)
    grid = rng.integers(-4, 5, size=(6000, 6)).astype(np.float32)  # many exact ties on the lattice
    c0 = grid[:48].astype(np.float64).copy()
    c0[10:20] = c0[0:10]  # duplicated centres
    want = oracle.lloyd(grid.astype(np.float64), c0, max_iters=8)
    got = run_path(native, grid, c0, 8, 1)
    check(want, got, "lattice ties")
    assert got["stats"]["rechecked"] > 0
    big = (rng.standard_normal((3000, 9)) * 1e20).astype(np.float32)
    c1 = big[:40].astype(np.float64)
    want = oracle.lloyd(big.astype(np.float64), c1, max_iters=6)
    got = run_path(native, big, c1, 6, 1)
    assert got["iterations"] == want["iterations"] and np.array_equal(got["labels"], want["labels"])
    assert rel_err(got["centers"] / 1e20, want["centers"] / 1e20) <= 1e-9
