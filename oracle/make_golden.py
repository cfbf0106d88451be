"""Generate tests/golden/*.npz by running the REAL reference in this container.

TEST INFRASTRUCTURE ONLY.  Usage (build container; /root/reference is not on
the GPU box, so the vectors are committed):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden.py

Each fixture records inputs (points, initial centres, k, max_iters, tol) and
the reference outputs of the hot path (labels, centres, counts, iterations,
converged) plus step-level vectors (assign_step / update_step / converged /
wcss / center_distances).  The generating calls are the reference's own public
functions (engine.iterate with assign_step/update_step closures, i.e. the
run_single path, engine.py:320-370), on inputs drawn with the reference test
suite's generators (pkg/tests/conftest.py:16-43) and datasets.generate_synthetic
(datasets.py:73-97).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

from kmeans_regimes import _kernels  # noqa: E402
from kmeans_regimes.datasets import generate_synthetic  # noqa: E402
from kmeans_regimes.engine import (  # noqa: E402
    KmeansConfig, assign_step, converged, diameter, init_centers, iterate, update_step,
)
from kmeans_regimes.model import Assignment, ClusterModel, Dataset, wcss  # noqa: E402

from conftest import random_coords  # noqa: E402  (reference test generator)


def run_iterate(coords, c0, max_iters=1000, tol=0.0):
    ds = Dataset(coords)
    cfg = KmeansConfig(k=c0.shape[0], max_iters=max_iters, tol=tol)
    model = ClusterModel(np.array(c0, dtype=np.float64, copy=True))
    model, assignment, iterations, done, _ = iterate(
        ds, cfg, model,
        lambda mdl: assign_step(ds, mdl),
        lambda a: update_step(ds, a, cfg.k, block=cfg.accum_block),
    )
    return {
        "labels": assignment.labels.copy(),
        "centers": model.centers.copy(),
        "counts": model.counts.copy(),
        "iterations": np.int64(iterations),
        "converged": np.bool_(done),
    }


def save(name, **arrays):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)


def lloyd_case(name, coords, c0, max_iters=1000, tol=0.0, compact_labels=False):
    res = run_iterate(coords, c0, max_iters, tol)
    labels = res["labels"].astype(np.uint16) if compact_labels else res["labels"]
    stored = coords.astype(np.float32) if np.array_equal(coords.astype(np.float32), coords) else coords
    save(name, coords=stored, c0=np.asarray(c0, dtype=np.float64), max_iters=np.int64(max_iters),
         tol=np.float64(tol), labels=labels, centers=res["centers"], counts=res["counts"],
         iterations=res["iterations"], converged=res["converged"])
    print(f"{name}: n={coords.shape[0]} m={coords.shape[1]} k={c0.shape[0]} "
          f"iters={int(res['iterations'])} conv={bool(res['converged'])}")


def main():
    _kernels.warmup()
    # 1. blob4 canonical instance (conftest.py:51-54), maximin init via the reference seeding
    blob4 = np.array([[0.0, 0.0], [0.0, 1.0], [10.0, 0.0], [10.0, 1.0]])
    ds = Dataset(blob4)
    c0 = init_centers(ds, KmeansConfig(k=2), diameter(ds)).centers
    lloyd_case("blob4", blob4, c0)

    # 2. tie → lowest index (test_engine.py:182-185)
    tie_x = np.array([[5.0, 0.0]])
    tie_c = np.array([[0.0, 0.0], [10.0, 0.0]])
    save("assign_tie", coords=tie_x, centers=tie_c,
         labels=assign_step(Dataset(tie_x), ClusterModel(tie_c.copy())).labels)

    # 3. repair known-answer (test_engine.py:227-235)
    rep_x = np.array([[0.0, 0.0], [1.0, 0.0], [8.0, 0.0]])
    a = Assignment(np.array([0, 0, 0]))
    mdl = update_step(Dataset(rep_x), a, 2)
    save("update_repair", coords=rep_x, labels_in=np.array([0, 0, 0], dtype=np.int64), k=np.int64(2),
         labels_out=a.labels.copy(), centers=mdl.centers, counts=mdl.counts)

    # 4. random fp64 instances (reference generators), maximin init from the reference
    rng = np.random.default_rng(20260821)
    rand = {}
    for t in range(40):
        n = int(rng.integers(10, 400))
        m = int(rng.integers(1, 12))
        coords = random_coords(rng, n, m)
        k = int(rng.integers(1, min(8, n) + 1))
        ds = Dataset(coords)
        try:
            c0 = init_centers(ds, KmeansConfig(k=k), diameter(ds)).centers
        except Exception:
            continue
        res = run_iterate(coords, c0)
        rand[t] = (coords, c0, res)
    np.savez_compressed(
        OUT / "random_fp64.npz",
        **{f"{key}_{t}": val for t, (coords, c0, res) in rand.items()
           for key, val in (("coords", coords), ("c0", c0), ("labels", res["labels"]),
                            ("centers", res["centers"]), ("counts", res["counts"]),
                            ("iterations", res["iterations"]), ("converged", res["converged"]))},
    )
    print(f"random_fp64: {len(rand)} instances")

    # 5. fp32-representable synthetic blobs (the bench's input family), first-K init
    for name, (n, m, k, seed) in {
        "synth_10k_5_4": (10_000, 5, 4, 0),        # BASELINE configs[0]
        "synth_20k_25_16": (20_000, 25, 16, 3),
        "synth_30k_10_8": (30_000, 10, 8, 1),
    }.items():
        coords = generate_synthetic(n, m, k, seed=seed).coords.astype(np.float32).astype(np.float64)
        lloyd_case(name, coords, coords[:k].copy(), compact_labels=True)

    # 6. max_iters cap (test_engine.py:341-345) and k = 1
    coords = random_coords(np.random.default_rng(7), 300, 2, kind=1)
    lloyd_case("maxiter1", coords, coords[:6].copy(), max_iters=1)
    lloyd_case("maxiter5", coords, coords[:6].copy(), max_iters=5)
    lloyd_case("k1", coords, coords[:1].copy())

    # 7. empty cluster inside the loop: duplicated initial centre → ties send
    # every point to the lower index, the duplicate starts empty and is repaired
    rng = np.random.default_rng(11)
    coords = random_coords(rng, 200, 3, kind=2)
    c0 = coords[[0, 1, 1, 2, 3]].copy()
    lloyd_case("dup_center_repair", coords, c0)
    coords = random_coords(rng, 500, 4, kind=0)
    c0 = np.repeat(coords[:1], 6, axis=0)   # all six identical: five empties at once
    lloyd_case("all_dup_repair", coords, c0)

    # 8. tol > 0
    coords = generate_synthetic(5000, 6, 5, seed=9).coords
    lloyd_case("tol_pos", coords, coords[:5].copy(), tol=1e-3)

    # 9. update_step vectors with random labels, incl. empties (test_engine.py:215-225)
    rng = np.random.default_rng(99)
    ups = {}
    for t in range(20):
        coords = random_coords(rng, int(rng.integers(6, 120)), int(rng.integers(1, 6)))
        k = int(rng.integers(1, 7))
        labels = rng.integers(max(1, k - (t % 3)), size=len(coords)).astype(np.int64)
        a = Assignment(labels.copy())
        mdl = update_step(Dataset(coords), a, k)
        ups[t] = dict(coords=coords, k=np.int64(k), labels_in=labels, labels_out=a.labels.copy(),
                      centers=mdl.centers, counts=mdl.counts)
    np.savez_compressed(OUT / "update_random.npz",
                        **{f"{key}_{t}": v for t, d in ups.items() for key, v in d.items()})

    # 10. assign_step vectors + converged + wcss + center_distances
    rng = np.random.default_rng(5)
    asg = {}
    for t in range(20):
        coords = random_coords(rng, int(rng.integers(4, 200)), int(rng.integers(1, 12)))
        k = int(rng.integers(1, 7))
        centers = coords[rng.choice(len(coords), size=min(k, len(coords)), replace=False)].copy()
        mdl = ClusterModel(centers.copy())
        lab = assign_step(Dataset(coords), mdl).labels
        out = np.empty((len(coords), centers.shape[0]))
        _kernels.center_distances(coords, centers, out)
        asg[t] = dict(coords=coords, centers=centers, labels=lab, counts=mdl.counts.copy(),
                      wcss=np.float64(wcss(Dataset(coords), mdl, Assignment(lab))), dist=out)
    np.savez_compressed(OUT / "assign_random.npz",
                        **{f"{key}_{t}": v for t, d in asg.items() for key, v in d.items()})
    conv_cases = [
        (np.array([[1.0, 2.0]]), np.array([[1.0, 2.0]]), 0.0),
        (np.array([[1.0, 2.0]]), np.array([[1.0, 2.0 + 1e-9]]), 0.0),
        (np.array([[1.0, 2.0]]), np.array([[1.0, 2.0 + 1e-9]]), 1e-6),
        (np.array([[0.0], [0.0]]), np.array([[0.0], [5.0]]), 1.0),
        (np.array([[0.0], [0.0]]), np.array([[0.0], [5.0]]), 5.0),
        (np.array([[1e-170, 0.0]]), np.array([[2e-170, 0.0]]), 0.0),   # d*d underflows → "equal"
        (np.array([[-0.0, 1.0]]), np.array([[0.0, 1.0]]), 0.0),        # signed zero
    ]
    np.savez_compressed(OUT / "converged_cases.npz",
                        **{f"{key}_{i}": v for i, (p, q, tol) in enumerate(conv_cases)
                           for key, v in (("prev", p), ("next", q), ("tol", np.float64(tol)),
                                          ("out", np.bool_(converged(ClusterModel(p), ClusterModel(q), tol))))})
    print("done")


def seeding():
    """Seeding phase + full run_single (engine.py:124-215, 346-370): diameter (optionally with a
    pair cap), maximin / random-far initial centres, the Lloyd result and its wcss, plus
    degenerate cases (fewer distinct points than k)."""
    from kmeans_regimes.engine import global_centroid_of, run_single  # noqa: E402
    from kmeans_regimes.exceptions import DegenerateDataError  # noqa: E402

    _kernels.warmup()
    rng = np.random.default_rng(424242)
    cases = {}
    specs = []
    for t in range(24):
        n = int(rng.integers(2, 600))
        m = int(rng.integers(1, 10))
        kind = int(rng.integers(0, 3))
        coords = random_coords(rng, n, m, kind=kind)
        if t % 2:
            coords = coords.astype(np.float32).astype(np.float64)
        k = int(rng.integers(1, min(9, n) + 1))
        init = "maximin" if t % 3 else "random-far"
        cap = None if t % 4 else int(rng.integers(1, max(2, n * (n - 1) // 2)))
        specs.append((coords, k, init, int(t), cap))
    for name, (n, m, k, seed) in {"s_synth_3k_5_4": (3000, 5, 4, 2), "s_synth_5k_25_16": (5000, 25, 16, 4)}.items():
        coords = generate_synthetic(n, m, k, seed=seed).coords.astype(np.float32).astype(np.float64)
        specs.append((coords, k, "maximin", seed, None))
        specs.append((coords, k, "random-far", seed, 20_000))
    dup = np.repeat(np.array([[1.0, 2.0], [3.0, 4.0]]), 5, axis=0)
    specs.append((dup, 3, "maximin", 0, None))          # 2 distinct points, k = 3 → degenerate
    specs.append((np.zeros((4, 3)), 2, "maximin", 0, None))  # diameter 0 → degenerate at the 2nd centre
    for t, (coords, k, init, seed, cap) in enumerate(specs):
        ds = Dataset(coords)
        cfg = KmeansConfig(k=k, init=init, seed=seed, diameter_pair_cap=cap)
        diam = diameter(ds, pair_cap=cap)
        rec = dict(coords=coords, k=np.int64(k), init=np.bytes_(init), seed=np.int64(seed),
                   cap=np.int64(-1 if cap is None else cap), d=np.float64(diam.d), i=np.int64(diam.i),
                   j=np.int64(diam.j), centroid=global_centroid_of(ds))
        try:
            c0 = init_centers(ds, cfg, diam).centers
            res = run_single(ds, cfg)
            rec.update(degenerate=np.bool_(False), c0=c0, labels=res.assignment.labels,
                       centers=res.model.centers, counts=res.model.counts, iterations=np.int64(res.iterations),
                       converged=np.bool_(res.converged),
                       inertia=np.float64(wcss(ds, res.model, res.assignment)))
        except DegenerateDataError:
            rec.update(degenerate=np.bool_(True))
        cases[t] = rec
    np.savez_compressed(OUT / "seeding.npz", **{f"{key}_{t}": v for t, d in cases.items() for key, v in d.items()},
                        count=np.int64(len(cases)))
    print(f"seeding: {len(cases)} cases ({sum(bool(d['degenerate']) for d in cases.values())} degenerate)")


def run_iterate_parallel(coords, c0, max_iters=1000, tol=0.0, workers=8):
    """engine.iterate with the run_multi closures (partition.assign_parallel / update_parallel,
    partition.py:215-261, 264-305) — bit-identical to run_single for any worker count
    (the reference's own cross-regime tests), and 8x faster at the benchmark sizes."""
    from concurrent.futures import ThreadPoolExecutor

    from kmeans_regimes.partition import assign_parallel, plan_chunks, update_parallel

    ds = Dataset(coords, copy=False)
    cfg = KmeansConfig(k=c0.shape[0], max_iters=max_iters, tol=tol)
    plan = plan_chunks(ds.n, workers)
    model = ClusterModel(np.array(c0, dtype=np.float64, copy=True))
    with ThreadPoolExecutor(max_workers=plan.n_workers) as pool:
        model, assignment, iterations, done, _ = iterate(
            ds, cfg, model,
            lambda mdl: assign_parallel(ds, mdl, plan, executor=pool),
            lambda a: update_parallel(ds, a, cfg.k, plan, block=cfg.accum_block, executor=pool),
        )
    return {"labels": assignment.labels, "centers": model.centers.copy(), "counts": model.counts.copy(),
            "iterations": np.int64(iterations), "converged": np.bool_(done)}


def bench_configs(which=("cfg2", "cfg3", "cfg3_20", "cfg4_20", "cfg5_3")):
    """Full-size goldens of the BASELINE.json benchmark configs (the GPU box regenerates the
    points with datasets.generate_synthetic_array — identical bytes — and checks them by digest):
    the reference loop from the first K rows, tol = 0.  Labels are stored in full (uint8/uint16)
    where they are small, otherwise as a SHA-256 digest of the int64 label array plus a strided
    sample.  cfg3 runs to convergence (539 iterations); the *_20 / *_3 cases stop at max_iters
    (the exhausted-run rule, engine.py:339-343)."""
    import hashlib
    import time

    specs = {
        "cfg2": (100_000, 10, 8, 1000),
        "cfg3": (2_000_000, 25, 16, 1000),
        "cfg3_20": (2_000_000, 25, 16, 20),
        "cfg4_20": (2_000_000, 25, 512, 20),
        "cfg5_3": (64_000_000, 25, 64, 3),
    }
    _kernels.warmup()
    cache = {}
    for name in which:
        n, m, k, iters = specs[name]
        key = (n, m, k)
        if key not in cache:
            cache.clear()
            x32 = generate_synthetic(n, m, k, seed=0).coords.astype(np.float32)
            cache[key] = (hashlib.sha256(x32.tobytes()).hexdigest(), x32.astype(np.float64))
        digest, coords = cache[key]
        c0 = coords[:k].copy()
        t0 = time.perf_counter()
        res = run_iterate_parallel(coords, c0, max_iters=iters)
        el = time.perf_counter() - t0
        lab = res["labels"]
        rec = dict(n=np.int64(n), m=np.int64(m), k=np.int64(k), seed=np.int64(0), max_iters=np.int64(iters),
                   tol=np.float64(0.0), coords_sha256=np.bytes_(digest), c0=c0,
                   labels_sha256=np.bytes_(hashlib.sha256(lab.astype(np.int64).tobytes()).hexdigest()),
                   labels_sample=lab[::997].astype(np.int64), centers=res["centers"], counts=res["counts"],
                   iterations=res["iterations"], converged=res["converged"], ref_seconds=np.float64(el))
        if n <= 2_000_000:
            rec["labels"] = lab.astype(np.uint8 if k <= 256 else np.uint16)
        save("bench_" + name, **rec)
        print(f"bench_{name}: n={n} m={m} k={k} iterations={int(res['iterations'])} "
              f"converged={bool(res['converged'])} ({el:.1f} s, 8 threads)", flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["seeding"]:
        seeding()
    elif sys.argv[1:2] == ["bench"]:
        bench_configs(tuple(sys.argv[2:]) or ("cfg2", "cfg3", "cfg3_20", "cfg4_20", "cfg5_3"))
    else:
        main()
        seeding()
