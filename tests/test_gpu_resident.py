"""The resident Lloyd loop (one cooperative launch for the whole iteration,
grid barrier between passes, per-CTA finish) against the launch-per-iteration
kernel and the C oracle.

Both paths must give bit-identical centres, counts, labels and iteration
counts: the totals are exact int64 fixed-point sums and every CTA derives the
same decisions from them.  KM_NO_RESIDENT=1 (read by km_lloyd at call time)
forces the launch-per-iteration path.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fit(x, c0, iters, tol=0.0, resident=True):
    from paper_1402_3788_b200 import _native

    if resident:
        os.environ.pop("KM_NO_RESIDENT", None)
    else:
        os.environ["KM_NO_RESIDENT"] = "1"
    try:
        eng = _native.NativeEngine(0)
        eng.load(x)
        centers, counts, labels, it, conv = eng.lloyd(c0, iters, tol)
        st = eng.stats()
        eng.close()
    finally:
        os.environ.pop("KM_NO_RESIDENT", None)
    return centers, counts, labels, it, conv, st


@pytest.mark.parametrize("n,m,k,iters,tol", [(300_000, 25, 16, 60, 0.0), (100_000, 10, 8, 1000, 0.0),
                                             (150_000, 5, 4, 1000, 1e-3), (80_000, 25, 64, 25, 0.0),
                                             (60_000, 13, 40, 30, 0.0), (7_777, 25, 16, 1000, 0.0)])
def test_resident_equals_per_iteration_launches(n, m, k, iters, tol):
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, k, seed=11 + n % 97, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    a = fit(x, c0, iters, tol, resident=True)
    b = fit(x, c0, iters, tol, resident=False)
    assert a[3] == b[3] and a[4] == b[4]
    assert np.array_equal(a[0], b[0]), "centres must be bit-identical"
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    # the resident run used few launches: one per empty-cluster repair round (+ the prep kernel)
    assert a[5]["host_syncs"] <= b[5]["host_syncs"]


def test_resident_repair_and_relaunch_vs_oracle():
    """Duplicated initial centres: the duplicates come out empty after the first update, the
    resident launch stops for the host repair, then a new launch continues the same loop."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(120_000, 25, 16, seed=5, dtype=np.float32)
    c0 = x[:16].astype(np.float64)
    c0[5] = c0[3]
    c0[9] = c0[3]
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=200, n_workers=8)
    centers, counts, labels, it, conv, st = fit(x, c0, 200)
    assert st["repairs"] >= 1
    assert it == want["iterations"] and conv == want["converged"]
    assert np.array_equal(labels, want["labels"]) and np.array_equal(counts, want["counts"])
    rel = np.max(np.abs(centers - want["centers"]) / np.maximum(np.abs(want["centers"]), 1.0))
    assert rel <= 1e-12


def test_resident_exhausted_counts_are_final_assignment():
    """max_iters reached without convergence: one more assign pass inside the launch, counts =
    bincount(L_T), labels = A(C_T) (engine.iterate's exhaustion rule)."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(200_000, 25, 16, seed=2, dtype=np.float32)
    c0 = x[:16].astype(np.float64)
    for iters in (1, 2, 7):
        want = oracle.lloyd(x.astype(np.float64), c0, max_iters=iters, n_workers=8)
        centers, counts, labels, it, conv, _ = fit(x, c0, iters)
        assert it == iters and not conv and not want["converged"]
        assert np.array_equal(labels, want["labels"]) and np.array_equal(counts, want["counts"])
        assert np.array_equal(np.bincount(labels, minlength=16), counts)


def test_sharded_nccl_world1_equals_resident():
    """The multi-GPU driver (row shards, NCCL allreduce, batched device-state loop) at world size 1
    must reproduce the single-GPU resident loop bit for bit — including a repair and exhaustion."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1402_3788_b200 import _native
    from paper_1402_3788_b200.datasets import generate_synthetic_array
    from paper_1402_3788_b200.distributed import TorchCollective, run_sharded

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        coll = TorchCollective()
        x = generate_synthetic_array(150_000, 25, 16, seed=9, dtype=np.float32)
        for c0, iters in ((x[:16].astype(np.float64), 1000), (x[:16].astype(np.float64), 9)):
            want = fit(x, c0, iters)
            eng = _native.NativeEngine(0)
            eng.load(x)
            got = run_sharded(eng, coll, c0, max_iters=iters)
            eng.close()
            assert got.iterations == want[3] and got.converged == want[4]
            assert np.array_equal(got.centers, want[0]) and np.array_equal(got.counts, want[1])
            assert np.array_equal(got.labels, want[2])
        c0 = x[:16].astype(np.float64)
        c0[7] = c0[2]  # an empty cluster after the first update: global repair through the collective
        want = fit(x, c0, 300)
        eng = _native.NativeEngine(0)
        eng.load(x)
        got = run_sharded(eng, coll, c0, max_iters=300)
        eng.close()
        assert want[5]["repairs"] >= 1
        assert got.iterations == want[3] and got.converged == want[4]
        assert np.array_equal(got.labels, want[2]) and np.array_equal(got.counts, want[1])
        assert np.array_equal(got.centers, want[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("max_iters,tol", [(1000, 0.0), (1000, 1e-3), (1000, 1e-2), (7, 0.0), (8, 0.0)])
def test_run_ahead_stop_points_vs_oracle(max_iters, tol):
    """n ≥ 500k: split first pass, then the resident loop whose tails run ahead into the next pass
    (transform + raw-slot refill).  Stopping right after such a tail — convergence at tol = 0 or at
    a coarse tol, or an exhausted run's final pass — must leave the result exactly the reference's
    (and the launch must end cleanly: the teardown waits for each raw slot's latest copy only)."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(600_000, 25, 16, seed=8, dtype=np.float32)
    c0 = x[:16].astype(np.float64)
    centers, counts, labels, it, conv, st = fit(x, c0, max_iters, tol, resident=True)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=max_iters, tol=tol, n_workers=16)
    assert it == want["iterations"] and conv == want["converged"]
    assert np.array_equal(labels, want["labels"]) and np.array_equal(counts, want["counts"])
    rel = np.max(np.abs(centers - want["centers"]) / np.maximum(np.abs(want["centers"]), 1.0))
    assert rel <= 1e-12
