"""The row-sharded resident loop with the in-kernel Δ exchange over peer memory
(km_peer_* / distributed._run_resident_peer) on one GPU: world size 1, the
rank's exchange buffer is its own (the same push → release flag → acquire →
sum code path the NVLink exchange runs at world > 1).  Results must be
bit-identical to the single-GPU resident loop (km_lloyd) and equal the C oracle:
converged runs, exhausted runs, and empty-cluster repairs (the kernel stops,
the host runs the global repair through the collective, the loop resumes).

This run has one GPU, so world > 1 is covered by construction and by the
host-side gloo tests of the same driver (tests/test_distributed_gloo.py)."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def coll():
    import torch.distributed as dist

    from paper_1402_3788_b200.distributed import TorchCollective

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield TorchCollective()
    dist.destroy_process_group()


def run_peer(coll, x, c0, max_iters, tol=0.0):
    from paper_1402_3788_b200 import _native
    from paper_1402_3788_b200.distributed import run_sharded

    eng = _native.NativeEngine(0)
    eng.load(x)
    r = run_sharded(eng, coll, c0, max_iters=max_iters, tol=tol)
    st = eng.stats()
    eng.close()
    return r, st


def run_single(x, c0, max_iters, tol=0.0):
    from paper_1402_3788_b200 import _native

    eng = _native.NativeEngine(0)
    eng.load(x)
    out = eng.lloyd(c0, max_iters, tol)
    eng.close()
    return out


@pytest.mark.parametrize("n,m,k,max_iters", [(200_000, 25, 16, 1000), (300_000, 10, 8, 7), (50_000, 5, 4, 1),
                                             (120_000, 25, 40, 12)])
def test_peer_loop_matches_single_gpu_and_oracle(coll, n, m, k, max_iters):
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(n, m, min(k, 16), seed=n % 97, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    r, st = run_peer(coll, x, c0, max_iters)
    centers, counts, labels, iters, conv = run_single(x, c0, max_iters)
    assert st["kernel_launches"] > 0
    assert r.iterations == iters and r.converged == conv
    assert np.array_equal(r.centers, centers) and np.array_equal(r.counts, counts)
    assert np.array_equal(r.labels, labels)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=max_iters, n_workers=8)
    assert iters == want["iterations"] and np.array_equal(labels, want["labels"])
    assert np.array_equal(counts, want["counts"])


def test_peer_loop_empty_cluster_repair(coll):
    """Duplicated initial centres: clusters start empty, the resident kernel stops with
    need_host, the global repair runs through the collective, the loop resumes."""
    from oracle import oracle
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(60_000, 6, 5, seed=4, dtype=np.float32)
    c0 = np.repeat(x[:1].astype(np.float64), 6, axis=0)
    c0[3] = x[7]
    r, _ = run_peer(coll, x, c0, 1000)
    want = oracle.lloyd(x.astype(np.float64), c0, max_iters=1000, n_workers=8)
    assert r.iterations == want["iterations"] and r.converged == want["converged"]
    assert np.array_equal(r.labels, want["labels"]) and np.array_equal(r.counts, want["counts"])
    rel = np.max(np.abs(r.centers - want["centers"]) / np.maximum(np.abs(want["centers"]), 1.0))
    assert rel <= 1e-12
