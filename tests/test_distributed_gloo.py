"""Row-sharded multi-rank driver (paper_1402_3788_b200.distributed) over
torch.distributed gloo, world_size 2 and 3, on CPU.

Each rank owns a contiguous shard (partition.plan_chunks rule) and a CPU
stand-in engine with the GPU engine's step contract; one allreduce of the
int64 partial buffer per iteration.  The gathered result must equal the
single-process reference run (oracle.lloyd): labels, iterations, converged
and counts exactly, centres to 1e-12 relative — including iterations with
empty-cluster repairs (global argmax across shards) and exhausted runs.
"""

import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, outdir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from fake_step_engine import FakeLoopEngine, FakeStepEngine
    from paper_1402_3788_b200.distributed import TorchCollective, run_sharded, shard_rows

    dist.init_process_group("gloo", rank=rank, world_size=world)
    for i, (x, c0, max_iters, tol, batched) in enumerate(cases):  # several cases per spawn (start-up cost)
        lo, hi = shard_rows(x.shape[0], world, rank)
        eng = (FakeLoopEngine if batched else FakeStepEngine)(x[lo:hi])
        res = run_sharded(eng, TorchCollective(), c0, max_iters=max_iters, tol=tol)
        assert not batched or hasattr(eng, "st"), "the batched device-state loop must have run"
        np.savez(Path(outdir) / f"case{i}_rank{rank}.npz", centers=res.centers, counts=res.counts, labels=res.labels,
                 iterations=res.iterations, converged=res.converged, row_offset=res.row_offset, lo=lo)
    dist.barrier()
    dist.destroy_process_group()


def run_world(world, cases):
    """cases: [(x, c0, max_iters, tol, batched)] → [(rank-0 result, gathered labels)]"""
    out = []
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), cases, d), nprocs=world, join=True)
        for i in range(len(cases)):
            parts = [dict(np.load(Path(d) / f"case{i}_rank{r}.npz")) for r in range(world)]
            for p in parts:
                assert int(p["row_offset"]) == int(p["lo"])
                assert np.array_equal(p["centers"], parts[0]["centers"]), "centres must be replicated bit-identically"
                assert np.array_equal(p["counts"], parts[0]["counts"])
                assert int(p["iterations"]) == int(parts[0]["iterations"])
            out.append((parts[0], np.concatenate([p["labels"] for p in parts])))
    return out


def _check_many(world, cases):
    from oracle import oracle

    for (x, c0, max_iters, tol, _), (got, labels) in zip(cases, run_world(world, cases)):
        want = oracle.lloyd(x, c0, max_iters=max_iters, tol=tol)
        assert int(got["iterations"]) == want["iterations"]
        assert bool(got["converged"]) == want["converged"]
        assert np.array_equal(labels, want["labels"])
        assert np.array_equal(got["counts"], want["counts"])
        rel = np.max(np.abs(got["centers"] - want["centers"]) / np.maximum(np.abs(want["centers"]), 1.0))
        assert rel <= 1e-12, rel


def _check(x, c0, world, max_iters=1000, tol=0.0, batched=False):
    _check_many(world, [(x, c0, max_iters, tol, batched)])


def test_shard_rows_rule():
    from paper_1402_3788_b200.distributed import shard_rows

    assert [shard_rows(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    spans = [shard_rows(1001, 8, r) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 1001
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


# --- the batched device-state loop (distributed._run_batched: several [allreduce, finish, pass]
# iterations per host round trip, gated kernels) — the branch the NCCL/GPU path takes -------------


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_single_process(world):
    """Both host loops of distributed.run_sharded — the per-iteration step loop and the batched
    device-state loop (_run_batched: several [allreduce, finish, pass] iterations per host round
    trip, gated kernels; the branch the NCCL/GPU path takes) — on converged runs, exhausted runs
    (max_iters 1 / 3 / 17: the final assign folded into the counts) and empty clusters (duplicated
    initial centres; the batched loop stops mid-batch, the host runs the global repair — argmax
    across shards — the check and the repaired assignment, then batching resumes)."""
    from conftest import golden
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    x = generate_synthetic_array(3001, 5, 4, seed=3, dtype=np.float32).astype(np.float64)
    y = generate_synthetic_array(2000, 6, 5, seed=8, dtype=np.float32).astype(np.float64)
    g1, g2 = golden("all_dup_repair"), golden("dup_center_repair")
    cases = []
    for batched in (False, True):
        cases += [(x, x[:4].copy(), 1000, 0.0, batched)]
        cases += [(y, y[:5].copy(), it, 0.0, batched) for it in (1, 3, 17)]
        cases += [(g["coords"].astype(np.float64), g["c0"], 1000, 0.0, batched) for g in (g1, g2)]
    _check_many(world, cases)
