"""Row-sharded multi-GPU Lloyd loop: one process per GPU, one allreduce per
iteration.

The reference's data-parallel strategy is 1/N row partitioning with ordered
merges (partition.py:84-100, 172-188, 237-261).  Here each rank holds a
contiguous row shard resident in its HBM; per iteration it runs the fused
assign+sum pass on its shard, the int64 fixed-point partial buffer
(k·m sums + k counts, 13 KB at k=64, m=25) is summed across ranks in place by
ONE allreduce (NCCL over NVLink via torch.distributed), and every rank runs the
identical finish kernel — integer sums make the result bit-identical on every
rank and for every GPU count, so centres stay replicated without a second
collective.  Only iterations with empty clusters exchange more: per empty
cluster one tiny all_gather of each rank's (max self-distance, global row,
donor label, row coordinates) to reproduce the reference's global
``np.argmax`` (first index) repair (engine.py:265-276).

The collective and the per-rank engine are injected, so the same driver runs
over NCCL with the CUDA engine in production and over gloo with a CPU
stand-in in the multi-process CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


class TorchCollective:
    """torch.distributed plumbing (NCCL on GPU, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
            else torch.device("cpu"))

    def allreduce_sum_(self, tensor):
        self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_scalar(self, value, op: str, dtype):
        t = self.torch.tensor([value], dtype=dtype, device=self.device)
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op), group=self.group)
        return t.item()

    def allgather_f64(self, vec: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64)).to(self.device)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def allgather_bytes(self, blob: bytes) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, bytes(blob), group=self.group)
        return out

    def exclusive_prefix(self, value: int) -> int:
        sizes = self.allgather_f64(np.array([float(value)]))[:, 0]
        return int(sizes[: self.rank].sum())


@dataclass
class ShardResult:
    centers: np.ndarray          # (k, m) float64, identical on every rank
    counts: np.ndarray           # (k,) int64, global
    labels: Optional[np.ndarray]  # this rank's (n_local,) int64 labels
    iterations: int
    converged: bool
    row_offset: int              # global index of this shard's first row


def partials_tensor(engine):
    """Device int64 tensor view of the engine's partial buffer (for NCCL)."""
    if hasattr(engine, "partials_tensor"):
        return engine.partials_tensor()
    import torch

    ptr, count = engine.step_partials()

    class _CAI:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<i8", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_CAI(), device="cuda")


def _global_repair(engine, coll, k, row_offset):
    empties = engine.step_empty_list(k)
    if len(empties) == 0:
        return 0
    engine.step_repair_prepare()
    m = engine.m
    for c in empties:
        d2, row, coords = engine.step_repair_candidate()
        donor = engine.step_label_of(row) if 0 <= row < engine.n else -1
        mine = np.concatenate([[d2, float(row_offset + row), float(donor)], coords])
        allc = coll.allgather_f64(mine)
        # np.argmax over the global array: largest d², then the lowest global row
        order = sorted(range(allc.shape[0]), key=lambda r: (-allc[r, 0], allc[r, 1]))
        w = order[0]
        win = allc[w]
        engine.step_repair_apply(int(c), w == coll.rank, int(win[1]) - row_offset, win[3:3 + m], int(win[2]))
    return len(empties)


def run_sharded(engine, coll, c0, max_iters=1000, tol=0.0, want_labels=True, resident=True) -> ShardResult:
    """engine.iterate semantics (engine.py:320-343) over row shards.

    `engine` holds this rank's shard (NativeEngine in production); `coll` is
    a TorchCollective.  Returns the replicated model and this rank's labels.

    Fast path (`resident`, CUDA engine, tensor-core shapes): one resident launch per GPU runs the
    loop and exchanges every iteration's Δ inside the kernel over NVLink peer memory
    (_run_resident_peer); the collective is only used to set up the IPC mappings, for the
    one-off agreements (n, max|x|) and for empty-cluster repairs.  Otherwise: per-iteration NCCL
    allreduce of the partial buffer (batched device-state loop, or the plain step loop).
    """
    c0 = np.ascontiguousarray(c0, dtype=np.float64)
    k = c0.shape[0]
    n_local = engine.n
    if getattr(coll, "device", None) is not None and coll.device.type == "cuda" and hasattr(engine, "set_stream"):
        # one stream for the engine's kernels and NCCL: no host sync between pass, allreduce and finish
        engine.set_stream(coll.torch.cuda.current_stream().cuda_stream)
    n_total = int(coll.allreduce_scalar(int(n_local), "SUM", coll.torch.int64))
    if k > n_total:
        from .exceptions import ContractViolationError

        raise ContractViolationError(f"k={k} exceeds sample count n={n_total}")
    row_offset = coll.exclusive_prefix(n_local)
    absmax = float(coll.allreduce_scalar(float(engine.points_info()["absmax"]), "MAX", coll.torch.float64))
    engine.set_frac_bits(engine.frac_bits_for(absmax, n_total))  # one global fixed-point scale
    if resident and hasattr(engine, "lloyd_peer") and _peer_capable(engine, k):
        return _run_resident_peer(engine, coll, c0, k, max_iters, tol, want_labels, row_offset)
    engine.step_begin(c0)
    part = partials_tensor(engine)
    if hasattr(engine, "loop_begin"):  # device-state loop: a few iterations per host round trip
        return _run_batched(engine, coll, part, k, max_iters, tol, want_labels, row_offset)
    engine.step_pass()                       # L0 = A(C0) + its sums
    t = 0
    converged = False
    while True:
        coll.allreduce_sum_(part)            # the one collective per iteration
        n_empty, conv = engine.step_finish(tol)
        t += 1
        if n_empty:
            _global_repair(engine, coll, k, row_offset)
            conv = engine.step_check(tol)
        if conv:
            converged = True
            break
        if t >= max_iters:
            engine.step_pass()               # L_T = A(C_T); counts = global bincount(L_T)
            coll.allreduce_sum_(part)
            engine.step_fold()
            break
        engine.step_pass()
    centers, counts, labels = engine.step_read(k, want_labels=want_labels)
    return ShardResult(centers, counts, labels, t, converged, row_offset)


def _run_batched(engine, coll, part, k, max_iters, tol, want_labels, row_offset) -> ShardResult:
    """The same loop with the device holding the state (DevState, as km_lloyd does): iterations
    are enqueued in batches of up to 16 [allreduce, finish, pass] and the state is read once per
    batch.  Kernels are gated on the state, so iterations enqueued past the end do no work and
    the allreduces then sum zeros.  Every rank reads the same state (replicated totals)."""
    engine.loop_begin(max_iters, tol)
    engine.loop_pass()                       # L0 = A(C0) + its sums
    batch = 1
    while True:
        for _ in range(batch):
            coll.allreduce_sum_(part)        # the one collective per iteration
            engine.loop_finish()             # update, empties, congruence, exhaustion (device)
            engine.loop_pass()               # next assignment (gated)
        t, done, conv, need_host = engine.loop_state()
        if done:
            break
        if need_host:                        # empty clusters: the global repair, then the test
            _global_repair(engine, coll, k, row_offset)
            engine.loop_check()
            t, done, conv, _ = engine.loop_state()
            if done:
                break
            engine.loop_pass()               # the assignment with the repaired centres
            batch = 1
            continue
        batch = min(batch * 2, 16)
    centers, counts, labels = engine.step_read(k, want_labels=want_labels)
    return ShardResult(centers, counts, labels, t, conv, row_offset)


def _peer_capable(engine, k) -> bool:
    """The resident peer loop runs the tensor-core pass: fp32 points, m <= 31, k <= 128."""
    info = engine.points_info()
    return info["point_bytes"] == 4 and info["m"] <= 31 and k <= 128


def _run_resident_peer(engine, coll, c0, k, max_iters, tol, want_labels, row_offset) -> ShardResult:
    """Every rank's resident kernel runs the Lloyd loop on its shard; per iteration its Δ goes to
    every rank's exchange buffer over NVLink (CUDA IPC, km_peer_*) and each rank sums the `world`
    rows itself — exact integers, so the model is bit-identical on every rank and to one GPU.  The
    kernels stop together (identical totals ⇒ identical decisions) when the loop is done or has
    empty clusters; those take the global repair here, then the loop resumes."""
    handle = engine.peer_init(coll.world, coll.rank, k)
    engine.peer_connect(coll.allgather_bytes(handle))
    t, done, conv, need_host = engine.lloyd_peer(c0, max_iters, tol)
    while not done:
        if need_host:
            _global_repair(engine, coll, k, row_offset)
            engine.loop_check()
            t, done, conv, _ = engine.loop_state()
            if done:
                break
        t, done, conv, need_host = engine.lloyd_peer_resume()
    centers, counts, labels = engine.step_read(k, want_labels=want_labels)
    return ShardResult(centers, counts, labels, t, conv, row_offset)


def shard_rows(n: int, world: int, rank: int):
    """Contiguous near-equal spans, first n % world get +1 (partition.plan_chunks, partition.py:84-100)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)
