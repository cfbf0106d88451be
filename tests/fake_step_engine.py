"""CPU stand-in for the per-rank CUDA engine's step API (test infrastructure).

Implements the NativeEngine step methods that paper_1402_3788_b200.distributed
drives (km_step_* in include/kmeans_b200.h) on a row shard held in host
memory, with the reference arithmetic (oracle/) and the same int64
fixed-point partial buffer.  Lets the multi-rank driver be tested with gloo
on CPU; the GPU engine implements the identical contract.
"""

import math

import numpy as np
import torch

from oracle import oracle


class FakeStepEngine:
    def __init__(self, shard: np.ndarray):
        self.x = np.ascontiguousarray(shard, dtype=np.float64)
        self.n, self.m = self.x.shape
        self.frac_bits = 0
        self.k = 0

    # -- data / scale -------------------------------------------------------
    def points_info(self):
        return {"n": self.n, "m": self.m, "point_bytes": 8, "absmax": float(np.abs(self.x).max())}

    def frac_bits_for(self, absmax, n_total):
        bound = max(absmax, 1e-300) * n_total
        _, ex = math.frexp(bound)
        return max(-60, min(1000, 62 - ex))

    def set_frac_bits(self, f):
        self.frac_bits = int(f)

    def _fixed(self, v):
        return np.rint(np.asarray(v, dtype=np.float64) * math.ldexp(1.0, self.frac_bits)).astype(np.int64)

    # -- step API ---------------------------------------------------------------
    def step_begin(self, c0):
        self.cur = np.array(c0, dtype=np.float64, copy=True)
        self.prev = self.cur.copy()
        self.k = self.cur.shape[0]
        self.part = torch.zeros(self.k * self.m + self.k, dtype=torch.int64)
        self.tot = np.zeros(self.k * self.m + self.k, dtype=np.int64)
        self.labels = np.zeros(self.n, dtype=np.int64)
        self.model_counts = np.zeros(self.k, dtype=np.int64)

    def partials_tensor(self):
        return self.part

    def step_pass(self):  # full sums of the shard (finish: tot = part)
        self.labels, counts = oracle.assign(self.x, self.cur)
        k, m = self.k, self.m
        sums = np.zeros((k, m), dtype=np.int64)
        np.add.at(sums, self.labels, self._fixed(self.x))
        buf = np.concatenate([sums.ravel(), counts.astype(np.int64)])
        self.part.copy_(torch.from_numpy(buf))

    def step_finish(self, tol):
        self.tot = self.part.numpy().copy()
        self.part.zero_()
        k, m = self.k, self.m
        sums = self.tot[: k * m].reshape(k, m)
        counts = self.tot[k * m:]
        self.prev = self.cur.copy()
        new = np.zeros((k, m))
        occ = counts > 0
        new[occ] = (sums[occ].astype(np.float64) * math.ldexp(1.0, -self.frac_bits)) / counts[occ, None]
        self.cur = new
        self.model_counts = counts.copy()
        n_empty = int((~occ).sum())
        conv = False if n_empty else oracle.converged(self.prev, self.cur, tol)
        return n_empty, conv

    def step_fold(self):
        self.tot = self.part.numpy().copy()
        self.part.zero_()
        self.model_counts = self.tot[self.k * self.m:].copy()

    def step_empty_list(self, k):
        return np.flatnonzero(self.model_counts == 0)

    def step_repair_prepare(self):
        self.d2 = oracle.self_distances(self.x, self.cur, self.labels)

    def step_repair_candidate(self):
        row = int(np.argmax(self.d2))
        return float(self.d2[row]), row, self.x[row].copy()

    def step_label_of(self, row):
        return int(self.labels[row])

    def step_repair_apply(self, cluster, owner, local_row, coords, donor):
        if owner:
            self.labels[local_row] = cluster
            self.d2[local_row] = 0.0
        self.model_counts[donor] -= 1
        self.model_counts[cluster] += 1
        self.cur[cluster] = coords

    def step_check(self, tol):
        return oracle.converged(self.prev, self.cur, tol)

    def step_read(self, k, want_labels=True):
        return self.cur.copy(), self.model_counts.copy(), (self.labels.copy() if want_labels else None)


class FakeLoopEngine(FakeStepEngine):
    """The device-state loop API on top of the step API (km_step_loop_* in include/kmeans_b200.h):
    the loop state lives "on the device" (here: in this object, mirroring DevState), passes and
    finishes are GATED on it — once the loop is done or waits for the host (empty clusters) they do
    no work and leave the partial buffer zero, exactly as the CUDA kernels do — so
    distributed._run_batched can enqueue several [allreduce, finish, pass] iterations per host
    round trip.  Same rules as lloyd_finish_kernel / lloyd_check_kernel (kmeans_finish.cuh):
    update + empties + congruence + exhaustion, and the exhausted run's final assign is folded
    into the counts (engine.py:339-343)."""

    def loop_begin(self, max_iters, tol):
        self.st = dict(t=0, done=0, converged=0, exhausted=0, need_host=0, max_iters=int(max_iters), tol=float(tol))
        self.gated_passes = 0

    def loop_pass(self):
        if self.st["done"] or self.st["need_host"]:
            self.gated_passes += 1
            return  # gated: the partial buffer stays zero (the allreduce then sums zeros)
        self.step_pass()

    def loop_finish(self):
        st = self.st
        if st["done"] or st["need_host"]:
            self.part.zero_()
            return
        if st["exhausted"]:  # the final assign pass of an exhausted run: counts = bincount(L_T)
            self.step_fold()
            st["done"] = 1
            return
        n_empty, conv = self.step_finish(st["tol"])
        st["t"] += 1
        if n_empty:
            st["need_host"] = 1
        elif conv:
            st["converged"] = st["done"] = 1
        elif st["t"] >= st["max_iters"]:
            st["exhausted"] = 1

    def loop_check(self):
        st = self.st
        st["need_host"] = 0
        if oracle.converged(self.prev, self.cur, st["tol"]):
            st["converged"] = st["done"] = 1
        elif st["t"] >= st["max_iters"]:
            st["exhausted"] = 1

    def loop_state(self):
        st = self.st
        return st["t"], bool(st["done"]), bool(st["converged"]), bool(st["need_host"])
