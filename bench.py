#!/usr/bin/env python
"""Benchmark of the B200 Lloyd hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], the headline): n = 2,000,000 points,
M = 25 features, K = 16 clusters, fp32 synthetic Gaussian blobs from the
reference generator (datasets.generate_synthetic, seed 0), initial centres =
the first K rows (the reference's first-K trajectory runs 539 updates before
it converges, so every timed iteration does full work).

One STEP = one Lloyd iteration = one fused assign+update pass over all points
+ the one-CTA finish (divide, empty clusters, congruence test).  The timed
region runs K steps as device-resident km_lloyd calls (≤ 500 iterations each,
restarted from C0), bracketed by barrier + cuda synchronize, timed with CUDA
events on the engine's stream, max over ranks.  Inputs (200 MB) exceed the
126 MB L2, so no flush is needed between iterations.

Printed JSON line: metric/value/unit (points·iterations/s, whole job),
ms_per_step, roofline (fused pass kernel vs measured HBM copy bandwidth),
cpu_baseline (the C restatement of the reference on this host's cores), e2e
(full fit to convergence through the C ABI from pinned host buffers, H2D and
D2H inside the timed region), clocks sampled during the timed region,
gpu_launches (kernels launched by the engine inside the timed region).

--impl reference: the reference's CPU path (its C restatement, oracle/, all
host threads) on the same config, rank 0 only.

N > 1 (torchrun): weak scaling, each rank holds its own 2M-point shard; one
NCCL allreduce of the k·m+k int64 partials per iteration.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n, m, k, description)
    "cfg1": (10_000, 5, 4, "n=10,000 M=5 K=4 (reference single-threaded CPU case)"),
    "cfg2": (100_000, 10, 8, "n=100,000 M=10 K=8 (single/multi regime boundary)"),
    "cfg3": (2_000_000, 25, 16, "n=2,000,000 M=25 K=16 fp32 blobs (paper headline shape), 1 B200"),
    "cfg4": (2_000_000, 25, 512, "n=2,000,000 M=25 K=512 (compute-bound large-K assignment)"),
    # the row-sharded config: 64M points on one GPU at N=1 (6.4 GB resident); under torchrun each rank
    # holds its own n-row shard (weak scaling, as the other configs)
    "cfg5": (64_000_000, 25, 64, "n=64,000,000 M=25 K=64 (row-shard config), one shard per GPU"),
}
METRIC = "Lloyd iters/sec & points·iters/sec at n=2M,M=25,K=16; HBM GB/s vs peak"
UNIT = "points*iters/s"
MAX_ITERS_PER_CALL = 500


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=50):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 f"-lms={self.period_ms}"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def traffic_from_profiles(cfg_name):
    """dram bytes per launch of the fused pass from the committed ncu summary (or None)."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------------
# CPU baseline: the reference path restated in C (oracle/), all host threads
# ------------------------------------------------------------------------------------------------
def cpu_lloyd_rate(x64, c0, budget_s, threads, min_rows=65_536, rows=None):
    """Time reference Lloyd iterations (assign_parallel + update_parallel) on a
    row sample; returns (points·iters/s, iterations, rows, seconds)."""
    from oracle import oracle

    n = x64.shape[0]
    if rows is None:
        rows = n
    rows = max(min(rows, n), min(min_rows, n))
    xs = np.ascontiguousarray(x64[:rows])
    centers = c0.copy()
    k = centers.shape[0]
    t0 = time.perf_counter()
    iters = 0
    while True:
        labels, _ = oracle.assign(xs, centers, n_workers=threads)
        centers, _, _ = oracle.update(xs, labels, k, n_workers=threads)
        iters += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return rows * iters / el, iters, rows, el


def run_reference(args, cfg_name):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    n, m, k, desc = CONFIGS[cfg_name]
    x = generate_synthetic_array(n, m, k, seed=0, dtype=np.float32).astype(np.float64)
    c0 = x[:k].copy()
    threads = os.cpu_count() or 1
    # size the per-step row sample so the whole K+W run takes about 90 s
    probe_rows = min(n, 200_000)
    rate, _, _, _ = cpu_lloyd_rate(x, c0, 0.5, threads, rows=probe_rows)
    per_row = 1.0 / rate
    budget = 90.0 / max(1, args.steps + args.warmup)
    rows = int(min(n, max(65_536, budget / per_row)))
    from oracle import oracle

    xs = np.ascontiguousarray(x[:rows])
    centers = c0.copy()
    for _ in range(args.warmup):
        labels, _ = oracle.assign(xs, centers, n_workers=threads)
        centers, _, _ = oracle.update(xs, labels, k, n_workers=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        labels, _ = oracle.assign(xs, centers, n_workers=threads)
        centers, _, _ = oracle.update(xs, labels, k, n_workers=threads)
    el = time.perf_counter() - t0
    value = rows * args.steps / el
    sample = f"{rows} of {n} rows per step (one Lloyd iteration: assign_parallel + update_parallel)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg_name + ": " + desc, "n": n, "m": m, "k": k, "init": "first K rows"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "notes": "reference CPU path restated in C (oracle/kmeans_oracle.c, pinned bit-exact to the numba "
                 "reference by tests/test_oracle_golden.py); the numba package itself cannot travel to this box",
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_ours(args, cfg_name):
    import torch

    from paper_1402_3788_b200 import _native
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    sharded = world > 1 or args.force_sharded
    if sharded:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    n, m, k, desc = CONFIGS[cfg_name]
    x = generate_synthetic_array(n, m, k, seed=rank, dtype=np.float32)
    c0 = x[:k].astype(np.float64)
    if sharded:
        t = torch.from_numpy(c0).cuda()
        dist.broadcast(t, 0)
        c0 = t.cpu().numpy()
    xd = torch.from_numpy(x).cuda()  # resident in HBM before the timed region
    stream = torch.cuda.current_stream()
    eng = _native.NativeEngine(local)
    eng.set_stream(stream.cuda_stream)
    eng.attach_device_f32(xd.data_ptr(), n, m)

    coll = None
    if sharded:
        from paper_1402_3788_b200.distributed import TorchCollective

        coll = TorchCollective()

    def lloyd(iters):
        if coll is None:
            _, _, _, it, conv = eng.lloyd(c0, iters, 0.0, want_labels=False)
            return it
        from paper_1402_3788_b200.distributed import run_sharded

        return run_sharded(eng, coll, c0, max_iters=iters, want_labels=False).iterations

    def k_steps(K):
        done = 0
        while done < K:
            done += lloyd(min(MAX_ITERS_PER_CALL, K - done))
        return done

    # warm-up (≥ W iterations, at least one full call)
    k_steps(max(args.warmup, 3))
    torch.cuda.synchronize()

    # repetitions of exactly K steps, long enough to sample clocks
    eng.reset_stats()
    eng.set_profiling(True)
    sampler = ClockSampler(local)
    sampler.start()
    rep_ms, total_iters = [], 0
    t_region = time.perf_counter()
    reps = 0
    while True:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        iters = k_steps(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if dist is not None:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        rep_ms.append(ms / iters)
        total_iters += iters
        reps += 1
        if reps >= args.max_reps or (time.perf_counter() - t_region) >= args.min_seconds:
            break
    clocks = sampler.stop()
    eng.set_profiling(False)
    st = eng.stats()
    ms_per_step = statistics.median(rep_ms)
    n_total = n * world
    value = n_total * 1e3 / ms_per_step
    launches = int(st["kernel_launches"]) // reps

    # roofline of the fused pass (the dominant kernel), device time from CUDA events in the timed region
    peak, peak_kind = measured_peaks()
    # device time of the fused pass (resident launches report launch time / passes); the row-sharded
    # step path has no per-pass events, so its roofline uses the whole step (pass + allreduce + finish)
    pass_ms = st["pass_ms_total"] / st["pass_timed"] if st["pass_timed"] else ms_per_step
    alg_bytes = n * (4 * m + 4)  # points read once (fp32) + int32 labels written once
    if k > 128:
        # compute-bound large-K regime: algorithmic 3·n·K·M flops per pass against the
        # FP32 pipe peak SMs × 128 lanes × 2 flops × the max SM clock
        props = torch.cuda.get_device_properties(local)
        f_max = (clocks or {}).get("sm_max_mhz") or 1965.0
        fp32_peak = props.multi_processor_count * 256 * f_max * 1e6 / 1e12
        alg_flops = 3.0 * n * k * m
        achieved = alg_flops / (pass_ms * 1e-3) / 1e12
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": None,
                    "kernel": "lloyd_pass_blocked_kernel (register-blocked FFMA2 SIMT pass)",
                    "kernel_ms_per_pass": pass_ms, "alg_flops_per_pass": alg_flops,
                    "peak_kind": f"FP32 pipe: {props.multi_processor_count} SMs x 128 lanes x 2 flops x {f_max:.0f} MHz",
                    "pass_share_of_step": pass_ms / ms_per_step,
                    "note": "expanded-form filter: M FMAs per (point, centre) = 2nKM flops executed; "
                            "3nKM is the reference recurrence's algorithmic count"}
    else:
        achieved = alg_bytes / (pass_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic_from_profiles(cfg_name), "kernel": "lloyd_pass_tc_kernel (resident loop; per-pass time = launch time / passes)",
                    "kernel_ms_per_pass": pass_ms, "alg_bytes_per_pass": alg_bytes, "peak_kind": peak_kind,
                    "pass_share_of_step": pass_ms / ms_per_step}

    # e2e: the public API from pinned host buffers, full fit to convergence
    e2e = None
    cpu = None
    if not args.skip_e2e:
        pinned = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
        pinned.numpy()[:] = x
        hx = pinned.numpy()
        eng2 = _native.NativeEngine(local)
        e2e_rates, e2e_iters = [], 0

        def one_fit():
            eng2.load(hx)  # H2D from pinned memory (+ device finiteness/absmax scan)
            if coll is None:
                centers, counts, labels, it, conv = eng2.lloyd(c0, 1000, 0.0, want_labels=True)
            else:
                from paper_1402_3788_b200.distributed import run_sharded

                r = run_sharded(eng2, coll, c0, max_iters=1000)
                it = r.iterations
            return it

        one_fit()  # warm-up
        for _ in range(args.e2e_steps):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            it = one_fit()
            el = time.perf_counter() - t0
            if dist is not None:
                tt = torch.tensor([el], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                el = float(tt.item())
            e2e_rates.append(n_total * it / el)
            e2e_iters = it
        eng2.close()
        e2e = {"value": statistics.median(e2e_rates), "unit": UNIT,
               "h2d_bytes_per_step": int(n * m * 4 + k * m * 8),
               "d2h_bytes_per_step": int(n * 8 + k * m * 8 + k * 8),
               "step": f"one full fit through the C ABI: H2D points from pinned host memory, km_lloyd to "
                       f"convergence ({e2e_iters} iterations), D2H int64 labels + centres + counts"}
    if rank == 0 and world == 1 and not args.skip_cpu:
        threads = os.cpu_count() or 1
        rate, iters, rows, el = cpu_lloyd_rate(x.astype(np.float64), c0, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{iters} Lloyd iterations over all {rows} rows (assign_parallel + update_parallel, "
                         f"{threads} threads, {el:.1f} s)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg_name + ": " + desc, "n_per_gpu": n, "m": m, "k": k,
                       "init": "first K rows (reference first-K trajectory)",
                       "l2": "no flush: 200 MB of points per GPU exceed the 126 MB L2",
                       "parallelism": f"dp{world} row shards, 1 allreduce/iter" if world > 1 else "single GPU",
                       "timing": f"median of {reps} repetitions of exactly {args.steps} steps"},
            "iters_per_sec": 1e3 / ms_per_step,
            "hbm_gbs_step": n * (4 * m + 4) / (ms_per_step * 1e-3) / 1e9,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches,
            "rechecked_points_per_iter": st["rechecked"] / max(1, st["passes"]),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--min-seconds", type=float, default=1.0)
    ap.add_argument("--max-reps", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--force-sharded", action="store_true",
                    help="testing: drive the row-sharded NCCL step path even at world size 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, args.config)
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
