#!/usr/bin/env python
"""Benchmark of the B200 Lloyd hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], the headline): n = 2,000,000 points,
M = 25 features, K = 16 clusters, fp32 synthetic Gaussian blobs from the
reference generator (datasets.generate_synthetic, seed 0), initial centres =
the first K rows (the reference's first-K trajectory runs 539 updates before
it converges, so every timed iteration does full work).  `--config` selects
the other BASELINE configs (cfg1, cfg2, cfg4 = K 512, cfg5 = 64M x 25 x 64).

One STEP = one Lloyd iteration = one fused assign+update pass over all points
+ the finish (divide, empty clusters, congruence test).  The timed region runs
exactly K steps as km_lloyd calls (≤ 500 iterations each, restarted from C0:
every repetition is iterations 1..K of the trajectory, including the first
pass of the call), bracketed by barrier + cuda synchronize, timed with CUDA
events on the engine's stream, max over ranks.  Inputs (200 MB) exceed the
126 MB L2, so no flush is needed between iterations.

Printed JSON line: metric/value/unit (points·iterations/s, whole job),
ms_per_step, roofline (the tensor-core pass vs the measured HBM copy
bandwidth; the FP32 pipe for K > 128), cpu_baseline (the C restatement of the
reference on this host's cores: all threads and one thread, with the CPU
model), e2e (full fit to convergence through the C ABI from pinned host
buffers, H2D and D2H inside the timed region), clocks sampled during the
timed region, gpu_launches (kernels the engine launched per timed repetition),
parity (iterations + SHA-256 of the centres after K iterations: identical for
every GPU count — exact integer sums).

--impl reference: the reference's CPU path (its C restatement, oracle/, all
host threads) on the same config, rank 0 only.

--gpus N > 1: row-sharded, one process per GPU (this script re-launches itself
under torch.distributed.run when WORLD_SIZE is not set).  `--scaling weak`
(default; cfg5: strong): every rank holds `n` rows of ONE dataset of N·n rows;
`--scaling strong`: the config's n rows split across the ranks (the
partition.plan_chunks rule).  One NCCL allreduce of the k·m+k int64 partials
per iteration (distributed.run_sharded).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import socket
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
    "cfg5": (64_000_000, 25, 64, "n=64,000,000 M=25 K=64 (row-sharded config, 6.4 GB)"),
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


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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

    def wait_first(self, timeout=10.0):
        """Block until nvidia-smi has printed its first sample (its start-up takes ~0.5 s), so the
        whole timed region is sampled."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.lines.clear()  # (that sample predates the timed region)

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


def scaling_mode(args):
    return args.scaling or ("strong" if args.config == "cfg5" else "weak")


def shard_plan(args, world, rank):
    """(total rows of the ONE dataset, this rank's [lo, hi))."""
    from paper_1402_3788_b200.distributed import shard_rows

    n = CONFIGS[args.config][0]
    total = n if scaling_mode(args) == "strong" else n * world
    lo, hi = shard_rows(total, world, rank)
    return total, lo, hi


def load_rows(args, world, rank):
    """This rank's rows (fp32) and C0 = the first K rows of the one dataset."""
    from paper_1402_3788_b200.datasets import generate_synthetic_array, generate_synthetic_shard

    _, m, k, _ = CONFIGS[args.config]
    total, lo, hi = shard_plan(args, world, rank)
    if world == 1:
        x = generate_synthetic_array(total, m, k, seed=0, dtype=np.float32)
        c0 = x[:k].astype(np.float64)
        return x, c0, total, lo, hi
    x = generate_synthetic_shard(total, m, k, 0, lo, hi)
    c0 = generate_synthetic_shard(total, m, k, 0, 0, k).astype(np.float64) if lo > 0 else x[:k].astype(np.float64)
    return x, c0, total, lo, hi


def config_block(args, world, total):
    n, m, k, desc = CONFIGS[args.config]
    return {"workload": args.config + ": " + desc, "n_total": total, "n_per_gpu": total // world, "m": m, "k": k,
            "init": "first K rows (reference first-K trajectory)", "tol": 0.0,
            "l2": "no flush: the points of every timed pass exceed the 126 MB L2" if total // world * m * 4 > 126e6
            else "inputs smaller than L2 (launch/L2-bound config): no flush, reported as it/s",
            "scaling": scaling_mode(args) if world > 1 else "single GPU",
            "parallelism": f"dp{world} row shards, 1 allreduce/iter" if world > 1 else "single GPU"}


# ------------------------------------------------------------------------------------------------
# CPU baseline: the reference path restated in C (oracle/)
# ------------------------------------------------------------------------------------------------
def cpu_lloyd_rate(x64, c0, budget_s, threads, max_iters=None):
    """Time reference Lloyd iterations (assign_parallel + update_parallel with `threads` workers,
    the run_multi closures; threads = 1 is run_single) over ALL rows until `budget_s` elapsed
    (at least one); returns (points·iters/s, iterations, seconds)."""
    from oracle import oracle

    n = x64.shape[0]
    centers = c0.copy()
    k = centers.shape[0]
    t0 = time.perf_counter()
    iters = 0
    while True:
        labels, _ = oracle.assign(x64, centers, n_workers=threads)
        centers, _, _ = oracle.update(x64, labels, k, n_workers=threads)
        iters += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_iters and iters >= max_iters):
            break
    return n * iters / el, iters, el


def cpu_baseline_block(x, c0, budget_s):
    threads = os.cpu_count() or 1
    x64 = x.astype(np.float64)
    rate, iters, el = cpu_lloyd_rate(x64, c0, budget_s, threads)
    r1, i1, e1 = cpu_lloyd_rate(x64, c0, budget_s, 1)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{iters} Lloyd iterations over all {x.shape[0]} rows (assign_parallel + update_parallel, "
                      f"{threads} threads, {el:.1f} s)",
            "single_thread": {"value": r1, "unit": UNIT, "cores": 1,
                              "sample": f"{i1} Lloyd iterations over all {x.shape[0]} rows (assign_step + "
                                        f"update_step, 1 thread, {e1:.1f} s)"},
            "cpu_model": cpu_model(), "host_threads": threads}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1402_3788_b200.datasets import generate_synthetic_array

    n, m, k, desc = CONFIGS[args.config]
    total = n if (world == 1 or scaling_mode(args) == "strong") else n * world
    x = generate_synthetic_array(total, m, k, seed=0, dtype=np.float32).astype(np.float64)
    c0 = x[:k].copy()
    threads = os.cpu_count() or 1
    from oracle import oracle

    # every step is a whole Lloyd iteration over ALL rows (same config as our arm, no row subsample);
    # only the NUMBER of timed steps is bounded so the run ends within a few minutes
    centers = c0.copy()
    t0 = time.perf_counter()
    labels, _ = oracle.assign(x, centers, n_workers=threads)
    centers, _, _ = oracle.update(x, labels, k, n_workers=threads)
    per_step = time.perf_counter() - t0
    budget = args.reference_seconds
    steps = max(1, min(args.steps, int(budget / max(per_step, 1e-9))))
    warm = min(args.warmup, max(0, int(budget / 4 / max(per_step, 1e-9))))
    for _ in range(warm):
        labels, _ = oracle.assign(x, centers, n_workers=threads)
        centers, _, _ = oracle.update(x, labels, k, n_workers=threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        labels, _ = oracle.assign(x, centers, n_workers=threads)
        centers, _, _ = oracle.update(x, labels, k, n_workers=threads)
    el = time.perf_counter() - t0
    value = total * steps / el
    sample = (f"{steps} of the requested {args.steps} steps timed (each a full Lloyd iteration over all {total} rows: "
              f"assign_parallel + update_parallel, {threads} threads) after {1 + warm} untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": 1 + warm, "ms_per_step": el / steps * 1e3,
        "higher_is_better": True, "scaling": scaling_mode(args) if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "same_config": True,
        "config": config_block(args, world, total),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "notes": "reference CPU path restated in C (oracle/kmeans_oracle.c, pinned bit-exact to the numba "
                 "reference by tests/test_oracle_golden.py); the numba package itself cannot travel to this box",
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    from paper_1402_3788_b200 import _native

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    sharded = world > 1 or args.force_sharded
    if sharded:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        # NCCL init logging on (stderr): the communicator's nranks / transport are checkable
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    n, m, k, desc = CONFIGS[args.config]
    x, c0, total, lo, hi = load_rows(args, world, rank)
    n_local = x.shape[0]
    xd = torch.from_numpy(x).cuda()  # resident in HBM before the timed region
    stream = torch.cuda.current_stream()
    eng = _native.NativeEngine(local)
    eng.set_stream(stream.cuda_stream)
    eng.attach_device_f32(xd.data_ptr(), n_local, m)

    coll = None
    if sharded:
        from paper_1402_3788_b200.distributed import TorchCollective

        coll = TorchCollective()

    def lloyd(iters, want_centers=False):
        if coll is None:
            centers, _, _, it, conv = eng.lloyd(c0, iters, 0.0, want_labels=False)
            return (it, centers) if want_centers else it
        from paper_1402_3788_b200.distributed import run_sharded

        r = run_sharded(eng, coll, c0, max_iters=iters, want_labels=False)
        return (r.iterations, r.centers) if want_centers else r.iterations

    def k_steps(K):
        done = 0
        while done < K:
            done += lloyd(min(MAX_ITERS_PER_CALL, K - done))
        return done

    # parity fingerprint of the timed trajectory (iterations 1..K from C0), outside the timed region:
    # exact integer sums make it identical for every GPU count and every scaling of the same dataset
    p_it, p_c = lloyd(min(args.steps, MAX_ITERS_PER_CALL), want_centers=True)
    parity = {"iterations": p_it, "centers_sha256": hashlib.sha256(np.ascontiguousarray(p_c).tobytes()).hexdigest(),
              "dataset_rows": total}

    # warm-up (≥ W iterations, at least one full call)
    k_steps(max(args.warmup, 3))
    torch.cuda.synchronize()

    # repetitions of exactly K steps, long enough to sample clocks
    sampler = ClockSampler(local)
    sampler.start()
    sampler.wait_first()
    eng.reset_stats()
    eng.set_profiling(True)
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
        # at least --min-seconds (clock samples) and 10 repetitions; --max-reps caps fast configs
        if reps >= args.max_reps or ((time.perf_counter() - t_region) >= args.min_seconds and reps >= 10):
            break
    clocks = sampler.stop()
    eng.set_profiling(False)
    st = eng.stats()
    ms_per_step = statistics.median(rep_ms)
    value = total * 1e3 / ms_per_step
    launches = int(st["kernel_launches"]) // reps

    # roofline of the dominant kernel, device time from CUDA events in the timed region: the first
    # pass + cluster sums + the resident launch (per-pass time = launch time / passes); the row-sharded
    # step path has no per-pass events, so its roofline uses the whole step (pass + allreduce + finish)
    peak, peak_kind = measured_peaks()
    pass_ms = st["pass_ms_total"] / st["pass_timed"] if st["pass_timed"] else ms_per_step
    alg_bytes = n_local * (4 * m + 4)  # points read once (fp32) + int32 labels written once
    if k > 128:
        # compute-bound large-K regime: algorithmic 3·n·K·M flops per pass against the
        # FP32 pipe peak SMs × 128 lanes × 2 flops × the max SM clock; the expanded-form filter
        # executes M FMAs per (point, centre) = 2·n·K·M flops, reported beside it
        props = torch.cuda.get_device_properties(local)
        f_max = (clocks or {}).get("sm_max_mhz") or 1965.0
        fp32_peak = props.multi_processor_count * 256 * f_max * 1e6 / 1e12
        alg_flops = 3.0 * n_local * k * m
        achieved = alg_flops / (pass_ms * 1e-3) / 1e12
        executed = 2.0 * n_local * k * m / (pass_ms * 1e-3) / 1e12
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": None,
                    "kernel": "lloyd_pass_blocked_kernel (register-blocked FFMA2 SIMT pass)",
                    "kernel_ms_per_pass": pass_ms, "alg_flops_per_pass": alg_flops,
                    "executed_tflops": executed, "executed_frac": executed / fp32_peak,
                    "peak_kind": f"FP32 pipe: {props.multi_processor_count} SMs x 128 lanes x 2 flops x {f_max:.0f} MHz",
                    "pass_share_of_step": pass_ms / ms_per_step,
                    "note": "frac = algorithmic 3nKM flops (the reference recurrence); executed_frac = the 2nKM "
                            "flops the expanded-form filter actually issues"}
    else:
        achieved = alg_bytes / (pass_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic_from_profiles(args.config),
                    "kernel": "lloyd_pass_tc_kernel (first pass + cluster sums + resident loop; per-pass time = "
                              "device time of the call's launches / passes)" if not sharded else
                              "whole sharded step (pass + NCCL allreduce + finish)",
                    "kernel_ms_per_pass": pass_ms, "alg_bytes_per_pass": alg_bytes, "peak_kind": peak_kind,
                    "pass_share_of_step": pass_ms / ms_per_step}

    # e2e: the public API from pinned host buffers, full fit to convergence
    e2e = None
    cpu = None
    if not args.skip_e2e:
        pinned = torch.empty((n_local, m), dtype=torch.float32, pin_memory=True)
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
            e2e_rates.append(total * it / el)
            e2e_iters = it
        eng2.close()
        e2e = {"value": statistics.median(e2e_rates), "unit": UNIT,
               "h2d_bytes_per_step": int(n_local * m * 4 + k * m * 8),
               "d2h_bytes_per_step": int(n_local * 8 + k * m * 8 + k * 8),
               "step": f"one full fit through the C ABI: H2D points from pinned host memory, km_lloyd to "
                       f"convergence ({e2e_iters} iterations), D2H int64 labels + centres + counts"
                       + (" (per rank)" if world > 1 else "")}
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline_block(x, c0, args.cpu_seconds)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling_mode(args) if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(config_block(args, world, total),
                           timing=f"median of {reps} repetitions of exactly {args.steps} steps"),
            "iters_per_sec": 1e3 / ms_per_step,
            "hbm_gbs_step": n_local * (4 * m + 4) / (ms_per_step * 1e-3) / 1e9,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "parity": parity,
            "rechecked_points_per_iter": st["rechecked"] / max(1, st["passes"]),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(args):
    """`--gpus N` (N > 1) started as a plain process: run this script under torch.distributed.run,
    one rank per GPU, rendezvous on 127.0.0.1; rank 0's JSON line is the output."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: weak = n rows per GPU (default), strong = n rows in total (default for cfg5)")
    ap.add_argument("--min-seconds", type=float, default=1.0)
    ap.add_argument("--max-reps", type=int, default=2000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--reference-seconds", type=float, default=60.0)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--force-sharded", action="store_true",
                    help="testing: drive the row-sharded NCCL step path even at world size 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        return relaunch_under_torchrun(args)
    if world and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
