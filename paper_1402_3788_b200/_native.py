"""ctypes binding of the C ABI (include/kmeans_b200.h) → libkmeans_b200.so.

This is the only way the package reaches the device.  If the library is not
built, or no sm_100 device is present, every entry point raises
DeviceUnavailableError — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

from .exceptions import (
    CapacityExceededError,
    ClusteringError,
    ContractViolationError,
    DeviceLostError,
    DeviceUnavailableError,
    ValidationFailureError,
)

import os as _os

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libkmeans_b200.so"
if _os.environ.get("KM_LIB_VARIANT"):  # tuning builds only (tools/); the product uses the default library
    LIB_PATH = Path(__file__).resolve().parent / "_lib" / "variants" / f"libkmeans_b200_{_os.environ['KM_LIB_VARIANT']}.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "kmeans_b200.h"

KM_OK = 0
_ERRORS = {
    1: ContractViolationError,
    2: ValidationFailureError,
    3: DeviceUnavailableError,
    4: DeviceLostError,
    5: CapacityExceededError,
    6: ClusteringError,
}

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F64 = ctypes.c_double


class KmStats(ctypes.Structure):
    _fields_ = [("passes", I64), ("rechecked", I64), ("repairs", I64), ("host_syncs", I64),
                ("frac_bits", I32), ("point_bytes", I32), ("kernel_launches", I64), ("changed", I64),
                ("pass_timed", I64), ("pass_ms_total", F64)]


# name -> (restype, argtypes); must list every symbol declared in the header
SIGNATURES = {
    "km_version": (ctypes.c_char_p, []),
    "km_device_count": (ctypes.c_int, [ctypes.POINTER(I32)]),
    "km_create": (ctypes.c_int, [I32, ctypes.POINTER(P)]),
    "km_destroy": (ctypes.c_int, [P]),
    "km_last_error": (ctypes.c_char_p, [P]),
    "km_set_stream": (ctypes.c_int, [P, P]),
    "km_load_points_f32": (ctypes.c_int, [P, P, I64, I32]),
    "km_load_points_f64": (ctypes.c_int, [P, P, I64, I32]),
    "km_attach_points_device_f32": (ctypes.c_int, [P, P, I64, I32]),
    "km_points_info": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32),
                                      ctypes.POINTER(F64)]),
    "km_assign": (ctypes.c_int, [P, P, I32, P, P]),
    "km_update": (ctypes.c_int, [P, P, I32, P, P]),
    "km_converged": (ctypes.c_int, [P, P, P, I32, I32, F64, ctypes.POINTER(I32)]),
    "km_lloyd": (ctypes.c_int, [P, P, I32, I32, F64, P, P, P, P, P]),
    "km_wcss": (ctypes.c_int, [P, P, I32, P, ctypes.POINTER(F64)]),
    "km_center_distances": (ctypes.c_int, [P, P, I32, P]),
    "km_diameter": (ctypes.c_int, [P, I64, ctypes.POINTER(F64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
    "km_max_pair_rows": (ctypes.c_int, [P, P, I64, ctypes.POINTER(F64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
    "km_block_sums": (ctypes.c_int, [P, P, I32, I64, I64, I64, P, P, ctypes.POINTER(I64)]),
    "km_step_loop_begin": (ctypes.c_int, [P, I32, F64]),
    "km_step_loop_pass": (ctypes.c_int, [P]),
    "km_step_loop_finish": (ctypes.c_int, [P]),
    "km_step_loop_check": (ctypes.c_int, [P]),
    "km_step_loop_state": (ctypes.c_int, [P, P]),
    "km_seed_reset": (ctypes.c_int, [P]),
    "km_seed_add": (ctypes.c_int, [P, I64, ctypes.POINTER(F64), ctypes.POINTER(I64)]),
    "km_seed_min_d2": (ctypes.c_int, [P, I64, ctypes.POINTER(F64)]),
    "km_set_frac_bits": (ctypes.c_int, [P, I32]),
    "km_frac_bits_for": (ctypes.c_int, [F64, I64, ctypes.POINTER(I32)]),
    "km_step_begin": (ctypes.c_int, [P, P, I32]),
    "km_step_partials": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(I64)]),
    "km_step_pass": (ctypes.c_int, [P]),
    "km_step_finish": (ctypes.c_int, [P, F64, P]),
    "km_step_repair_prepare": (ctypes.c_int, [P]),
    "km_step_repair_candidate": (ctypes.c_int, [P, ctypes.POINTER(F64), ctypes.POINTER(I64), P]),
    "km_step_repair_apply": (ctypes.c_int, [P, I32, I32, I64, P, I32]),
    "km_step_fold": (ctypes.c_int, [P]),
    "km_step_empty_list": (ctypes.c_int, [P, P, ctypes.POINTER(I32)]),
    "km_step_label_of": (ctypes.c_int, [P, I64, ctypes.POINTER(I32)]),
    "km_step_check": (ctypes.c_int, [P, F64, ctypes.POINTER(I32)]),
    "km_step_read": (ctypes.c_int, [P, P, P, P]),
    "km_peer_init": (ctypes.c_int, [P, I32, I32, I32, P]),
    "km_peer_connect": (ctypes.c_int, [P, P]),
    "km_lloyd_peer": (ctypes.c_int, [P, P, I32, I32, F64, P]),
    "km_lloyd_peer_resume": (ctypes.c_int, [P, P]),
    "km_get_stats": (ctypes.c_int, [P, ctypes.POINTER(KmStats)]),
    "km_reset_stats": (ctypes.c_int, [P]),
    "km_set_kernel_path": (ctypes.c_int, [P, I32]),
    "km_kernel_path": (ctypes.c_int, [P, ctypes.POINTER(I32)]),
    "km_debug_filter_scores": (ctypes.c_int, [P, P, I32, P]),
    "km_set_profiling": (ctypes.c_int, [P, I32]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libkmeans_b200.so (raises DeviceUnavailableError if it is not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceUnavailableError(
                f"CUDA engine not built ({LIB_PATH} missing); run `python -m paper_1402_3788_b200.build` "
                "(no CPU fallback exists)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(P)


def device_count() -> int:
    lib = load_library()
    out = I32(0)
    lib.km_device_count(ctypes.byref(out))
    return int(out.value)


class NativeEngine:
    """One km_engine handle: one device, one stream, resident points."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = P()
        rc = self._lib.km_create(int(device), ctypes.byref(h))
        if rc != KM_OK:
            msg = self._lib.km_last_error(None).decode()
            raise _ERRORS.get(rc, ClusteringError)(msg)
        self._h = h
        self.device = device
        self.n = 0
        self.m = 0
        # (iterations, converged) of km_lloyd, written through a cached address
        self._res = np.zeros(2, dtype=np.int32)
        self._res_p = self._res.__array_interface__["data"][0]

    # -- plumbing ---------------------------------------------------------
    def _check(self, rc):
        if rc != KM_OK:
            msg = self._lib.km_last_error(self._h).decode()
            raise _ERRORS.get(rc, ClusteringError)(msg)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.km_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        self._check(self._lib.km_set_stream(self._h, P(stream_handle) if stream_handle else None))

    # -- data -------------------------------------------------------------
    def load(self, coords: np.ndarray):
        coords = np.ascontiguousarray(coords)
        n, m = coords.shape
        if coords.dtype == np.float32:
            self._check(self._lib.km_load_points_f32(self._h, _ptr(coords), n, m))
        else:
            coords = np.ascontiguousarray(coords, dtype=np.float64)
            self._check(self._lib.km_load_points_f64(self._h, _ptr(coords), n, m))
        self.n, self.m = n, m

    def attach_device_f32(self, dev_ptr: int, n: int, m: int):
        self._check(self._lib.km_attach_points_device_f32(self._h, P(dev_ptr), int(n), int(m)))
        self.n, self.m = int(n), int(m)

    def points_info(self):
        n, m, pb, mx = I64(), I32(), I32(), F64()
        self._check(self._lib.km_points_info(self._h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(pb),
                                             ctypes.byref(mx)))
        return {"n": n.value, "m": m.value, "point_bytes": pb.value, "absmax": mx.value}

    # -- hot-path steps -----------------------------------------------------
    def assign(self, centers: np.ndarray):
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        k = centers.shape[0]
        labels = np.empty(self.n, dtype=np.int64)
        counts = np.empty(k, dtype=np.int64)
        self._check(self._lib.km_assign(self._h, _ptr(centers), k, _ptr(labels), _ptr(counts)))
        return labels, counts

    def update(self, labels: np.ndarray, k: int):
        """Returns (centers, counts); `labels` (int64, C-contiguous) is modified in place by the repair."""
        if labels.dtype != np.int64 or not labels.flags.c_contiguous:
            raise ContractViolationError("labels must be a C-contiguous int64 array")
        centers = np.empty((k, self.m), dtype=np.float64)
        counts = np.empty(k, dtype=np.int64)
        self._check(self._lib.km_update(self._h, _ptr(labels), int(k), _ptr(centers), _ptr(counts)))
        return centers, counts

    def converged(self, prev: np.ndarray, nxt: np.ndarray, tol: float) -> bool:
        prev = np.ascontiguousarray(prev, dtype=np.float64)
        nxt = np.ascontiguousarray(nxt, dtype=np.float64)
        out = I32(0)
        k, m = prev.shape
        self._check(self._lib.km_converged(self._h, _ptr(prev), _ptr(nxt), k, m, float(tol), ctypes.byref(out)))
        return bool(out.value)

    def lloyd(self, c0: np.ndarray, max_iters: int, tol: float, want_labels: bool = True):
        # (lean: this call is inside every timed bench step — one output buffer for the centres
        # and counts, raw addresses instead of ctypes pointer objects)
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        k = c0.shape[0]
        km = k * self.m
        out = np.empty(km + k, dtype=np.float64)
        po = out.__array_interface__["data"][0]
        labels = np.empty(self.n, dtype=np.int64) if want_labels else None
        rc = self._lib.km_lloyd(self._h, c0.__array_interface__["data"][0], k, int(max_iters), float(tol), po,
                                po + 8 * km, labels.__array_interface__["data"][0] if labels is not None else None,
                                self._res_p, self._res_p + 4)
        if rc != KM_OK:
            self._check(rc)
        return (out[:km].reshape(k, self.m), out[km:].view(np.int64), labels, int(self._res[0]),
                bool(self._res[1]))

    def wcss(self, centers: np.ndarray, labels: np.ndarray) -> float:
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        out = F64(0)
        self._check(self._lib.km_wcss(self._h, _ptr(centers), centers.shape[0], _ptr(labels), ctypes.byref(out)))
        return float(out.value)

    def center_distances(self, centers: np.ndarray) -> np.ndarray:
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        out = np.empty((self.n, centers.shape[0]), dtype=np.float64)
        self._check(self._lib.km_center_distances(self._h, _ptr(centers), centers.shape[0], _ptr(out)))
        return out

    # -- batched step loop (multi-GPU driver without a host round trip per iteration) --
    def loop_begin(self, max_iters, tol):
        self._check(self._lib.km_step_loop_begin(self._h, int(max_iters), float(tol)))

    def loop_pass(self):
        self._check(self._lib.km_step_loop_pass(self._h))

    def loop_finish(self):
        self._check(self._lib.km_step_loop_finish(self._h))

    def loop_check(self):
        self._check(self._lib.km_step_loop_check(self._h))

    # -- row-sharded resident loop, in-kernel NVLink exchange (km_peer_*) ----------------------
    def peer_init(self, world: int, rank: int, k: int) -> bytes:
        """Allocate this rank's exchange buffer; returns its 64-byte CUDA IPC handle."""
        h = ctypes.create_string_buffer(64)
        self._check(self._lib.km_peer_init(self._h, int(world), int(rank), int(k), h))
        return h.raw

    def peer_connect(self, handles) -> None:
        """Map every rank's exchange buffer (handles in rank order, 64 bytes each)."""
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles))
        self._check(self._lib.km_peer_connect(self._h, buf))

    def lloyd_peer(self, c0: np.ndarray, max_iters: int, tol: float):
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        out = np.zeros(4, dtype=np.int32)
        self._check(self._lib.km_lloyd_peer(self._h, _ptr(c0), c0.shape[0], int(max_iters), float(tol), _ptr(out)))
        return int(out[0]), bool(out[1]), bool(out[2]), bool(out[3])

    def lloyd_peer_resume(self):
        out = np.zeros(4, dtype=np.int32)
        self._check(self._lib.km_lloyd_peer_resume(self._h, _ptr(out)))
        return int(out[0]), bool(out[1]), bool(out[2]), bool(out[3])

    def loop_state(self):
        """(t, done, converged, need_host) — one device→host read."""
        out = np.zeros(4, dtype=np.int32)
        self._check(self._lib.km_step_loop_state(self._h, _ptr(out)))
        return int(out[0]), bool(out[1]), bool(out[2]), bool(out[3])

    # -- seeding -------------------------------------------------
    def diameter(self, pair_cap=None):
        """(d, i, j): largest pairwise distance over engine.scan_rows(n, pair_cap) rows."""
        d, i, j = F64(), I64(), I64()
        cap = 0 if pair_cap is None else int(pair_cap)
        self._check(self._lib.km_diameter(self._h, cap, ctypes.byref(d), ctypes.byref(i), ctypes.byref(j)))
        return d.value, i.value, j.value

    # -- device jobs (device.py:117-239) ----------------------------
    def max_pair_rows(self, rows):
        """MAX_PAIR job: (d2, i, j) over the ascending `rows` × columns j > i; (-1.0, -1, -1) if none."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        d2, i, j = F64(), I64(), I64()
        self._check(self._lib.km_max_pair_rows(self._h, _ptr(rows), rows.shape[0], ctypes.byref(d2),
                                               ctypes.byref(i), ctypes.byref(j)))
        return d2.value, i.value, j.value

    def block_sums(self, start, stop, block, labels=None, k=0):
        """COORD_SUM (labels None): (nb, m) sums.  CLUSTER_SUM: ((nb, k, m) sums, (nb, k) counts).
        A label outside [0, k) raises ValidationFailureError naming the first such sample."""
        nb = -(-(int(stop) - int(start)) // int(block)) if stop > start else 0
        bad = I64(-1)
        if labels is None:
            sums = np.zeros((nb, self.m), dtype=np.float64)
            self._check(self._lib.km_block_sums(self._h, None, 1, int(start), int(stop), int(block), _ptr(sums),
                                                None, ctypes.byref(bad)))
            return sums, None
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        if labels.shape[0] < stop:
            raise ContractViolationError(f"labels cover {labels.shape[0]} samples, job needs {stop}")
        sums = np.zeros((nb, int(k), self.m), dtype=np.float64)
        counts = np.zeros((nb, int(k)), dtype=np.int64)
        self._check(self._lib.km_block_sums(self._h, _ptr(labels), int(k), int(start), int(stop), int(block),
                                            _ptr(sums), _ptr(counts), ctypes.byref(bad)))
        return sums, counts

    def seed_reset(self):
        self._check(self._lib.km_seed_reset(self._h))

    def seed_add(self, c: int):
        """Lower min_d2 with sample c; returns (max min_d2, its first index)."""
        v, i = F64(), I64()
        self._check(self._lib.km_seed_add(self._h, int(c), ctypes.byref(v), ctypes.byref(i)))
        return v.value, i.value

    def seed_min_d2(self, i: int) -> float:
        v = F64()
        self._check(self._lib.km_seed_min_d2(self._h, int(i), ctypes.byref(v)))
        return v.value

    # -- step API (multi-GPU) -------------------------------------------------
    def set_frac_bits(self, f: int):
        self._check(self._lib.km_set_frac_bits(self._h, int(f)))

    def frac_bits_for(self, absmax: float, n_total: int) -> int:
        out = I32(0)
        self._check(self._lib.km_frac_bits_for(float(absmax), int(n_total), ctypes.byref(out)))
        return int(out.value)

    def step_begin(self, c0: np.ndarray):
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        self._check(self._lib.km_step_begin(self._h, _ptr(c0), c0.shape[0]))

    def step_partials(self):
        ptr, cnt = P(), I64()
        self._check(self._lib.km_step_partials(self._h, ctypes.byref(ptr), ctypes.byref(cnt)))
        return int(ptr.value), int(cnt.value)

    def step_pass(self):
        self._check(self._lib.km_step_pass(self._h))

    def step_finish(self, tol: float):
        st = np.zeros(2, dtype=np.int32)
        self._check(self._lib.km_step_finish(self._h, float(tol), _ptr(st)))
        return int(st[0]), bool(st[1])

    def step_fold(self):
        self._check(self._lib.km_step_fold(self._h))

    def step_repair_prepare(self):
        self._check(self._lib.km_step_repair_prepare(self._h))

    def step_repair_candidate(self):
        d2, row = F64(), I64()
        coords = np.zeros(self.m, dtype=np.float64)
        self._check(self._lib.km_step_repair_candidate(self._h, ctypes.byref(d2), ctypes.byref(row), _ptr(coords)))
        return float(d2.value), int(row.value), coords

    def step_repair_apply(self, cluster: int, owner: bool, local_row: int, coords: np.ndarray, donor: int):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        self._check(self._lib.km_step_repair_apply(self._h, int(cluster), int(bool(owner)), int(local_row),
                                                   _ptr(coords), int(donor)))

    def step_empty_list(self, k: int):
        out = np.zeros(k, dtype=np.int32)
        cnt = I32(0)
        self._check(self._lib.km_step_empty_list(self._h, _ptr(out), ctypes.byref(cnt)))
        return out[: cnt.value].astype(np.int64)

    def step_label_of(self, local_row: int) -> int:
        out = I32(0)
        self._check(self._lib.km_step_label_of(self._h, int(local_row), ctypes.byref(out)))
        return int(out.value)

    def step_check(self, tol: float) -> bool:
        out = I32(0)
        self._check(self._lib.km_step_check(self._h, float(tol), ctypes.byref(out)))
        return bool(out.value)

    def step_read(self, k: int, want_labels: bool = True):
        centers = np.empty((k, self.m), dtype=np.float64)
        counts = np.empty(k, dtype=np.int64)
        labels = np.empty(self.n, dtype=np.int64) if want_labels else None
        self._check(self._lib.km_step_read(self._h, _ptr(centers), _ptr(counts),
                                           _ptr(labels) if labels is not None else None))
        return centers, counts, labels

    def set_profiling(self, enable: bool):
        self._check(self._lib.km_set_profiling(self._h, int(bool(enable))))

    def set_kernel_path(self, path: int):
        """0 = auto (tensor core when eligible), 1 = SIMT only, 2 = tensor core required."""
        self._check(self._lib.km_set_kernel_path(self._h, int(path)))

    def kernel_path(self) -> int:
        out = I32(0)
        self._check(self._lib.km_kernel_path(self._h, ctypes.byref(out)))
        return int(out.value)

    def debug_filter_scores(self, centers: np.ndarray) -> np.ndarray:
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        out = np.empty((self.n, centers.shape[0]), dtype=np.float32)
        self._check(self._lib.km_debug_filter_scores(self._h, _ptr(centers), centers.shape[0], _ptr(out)))
        return out

    def reset_stats(self):
        self._check(self._lib.km_reset_stats(self._h))

    def partials_tensor(self):
        """torch int64 CUDA tensor aliasing the device partial buffer (k·m sums + k counts)."""
        import torch

        ptr, count = self.step_partials()

        class _CAI:
            __cuda_array_interface__ = {"shape": (count,), "typestr": "<i8", "data": (ptr, False), "version": 3}

        return torch.as_tensor(_CAI(), device=f"cuda:{self.device}")

    def stats(self) -> dict:
        s = KmStats()
        self._check(self._lib.km_get_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in KmStats._fields_}
