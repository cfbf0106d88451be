"""In-tree build of the native pieces (nvcc / gcc called directly, no JIT cache).

* ``paper_1402_3788_b200/_lib/libkmeans_b200.so`` — CUDA engine + C ABI,
  compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``).
* ``oracle/_build/libkmeans_oracle.so`` — the CPU restatement used by tests and
  by bench.py's cpu_baseline leg (test infrastructure, never the product path).

Both outputs are git-ignored and travel to the GPU box with the snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libkmeans_b200.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libkmeans_oracle.so"

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the engine")


def _sources():
    return (sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h"))
            + [ROOT / "include" / "kmeans_b200.h"])


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build_engine(force: bool = False, verbose: bool = False, defines=(), out: Path = None) -> Path:
    """Compile every csrc/*.cu to an object in parallel, then link the shared library.

    ``defines``/``out`` build a tuning variant (e.g. KM_WAIT_MODE=1) into another file.
    """
    lib = out or LIB
    if not force and not _stale(lib, _sources()):
        return lib
    from concurrent.futures import ThreadPoolExecutor

    LIBDIR.mkdir(parents=True, exist_ok=True)
    objdir = LIBDIR / ("obj" if out is None else "obj_" + lib.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    common = [nvcc, *NVCC_ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v" if verbose else "-O3",
              "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "-I", str(ROOT / "include"),
              *[f"-D{d}" for d in defines]]
    units = sorted(CSRC.glob("*.cu"))

    def compile_one(src: Path):
        obj = objdir / (src.stem + ".o")
        cmd = [*common, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=len(units)) as pool:
        results = list(pool.map(compile_one, units))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *NVCC_ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC",
           *[str(o) for o, _ in results], "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


def build_oracle(force: bool = False) -> Path:
    src = ORACLE_DIR / "kmeans_oracle.c"
    if not force and not _stale(ORACLE_LIB, [src]):
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = ORACLE_LIB.with_suffix(".so.tmp")
    # -ffp-contract=off: no FMA contraction, the reference's numba kernels are
    # compiled without fastmath (_kernels.py:5-9).
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-pthread", str(src), "-o", str(tmp), "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, ORACLE_LIB)
    return ORACLE_LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_engine(force=force, verbose=verbose)
    if (ORACLE_DIR / "kmeans_oracle.c").exists():
        build_oracle(force=force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
