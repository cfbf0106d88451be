"""The C-ABI library loads on CPU and exports every symbol include/kmeans_b200.h
declares; without a GPU, engine creation fails loudly (no CPU fallback)."""

import ctypes
import re
from pathlib import Path

import pytest

from conftest import ROOT, gpu_available


def header_symbols():
    text = (ROOT / "include" / "kmeans_b200.h").read_text()
    return sorted(set(re.findall(r"KM_API\s+[\w\s\*]+?\b(km_\w+)\s*\(", text)))


def test_header_declares_symbols():
    syms = header_symbols()
    assert "km_lloyd" in syms and "km_assign" in syms and "km_update" in syms
    assert len(syms) >= 30


def test_library_exports_every_header_symbol():
    from paper_1402_3788_b200 import _native

    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"


def test_binding_covers_header():
    from paper_1402_3788_b200 import _native

    assert set(header_symbols()) == set(_native.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess

    from paper_1402_3788_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_version_string():
    from paper_1402_3788_b200 import _native

    lib = _native.load_library()
    assert b"sm_100a" in lib.km_version()


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    from paper_1402_3788_b200 import DeviceUnavailableError
    from paper_1402_3788_b200._native import NativeEngine

    with pytest.raises(DeviceUnavailableError):
        NativeEngine(0)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_product_path_has_no_cpu_fallback():
    import numpy as np

    from paper_1402_3788_b200 import ClusterModel, Dataset, DeviceUnavailableError, assign_step

    with pytest.raises(DeviceUnavailableError):
        assign_step(Dataset(np.zeros((4, 2))), ClusterModel(np.zeros((2, 2))))


def test_product_package_never_imports_oracle():
    pkg = ROOT / "paper_1402_3788_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "import oracle" not in text and "from oracle" not in text, py
