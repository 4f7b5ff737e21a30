"""The C-ABI library loads without a GPU and exports every declared symbol;
without a device every entry point fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eigenid_b200.h")
LIB = os.path.join(ROOT, "paper_2002_04989_b200", "libeigenid_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(eigenid_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("eigenid_gpu_create", "eigenid_gpu_all_magnitudes",
                 "eigenid_gpu_eigenvalues", "eigenid_gpu_identity",
                 "eigenid_gpu_all_magnitudes_device"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(lib, name), name


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_python_binding_covers_header():
    from paper_2002_04989_b200 import _native
    assert set(declared()) == set(_native.SIGNATURES)
    lib = _native.load()
    assert lib.eigenid_gpu_abi_version() == 1


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_no_cpu_fallback_without_device():
    from paper_2002_04989_b200 import DeviceError, IdentityEngine, _native
    lib = _native.load()
    if lib.eigenid_gpu_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(DeviceError):
        IdentityEngine()
    ctx = ctypes.c_void_p()
    err = _native.GpuErr()
    assert lib.eigenid_gpu_create(ctypes.byref(ctx), 0, ctypes.byref(err)) == 20
