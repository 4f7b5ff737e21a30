"""ctypes binding of the C-ABI (include/eigenid_b200.h).

Loads the in-tree libeigenid_b200.so built by build.py.  A missing library or
device raises immediately — the product never falls back to CPU code.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libeigenid_b200.so")

_dp = C.POINTER(C.c_double)


class GpuErr(C.Structure):
    _fields_ = [("code", C.c_int), ("index", C.c_int64), ("gap", C.c_double),
                ("cuda_error", C.c_int), ("msg", C.c_char * 256)]


class GpuConfig(C.Structure):
    _fields_ = [("batch_size", C.c_size_t), ("degeneracy_tol", C.c_double),
                ("log_domain", C.c_int)]


class GpuMagnitude(C.Structure):
    """eigenid_gpu_magnitude = MagnitudeResult (identity.hpp:66-74)."""
    _fields_ = [("value", C.c_double), ("raw_value", C.c_double), ("i", C.c_uint64),
                ("j", C.c_uint64), ("method", C.c_int), ("condition_flag", C.c_double)]


# every symbol the header declares, with its signature
SIGNATURES = {
    "eigenid_gpu_abi_version": (C.c_int, []),
    "eigenid_gpu_device_count": (C.c_int, []),
    "eigenid_gpu_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(GpuErr)]),
    "eigenid_gpu_destroy": (C.c_int, [C.c_void_p]),
    "eigenid_gpu_stream": (C.c_void_p, [C.c_void_p]),
    "eigenid_gpu_sync": (C.c_int, [C.c_void_p, C.POINTER(GpuErr)]),
    "eigenid_gpu_eigenvalues": (C.c_int, [C.c_void_p, _dp, C.c_size_t, _dp,
                                          C.POINTER(GpuErr)]),
    "eigenid_gpu_all_magnitudes": (C.c_int, [C.c_void_p, _dp, C.c_size_t,
                                             C.POINTER(GpuConfig), _dp, _dp, _dp,
                                             C.POINTER(GpuErr)]),
    "eigenid_gpu_all_magnitudes_batched": (C.c_int, [C.c_void_p, _dp, C.c_size_t,
                                                     C.c_size_t, C.POINTER(GpuConfig),
                                                     _dp, C.POINTER(GpuErr)]),
    "eigenid_gpu_minor_spectra": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t,
                                            C.c_size_t, _dp, _dp, C.POINTER(GpuErr)]),
    "eigenid_gpu_identity": (C.c_int, [C.c_void_p, _dp, _dp, C.c_size_t, C.c_size_t,
                                       C.c_size_t, C.POINTER(GpuConfig), _dp,
                                       C.POINTER(GpuErr)]),
    "eigenid_gpu_vector_magnitudes": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t,
                                                C.POINTER(GpuConfig), _dp, _dp,
                                                C.POINTER(GpuErr)]),
    "eigenid_gpu_recover_signs": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t, _dp,
                                            C.c_size_t, C.c_double, C.c_double, _dp,
                                            C.POINTER(GpuErr)]),
    "eigenid_gpu_recover_signs_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t,
                                                   C.c_void_p, C.c_double, C.c_double,
                                                   C.c_void_p, C.POINTER(GpuErr)]),
    "eigenid_gpu_component_magnitude": (C.c_int, [C.c_void_p, _dp, C.c_size_t,
                                                  C.c_size_t, C.c_size_t, _dp, _dp,
                                                  C.POINTER(GpuConfig), _dp, _dp,
                                                  C.POINTER(C.c_int),
                                                  C.POINTER(GpuErr)]),
    "eigenid_gpu_solve_count": (C.c_size_t, [C.c_void_p]),
    "eigenid_gpu_reset_solve_count": (None, [C.c_void_p]),
    "eigenid_gpu_all_magnitudes_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t,
                                                    C.c_size_t, C.c_size_t,
                                                    C.POINTER(GpuConfig), C.c_void_p,
                                                    C.c_void_p, C.c_void_p,
                                                    C.POINTER(GpuErr)]),
    "eigenid_gpu_all_magnitudes_batched_device": (C.c_int, [C.c_void_p, C.c_void_p,
                                                            C.c_size_t, C.c_size_t,
                                                            C.POINTER(GpuConfig),
                                                            C.c_void_p,
                                                            C.POINTER(GpuErr)]),
    "eigenid_gpu_identity_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_size_t, C.c_size_t, C.c_size_t,
                                              C.POINTER(GpuConfig), C.c_void_p,
                                              C.POINTER(GpuErr)]),
    "eigenid_gpu_c5_mu_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p,
                                           C.c_size_t, C.c_size_t, C.c_size_t,
                                           C.c_void_p, C.POINTER(GpuErr)]),
    "eigenid_gpu_launch_count": (C.c_uint64, [C.c_void_p]),
    "eigenid_random_symmetric": (None, [C.c_uint64, C.c_size_t, C.c_int, _dp]),
    "eigenid_seeded_draws": (None, [C.c_uint64, C.c_size_t, C.c_int, _dp]),
    "eigenid_c3_matrix": (None, [C.c_uint64, C.c_size_t, _dp]),
    "eigenid_gpu_set_profiling": (None, [C.c_void_p, C.c_int]),
    "eigenid_gpu_create_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                           C.POINTER(GpuErr)]),
    "eigenid_gpu_num_devices": (C.c_int, [C.c_void_p]),
    "eigenid_gpu_device_stream": (C.c_void_p, [C.c_void_p, C.c_int]),
    "eigenid_gpu_all_magnitudes_multi_device": (C.c_int, [C.c_void_p,
                                                          C.POINTER(C.c_void_p),
                                                          C.c_size_t,
                                                          C.POINTER(GpuConfig),
                                                          C.POINTER(C.c_void_p),
                                                          C.POINTER(GpuErr)]),
    "eigenid_gpu_component": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t,
                                        C.c_size_t, _dp, _dp, C.POINTER(GpuConfig),
                                        C.c_int, C.POINTER(GpuMagnitude),
                                        C.POINTER(GpuErr)]),
    "eigenid_gpu_vector": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t,
                                     C.POINTER(GpuConfig), C.POINTER(GpuMagnitude),
                                     C.POINTER(GpuErr)]),
    "eigenid_gpu_log_domain_product": (C.c_int, [C.c_void_p, _dp, _dp, C.c_size_t, _dp,
                                                 C.POINTER(GpuErr)]),
    "eigenid_gpu_tridiagonalize": (C.c_int, [C.c_void_p, _dp, C.c_size_t, _dp, _dp,
                                             C.POINTER(GpuErr)]),
    "eigenid_gpu_tridiagonal_eigenvalues": (C.c_int, [C.c_void_p, _dp, _dp, C.c_size_t,
                                                      _dp, C.POINTER(GpuErr)]),
    "eigenid_gpu_stage_times": (C.c_int, [C.c_void_p, _dp, C.c_int]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Loads the CUDA library (raises DeviceError if it was not built).
    EIGENID_LIB selects another build of the same library (A/B timing of
    kernel variants, tools/variant_run.sh)."""
    global _lib
    path = path or os.environ.get("EIGENID_LIB") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise errors.DeviceError(
                f"{path} is missing: run __graft_entry__.build() "
                "(the B200 path has no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(st: int, err: GpuErr):
    if st:
        errors.raise_for(st, err.msg.decode(errors="replace"), err.gap,
                         err.cuda_error)


def dptr(a) -> _dp:
    return a.ctypes.data_as(_dp)
