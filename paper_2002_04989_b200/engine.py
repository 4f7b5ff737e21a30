"""Python mirror of the reference's public API for the hot path.

Same names, argument meaning and error behaviour as
proj/include/eigenid/{matrix,eigensolve,identity}.hpp, implemented over the
C-ABI (include/eigenid_b200.h) — every computation runs in the sm_100a
kernels of libeigenid_b200.so; nothing here computes eigenvalues or
products on the CPU.

    SymmetricMatrix.build        matrix.hpp:21-22, matrix.cpp:10-38
    SymmetricMatrix.minor_matrix matrix.hpp:35-37, matrix.cpp:51-68
    eigenvalues(a)               eigensolve.hpp:46, eigensolve.cpp:130-132
    IdentityConfig               identity.hpp:81-93
    IdentityEngine.all_magnitudes identity.hpp:133-135, identity.cpp:294-316
    eigenvalue_solve_count       identity.hpp:137-144
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _native, errors

KSTRICT, KSYMMETRIZE = "strict", "symmetrize"


class SymmetricMatrix:
    """Dense real symmetric n x n matrix, row-major, immutable
    (matrix.hpp:13-47)."""

    def __init__(self, n: int, entries: np.ndarray):
        self._n = n
        self._e = entries
        self._e.setflags(write=False)

    @staticmethod
    def build(n: int, entries, policy: str = KSTRICT) -> "SymmetricMatrix":
        """matrix.cpp:10-38: DimensionMismatch / NonFiniteEntry /
        AsymmetricInput (strict) or (A + A^T)/2 off the diagonal (symmetrize)."""
        if n < 1:
            raise errors.DimensionMismatch("matrix dimension must be >= 1")
        e = np.array(entries, dtype=np.float64).reshape(-1)
        if e.size != n * n:
            raise errors.DimensionMismatch(
                f"expected {n * n} entries, got {e.size}")
        if not np.all(np.isfinite(e)):
            raise errors.NonFiniteEntry("matrix entry is not finite")
        m = e.reshape(n, n)
        up = np.triu_indices(n, 1)
        asym = np.abs(m[up] - m.T[up])
        max_asym = float(asym.max()) if asym.size else 0.0
        if max_asym > 0.0:
            if policy == KSTRICT:
                raise errors.AsymmetricInput(
                    f"input is not symmetric (max |a_rc - a_cr| = {max_asym:f})")
            mid = 0.5 * (m[up] + m.T[up])
            m = m.copy()
            m[up] = mid
            m.T[up] = mid
            e = m.reshape(-1)
        return SymmetricMatrix(n, np.ascontiguousarray(e))

    @staticmethod
    def diagonal(d) -> "SymmetricMatrix":
        d = np.asarray(d, dtype=np.float64)
        return SymmetricMatrix.build(d.size, np.diag(d))

    @staticmethod
    def identity(n: int) -> "SymmetricMatrix":
        return SymmetricMatrix.diagonal(np.ones(n))

    def n(self) -> int:
        return self._n

    def entries(self) -> np.ndarray:
        return self._e

    def array(self) -> np.ndarray:
        return self._e.reshape(self._n, self._n)

    def __call__(self, r: int, c: int) -> float:
        return float(self._e[r * self._n + c])

    def minor_matrix(self, j: int) -> "SymmetricMatrix":
        """matrix.cpp:51-68."""
        if self._n == 1:
            raise errors.MatrixTooSmall("cannot take a minor of a 1x1 matrix")
        if j >= self._n or j < 0:
            raise errors.IndexOutOfRange(
                f"minor index {j} out of range for n = {self._n}")
        keep = np.r_[0:j, j + 1:self._n]
        m = self.array()[np.ix_(keep, keep)]
        return SymmetricMatrix(self._n - 1, np.ascontiguousarray(m).reshape(-1))

    def scaled(self, factor: float) -> "SymmetricMatrix":
        return SymmetricMatrix(self._n, self._e * factor)

    def frobenius_norm(self) -> float:
        return float(np.sqrt(np.sum(self._e * self._e)))

    def trace(self) -> float:
        return float(np.trace(self.array()))


def random_symmetric(seed: int, n: int, dist: str = "gaussian") -> np.ndarray:
    """random_symmetric (matrix_io.cpp:171-181): the reference's seeded
    generator (mt19937_64, Box-Muller / uniform(-1,1), build(kSymmetrize)),
    bit-identical; host code in the C-ABI library."""
    out = np.empty((n, n), np.float64)
    _native.load().eigenid_random_symmetric(seed, n, 1 if dist == "uniform" else 0,
                                            _native.dptr(out))
    return out


def seeded_draws(seed: int, count: int, dist: str = "gaussian") -> np.ndarray:
    """The reference's raw SeededDraws stream (matrix_io.cpp:44-65)."""
    out = np.empty(count, np.float64)
    _native.load().eigenid_seeded_draws(seed, count, 1 if dist == "uniform" else 0,
                                        _native.dptr(out))
    return out


def c3_matrix(n: int = 1024, seed: int = 3) -> np.ndarray:
    """C3 input: Q diag(linspace(-1, 1)) Q^T, Q the sign-fixed
    Householder QR factor of a seeded Gaussian matrix, symmetrised; plain
    deterministic host loops in the C-ABI library (same bytes on any CPU)."""
    out = np.empty((n, n), np.float64)
    _native.load().eigenid_c3_matrix(seed, n, _native.dptr(out))
    return out


def c5_lambda(seed: int, n: int) -> np.ndarray:
    """C5 synthetic spectrum: n uniform(-1,1) draws, sorted,
    ties re-drawn from the same stream (strictly increasing)."""
    draws = seeded_draws(seed, 2 * n, "uniform")
    lam = np.sort(draws[:n])
    extra = iter(draws[n:])
    while True:
        tie = np.nonzero(lam[1:] == lam[:-1])[0]
        if tie.size == 0:
            return lam
        for k in tie:
            lam[k + 1] = next(extra)
        lam = np.sort(lam)


METHODS = {0: "baseline", 1: "batched", 2: "batched-parallel", 3: "log-domain"}


def log_domain_product(numerator, denominator, device: int = 0) -> float:
    """log_domain_product (identity.cpp:98-122) of explicit factor lists, on
    the device."""
    num = np.ascontiguousarray(numerator, np.float64)
    den = np.ascontiguousarray(denominator, np.float64)
    if num.size != den.size:
        raise errors.DimensionMismatch("factor lists differ in length")
    dev = Device.get(device)
    out = C.c_double()
    err = _native.GpuErr()
    _native.check(dev.lib.eigenid_gpu_log_domain_product(
        dev.ctx, _native.dptr(num), _native.dptr(den), num.size, C.byref(out),
        C.byref(err)), err)
    return out.value


def tridiagonalize(a, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """tridiagonalize (eigensolve.hpp:41): (diag, offdiag) of the device
    reduction — orthogonally similar to A, not tred1's sequence."""
    n, e = _as_matrix(a)
    dev = Device.get(device)
    d = np.empty(n, np.float64)
    off = np.empty(max(n - 1, 1), np.float64)
    err = _native.GpuErr()
    _native.check(dev.lib.eigenid_gpu_tridiagonalize(dev.ctx, _native.dptr(e), n,
                                                     _native.dptr(d), _native.dptr(off),
                                                     C.byref(err)), err)
    return d, off[: n - 1]


def tridiagonal_eigenvalues(diag, offdiag, device: int = 0) -> np.ndarray:
    """eigenvalues(TridiagonalForm) (eigensolve.cpp:72-128) by device Sturm
    bisection, ascending."""
    d = np.ascontiguousarray(diag, np.float64)
    off = np.ascontiguousarray(offdiag, np.float64)
    n = d.size
    if n > 0 and off.size != n - 1:
        raise errors.DimensionMismatch("tridiagonal form needs n-1 off-diagonal values")
    dev = Device.get(device)
    out = np.empty(n, np.float64)
    err = _native.GpuErr()
    _native.check(dev.lib.eigenid_gpu_tridiagonal_eigenvalues(
        dev.ctx, _native.dptr(d), _native.dptr(off) if off.size else None, n,
        _native.dptr(out), C.byref(err)), err)
    return out


def _as_matrix(a) -> tuple[int, np.ndarray]:
    if isinstance(a, SymmetricMatrix):
        return a.n(), np.ascontiguousarray(a.entries())
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise errors.DimensionMismatch("expected a square matrix")
    return arr.shape[0], arr.reshape(-1)


@dataclass
class IdentityConfig:
    """identity.hpp:81-93.  `workers` is accepted for source compatibility and
    has no device meaning (the CUDA grid replaces the thread pool)."""
    batch_size: int = 64
    workers: int = 0
    degeneracy_tol: float = 1e-12
    evaluation: str = "paired-batched"  # or "log-domain"

    def _c(self) -> _native.GpuConfig:
        return _native.GpuConfig(int(self.batch_size), float(self.degeneracy_tol),
                                 1 if self.evaluation == "log-domain" else 0)


class Device:
    """One C-ABI context (device buffers + stream), shared by engines on the
    same GPU like the reference's per-engine pool (SPEC D5)."""

    _instances: dict[int, "Device"] = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0, num_gpus: int = 1, multi: bool = False):
        self.lib = _native.load()
        self.ctx = C.c_void_p()
        err = _native.GpuErr()
        if num_gpus == 1 and not multi:
            _native.check(self.lib.eigenid_gpu_create(C.byref(self.ctx), device,
                                                      C.byref(err)), err)
        else:  # devices device .. device+num_gpus-1, one NCCL communicator
            _native.check(self.lib.eigenid_gpu_create_multi(
                C.byref(self.ctx), device, num_gpus, C.byref(err)), err)
        self.device = device
        self.num_gpus = num_gpus

    @classmethod
    def get(cls, device: int = 0) -> "Device":
        with cls._lock:
            if device not in cls._instances:
                cls._instances[device] = Device(device)
            return cls._instances[device]

    def stream(self) -> int:
        return int(self.lib.eigenid_gpu_stream(self.ctx) or 0)

    def launch_count(self) -> int:
        return int(self.lib.eigenid_gpu_launch_count(self.ctx))

    def sync(self):
        err = _native.GpuErr()
        _native.check(self.lib.eigenid_gpu_sync(self.ctx, C.byref(err)), err)

    def set_profiling(self, on: bool) -> None:
        self.lib.eigenid_gpu_set_profiling(self.ctx, 1 if on else 0)

    def stage_times(self) -> dict:
        """ms per stage of the last large-n call (needs set_profiling)."""
        buf = (C.c_double * 5)()
        k = self.lib.eigenid_gpu_stage_times(self.ctx, buf, 5)
        names = ["stage1", "stage2", "lambda_A", "bisect_minors", "identity"]
        return {names[t]: buf[t] for t in range(k)}

    def __del__(self):
        try:
            if self.ctx:
                self.lib.eigenid_gpu_destroy(self.ctx)
        except Exception:
            pass


def eigenvalues(a, device: int = 0) -> np.ndarray:
    """Spectrum eigenvalues(const SymmetricMatrix&): ascending eigenvalues,
    computed on the GPU (stage 1 + stage 2 + Sturm bisection)."""
    n, e = _as_matrix(a)
    dev = Device.get(device)
    out = np.empty(n, np.float64)
    err = _native.GpuErr()
    _native.check(dev.lib.eigenid_gpu_eigenvalues(dev.ctx, _native.dptr(e), n,
                                                  _native.dptr(out), C.byref(err)),
                  err)
    return out


def recover_signs(a, i: int, magnitudes, lambda_i: float, sign_tol: float = 1e-10,
                  device: int = 0) -> np.ndarray:
    """recover_signs (identity.hpp:159-166, signs.cpp:48-120): the signed
    eigenvector i from its squared magnitudes, solved on the GPU.  Raises
    DimensionMismatch for a wrong-length magnitude vector and
    SignRecoveryFailure for a singular anchor system or a residual above
    1e-6 ||A||_F, as the reference does."""
    n, e = _as_matrix(a)
    mags = np.ascontiguousarray(magnitudes, np.float64).reshape(-1)
    dev = Device.get(device)
    out = np.empty(n, np.float64)
    err = _native.GpuErr()
    _native.check(dev.lib.eigenid_gpu_recover_signs(
        dev.ctx, _native.dptr(e), n, i, _native.dptr(mags), mags.size, lambda_i,
        sign_tol, _native.dptr(out), C.byref(err)), err)
    return out


class IdentityEngine:
    """identity.hpp:99-157, the all-magnitudes path on the GPU."""

    def __init__(self, cfg: IdentityConfig | None = None, device: int = 0,
                 num_gpus: int | None = None):
        self._cfg = cfg or IdentityConfig()
        if self._cfg.batch_size < 1:
            raise errors.ConfigError("batch size must be >= 1")
        if not self._cfg.degeneracy_tol >= 0.0:
            raise errors.ConfigError("degeneracy tolerance must be >= 0")
        if num_gpus is not None and num_gpus < 1:
            raise errors.ConfigError("num_gpus must be >= 1")
        # num_gpus given: an engine-owned multi-device context over devices
        # device .. device+num_gpus-1 (NCCL communicator, even for one GPU);
        # all_magnitudes shards the minors and all-gathers rows with NCCL.
        # None: the process-wide context of `device`.
        self._dev = Device.get(device) if num_gpus is None else Device(device, num_gpus,
                                                                         multi=True)
        self._solves = 0
        self._solves_lock = threading.Lock()

    def config(self) -> IdentityConfig:
        return self._cfg

    @property
    def device(self) -> Device:
        return self._dev

    # -- instrumentation (identity.hpp:137-144)
    def eigenvalue_solve_count(self) -> int:
        return self._solves

    def reset_solve_count(self) -> None:
        self._solves = 0

    def _count(self, before: int):
        after = int(self._dev.lib.eigenid_gpu_solve_count(self._dev.ctx))
        with self._solves_lock:
            self._solves += after - before

    def _before(self) -> int:
        return int(self._dev.lib.eigenid_gpu_solve_count(self._dev.ctx))

    def all_magnitudes(self, a, return_spectra: bool = False):
        """Row-major n*n vector, entry [j*n + i] = |v_ij|^2
        (identity.cpp:294-316)."""
        n, e = _as_matrix(a)
        lib = self._dev.lib
        out = np.empty(n * n, np.float64)
        lam = np.empty(max(n, 1), np.float64)
        mu = np.empty(max(n * (n - 1), 1), np.float64) if return_spectra else None
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = lib.eigenid_gpu_all_magnitudes(
            self._dev.ctx, _native.dptr(e), n, C.byref(cfg), _native.dptr(out),
            _native.dptr(lam), _native.dptr(mu) if mu is not None else None,
            C.byref(err))
        self._count(b)
        _native.check(st, err)
        if return_spectra:
            return out, lam[:n], mu[: n * (n - 1)].reshape(n, n - 1)
        return out

    def all_magnitudes_batched(self, a_batch) -> np.ndarray:
        """count x n x n independent matrices -> count x n*n (config C2)."""
        a_batch = np.ascontiguousarray(np.asarray(a_batch, dtype=np.float64))
        count, n = a_batch.shape[0], a_batch.shape[1]
        out = np.empty((count, n * n), np.float64)
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_all_magnitudes_batched(
            self._dev.ctx, _native.dptr(a_batch), count, n, C.byref(cfg),
            _native.dptr(out), C.byref(err))
        self._count(b)
        _native.check(st, err)
        return out

    def vector_magnitudes(self, a, i: int, return_raw: bool = False):
        """|v_ij|^2 for j = 0..n-1 (identity.cpp:276-292): n+1 solves."""
        n, e = _as_matrix(a)
        out = np.empty(n, np.float64)
        raw = np.empty(n, np.float64)
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_vector_magnitudes(
            self._dev.ctx, _native.dptr(e), n, i, C.byref(cfg), _native.dptr(out),
            _native.dptr(raw), C.byref(err))
        self._count(b)
        _native.check(st, err)
        return (out, raw) if return_raw else out

    def component_magnitude(self, a, i: int, j: int, cached_lambda=None,
                            cached_mu=None):
        """(value, raw_value, method) of |v_ij|^2 (identity.cpp:240-251);
        cached spectra skip the two solves (SPEC D6)."""
        if isinstance(a, SymmetricMatrix) or a is not None:
            n, e = _as_matrix(a)
        else:
            n, e = len(cached_lambda), np.zeros(1)
        lam = None if cached_lambda is None else np.ascontiguousarray(cached_lambda, np.float64)
        mu = None if cached_mu is None else np.ascontiguousarray(cached_mu, np.float64)
        v, r, m = C.c_double(), C.c_double(), C.c_int()
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_component_magnitude(
            self._dev.ctx, _native.dptr(e), n, i, j,
            _native.dptr(lam) if lam is not None else None,
            _native.dptr(mu) if mu is not None else None, C.byref(cfg),
            C.byref(v), C.byref(r), C.byref(m), C.byref(err))
        self._count(b)
        _native.check(st, err)
        return v.value, r.value, m.value

    def _component(self, a, i, j, cached_lambda, cached_mu, variant) -> dict:
        n, e = _as_matrix(a)
        lam = None if cached_lambda is None else np.ascontiguousarray(cached_lambda, np.float64)
        mu = None if cached_mu is None else np.ascontiguousarray(cached_mu, np.float64)
        m = _native.GpuMagnitude()
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_component(
            self._dev.ctx, _native.dptr(e), n, i, j,
            _native.dptr(lam) if lam is not None else None,
            _native.dptr(mu) if mu is not None else None, C.byref(cfg), variant,
            C.byref(m), C.byref(err))
        self._count(b)
        _native.check(st, err)
        return {"value": m.value, "raw_value": m.raw_value, "i": i, "j": j,
                "method": METHODS[m.method], "condition_flag": m.condition_flag}

    def component_magnitude_baseline(self, a, i: int, j: int) -> dict:
        """MagnitudeResult of component_magnitude_baseline (identity.cpp:151-183):
        natural pairing, sequential running products on the device, 2 solves;
        NonFiniteIntermediate when a product leaves the finite range."""
        return self._component(a, i, j, None, None, 2)

    def component_result(self, a, i: int, j: int, cached_lambda=None,
                         cached_mu=None) -> dict:
        """Full MagnitudeResult of component_magnitude (identity.cpp:240-251)."""
        return self._component(a, i, j, cached_lambda, cached_mu, 0)

    def vector_results(self, a, i: int) -> list[dict]:
        """vector_magnitudes (identity.cpp:276-292) as MagnitudeResult dicts."""
        n, e = _as_matrix(a)
        out = (_native.GpuMagnitude * n)()
        err = _native.GpuErr()
        cfg = self._cfg._c()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_vector(self._dev.ctx, _native.dptr(e), n, i,
                                              C.byref(cfg), out, C.byref(err))
        self._count(b)
        _native.check(st, err)
        return [{"value": m.value, "raw_value": m.raw_value, "i": i, "j": j,
                 "method": METHODS[m.method], "condition_flag": m.condition_flag}
                for j, m in enumerate(out)]

    def log_domain_magnitude(self, a, i: int, j: int, cached_lambda=None,
                             cached_mu=None):
        """log_domain_magnitude (identity.cpp:253-274)."""
        saved = self._cfg.evaluation
        self._cfg.evaluation = "log-domain"
        try:
            return self.component_magnitude(a, i, j, cached_lambda, cached_mu)
        finally:
            self._cfg.evaluation = saved

    def minor_spectra(self, a, j0: int = 0, j1: int | None = None):
        """lambda(A) and the ascending spectra of minors j0..j1-1."""
        n, e = _as_matrix(a)
        j1 = n if j1 is None else j1
        lam = np.empty(n, np.float64)
        mu = np.empty((max(j1 - j0, 1), n - 1), np.float64)
        err = _native.GpuErr()
        b = self._before()
        st = self._dev.lib.eigenid_gpu_minor_spectra(
            self._dev.ctx, _native.dptr(e), n, j0, j1, _native.dptr(lam),
            _native.dptr(mu), C.byref(err))
        self._count(b)
        _native.check(st, err)
        return lam, mu[: j1 - j0]

    def identity(self, lam, mu_rows, j0: int = 0) -> np.ndarray:
        """Identity stage only from given spectra (rows j0..j0+len(mu_rows))."""
        lam = np.ascontiguousarray(lam, np.float64)
        mu_rows = np.ascontiguousarray(mu_rows, np.float64)
        n = lam.shape[0]
        rows = mu_rows.shape[0]
        out = np.empty((rows, n), np.float64)
        err = _native.GpuErr()
        cfg = self._cfg._c()
        _native.check(self._dev.lib.eigenid_gpu_identity(
            self._dev.ctx, _native.dptr(lam), _native.dptr(mu_rows), n, j0,
            j0 + rows, C.byref(cfg), _native.dptr(out), C.byref(err)), err)
        return out

    # -- device-resident entry points (torch tensors or raw pointers)
    def all_magnitudes_device(self, a_ptr: int, n: int, j0: int, j1: int,
                              out_ptr: int, lam_ptr: int = 0, mu_ptr: int = 0):
        err = _native.GpuErr()
        cfg = self._cfg._c()
        _native.check(self._dev.lib.eigenid_gpu_all_magnitudes_device(
            self._dev.ctx, a_ptr, n, j0, j1, C.byref(cfg), out_ptr,
            lam_ptr or None, mu_ptr or None, C.byref(err)), err)

    def identity_device(self, lam_ptr: int, mu_ptr: int, n: int, j0: int,
                        j1: int, out_ptr: int):
        err = _native.GpuErr()
        cfg = self._cfg._c()
        _native.check(self._dev.lib.eigenid_gpu_identity_device(
            self._dev.ctx, lam_ptr, mu_ptr, n, j0, j1, C.byref(cfg), out_ptr,
            C.byref(err)), err)

    def batched_device(self, a_ptr: int, count: int, n: int, out_ptr: int):
        err = _native.GpuErr()
        cfg = self._cfg._c()
        _native.check(self._dev.lib.eigenid_gpu_all_magnitudes_batched_device(
            self._dev.ctx, a_ptr, count, n, C.byref(cfg), out_ptr, C.byref(err)),
            err)

    def c5_mu_device(self, seed: int, lam_ptr: int, n: int, j0: int, j1: int,
                     mu_ptr: int):
        err = _native.GpuErr()
        _native.check(self._dev.lib.eigenid_gpu_c5_mu_device(
            self._dev.ctx, seed, lam_ptr, n, j0, j1, mu_ptr, C.byref(err)), err)

    def sync(self):
        self._dev.sync()
