"""ctypes access to the CPU checker (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so, the plain-C restatement of the reference
hot path (oracle.c); `Reference` wraps oracle/_ref/libeigenid_ref.so, the
unmodified reference compiled from /root/reference/proj/src.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module — the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libeigenid_ref.so")

_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)


class OrcErr(C.Structure):
    _fields_ = [("code", C.c_int), ("index", C.c_int64), ("gap", C.c_double),
                ("msg", C.c_char * 256)]


class OracleError(RuntimeError):
    def __init__(self, code, index, gap, msg):
        super().__init__(f"[{code}] {msg}")
        self.code, self.index, self.gap = code, index, gap


def _p(a):
    return a.ctypes.data_as(_dp)


def _check(st, err):
    if st:
        raise OracleError(err.code, err.index, err.gap,
                          err.msg.decode(errors="replace"))


class Oracle:
    """The plain-C restatement (kind "port")."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run make -f oracle/Makefile")
        L = self.lib = C.CDLL(path)
        L.orc_random_symmetric.argtypes = [C.c_uint64, C.c_size_t, C.c_int, _dp]
        L.orc_gaussian_stream.argtypes = [C.c_uint64, C.c_size_t, _dp]
        L.orc_c3_matrix.argtypes = [C.c_uint64, C.c_size_t, _dp]
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_minor.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
        L.orc_c5_lambda.argtypes = [C.c_uint64, C.c_size_t, _dp]
        L.orc_c5_mu_row.argtypes = [C.c_uint64, _dp, C.c_size_t, C.c_size_t, _dp]
        L.orc_tridiagonalize.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _dp]
        L.orc_ql.argtypes = [_dp, _dp, C.c_size_t, C.POINTER(OrcErr)]
        L.orc_eigenvalues.argtypes = [_dp, C.c_size_t, _dp, C.POINTER(OrcErr)]
        L.orc_check_fully_nondegenerate.argtypes = [_dp, C.c_size_t, C.c_double,
                                                    C.POINTER(OrcErr)]
        L.orc_evaluate.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                   C.c_double, C.c_int, _dp, _dp,
                                   C.POINTER(C.c_int), C.POINTER(OrcErr)]
        L.orc_log_domain_product.argtypes = [_dp, _dp, C.c_size_t, _dp,
                                             C.POINTER(OrcErr)]
        L.orc_identity_rows.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t,
                                        C.c_size_t, C.c_size_t, C.c_double,
                                        C.c_int, C.c_int, _dp, C.POINTER(OrcErr)]
        L.orc_all_magnitudes.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_double,
                                         C.c_int, C.c_int, _dp, _dp, _dp,
                                         C.POINTER(OrcErr)]
        L.orc_recover_signs.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t,
                                         C.c_double, C.c_double, _dp, C.POINTER(OrcErr)]
        L.orc_minor_spectra.argtypes = [_dp, C.c_size_t, _szp, C.c_size_t,
                                        C.c_int, _dp, C.POINTER(OrcErr)]

    # ---- inputs
    def random_symmetric(self, seed: int, n: int, uniform: bool = False):
        out = np.empty((n, n), np.float64)
        self.lib.orc_random_symmetric(seed, n, int(uniform), _p(out))
        return out

    def c3_matrix(self, n: int = 1024, seed: int = 3):
        """SURVEY §8 d3 input (bit-identical to the product's eigenid_c3_matrix)."""
        out = np.empty((n, n), np.float64)
        self.lib.orc_c3_matrix(seed, n, _p(out))
        return out

    def gaussian_stream(self, seed: int, count: int):
        out = np.empty(count, np.float64)
        self.lib.orc_gaussian_stream(seed, count, _p(out))
        return out

    def splitmix64(self, x: int) -> int:
        return int(self.lib.orc_splitmix64(x))

    def minor(self, a, j: int):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        out = np.empty((n - 1, n - 1), np.float64)
        self.lib.orc_minor(_p(a), n, j, _p(out))
        return out

    def c5_lambda(self, seed: int, n: int):
        out = np.empty(n, np.float64)
        self.lib.orc_c5_lambda(seed, n, _p(out))
        return out

    def c5_mu_rows(self, seed: int, lam, rows):
        lam = np.ascontiguousarray(lam, np.float64)
        n = lam.shape[0]
        out = np.empty((len(rows), n - 1), np.float64)
        for r, j in enumerate(rows):
            self.lib.orc_c5_mu_row(seed, _p(lam), n, int(j), _p(out[r]))
        return out

    # ---- eigensolver
    def tridiagonalize(self, a, max_steps: int | None = None):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        d = np.empty(n, np.float64)
        e = np.empty(max(n - 1, 1), np.float64)
        steps = (1 << 64) - 1 if max_steps is None else max_steps
        self.lib.orc_tridiagonalize(_p(a), n, steps, _p(d), _p(e))
        return d, e[: n - 1]

    def ql(self, d, e):
        d = np.array(d, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        if e.size == 0:
            e = np.zeros(1)
        err = OrcErr()
        _check(self.lib.orc_ql(_p(d), _p(e), d.shape[0], C.byref(err)), err)
        return d

    def eigenvalues(self, a):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        out = np.empty(n, np.float64)
        err = OrcErr()
        _check(self.lib.orc_eigenvalues(_p(a), n, _p(out), C.byref(err)), err)
        return out

    # ---- identity engine
    def check_fully_nondegenerate(self, s, tol=1e-12):
        s = np.ascontiguousarray(s, np.float64)
        err = OrcErr()
        _check(self.lib.orc_check_fully_nondegenerate(_p(s), s.shape[0], tol,
                                                      C.byref(err)), err)

    def evaluate(self, lam, mu, i, batch=64, tol=1e-12, log_domain=False):
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        raw, val, meth = C.c_double(), C.c_double(), C.c_int()
        err = OrcErr()
        _check(self.lib.orc_evaluate(_p(lam), _p(mu), lam.shape[0], i, batch, tol,
                                     int(log_domain), C.byref(raw), C.byref(val),
                                     C.byref(meth), C.byref(err)), err)
        return val.value, raw.value, meth.value

    def log_domain_product(self, num, den):
        num = np.ascontiguousarray(num, np.float64)
        den = np.ascontiguousarray(den, np.float64)
        out = C.c_double()
        err = OrcErr()
        _check(self.lib.orc_log_domain_product(_p(num), _p(den), num.shape[0],
                                               C.byref(out), C.byref(err)), err)
        return out.value

    def identity_rows(self, lam, mu_rows, batch=64, tol=1e-12, log_domain=False,
                      threads=None):
        lam = np.ascontiguousarray(lam, np.float64)
        mu_rows = np.ascontiguousarray(mu_rows, np.float64)
        n = lam.shape[0]
        rows = mu_rows.shape[0]
        out = np.empty((rows, n), np.float64)
        err = OrcErr()
        _check(self.lib.orc_identity_rows(_p(lam), _p(mu_rows), n, 0, rows, batch,
                                          tol, int(log_domain),
                                          threads or os.cpu_count() or 1,
                                          _p(out), C.byref(err)), err)
        return out

    def all_magnitudes(self, a, batch=64, tol=1e-12, log_domain=False,
                       threads=None, return_spectra=False):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        out = np.empty((n, n), np.float64)
        lam = np.empty(max(n, 1), np.float64)
        mu = np.empty(max(n * (n - 1), 1), np.float64)
        err = OrcErr()
        _check(self.lib.orc_all_magnitudes(_p(a), n, batch, tol, int(log_domain),
                                           threads or os.cpu_count() or 1,
                                           _p(out), _p(lam), _p(mu),
                                           C.byref(err)), err)
        if return_spectra:
            return out, lam[:n], mu[: n * (n - 1)].reshape(n, n - 1)
        return out

    def recover_signs(self, a, i, mags, lambda_i, sign_tol=1e-10):
        """signs.cpp:48-120."""
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        mags = np.ascontiguousarray(mags, np.float64)
        out = np.empty(n)
        err = OrcErr()
        _check(self.lib.orc_recover_signs(_p(a), n, i, _p(mags), mags.size, lambda_i,
                                        sign_tol, _p(out), C.byref(err)), err)
        return out

    def minor_spectra(self, a, js, threads=None):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        js_arr = (C.c_size_t * len(js))(*[int(j) for j in js])
        out = np.empty((len(js), n - 1), np.float64)
        err = OrcErr()
        _check(self.lib.orc_minor_spectra(_p(a), n, js_arr, len(js),
                                          threads or os.cpu_count() or 1, _p(out),
                                          C.byref(err)), err)
        return out


class Reference:
    """The unmodified reference library (kind "reference")."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run make -f oracle/Makefile")
        L = self.lib = C.CDLL(path)
        E = C.POINTER(OrcErr)
        L.ref_random_symmetric.argtypes = [C.c_uint64, C.c_size_t, C.c_int, _dp]
        L.ref_tridiagonalize.argtypes = [_dp, C.c_size_t, _dp, _dp]
        L.ref_eigenvalues.argtypes = [_dp, C.c_size_t, _dp, E]
        L.ref_all_magnitudes.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                         C.c_double, C.c_int, _dp,
                                         C.POINTER(C.c_size_t), E]
        L.ref_component_magnitude_cached.argtypes = [
            C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp, C.c_size_t, C.c_double,
            _dp, _dp, C.POINTER(C.c_int), E]
        L.ref_minor_spectra.argtypes = [_dp, C.c_size_t, _szp, C.c_size_t,
                                        C.c_size_t, _dp, E]
        L.ref_identity_rows.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t,
                                        C.c_size_t, C.c_double, C.c_size_t, _dp, E]
        L.ref_jacobi.argtypes = [_dp, C.c_size_t, _dp, _dp, E]
        L.ref_recover_signs.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t,
                                        C.c_double, C.c_double, _dp, E]

    def random_symmetric(self, seed, n, uniform=False):
        out = np.empty((n, n), np.float64)
        self.lib.ref_random_symmetric(seed, n, int(uniform), _p(out))
        return out

    def tridiagonalize(self, a):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        d = np.empty(n)
        e = np.empty(max(n - 1, 1))
        self.lib.ref_tridiagonalize(_p(a), n, _p(d), _p(e))
        return d, e[: n - 1]

    def eigenvalues(self, a):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        out = np.empty(n)
        err = OrcErr()
        _check(self.lib.ref_eigenvalues(_p(a), n, _p(out), C.byref(err)), err)
        return out

    def all_magnitudes(self, a, batch=64, workers=0, tol=1e-12, log_domain=False):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        out = np.empty((n, n))
        solves = C.c_size_t()
        err = OrcErr()
        _check(self.lib.ref_all_magnitudes(_p(a), n, batch, workers, tol,
                                           int(log_domain), _p(out),
                                           C.byref(solves), C.byref(err)), err)
        self.last_solves = solves.value
        return out

    def component_magnitude_cached(self, lam, mu, i, j, batch=64, tol=1e-12):
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        v, r, m = C.c_double(), C.c_double(), C.c_int()
        err = OrcErr()
        _check(self.lib.ref_component_magnitude_cached(
            lam.shape[0], i, j, _p(lam), _p(mu), batch, tol, C.byref(v),
            C.byref(r), C.byref(m), C.byref(err)), err)
        return v.value, r.value, m.value

    def minor_spectra(self, a, js, workers=0):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        js_arr = (C.c_size_t * len(js))(*[int(j) for j in js])
        out = np.empty((len(js), n - 1))
        err = OrcErr()
        _check(self.lib.ref_minor_spectra(_p(a), n, js_arr, len(js),
                                          workers or os.cpu_count() or 1, _p(out),
                                          C.byref(err)), err)
        return out

    def identity_rows(self, lam, mu_rows, batch=64, tol=1e-12, workers=0):
        lam = np.ascontiguousarray(lam, np.float64)
        mu_rows = np.ascontiguousarray(mu_rows, np.float64)
        n = lam.shape[0]
        out = np.empty((mu_rows.shape[0], n))
        err = OrcErr()
        _check(self.lib.ref_identity_rows(_p(lam), _p(mu_rows), n, mu_rows.shape[0],
                                          batch, tol, workers or os.cpu_count() or 1,
                                          _p(out), C.byref(err)), err)
        return out

    def recover_signs(self, a, i, mags, lambda_i, sign_tol=1e-10):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        mags = np.ascontiguousarray(mags, np.float64)
        out = np.empty(n)
        err = OrcErr()
        _check(self.lib.ref_recover_signs(_p(a), n, i, _p(mags), mags.size, lambda_i,
                                        sign_tol, _p(out), C.byref(err)), err)
        return out

    def jacobi(self, a, vectors=True):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        ev = np.empty(n)
        vec = np.empty((n, n)) if vectors else None
        err = OrcErr()
        _check(self.lib.ref_jacobi(_p(a), n, _p(ev),
                                   _p(vec) if vectors else None, C.byref(err)), err)
        return (ev, vec) if vectors else ev
