"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU oracle.

Two libraries, both built by ``oracle/Makefile``:

* ``liboracle.so``            -- the C restatement (``fastleg_oracle.c``), ``fo_*``.
* ``_ref/libfastleg_ref.so``  -- the unmodified reference headers compiled in
  place against the FFTW-API shim, ``fr_*``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module, and only as the checker / the timed CPU baseline. The
product (``paper_1505_00354_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CHEB1, CHEBSTAR = 0, 1

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    """Non-zero return code from the oracle (1 invalid_argument, 2 domain_error,
    3 overflow_error, 4 runtime_error)."""

    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: oracle status {code}")
        self.code = code


def _check(rc: int, where: str) -> None:
    if rc:
        raise OracleError(rc, where)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _load(path: str) -> C.CDLL | None:
    return C.CDLL(path) if os.path.exists(path) else None


_lib = _load(os.path.join(HERE, "liboracle.so"))
_ref = _load(os.path.join(HERE, "_ref", "libfastleg_ref.so"))


def have_ref() -> bool:
    return _ref is not None


def _sig(lib, name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


class _Oracle:
    """Uniform facade over either library (prefix fo_ or fr_)."""

    def __init__(self, lib: C.CDLL, is_ref: bool):
        self.lib = lib
        self.is_ref = is_ref
        L, sz, i, d = lib, C.c_size_t, C.c_int, C.c_double
        p = "fr_" if is_ref else "fo_"
        self._nodes = _sig(L, p + "legendre_nodes_weights", i, sz, _dp, _dp, _dp)
        if is_ref:
            self._trig = _sig(L, "fr_trig", i, i, sz, i, _dp, _dp)
            self._ndct = _sig(L, "fr_ndct", i, i, sz, i, i, _dp, _dp, _dp)
            self._l2c = _sig(L, "fr_leg2cheb", i, i, sz, _dp, _dp)
            self._dlt = _sig(L, "fr_dlt_grid", i, sz, i, d, _dp, _dp, _dp, _dp, _dp)
            self._idlt = _sig(L, "fr_idlt_grid", i, sz, i, d, _dp, _dp, _dp, _dp, _dp)
            self._lam = _sig(L, "fr_lambda_table", i, sz, _dp)
            self._rnd = _sig(L, "fr_random_decaying", None, sz, d, C.c_uint64, _dp)
            self._mtn = _sig(L, "fr_mt19937_64_nth", C.c_uint64, C.c_uint64, C.c_uint64)
            self._eld = _sig(L, "fr_eval_legendre_direct", i, sz, _dp, sz, _dp, _dp)
            self._ecd = _sig(L, "fr_eval_chebyshev_direct", i, sz, _dp, sz, _dp, _dp)
            self._ccl = _sig(L, "fr_cheb_coeffs_of_legendre", i, sz, sz, _dp)
            self._mtt = _sig(L, "fr_min_taylor_terms", i, i, d, C.POINTER(C.c_int))
            self._ttb = _sig(L, "fr_taylor_term_bound", d, i, i)
            self._eb = _sig(L, "fr_ndct_error_bound", d, sz, i, i, _dp, _dp)
            self._entry = _sig(L, "fr_leg2cheb_entry", d, sz, sz, sz)
        else:
            self._trigs = [_sig(L, "fo_" + nm, i, sz, i, _dp, _dp) for nm in
                           ("dct_iii", "dst_iii", "dct_iii_transpose", "dst_iii_transpose")]
            self._ndf = _sig(L, "fo_ndct_apply", i, sz, i, i, _dp, _dp, _dp)
            self._ndt = _sig(L, "fo_ndct_apply_transpose", i, sz, i, i, _dp, _dp, _dp)
            self._l2f = _sig(L, "fo_leg2cheb_apply", i, sz, _dp, sz, _dp, _dp)
            self._l2t = _sig(L, "fo_leg2cheb_apply_transpose", i, sz, _dp, sz, _dp, _dp)
            self._dltg = _sig(L, "fo_dlt_grid", i, sz, i, i, _dp, _dp, _dp)
            self._idltg = _sig(L, "fo_idlt_grid", i, sz, i, i, _dp, _dp, _dp, _dp)
            self._lamt = _sig(L, "fo_lambda_table", None, sz, _dp)
            self._rnd = _sig(L, "fo_random_decaying", None, sz, d, C.c_uint64, _dp)
            self._uni = _sig(L, "fo_uniform_pm1", None, sz, C.c_uint64, _dp)
            self._mtn = _sig(L, "fo_mt19937_64_nth", C.c_uint64, C.c_uint64, C.c_uint64)
            self._eld = _sig(L, "fo_eval_legendre_direct", i, sz, _dp, sz, _dp, _dp)
            self._ecd = _sig(L, "fo_eval_chebyshev_direct", i, sz, _dp, sz, _dp, _dp)
            self._idd = _sig(L, "fo_idlt_direct", i, sz, _dp, _dp, _dp, _dp)
            self._ccl = _sig(L, "fo_cheb_coeffs_of_legendre", i, sz, sz, _dp)
            self._mtt = _sig(L, "fo_min_taylor_terms", i, i, d, C.POINTER(C.c_int))
            self._ttb = _sig(L, "fo_taylor_term_bound", d, i, i)
            self._eb = _sig(L, "fo_ndct_error_bound", d, sz, i, i, _dp, _dp)
            self._entry = _sig(L, "fo_leg2cheb_entry", d, sz, sz, _dp, sz)
            self._lr = _sig(L, "fo_lambda_ratio", i, d, _dp, sz, C.POINTER(C.c_double))
            self._refg = _sig(L, "fo_reference_grid", i, sz, i, _dp, _dp, _dp)
            self._refa = _sig(L, "fo_reference_angle", d, sz, i, sz)

    # quadrature.hpp
    def nodes_weights(self, n: int):
        th, x, w = (np.empty(n) for _ in range(3))
        _check(self._nodes(n, th, x, w), "legendre_nodes_weights")
        return th, x, w

    # trig.hpp; op 0 dct_iii, 1 dst_iii, 2 dct_iii_transpose, 3 dst_iii_transpose
    def trig(self, op: int, v, kind: int) -> np.ndarray:
        v = _f64(v)
        out = np.empty(len(v))
        if self.is_ref:
            _check(self._trig(op, len(v), kind, v, out), "trig")
        else:
            _check(self._trigs[op](len(v), kind, v, out), "trig")
        return out

    # ndct.hpp
    def ndct(self, v, kind: int, num_terms: int, delta, transpose: bool = False) -> np.ndarray:
        v, delta = _f64(v), _f64(delta)
        out = np.empty(len(v))
        if self.is_ref:
            _check(self._ndct(int(transpose), len(v), kind, num_terms, delta, v, out), "ndct")
        else:
            fn = self._ndt if transpose else self._ndf
            _check(fn(len(v), kind, num_terms, delta, v, out), "ndct")
        return out

    def min_taylor_terms(self, kind: int, tol: float) -> int:
        t = C.c_int(0)
        _check(self._mtt(kind, tol, C.byref(t)), "min_taylor_terms")
        return t.value

    def taylor_term_bound(self, kind: int, terms: int) -> float:
        return self._ttb(kind, terms)

    def ndct_error_bound(self, c, kind: int, num_terms: int, delta) -> float:
        c, delta = _f64(c), _f64(delta)
        return self._eb(len(c), kind, num_terms, delta, c)

    # conversion.hpp
    def lambda_table(self, max_index: int) -> np.ndarray:
        t = np.empty(max_index + 1)
        if self.is_ref:
            _check(self._lam(max_index, t), "lambda")
        else:
            self._lamt(max_index, t)
        return t

    def leg2cheb_entry(self, k: int, n: int, max_index: int) -> float:
        if self.is_ref:
            return self._entry(k, n, max_index)
        return self._entry(k, n, self.lambda_table(max_index), max_index)

    def leg2cheb(self, v, transpose: bool = False) -> np.ndarray:
        v = _f64(v)
        n = len(v)
        out = np.empty(n)
        if self.is_ref:
            _check(self._l2c(int(transpose), n, v, out), "leg2cheb")
        else:
            t = self.lambda_table(max(n - 1, 0))
            fn = self._l2t if transpose else self._l2f
            _check(fn(n, t, max(n - 1, 0), v, out), "leg2cheb")
        return out

    # transforms.hpp with an injected grid
    def dlt_grid(self, c, kind: int, tol: float, theta, x, w) -> np.ndarray:
        c = _f64(c)
        n = len(c)
        f = np.empty(n)
        if self.is_ref:
            _check(self._dlt(n, kind, tol, _f64(theta), _f64(x), _f64(w), c, f), "dlt")
        else:
            L = self.min_taylor_terms(kind, tol)
            delta = self.reference_delta(n, kind, theta)
            _check(self._dltg(n, kind, L, delta, c, f), "dlt")
        return f

    def idlt_grid(self, f, kind: int, tol: float, theta, x, w) -> np.ndarray:
        f = _f64(f)
        n = len(f)
        c = np.empty(n)
        if self.is_ref:
            _check(self._idlt(n, kind, tol, _f64(theta), _f64(x), _f64(w), f, c), "idlt")
        else:
            L = self.min_taylor_terms(kind, tol)
            delta = self.reference_delta(n, kind, theta)
            _check(self._idltg(n, kind, L, delta, _f64(w), f, c), "idlt")
        return c

    def reference_delta(self, n: int, kind: int, theta) -> np.ndarray:
        """delta_theta of quadrature.hpp:147-158 (restatement only)."""
        if self.is_ref:
            return _ORACLE_C.reference_delta(n, kind, theta)
        ts, d = np.empty(n), np.empty(n)
        _check(self._refg(n, kind, _f64(theta), ts, d), "reference_grid")
        return d

    # oracle.hpp
    def eval_legendre_direct(self, c, xs) -> np.ndarray:
        c, xs = _f64(c), _f64(xs)
        out = np.empty(len(xs))
        _check(self._eld(len(c), c, len(xs), xs, out), "eval_legendre_direct")
        return out

    def eval_chebyshev_direct(self, c, xs) -> np.ndarray:
        c, xs = _f64(c), _f64(xs)
        out = np.empty(len(xs))
        _check(self._ecd(len(c), c, len(xs), xs, out), "eval_chebyshev_direct")
        return out

    def cheb_coeffs_of_legendre(self, n: int, m: int) -> np.ndarray:
        out = np.empty(n + 1)
        _check(self._ccl(n, m, out), "cheb_coeffs_of_legendre")
        return out

    # random.hpp
    def random_decaying(self, n: int, decay: float, seed: int) -> np.ndarray:
        out = np.empty(n)
        self._rnd(n, decay, seed, out)
        return out

    def mt19937_64_nth(self, seed: int, count: int) -> int:
        return int(self._mtn(seed, count))


ORACLE = _Oracle(_lib, False) if _lib is not None else None
_ORACLE_C = ORACLE
REF = _Oracle(_ref, True) if _ref is not None else None


def uniform_pm1(n: int, seed: int) -> np.ndarray:
    out = np.empty(n)
    ORACLE._uni(n, seed, out)
    return out


def idlt_direct(f, x, w) -> np.ndarray:
    f = _f64(f)
    out = np.empty(len(f))
    _check(ORACLE._idd(len(f), f, _f64(x), _f64(w), out), "idlt_direct")
    return out


def lambda_ratio(z: float, max_index: int) -> float:
    t = ORACLE.lambda_table(max_index)
    out = C.c_double(0)
    _check(ORACLE._lr(z, t, max_index, C.byref(out)), "lambda_ratio")
    return out.value
