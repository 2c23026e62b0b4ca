"""Python mirror of the reference header API (proj/include/fastleg/*.hpp) over
the C ABI of libfastleg_b200.

Names, argument meaning, validation order and error types follow the
reference (each function cites the reference file:line it stands in for).
Values may be

* NumPy arrays / sequences (host; shape (n,) = the reference call, or
  (batch, n) = `batch` independent columns), staged through device memory by
  the library, or
* CUDA ``torch.Tensor`` s of dtype float64 and shape (n,) or (batch, n)
  (device-resident, zero-copy, on torch's current stream).

Everything numeric runs in the CUDA library; the scalar helpers
(reference_angle, taylor_term_bound, min_taylor_terms, lambda_ratio,
leg2cheb_entry) are host arithmetic exactly as in the reference headers.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np

from . import _lib
from ._lib import LIB, check

default_tolerance = 2.0 ** -52  # types.hpp:8
max_taylor_terms = 30           # ndct.hpp:46
_PI = 3.14159265358979323846264338327950288  # types.hpp:36


class GridKind(enum.IntEnum):  # types.hpp:14
    cheb1 = _lib.CHEB1
    chebstar = _lib.CHEBSTAR


class Basis(enum.IntEnum):  # types.hpp:16
    legendre = 0
    chebyshev = 1


@dataclass
class CoefficientVector:  # types.hpp:19-24
    basis: Basis = Basis.legendre
    values: Any = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return _ncols_n(self.values)[1]


def legendre_coefficients(values) -> CoefficientVector:  # types.hpp:26-28
    return CoefficientVector(Basis.legendre, values)


def chebyshev_coefficients(values) -> CoefficientVector:  # types.hpp:30-32
    return CoefficientVector(Basis.chebyshev, values)


@dataclass
class LegendreGrid:  # quadrature.hpp:16-21
    size: int = 0
    theta: Any = None
    x: Any = None
    weights: Any = None


@dataclass
class ReferenceGrid:  # quadrature.hpp:25-30
    size: int = 0
    kind: GridKind = GridKind.chebstar
    theta_star: Any = None
    delta_theta: Any = None


@dataclass
class TaylorPlan:  # ndct.hpp:27-33
    size: int = 0
    kind: GridKind = GridKind.chebstar
    tolerance: float = 0.0
    num_terms: int = 0
    reference: ReferenceGrid = field(default_factory=ReferenceGrid)


# ---------------------------------------------------------------------------
# array plumbing
# ---------------------------------------------------------------------------

def _is_torch_cuda(a) -> bool:
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _ncols_n(a) -> tuple[int, int]:
    shape = tuple(a.shape) if hasattr(a, "shape") else (len(a),)
    if len(shape) == 1:
        return 1, shape[0]
    if len(shape) == 2:
        return shape[0], shape[1]
    raise _lib.InvalidArgument("fastleg: expected a 1-D vector or a (batch, n) block")


class _Arr:
    """A host (NumPy) or device (torch) float64 block and its raw pointer."""

    def __init__(self, a, *, out_like: "_Arr | None" = None, shape=None):
        if out_like is not None:
            if out_like.device:
                import torch
                self.obj = torch.empty(shape, dtype=torch.float64, device=out_like.obj.device)
            else:
                self.obj = np.empty(shape, dtype=np.float64)
        elif _is_torch_cuda(a):
            import torch
            if a.dtype != torch.float64:
                raise _lib.InvalidArgument("fastleg: device tensors must be float64")
            self.obj = a.contiguous()
        else:
            self.obj = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        self.device = _is_torch_cuda(self.obj)

    @property
    def ptr(self) -> int:
        if self.device:
            return self.obj.data_ptr()
        return self.obj.ctypes.data

    @property
    def n(self) -> int:
        """Number of elements."""
        return int(self.obj.numel()) if self.device else int(self.obj.size)

    @property
    def stream(self):
        if self.device:
            import torch
            return C.c_void_p(torch.cuda.current_stream(self.obj.device).cuda_stream)
        return None


def _vp(p: int) -> C.c_void_p:
    return C.c_void_p(p)


def _host(a) -> np.ndarray:
    if _is_torch_cuda(a):
        return a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------------
# quadrature.hpp
# ---------------------------------------------------------------------------

def reference_angle(n: int, kind: GridKind, k: int) -> float:  # quadrature.hpp:32-36
    if kind == GridKind.cheb1:
        return (float(k) + 0.5) * _PI / float(n)
    return (float(k) + 0.75) * _PI / (float(n) + 0.5)


def legendre_nodes_weights(n: int, device=None) -> LegendreGrid:  # quadrature.hpp:76-143
    """Gauss-Legendre grid from the one-thread-per-node kernel. ``device`` =
    a torch device to keep the grid resident there (else NumPy arrays)."""
    if device is not None:
        import torch
        th, x, w = (torch.empty(max(n, 1), dtype=torch.float64, device=device) for _ in range(3))
        check(LIB.fl_nodes_weights(n, _vp(th.data_ptr()), _vp(x.data_ptr()), _vp(w.data_ptr()),
                                   _vp(torch.cuda.current_stream(device).cuda_stream)))
        return LegendreGrid(n, th[:n], x[:n], w[:n])
    th, x, w = (np.empty(max(n, 1)) for _ in range(3))
    check(LIB.fl_nodes_weights(n, _vp(th.ctypes.data), _vp(x.ctypes.data), _vp(w.ctypes.data), None))
    return LegendreGrid(n, th[:n], x[:n], w[:n])


def reference_grid(grid: LegendreGrid, kind: GridKind) -> ReferenceGrid:  # quadrature.hpp:147-158
    th = _Arr(grid.theta)
    n = grid.size
    ts = _Arr(None, out_like=th, shape=(n,))
    dl = _Arr(None, out_like=th, shape=(n,))
    check(LIB.fl_reference_grid(n, int(kind), _vp(th.ptr), _vp(ts.ptr), _vp(dl.ptr), th.stream))
    return ReferenceGrid(n, GridKind(kind), ts.obj, dl.obj)


# ---------------------------------------------------------------------------
# trig.hpp
# ---------------------------------------------------------------------------

def _trig(op: int, c, kind: GridKind):
    a = _Arr(c)
    batch, n = _ncols_n(a.obj)
    out = _Arr(None, out_like=a, shape=a.obj.shape)
    check(LIB.fl_trig(op, int(kind), n, _vp(a.ptr), _vp(out.ptr), batch, n, a.stream))
    return out.obj


def dct_iii(c, kind: GridKind):  # trig.hpp:55-74
    return _trig(_lib.DCT_III, c, kind)


def dst_iii(c, kind: GridKind):  # trig.hpp:76-95
    return _trig(_lib.DST_III, c, kind)


def dct_iii_transpose(g, kind: GridKind):  # trig.hpp:100-116
    return _trig(_lib.DCT_III_T, g, kind)


def dst_iii_transpose(g, kind: GridKind):  # trig.hpp:118-136
    return _trig(_lib.DST_III_T, g, kind)


# ---------------------------------------------------------------------------
# ndct.hpp
# ---------------------------------------------------------------------------

def _q(kind: GridKind) -> float:
    return 0.83845 if kind == GridKind.cheb1 else 1.0 / (6.0 * _PI)


def taylor_term_bound(kind: GridKind, num_terms: int) -> float:  # ndct.hpp:38-44
    if num_terms < 0:
        raise _lib.InvalidArgument("taylor_term_bound: negative term count")
    q, b = _q(kind), 1.0
    for l in range(1, num_terms + 1):
        b *= q / float(l)
    return b


def min_taylor_terms(kind: GridKind, tolerance: float) -> int:  # ndct.hpp:49-59
    if not (tolerance > 0.0 and tolerance < 1.0):
        raise _lib.InvalidArgument("min_taylor_terms: tolerance must lie in (0, 1)")
    q, b = _q(kind), 1.0
    for l in range(1, max_taylor_terms + 1):
        b *= q / float(l)
        if b <= tolerance:
            return l
    raise _lib.DomainError("min_taylor_terms: tolerance unattainable with <= 30 terms")


def plan_ndct(grid_or_n, kind: GridKind, tolerance: float) -> TaylorPlan:  # ndct.hpp:61-73
    grid = grid_or_n if isinstance(grid_or_n, LegendreGrid) else legendre_nodes_weights(int(grid_or_n))
    plan = TaylorPlan(grid.size, GridKind(kind), tolerance, min_taylor_terms(kind, tolerance))
    plan.reference = reference_grid(grid, kind)
    return plan


def _ndct(plan: TaylorPlan, v, transpose: int, where: str):
    a = _Arr(v)
    batch, n = _ncols_n(a.obj)
    if n != plan.size:  # ndct.hpp:81-82
        raise _lib.InvalidArgument(f"{where}: input size does not match plan")
    delta = _Arr(plan.reference.delta_theta if a.device or not _is_torch_cuda(plan.reference.delta_theta)
                 else _host(plan.reference.delta_theta))
    if a.device and not delta.device:
        import torch
        delta = _Arr(torch.as_tensor(delta.obj, device=a.obj.device))
    out = _Arr(None, out_like=a, shape=a.obj.shape)
    check(LIB.fl_ndct(transpose, int(plan.kind), n, int(plan.num_terms), _vp(delta.ptr),
                      _vp(a.ptr), _vp(out.ptr), batch, n, a.stream))
    return out.obj


def ndct_apply(plan: TaylorPlan, coeffs):  # ndct.hpp:98-117
    return _ndct(plan, coeffs, 0, "ndct_apply")


def ndct_apply_transpose(plan: TaylorPlan, values):  # ndct.hpp:121-143
    return _ndct(plan, values, 1, "ndct_apply_transpose")


def ndct_error_bound(plan: TaylorPlan, coeffs) -> float:  # ndct.hpp:147-155
    """Certified bound; the O(N) reductions (max |delta|, ||c||_1) run on the
    device through the batched ndct entry's error-bound helper."""
    d = _Arr(plan.reference.delta_theta)
    c = _Arr(coeffs)
    out = C.c_double(0.0)
    check(LIB.fl_ndct_error_bound(int(plan.size), int(plan.kind), int(plan.num_terms), _vp(d.ptr),
                                  d.n, _vp(c.ptr), c.n, C.byref(out), c.stream or d.stream))
    return out.value


# ---------------------------------------------------------------------------
# conversion.hpp
# ---------------------------------------------------------------------------

class LambdaCache:  # conversion.hpp:23-37
    """Lambda(z) = Gamma(z+1/2)/Gamma(z+1), z = 0..max_index, built on the device."""

    def __init__(self, max_index: int):
        self._t = np.empty(max_index + 1)
        check(LIB.fl_lambda_table(max_index, _vp(self._t.ctypes.data), None))

    def __getitem__(self, z: int) -> float:
        return float(self._t[z])

    def max_index(self) -> int:
        return len(self._t) - 1

    @property
    def table(self) -> np.ndarray:
        return self._t


def _lambda_asymptotic(z: float) -> float:  # conversion.hpp:43-56
    k = [-1 / 8, 1 / 128, 5 / 1024, -21 / 32768, -399 / 262144, 869 / 4194304, 39325 / 33554432,
         -334477 / 2147483648]
    r = 1.0 / z
    s = k[7]
    for c in reversed(k[:7]):
        s = c + r * s
    return (1.0 + r * s) / math.sqrt(z)


def lambda_ratio(z: float, cache: LambdaCache) -> float:  # conversion.hpp:63-73
    if not (z >= 0.0):
        raise _lib.DomainError("lambda_ratio: argument must be non-negative")
    zf = math.floor(z)
    if z == zf and zf <= cache.max_index():
        return cache[int(zf)]
    if z >= 30.0:
        return _lambda_asymptotic(z)
    frac = z - zf
    value = math.exp(math.lgamma(frac + 0.5) - math.lgamma(frac + 1.0))
    w = frac
    while w < z - 0.5:
        value *= (w + 0.5) / (w + 1.0)
        w += 1.0
    return value


def leg2cheb_entry(k: int, n: int, cache: LambdaCache) -> float:  # conversion.hpp:76-81
    if k > n or (k + n) % 2 != 0:
        return 0.0
    pref = (1.0 if k == 0 else 2.0) / _PI
    return pref * lambda_ratio(float((n - k) // 2), cache) * lambda_ratio(float((n + k) // 2), cache)


def _l2c(v, cache: LambdaCache | None, transpose: int):
    a = _Arr(v)
    batch, n = _ncols_n(a.obj)
    if cache is None:
        cache = LambdaCache(n - 1 if n else 0)
    t = cache.table
    out = _Arr(None, out_like=a, shape=a.obj.shape)
    check(LIB.fl_leg2cheb(transpose, n, _vp(t.ctypes.data), len(t), _vp(a.ptr), _vp(out.ptr), batch,
                          n, a.stream))
    return out.obj


def leg2cheb_apply(c: CoefficientVector, cache: LambdaCache | None = None) -> CoefficientVector:
    """conversion.hpp:100-118"""
    if c.basis != Basis.legendre:
        raise _lib.InvalidArgument("leg2cheb_apply: expected Legendre coefficients")
    return chebyshev_coefficients(_l2c(c.values, cache, 0))


def leg2cheb_apply_transpose(v, cache: LambdaCache | None = None):  # conversion.hpp:121-140
    return _l2c(v, cache, 1)


# ---------------------------------------------------------------------------
# transforms.hpp
# ---------------------------------------------------------------------------

class TransformConfig:  # transforms.hpp:19-38
    """Immutable per-size bundle: device-resident grid, NDCT plan, Lambda table."""

    def __init__(self, n: int, tolerance: float = default_tolerance, kind: GridKind = GridKind.chebstar,
                 *, grid: LegendreGrid | None = None, ndct_mode: int | None = None):
        h = C.c_void_p()
        if grid is None:
            check(LIB.fl_plan_create(n, tolerance, int(kind), C.byref(h)))
        else:
            th, x, w = (_Arr(a) for a in (grid.theta, grid.x, grid.weights))
            check(LIB.fl_plan_create_from_grid(n, tolerance, int(kind), _vp(th.ptr), _vp(x.ptr),
                                               _vp(w.ptr), C.byref(h)))
        self._h = h
        if ndct_mode is not None:
            check(LIB.fl_plan_set_ndct_mode(h, int(ndct_mode)))
        self._grid = None
        self._plan = None
        self._lambda = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            LIB.fl_plan_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def size(self) -> int:
        return int(LIB.fl_plan_size(self._h))

    def kind(self) -> GridKind:
        return GridKind(LIB.fl_plan_kind(self._h))

    def tolerance(self) -> float:
        return float(LIB.fl_plan_tolerance(self._h))

    def ndct_mode(self) -> int:
        return int(LIB.fl_plan_ndct_mode(self._h))

    def set_ndct_mode(self, mode: int) -> None:
        check(LIB.fl_plan_set_ndct_mode(self._h, int(mode)))

    def set_leg2cheb_mode(self, mode: int) -> None:
        """LEG2CHEB_DIRECT (reference O(N^2) product), LEG2CHEB_FAST (default:
        the asymptotic expansion for power-of-two n >= 2^16, else
        Toeplitz-Hankel), LEG2CHEB_TOEPLITZ (Toeplitz-Hankel, n >= 2^14) or
        LEG2CHEB_ASYMPTOTIC (Hale-Townsend asymptotic expansion, power-of-two
        n in [2^10, 2^26]); the fast modes apply to <= 16 columns."""
        check(LIB.fl_plan_set_leg2cheb_mode(self._h, int(mode)))

    def leg2cheb_rank(self, parity: int = 0) -> int:
        return int(LIB.fl_plan_leg2cheb_rank(self._h, int(parity)))

    def leg2cheb_asy_info(self) -> dict:
        """The asymptotic conversion's shape: expansion terms M, levels,
        length-N transforms per column, recurrence (point, degree) steps / N."""
        m, lv, tr = C.c_int(), C.c_int(), C.c_int()
        st = C.c_double()
        check(LIB.fl_plan_leg2cheb_asy_info(self._h, C.byref(m), C.byref(lv), C.byref(tr), C.byref(st)))
        return {"terms": m.value, "levels": lv.value, "transforms": tr.value,
                "recurrence_steps_per_n": st.value}

    def set_gemm_mode(self, mode: int) -> None:
        """GEMM_INT8_SPLIT (default: exact split-integer conversion product on
        the int8 tensor cores, n % 256 == 0, 512 <= n <= 16384, > 16 columns)
        or GEMM_FP64 (fp64 tensor cores)."""
        check(LIB.fl_plan_set_gemm_mode(self._h, int(mode)))

    def gemm_mode(self) -> int:
        return int(LIB.fl_plan_gemm_mode(self._h))

    def set_dlt_method(self, method: int) -> None:
        """DLT_DIRECT (default: one dense split-int8 product per parity,
        f = P c, for n % 256 == 0, 512 <= n <= 8192, > 16 columns) or
        DLT_FACTORED (the reference's conversion + NDCT)."""
        check(LIB.fl_plan_set_dlt_method(self._h, int(method)))

    def dlt_method(self) -> int:
        return int(LIB.fl_plan_dlt_method(self._h))

    def uses_direct(self, batch: int) -> bool:
        return bool(LIB.fl_plan_uses_direct(self._h, int(batch)))

    def grid(self) -> LegendreGrid:
        if self._grid is None:
            n = self.size()
            th, x, w = (np.empty(n) for _ in range(3))
            check(LIB.fl_plan_grid(self._h, _vp(th.ctypes.data), _vp(x.ctypes.data), _vp(w.ctypes.data)))
            self._grid = LegendreGrid(n, th, x, w)
        return self._grid

    def plan(self) -> TaylorPlan:
        if self._plan is None:
            n = self.size()
            ts, dl = np.empty(n), np.empty(n)
            check(LIB.fl_plan_reference(self._h, _vp(ts.ctypes.data), _vp(dl.ctypes.data)))
            self._plan = TaylorPlan(n, self.kind(), self.tolerance(), int(LIB.fl_plan_num_terms(self._h)),
                                    ReferenceGrid(n, self.kind(), ts, dl))
        return self._plan

    def lambda_(self) -> LambdaCache:
        if self._lambda is None:
            self._lambda = LambdaCache(max(self.size() - 1, 0))
        return self._lambda

    def _stage(self, fn, x, transpose: int):
        a = _Arr(x)
        batch, n = _ncols_n(a.obj)
        if n != self.size():
            raise _lib.InvalidArgument("fastleg: input size does not match config")
        out = _Arr(None, out_like=a, shape=a.obj.shape)
        check(fn(self._h, int(transpose), _vp(a.ptr), _vp(out.ptr), batch, n, a.stream))
        return out.obj

    def convert(self, x, transpose: bool = False):
        """The plan's conversion step exactly as dlt / idlt run it
        (fl_plan_leg2cheb): M x (transforms.hpp:47), or (m + 1/2) M^T x
        (the last step of transforms.hpp:62) with transpose=True."""
        return self._stage(LIB.fl_plan_leg2cheb, x, int(transpose))

    def ndct(self, x, transpose: bool = False):
        """The plan's NDCT step exactly as dlt / idlt run it (fl_plan_ndct,
        same fast / literal mode): NDCT(x) (transforms.hpp:48), or the
        unweighted NDCT^T(x) of transforms.hpp:60 with transpose=True."""
        return self._stage(LIB.fl_plan_ndct, x, int(transpose))


def dlt(c: CoefficientVector | Any, config: TransformConfig):  # transforms.hpp:42-49
    if isinstance(c, CoefficientVector):
        if c.basis != Basis.legendre:
            raise _lib.InvalidArgument("dlt: expected Legendre coefficients")
        c = c.values
    a = _Arr(c)
    batch, n = _ncols_n(a.obj)
    if n != config.size():
        raise _lib.InvalidArgument("dlt: coefficient size does not match config")
    out = _Arr(None, out_like=a, shape=a.obj.shape)
    check(LIB.fl_dlt(config.handle, _vp(a.ptr), _vp(out.ptr), batch, n, a.stream))
    return out.obj


def idlt(f, config: TransformConfig) -> CoefficientVector:  # transforms.hpp:54-64
    a = _Arr(f)
    batch, n = _ncols_n(a.obj)
    if n != config.size():
        raise _lib.InvalidArgument("idlt: value size does not match config")
    out = _Arr(None, out_like=a, shape=a.obj.shape)
    check(LIB.fl_idlt(config.handle, _vp(a.ptr), _vp(out.ptr), batch, n, a.stream))
    return legendre_coefficients(out.obj)


# ---------------------------------------------------------------------------
# oracle.hpp (direct O(N^2) evaluations, as device kernels)
# ---------------------------------------------------------------------------

def _direct_eval(c: CoefficientVector, xs, chebyshev: int, where: str):
    want = Basis.chebyshev if chebyshev else Basis.legendre
    if c.basis != want:
        raise _lib.InvalidArgument(f"{where}: expected {want.name.capitalize()} coefficients")
    cv, x = _Arr(c.values), _Arr(xs)
    n, m = _ncols_n(cv.obj)[1], _ncols_n(x.obj)[1]
    out = _Arr(None, out_like=x, shape=(m,))
    fn = LIB.fl_eval_chebyshev_direct if chebyshev else LIB.fl_eval_legendre_direct
    check(fn(_vp(cv.ptr), n, _vp(x.ptr), m, _vp(out.ptr), x.stream))
    return out.obj


def eval_legendre_direct(c: CoefficientVector, xs):  # oracle.hpp:19-48
    return _direct_eval(c, xs, 0, "eval_legendre_direct")


def eval_chebyshev_direct(c: CoefficientVector, xs):  # oracle.hpp:52-79
    return _direct_eval(c, xs, 1, "eval_chebyshev_direct")


def idlt_direct(f, grid: LegendreGrid) -> CoefficientVector:  # oracle.hpp:84-116
    a = _Arr(f)
    n = _ncols_n(a.obj)[1]
    if n != grid.size:
        raise _lib.InvalidArgument("idlt_direct: value/grid size mismatch")
    x, w = _Arr(grid.x), _Arr(grid.weights)
    out = _Arr(None, out_like=a, shape=(n,))
    check(LIB.fl_idlt_direct(_vp(a.ptr), n, _vp(x.ptr), _vp(w.ptr), _vp(out.ptr), a.stream))
    return legendre_coefficients(out.obj)


def cheb_coeffs_of_legendre(n: int, m: int) -> np.ndarray:  # oracle.hpp:122-153
    out = np.empty(n + 1)
    check(LIB.fl_cheb_coeffs_of_legendre(n, m, _vp(out.ctypes.data), None))
    return out


# ---------------------------------------------------------------------------
# random.hpp (host input generators)
# ---------------------------------------------------------------------------

def random_decaying(n: int, decay: float, seed: int, batch: int = 1, threads: int = 0) -> np.ndarray:
    """random.hpp:45-55; column j of a batch uses seed + j."""
    out = np.empty((batch, n)) if batch > 1 else np.empty(n)
    LIB.fl_random_decaying(n, decay, seed, _vp(out.ctypes.data), batch, threads)
    return out


def random_uniform_pm1(n: int, seed: int, batch: int = 1, threads: int = 0) -> np.ndarray:
    """SURVEY.md 8d C4 recipe: 2 * ((mt19937_64() >> 11) * 2^-53) - 1, column j seeded seed + j."""
    out = np.empty((batch, n)) if batch > 1 else np.empty(n)
    LIB.fl_random_uniform_pm1(n, seed, _vp(out.ctypes.data), batch, threads)
    return out


# ---------------------------------------------------------------------------
# vector_io.hpp, staged through pinned buffers
# ---------------------------------------------------------------------------

VECTOR_CSV, VECTOR_RAW_BINARY = 0, 1


def load_vector(path: str, fmt: int = VECTOR_RAW_BINARY, device=None):  # vector_io.hpp:66-102
    """Read a csv / FLEGVEC1 vector; ``device`` (a torch device) -> the values
    land in device memory through overlapped pinned chunks, else NumPy."""
    cnt = C.c_size_t(0)
    # first pass learns the length (capacity 0 raises invalid_argument for n > 0)
    rc = LIB.fl_load_vector(str(path).encode(), int(fmt), None, 0, C.byref(cnt), None)
    if rc not in (_lib.FL_OK, _lib.FL_INVALID_ARGUMENT):
        check(rc)
    n = cnt.value
    if device is not None:
        import torch
        out = torch.empty(max(n, 1), dtype=torch.float64, device=device)
        check(LIB.fl_load_vector(str(path).encode(), int(fmt), _vp(out.data_ptr()), n, C.byref(cnt),
                                 _vp(torch.cuda.current_stream(out.device).cuda_stream)))
        return out[:n]
    out = np.empty(max(n, 1))
    check(LIB.fl_load_vector(str(path).encode(), int(fmt), _vp(out.ctypes.data), n, C.byref(cnt), None))
    return out[:n]


def save_vector(path: str, values, fmt: int = VECTOR_RAW_BINARY) -> None:  # vector_io.hpp:49-64
    a = _Arr(values)
    check(LIB.fl_save_vector(str(path).encode(), int(fmt), _vp(a.ptr), a.n, a.stream))
