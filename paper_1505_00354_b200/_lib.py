"""ctypes binding of libfastleg_b200.so (the C ABI in include/fastleg_b200.h).

The library is the product: there is no Python or CPU fallback. Importing
this module without the built .so raises; calling a compute entry point
without a CUDA device returns FL_CUDA_ERROR, raised here as
``FastlegCudaError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLB_LIB_PATH") or os.path.join(HERE, "libfastleg_b200.so")

FL_OK, FL_INVALID_ARGUMENT, FL_DOMAIN_ERROR, FL_OVERFLOW_ERROR, FL_RUNTIME_ERROR, FL_CUDA_ERROR = range(6)
CHEB1, CHEBSTAR = 0, 1
DCT_III, DST_III, DCT_III_T, DST_III_T = range(4)
NDCT_LITERAL, NDCT_FAST = 0, 1
LEG2CHEB_DIRECT, LEG2CHEB_FAST, LEG2CHEB_ASYMPTOTIC, LEG2CHEB_TOEPLITZ = 0, 1, 2, 3
GEMM_FP64, GEMM_INT8_SPLIT = 0, 1
DLT_FACTORED, DLT_DIRECT = 0, 1


class FastlegError(Exception):
    """Base of the errors raised through the C ABI."""


class InvalidArgument(FastlegError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(FastlegError, ValueError):
    """std::domain_error in the reference."""


class OverflowErrorFL(FastlegError, OverflowError):
    """std::overflow_error in the reference."""


class RuntimeErrorFL(FastlegError, RuntimeError):
    """std::runtime_error in the reference."""


class FastlegCudaError(FastlegError, RuntimeError):
    """CUDA failure or no device (no CPU fallback exists)."""


_EXC = {
    FL_INVALID_ARGUMENT: InvalidArgument,
    FL_DOMAIN_ERROR: DomainError,
    FL_OVERFLOW_ERROR: OverflowErrorFL,
    FL_RUNTIME_ERROR: RuntimeErrorFL,
    FL_CUDA_ERROR: FastlegCudaError,
}

# every symbol include/fastleg_b200.h declares
EXPORTS = [
    "fl_last_error", "fl_device_available", "fl_nodes_weights", "fl_reference_grid",
    "fl_lambda_table", "fl_trig", "fl_ndct", "fl_ndct_error_bound", "fl_leg2cheb", "fl_plan_create",
    "fl_plan_create_from_grid", "fl_plan_destroy", "fl_plan_size", "fl_plan_kind",
    "fl_plan_tolerance", "fl_plan_num_terms", "fl_plan_grid", "fl_plan_reference",
    "fl_plan_lambda", "fl_dlt", "fl_idlt", "fl_plan_set_ndct_mode", "fl_plan_ndct_mode",
    "fl_random_decaying", "fl_random_uniform_pm1", "fl_kernel_launch_count",
    "fl_eval_legendre_direct", "fl_eval_chebyshev_direct", "fl_idlt_direct",
    "fl_cheb_coeffs_of_legendre", "fl_plan_set_leg2cheb_mode", "fl_plan_leg2cheb_rank",
    "fl_plan_stage_terms", "fl_dlt_stage", "fl_plan_set_gemm_mode", "fl_plan_gemm_mode",
    "fl_plan_leg2cheb", "fl_plan_ndct", "fl_plan_ndct_terms", "fl_set_free_ndct_mode",
    "fl_free_ndct_mode", "fl_plan_set_dlt_method", "fl_plan_dlt_method", "fl_plan_uses_direct",
    "fl_load_vector", "fl_save_vector", "fl_plan_leg2cheb_asy_info", "fl_plan_stage_cost",
    "fl_fs_create", "fl_fs_destroy", "fl_fs_info", "fl_fs_coef_count", "fl_fs_work_elems",
    "fl_fs_to_residue", "fl_fs_from_residue", "fl_fs_values", "fl_fs_ndct_part", "fl_fs_check",
]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, sz, i, d, dp, u64 = C.c_void_p, C.c_size_t, C.c_int, C.c_double, C.c_void_p, C.c_uint64
    sigs = {
        "fl_last_error": (C.c_char_p, []),
        "fl_device_available": (i, []),
        "fl_nodes_weights": (i, [sz, dp, dp, dp, vp]),
        "fl_reference_grid": (i, [sz, i, dp, dp, dp, vp]),
        "fl_lambda_table": (i, [sz, dp, vp]),
        "fl_trig": (i, [i, i, sz, dp, dp, sz, sz, vp]),
        "fl_ndct": (i, [i, i, sz, i, dp, dp, dp, sz, sz, vp]),
        "fl_ndct_error_bound": (i, [sz, i, i, dp, sz, dp, sz, C.POINTER(d), vp]),
        "fl_leg2cheb": (i, [i, sz, dp, sz, dp, dp, sz, sz, vp]),
        "fl_plan_create": (i, [sz, d, i, C.POINTER(vp)]),
        "fl_plan_create_from_grid": (i, [sz, d, i, dp, dp, dp, C.POINTER(vp)]),
        "fl_plan_destroy": (i, [vp]),
        "fl_plan_size": (sz, [vp]),
        "fl_plan_kind": (i, [vp]),
        "fl_plan_tolerance": (d, [vp]),
        "fl_plan_num_terms": (i, [vp]),
        "fl_plan_grid": (i, [vp, dp, dp, dp]),
        "fl_plan_reference": (i, [vp, dp, dp]),
        "fl_plan_lambda": (i, [vp, dp]),
        "fl_dlt": (i, [vp, dp, dp, sz, sz, vp]),
        "fl_idlt": (i, [vp, dp, dp, sz, sz, vp]),
        "fl_plan_set_ndct_mode": (i, [vp, i]),
        "fl_plan_ndct_mode": (i, [vp]),
        "fl_random_decaying": (None, [sz, d, u64, dp, sz, i]),
        "fl_random_uniform_pm1": (None, [sz, u64, dp, sz, i]),
        "fl_kernel_launch_count": (u64, []),
        "fl_eval_legendre_direct": (i, [dp, sz, dp, sz, dp, vp]),
        "fl_eval_chebyshev_direct": (i, [dp, sz, dp, sz, dp, vp]),
        "fl_idlt_direct": (i, [dp, sz, dp, dp, dp, vp]),
        "fl_cheb_coeffs_of_legendre": (i, [sz, sz, dp, vp]),
        "fl_plan_set_leg2cheb_mode": (i, [vp, i]),
        "fl_plan_leg2cheb_rank": (i, [vp, i]),
        "fl_plan_stage_terms": (i, [vp, i, C.POINTER(i)]),
        "fl_dlt_stage": (i, [vp, i, i, i, i, dp, dp, vp]),
        "fl_plan_set_gemm_mode": (i, [vp, i]),
        "fl_plan_gemm_mode": (i, [vp]),
        "fl_plan_leg2cheb": (i, [vp, i, dp, dp, sz, sz, vp]),
        "fl_plan_ndct": (i, [vp, i, dp, dp, sz, sz, vp]),
        "fl_plan_ndct_terms": (i, [vp]),
        "fl_set_free_ndct_mode": (i, [i]),
        "fl_free_ndct_mode": (i, []),
        "fl_plan_set_dlt_method": (i, [vp, i]),
        "fl_plan_dlt_method": (i, [vp]),
        "fl_plan_uses_direct": (i, [vp, sz]),
        "fl_load_vector": (i, [C.c_char_p, i, dp, sz, C.POINTER(sz), vp]),
        "fl_save_vector": (i, [C.c_char_p, i, dp, sz, vp]),
        "fl_plan_leg2cheb_asy_info": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(d)]),
        "fl_plan_stage_cost": (i, [vp, i, i, C.POINTER(d)]),
        "fl_fs_create": (i, [vp, i, i, C.POINTER(vp)]),
        "fl_fs_destroy": (i, [vp]),
        "fl_fs_info": (i, [vp, C.POINTER(sz)]),
        "fl_fs_coef_count": (i, [vp, i, i, i, C.POINTER(sz)]),
        "fl_fs_work_elems": (sz, [vp, i]),
        "fl_fs_to_residue": (i, [vp, dp, dp, vp]),
        "fl_fs_from_residue": (i, [vp, dp, dp, vp]),
        "fl_fs_values": (i, [vp, i, dp, dp, vp]),
        "fl_fs_ndct_part": (i, [vp, i, i, i, i, vp, vp, vp, i, vp]),
        "fl_fs_check": (i, [vp, i, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def check(status: int) -> None:
    if status != FL_OK:
        msg = LIB.fl_last_error().decode()
        raise _EXC.get(status, FastlegError)(msg)


def device_available() -> bool:
    return bool(LIB.fl_device_available())


def set_free_ndct_mode(mode: int) -> None:
    """NDCT_FAST (default) or NDCT_LITERAL for the free functions ndct_apply /
    ndct_apply_transpose and the chebstar dct_iii / dst_iii / transposes
    (include/fastleg_b200.h, fl_set_free_ndct_mode)."""
    check(LIB.fl_set_free_ndct_mode(int(mode)))


def free_ndct_mode() -> int:
    return int(LIB.fl_free_ndct_mode())


def launch_count() -> int:
    return int(LIB.fl_kernel_launch_count())
