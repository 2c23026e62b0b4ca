"""fastleg-b200: B200-native fast discrete Legendre transform (DLT/IDLT).

A drop-in for the hot path of the reference ``fastleg`` library
(arXiv 1505.00354, Hale & Townsend): Gauss-Legendre nodes/weights,
Legendre->Chebyshev conversion, the Taylor-series NDCT and the fp64 DCT/DST
engine, as hand-written sm_100a CUDA kernels behind the C ABI in
``include/fastleg_b200.h``. This package is the Python mirror of the
reference's header API; ``include/fastleg/*.hpp`` is the C++ one.
"""
from ._lib import (  # noqa: F401
    DomainError, FastlegCudaError, FastlegError, InvalidArgument, OverflowErrorFL,
    RuntimeErrorFL, device_available, launch_count, set_free_ndct_mode, free_ndct_mode, NDCT_FAST,
    NDCT_LITERAL, LEG2CHEB_DIRECT, LEG2CHEB_FAST, LEG2CHEB_ASYMPTOTIC, LEG2CHEB_TOEPLITZ, GEMM_FP64, GEMM_INT8_SPLIT, DLT_FACTORED, DLT_DIRECT,
)
from .api import *  # noqa: F401,F403
from .api import (  # noqa: F401
    Basis, CoefficientVector, GridKind, LambdaCache, LegendreGrid, ReferenceGrid, TaylorPlan,
    TransformConfig, chebyshev_coefficients, dct_iii, dct_iii_transpose, default_tolerance, dlt,
    dst_iii, dst_iii_transpose, idlt, lambda_ratio, leg2cheb_apply, leg2cheb_apply_transpose,
    leg2cheb_entry, legendre_coefficients, legendre_nodes_weights, max_taylor_terms,
    min_taylor_terms, ndct_apply, ndct_apply_transpose, ndct_error_bound, plan_ndct,
    random_decaying, random_uniform_pm1, reference_angle, reference_grid, taylor_term_bound,
    eval_legendre_direct, eval_chebyshev_direct, idlt_direct, cheb_coeffs_of_legendre,
    load_vector, save_vector, VECTOR_CSV, VECTOR_RAW_BINARY,
)
