"""The split-integer conversion product (FL_GEMM_INT8_SPLIT, tcgen05 kind::i8)
inside dlt/idlt: parity against the CPU oracle on the injected grid, against
the fp64 tensor-core product, and the edge cases of the scaling (zero,
decaying and non-finite columns, ragged column counts, strided device input).
Tolerance for parity is the north star's 1e-13 log2(N) ||input||_1; the
split-vs-fp64 agreement is held to 1e-15 (uniform inputs) / 1e-14 (decaying)
||input||_1: both are fp64-level.
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import CHEB1, CHEBSTAR, ORACLE as O
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib

pytestmark = pytest.mark.gpu
K = {CHEB1: fl.GridKind.cheb1, CHEBSTAR: fl.GridKind.chebstar}


def tol_n(n):
    return 1e-13 * max(math.log2(n), 1.0)


def rel(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / (scale if scale > 0 else 1.0)


def both(cfg, c):
    """dlt and idlt of the (batch, n) block c with the split and the fp64
    conversion product (the factored path: conversion + NDCT)."""
    cfg.set_dlt_method(fl.DLT_FACTORED)
    out = {}
    for mode in (fl.GEMM_INT8_SPLIT, fl.GEMM_FP64):
        cfg.set_gemm_mode(mode)
        out[mode] = (fl.dlt(c, cfg), fl.idlt(c, cfg).values)
    cfg.set_gemm_mode(fl.GEMM_INT8_SPLIT)
    return out


def test_default_mode_and_validation():
    cfg = fl.TransformConfig(1024)
    assert cfg.gemm_mode() == fl.GEMM_INT8_SPLIT
    with pytest.raises(fl.InvalidArgument):
        cfg.set_gemm_mode(7)
    cfg.set_gemm_mode(fl.GEMM_FP64)
    assert cfg.gemm_mode() == fl.GEMM_FP64


@pytest.mark.parametrize("n", [512, 1024, 4096])
def test_split_vs_oracle_injected_grid(n):
    """40 columns (not a multiple of the 64-column tile) through the split
    product, both grid kinds, DLT and IDLT against the oracle."""
    for kind in (CHEB1, CHEBSTAR):
        cfg = fl.TransformConfig(n, fl.default_tolerance, K[kind])
        g = cfg.grid()
        c = fl.random_uniform_pm1(n, 4100 + n, batch=40)
        f = fl.dlt(c, cfg)
        back = fl.idlt(f, cfg).values
        for j in (0, 17, 39):
            ref_f = O.dlt_grid(c[j], kind, fl.default_tolerance, g.theta, g.x, g.weights)
            assert rel(f[j], ref_f, np.abs(c[j]).sum()) <= tol_n(n), (kind, j)
            ref_b = O.idlt_grid(f[j], kind, fl.default_tolerance, g.theta, g.x, g.weights)
            assert rel(back[j], ref_b, np.abs(f[j]).sum()) <= tol_n(n), (kind, j)
            assert np.max(np.abs(back[j] - c[j])) <= 1e-10 * np.max(np.abs(c[j]))


@pytest.mark.parametrize("n,batch", [(512, 17), (2048, 200), (4096, 130)])
def test_split_matches_fp64_product(n, batch):
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 77, batch=batch)
    r = both(cfg, c)
    for k in (0, 1):
        a, b = r[fl.GEMM_INT8_SPLIT][k], r[fl.GEMM_FP64][k]
        for j in range(batch):
            assert rel(a[j], b[j], np.abs(c[j]).sum()) <= 1e-15, (k, j)


def test_split_digit_carries():
    """8-bit digits: a residual in [127.5, 128] / 256 rounds to a digit of
    +128, which is stored as -128 with a carry into the next higher digit
    (l2c_ozaki.cu split_digits). Columns built so that (nearly) every entry
    carries, some in chains (consecutive 0.999.../256 residuals), must still
    match the fp64 product."""
    n, batch = 1024, 24
    cfg = fl.TransformConfig(n)
    rng = np.random.default_rng(5)
    c = np.empty((batch, n))
    for j in range(batch):
        # per-parity max in [1, 2): scale 2^3, r = x / 8 = (d0 + tail) / 256.
        # tail 0.499: digit 1 rounds 127.74 -> 128 (one carry); tail
        # (127 + 0.499) / 256: digit 1 = 127, digit 2 = 128 -> a carry chain
        # 2 -> 1 -> 0 in the odd columns
        d0 = rng.integers(-60, 60, n).astype(float)
        tail = (127.0 + 0.499) / 256.0 if j % 2 else 0.499
        c[j] = 8.0 * (d0 + np.sign(d0 + 0.5) * tail) / 256.0
        c[j, 0] = c[j, 1] = 1.0
    r = both(cfg, c)
    for k in (0, 1):
        a, b = r[fl.GEMM_INT8_SPLIT][k], r[fl.GEMM_FP64][k]
        for j in range(batch):
            assert rel(a[j], b[j], np.abs(c[j]).sum()) <= 1e-15, (k, j)


def test_split_decaying_and_zero_columns():
    """Large per-column dynamic range (decaying coefficients, scales 1e-200 ..
    1e200) and all-zero columns: the power-of-two scaling keeps every column
    at fp64 level and zero columns give exact zeros. The split drops digit
    pairs below 2^-56 of max|M row| max|c| per term, so on a decaying column
    its error grows like (N/2) 2^-56 max|c| / ||c||_1 (~2e-15 here, against
    ~4e-16 for the fp64 product): fp64 level, and three orders below the
    north star's 1e-13 log2 N."""
    n, batch = 1024, 24
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    c = fl.random_decaying(n, 1.0, 5, batch=batch)
    c[3] = 0.0
    c[4] *= 1e-200
    c[5] *= 1e200
    r = both(cfg, c)
    a, b = r[fl.GEMM_INT8_SPLIT][0], r[fl.GEMM_FP64][0]
    assert np.all(a[3] == 0.0) and np.all(r[fl.GEMM_INT8_SPLIT][1][3] == 0.0)
    worst = [0.0, 0.0]
    for j in range(batch):
        if j == 3:
            continue
        l1 = np.abs(c[j]).sum()
        ref = O.dlt_grid(c[j], CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        e_split, e_fp64 = rel(a[j], ref, l1), rel(b[j], ref, l1)
        assert e_split <= 4e-15, (j, e_split, e_fp64)  # ~20 eps: fp64 level
        bound = (n / 2) * 2.0 ** -55 * 4.0 * np.abs(c[j]).max() / l1 + 2e-16
        assert e_split <= max(2.0 * e_fp64, bound), (j, e_split, e_fp64, bound)
        worst = [max(worst[0], e_split), max(worst[1], e_fp64)]
        assert rel(a[j], b[j], l1) <= 1e-14, j
        ib, ia = r[fl.GEMM_FP64][1][j], r[fl.GEMM_INT8_SPLIT][1][j]
        assert rel(ia, ib, l1) <= 1e-14, j
    assert worst[0] <= 4e-15 and worst[1] <= 4e-15, worst


def test_split_nonfinite_column_reported():
    n = 512
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 5, batch=32)
    c[7, 100] = np.nan
    with pytest.raises(fl.InvalidArgument):
        fl.dlt(c, cfg)
    c[7, 100] = np.inf
    with pytest.raises(fl.InvalidArgument):
        fl.idlt(c, cfg)


def test_split_strided_device_input():
    """Device columns of stride ld > n (fl_dlt packs them for the product)."""
    import torch
    n, batch, ld = 1024, 48, 1024 + 40
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 9, batch=batch)
    ref = fl.dlt(c, cfg)
    blk = torch.zeros(batch, ld, dtype=torch.float64, device="cuda")
    blk[:, :n] = torch.from_numpy(c).cuda()
    out = torch.full((batch, ld), 7.0, dtype=torch.float64, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(blk.data_ptr()), C.c_void_p(out.data_ptr()),
                               batch, ld, s))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(got[:, :n], ref)
    assert np.all(got[:, n:] == 7.0)


def test_unsupported_sizes_use_fp64_product():
    """n not a multiple of 256: the mode is accepted, the fp64 product runs."""
    for n in (600, 1000):
        cfg = fl.TransformConfig(n)
        c = fl.random_uniform_pm1(n, 3, batch=20)
        f = fl.dlt(c, cfg)
        g = cfg.grid()
        ref = O.dlt_grid(c[11], CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        assert rel(f[11], ref, np.abs(c[11]).sum()) <= tol_n(n)
