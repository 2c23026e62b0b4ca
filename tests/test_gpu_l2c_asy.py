"""The asymptotic-expansion Legendre -> Chebyshev conversion (plan mode
LEG2CHEB_ASYMPTOTIC, csrc/l2c_asy.cu; north-star subsystem 2) against the
reference's direct product (conversion.hpp:100-140 through the oracle), the
Toeplitz-Hankel conversion, and inside dlt / idlt against the oracle's
transforms (transforms.hpp:42-64). Tolerance: ||gpu - ref||_inf / ||c||_1 <=
1e-13 log2 N."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_1505_00354_b200")
from oracle import ORACLE as O  # noqa: E402


def tol_n(n):
    return 1e-13 * math.log2(n)


def rel_err(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / scale)


def asy_config(n, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        cfg = fl.TransformConfig(n)
        cfg.set_leg2cheb_mode(fl.LEG2CHEB_ASYMPTOTIC)
        info = cfg.leg2cheb_asy_info()  # builds the tables under this environment
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return cfg, info


@pytest.mark.parametrize("n", [1 << k for k in range(10, 17)])
def test_asy_conversion_vs_oracle(n):
    cfg, info = asy_config(n)
    rng = np.random.default_rng(n)
    c = np.stack([rng.standard_normal(n) / np.sqrt(np.arange(n) + 1.0), rng.uniform(-1, 1, n),
                  fl.random_decaying(n, 1.0, 3)])
    f = cfg.convert(c)
    t = cfg.convert(c, transpose=True)
    scale = np.arange(n) + 0.5
    for j in range(len(c)):
        s = np.abs(c[j]).sum()
        assert rel_err(f[j], O.leg2cheb(c[j]), s) <= tol_n(n), (j, info)
        assert rel_err(t[j], scale * O.leg2cheb(c[j], True), s * n) <= tol_n(n), (j, info)


@pytest.mark.parametrize("env", [
    {"FLB_ASY_M": 14, "FLB_ASY_R": 4},
    {"FLB_ASY_M": 18, "FLB_ASY_R": 8},
    {"FLB_ASY_M": 10, "FLB_ASY_R": 8, "FLB_ASY_LEVELS": 1},  # most points by the chunked recurrence
    {"FLB_ASY_M": 10, "FLB_ASY_R": 8, "FLB_ASY_LEVELS": 0},  # the recurrence alone (O(N^2))
])
def test_asy_conversion_settings(env):
    """Other term counts / level ratios, and truncated level sets that move
    the work into the chunked transfer-matrix recurrence (many chunks per
    point: transfer, prefix and restart kernels)."""
    n = 1 << 14
    cfg, info = asy_config(n, **env)
    if env.get("FLB_ASY_LEVELS") == 0:
        assert info["levels"] == 0 and info["recurrence_steps_per_n"] == n
    c = fl.random_decaying(n, 0.5, 7, batch=2)
    f = cfg.convert(c)
    t = cfg.convert(c, transpose=True)
    for j in range(2):
        s = np.abs(c[j]).sum()
        assert rel_err(f[j], O.leg2cheb(c[j]), s) <= tol_n(n), info
        assert rel_err(t[j], (np.arange(n) + 0.5) * O.leg2cheb(c[j], True), s * n) <= tol_n(n), info


@pytest.mark.parametrize("n", [1 << 18, 1 << 20])
def test_asy_vs_toeplitz_hankel_and_sampled_rows(n):
    """Large N: against the Toeplitz-Hankel conversion of the same plan (full
    vector) and sampled rows of conversion.hpp:106-111 / :126-133 (O(N) each)."""
    cfg, info = asy_config(n)
    c = fl.random_decaying(n, 1.0, 3)
    f = cfg.convert(c)
    t = cfg.convert(c, transpose=True)
    cfg.set_leg2cheb_mode(fl.LEG2CHEB_TOEPLITZ)
    f_th = cfg.convert(c)
    t_th = cfg.convert(c, transpose=True)
    s = np.abs(c).sum()
    assert rel_err(f, f_th, s) <= tol_n(n), info
    assert rel_err(t, t_th, s * n) <= tol_n(n), info
    lam = O.lambda_table(n - 1)
    sl = lam / lam[0]
    for k in (0, 1, 2, 3, 777, n // 3, n // 2, n - 4, n - 3, n - 2, n - 1):
        j = np.arange((n - k + 1) // 2)
        ref = (1.0 if k == 0 else 2.0) * np.sum(sl[j] * sl[k + j] * c[k + 2 * j])
        assert abs(f[k] - ref) <= tol_n(n) * s, k
        jt = np.arange((k + 1) // 2) if k % 2 else np.arange(k // 2)
        reft = 2.0 * np.sum(sl[jt] * sl[k - jt] * c[k - 2 * jt])
        if k % 2 == 0:
            reft += sl[k // 2] * sl[k - k // 2] * c[0]
        assert abs(t[k] - (k + 0.5) * reft) <= tol_n(n) * s * n, k


@pytest.mark.parametrize("kind", [fl.GridKind.chebstar, fl.GridKind.cheb1])
def test_asy_inside_dlt_idlt(kind):
    """dlt / idlt of a plan in asymptotic mode against the oracle's transforms
    on the same injected grid."""
    n = 1 << 15
    cfg = fl.TransformConfig(n, fl.default_tolerance, kind)
    cfg.set_leg2cheb_mode(fl.LEG2CHEB_ASYMPTOTIC)
    g = cfg.grid()
    c = fl.random_decaying(n, 1.0, 5)
    f = fl.dlt(fl.legendre_coefficients(c), cfg)
    b = fl.idlt(f, cfg).values
    ref_f = O.dlt_grid(c, int(kind), fl.default_tolerance, g.theta, g.x, g.weights)
    ref_b = O.idlt_grid(f, int(kind), fl.default_tolerance, g.theta, g.x, g.weights)
    assert rel_err(f, ref_f, np.abs(c).sum()) <= tol_n(n)
    assert rel_err(b, ref_b, np.abs(f).sum()) <= tol_n(n)


def test_asy_deterministic():
    """Bit-identical results on repetition (no atomics: fixed-order partial sums)."""
    n = 1 << 16
    cfg, _ = asy_config(n, FLB_ASY_LEVELS=2)
    c = fl.random_decaying(n, 1.0, 9)
    a = [cfg.convert(c) for _ in range(3)]
    b = [cfg.convert(c, transpose=True) for _ in range(3)]
    assert all(np.array_equal(a[0], x) for x in a[1:])
    assert all(np.array_equal(b[0], x) for x in b[1:])


def test_asy_stage_slices_sum_to_full():
    """The term-parallel C5 split (fl_dlt_stage, FL_STAGE_LEG2CHEB): partial
    conversions over weighted slices of the (level, m) terms and recurrence
    bands sum to the full conversion (forward and transposed)."""
    import torch
    from paper_1505_00354_b200 import distributed as D
    n = 1 << 20
    cfg = fl.TransformConfig(n)  # FAST mode: the expansion at 2^20
    count = D.stage_terms(cfg, D.STAGE_LEG2CHEB)
    info = cfg.leg2cheb_asy_info()
    assert count > info["levels"] * info["terms"]
    costs = D.stage_costs(cfg, D.STAGE_LEG2CHEB, count)
    x = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
    for inverse in (0, 1):
        full = torch.empty_like(x)
        D.gpu_stage(cfg, inverse, D.STAGE_LEG2CHEB, 0, count, x, full)
        for world in (2, 3, 8):
            acc = torch.zeros_like(x)
            for r in range(world):
                lo, hi = D.weighted_slice(costs, world, r)
                part = torch.empty_like(x)
                D.gpu_stage(cfg, inverse, D.STAGE_LEG2CHEB, lo, hi, x, part)
                acc += part
            s = float(x.abs().sum()) * (n if inverse else 1)
            assert float((acc - full).abs().max()) / s <= 1e-15 * math.log2(n), (inverse, world)
        ref = cfg.convert(x.cpu().numpy(), transpose=bool(inverse))
        assert float(np.abs(full.cpu().numpy() - ref).max()) / s <= 1e-15 * math.log2(n)
