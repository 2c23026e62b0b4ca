"""The direct DLT / IDLT (FL_DLT_DIRECT, the default for > 16 columns at
n % 256 == 0, 512 <= n <= 8192): f = P c and c = D_s P^T D_w f as one dense
split-int8 tcgen05 product per parity, P_kn = P_n(cos theta_k) at the
reference's evaluation angles. Parity against the CPU oracle (the
reference's factored algorithm, transforms.hpp:42-64, on the same injected
grid) at the north star's 1e-13 log2 N; agreement with the factored GPU
path; the edge cases of the batched entry (strides, non-finite columns,
pinned host pipeline, few columns -> factored)."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import CHEB1, CHEBSTAR, ORACLE as O
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib

pytestmark = pytest.mark.gpu
K = {CHEB1: fl.GridKind.cheb1, CHEBSTAR: fl.GridKind.chebstar}
TOL = fl.default_tolerance


def tol_n(n):
    return 1e-13 * max(math.log2(n), 1.0)


def rel(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / (scale if scale > 0 else 1.0)


@pytest.mark.parametrize("n", [512, 768, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("kind", [CHEB1, CHEBSTAR])
def test_direct_vs_oracle_and_factored(n, kind):
    import torch
    cfg = fl.TransformConfig(n, TOL, K[kind])
    assert cfg.uses_direct(40) and not cfg.uses_direct(16)
    g = cfg.grid()
    c = np.concatenate([fl.random_decaying(n, 0.5, 60 + n, batch=20),
                        fl.random_uniform_pm1(n, 4000 + n, batch=20)])
    v = fl.random_decaying(n, 0.0, 70 + n, batch=40)
    f = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
    b = fl.idlt(torch.from_numpy(v).cuda(), cfg).values.cpu().numpy()
    t = tol_n(n)
    for j in (0, 7, 19, 20, 39):
        ref = O.dlt_grid(c[j], kind, TOL, g.theta, g.x, g.weights)
        assert rel(f[j], ref, np.abs(c[j]).sum()) <= t, ("dlt", j)
        refb = O.idlt_grid(v[j], kind, TOL, g.theta, g.x, g.weights)
        assert rel(b[j], refb, np.abs(v[j]).sum()) <= t, ("idlt", j)
    cfg.set_dlt_method(fl.DLT_FACTORED)
    assert not cfg.uses_direct(40)
    f2 = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
    b2 = fl.idlt(torch.from_numpy(v).cuda(), cfg).values.cpu().numpy()
    for j in range(40):
        assert rel(f[j], f2[j], np.abs(c[j]).sum()) <= t, j
        assert rel(b[j], b2[j], np.abs(v[j]).sum()) <= t, j


def test_direct_round_trip_and_batch_invariance():
    import torch
    n = 4096
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4100, batch=300)
    dev = torch.from_numpy(c).cuda()
    f = fl.dlt(dev, cfg)
    back = fl.idlt(f, cfg).values.cpu().numpy()
    assert np.max(np.abs(back - c)) <= 1e-10 * np.max(np.abs(c))  # acceptance.cpp:193-211
    f17 = fl.dlt(dev[:17].contiguous(), cfg).cpu().numpy()
    assert np.array_equal(f17, f.cpu().numpy()[:17])


@pytest.mark.parametrize("extra", [0, 1, 2])
def test_direct_strides_and_offsets(extra):
    """ld = n, n + 1 (odd: every other column 8-byte aligned only), n + 2,
    and a view at an odd element offset: equal to the contiguous call bit for
    bit, padding untouched."""
    import torch
    n, batch = 2048, 33
    ld = n + extra
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 17, batch=batch)
    base = torch.zeros(batch * ld + 1, dtype=torch.float64, device="cuda")
    x = base[1:].view(batch, ld) if extra == 1 else base[:batch * ld].view(batch, ld)
    x[:, :n] = torch.from_numpy(c).cuda()
    y = torch.full((batch, ld), 7.0, dtype=torch.float64, device="cuda")
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), batch, ld, None))
    ref = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
    yh = y.cpu().numpy()
    assert np.array_equal(yh[:, :n], ref)
    assert np.all(yh[:, n:] == 7.0)
    z = torch.full((batch, ld), 5.0, dtype=torch.float64, device="cuda")
    _lib.check(_lib.LIB.fl_idlt(cfg.handle, C.c_void_p(y.data_ptr()), C.c_void_p(z.data_ptr()), batch, ld, None))
    refb = fl.idlt(torch.from_numpy(ref).cuda(), cfg).values.cpu().numpy()
    assert np.array_equal(z.cpu().numpy()[:, :n], refb)


def test_direct_nonfinite_column_raises():
    n, batch = 1024, 20
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 3, batch=batch)
    c[11, 5] = np.nan
    with pytest.raises(fl.InvalidArgument, match="ndct_apply: non-finite input"):
        fl.dlt(c, cfg)
    c[11, 5] = np.inf
    with pytest.raises(fl.InvalidArgument, match="ndct_apply_transpose: non-finite input"):
        fl.idlt(c, cfg)


def test_direct_zero_and_scaled_columns():
    """Per-column power-of-two scaling: an all-zero column gives exact zeros,
    columns scaled by 2^-600 / 2^600 give the scaled result exactly."""
    n, batch = 1024, 24
    cfg = fl.TransformConfig(n)
    c = fl.random_decaying(n, 1.0, 5, batch=batch)
    c[3] = 0.0
    c[4] = c[6] * 2.0 ** -600
    c[5] = c[6] * 2.0 ** 600
    f = fl.dlt(c, cfg)
    assert np.all(f[3] == 0.0)
    assert np.array_equal(f[4], f[6] * 2.0 ** -600) and np.array_equal(f[5], f[6] * 2.0 ** 600)


@pytest.mark.parametrize("n", [256, 258, 300, 512, 1000, 1002, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("kind", [CHEB1, CHEBSTAR])
def test_direct_few_columns_fp64_table(n, kind):
    """<= 16 columns (C1 and the C3 sweep up to 8192): the direct method as
    fp64 products over the plan's table of P_n(x_k) (dense_gemv.cu), against
    the oracle and the factored GPU path; one column and 3 / 16 columns with a
    stride (host and device buffers)."""
    import torch
    cfg = fl.TransformConfig(n, TOL, K[kind])
    g = cfg.grid()
    c = fl.random_decaying(n, 0.5, 80 + n, batch=16)
    v = fl.random_decaying(n, 0.0, 90 + n, batch=16)
    t = tol_n(n)
    f1 = fl.dlt(c[0], cfg)
    b1 = fl.idlt(v[0], cfg).values
    assert rel(f1, O.dlt_grid(c[0], kind, TOL, g.theta, g.x, g.weights), np.abs(c[0]).sum()) <= t
    assert rel(b1, O.idlt_grid(v[0], kind, TOL, g.theta, g.x, g.weights), np.abs(v[0]).sum()) <= t
    f16 = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
    b16 = fl.idlt(torch.from_numpy(v).cuda(), cfg).values.cpu().numpy()
    f3 = fl.dlt(c[:3], cfg)
    for j in (0, 5, 15):
        assert rel(f16[j], O.dlt_grid(c[j], kind, TOL, g.theta, g.x, g.weights), np.abs(c[j]).sum()) <= t, j
        assert rel(b16[j], O.idlt_grid(v[j], kind, TOL, g.theta, g.x, g.weights),
                   np.abs(v[j]).sum()) <= t, j
    assert np.array_equal(f16[0], f1) and np.array_equal(f3[2], f16[2])  # batch-invariant
    cfg.set_dlt_method(fl.DLT_FACTORED)
    f2 = fl.dlt(c[:3], cfg)
    b2 = fl.idlt(v[:3], cfg).values
    for j in range(3):
        assert rel(f3[j], f2[j], np.abs(c[j]).sum()) <= t, j
        assert rel(b16[j], b2[j], np.abs(v[j]).sum()) <= t, j


def test_direct_few_columns_edge_cases():
    """Strided device columns, non-finite inputs (the reference's
    invalid_argument), bit-identical repetition."""
    import torch
    n = 1024
    cfg = fl.TransformConfig(n)
    c = fl.random_decaying(n, 0.5, 7, batch=5)
    base = fl.dlt(c, cfg)
    wide = torch.zeros(5, n + 37, dtype=torch.float64, device="cuda")
    wide[:, :n] = torch.from_numpy(c).cuda()
    out = torch.zeros(5, n + 37, dtype=torch.float64, device="cuda")  # one stride for both
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(wide.data_ptr()), C.c_void_p(out.data_ptr()), 5, n + 37,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    assert np.array_equal(out[:, :n].cpu().numpy(), base)
    assert all(np.array_equal(fl.dlt(c, cfg), base) for _ in range(3))
    bad = c.copy()
    bad[3, 17] = np.nan
    with pytest.raises(fl.InvalidArgument, match="ndct_apply: non-finite input"):
        fl.dlt(bad, cfg)
    bad[3, 17] = np.inf
    with pytest.raises(fl.InvalidArgument, match="ndct_apply_transpose: non-finite input"):
        fl.idlt(bad, cfg)
