"""GPU parity: every hot-path entry point of the C ABI against the CPU oracle
(the C restatement, itself pinned bit-for-bit to the compiled reference in
test_oracle_pins.py) on the same seeded inputs and the same injected grid
(SURVEY.md 8c protocol 1), plus the reference tests' own known answers.

Tolerances (the north star's): NDCT/DLT/leg2cheb ||gpu - oracle||_inf /
||input||_1 <= 1e-13 log2(N); IDLT normalised by ||f||_1;
DCT engine 100 eps N ||c||_1 (test_trig.cpp:131-155); adjoints 1e-12
(acceptance.cpp:215-241); node ordering/reflection bit-exact.
"""
import math

import numpy as np
import pytest

from conftest import EPS, unhex
from oracle import CHEB1, CHEBSTAR, ORACLE as O
import oracle
import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu
K = {CHEB1: fl.GridKind.cheb1, CHEBSTAR: fl.GridKind.chebstar}


def tol_n(n):
    return 1e-13 * max(math.log2(n), 1.0)


def rel_err(a, b, scale):
    scale = scale if scale > 0 else 1.0
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale if len(np.ravel(a)) else 0.0


def angles(kind, n):
    k = np.arange(n)
    return (k + 0.5) * np.pi / n if kind == CHEB1 else (k + 0.75) * np.pi / (n + 0.5)


# --------------------------------------------------------------------------- nodes

def test_nodes_closed_forms():  # test_quadrature.cpp:59-89
    g = fl.legendre_nodes_weights(1)
    assert g.theta[0] == 0.5 * math.pi and g.x[0] == 0.0 and g.weights[0] == 2.0
    g = fl.legendre_nodes_weights(2)
    assert abs(g.x[0] - 1 / math.sqrt(3)) <= 4 * EPS and g.x[1] == -g.x[0]
    assert np.all(np.abs(g.weights - 1.0) <= 4 * EPS)
    g = fl.legendre_nodes_weights(3)
    assert abs(g.x[0] - math.sqrt(0.6)) <= 8 * EPS and g.x[1] == 0.0
    assert abs(g.weights[0] - 5 / 9) <= 8 * EPS and abs(g.weights[1] - 8 / 9) <= 8 * EPS
    with pytest.raises(fl.InvalidArgument):
        fl.legendre_nodes_weights(0)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 16, 17, 20, 64, 127, 128, 129, 257, 1000, 4096, 10000, 65537])
def test_nodes_structure_bitexact(n):
    """Ordering, exact reflection and odd-N middle (quadrature.hpp:126-141),
    sum of weights (test_quadrature.cpp:99-128)."""
    g = fl.legendre_nodes_weights(n)
    th, x, w = g.theta, g.x, g.weights
    assert np.all(np.diff(th) > 0) and np.all(np.diff(x) < 0)
    assert np.all(th > 0) and np.all(th < math.pi)
    h = n // 2
    for k in range(h):
        assert th[n - 1 - k] == math.pi - th[k]
        assert x[n - 1 - k] == -x[k]
        assert w[n - 1 - k] == w[k]
    if n % 2:
        assert th[h] == 0.5 * math.pi and x[h] == 0.0
    assert abs(w.sum() - 2.0) <= 16 * EPS * n


def test_nodes_vs_truth(nodes_truth):
    """The asymptotic/double-double node kernel against 40-digit truth."""
    worst_t, worst_w = 0.0, 0.0
    for n, rows in nodes_truth["nodes"].items():
        g = fl.legendre_nodes_weights(int(n))
        for r in rows:
            t, wt = float(r["theta"]), float(r["w"])
            et = abs(g.theta[r["k"]] - t) / np.spacing(t)
            ew = abs(g.weights[r["k"]] - wt) / wt
            worst_t, worst_w = max(worst_t, et), max(worst_w, ew)
            assert et <= 2.0, (n, r["k"], et)
            assert ew <= 4e-15, (n, r["k"], ew)
    print(f"nodes vs truth: worst {worst_t:.2f} ulp(theta), weight rel {worst_w:.2e}")


@pytest.mark.parametrize("n", [5, 64, 100, 1000, 4096])
def test_nodes_vs_reference_model(n):
    """Against the reference's own Newton nodes: |dtheta| <= 4 eps/sin(theta)
    (the reference's error)."""
    th, x, w = O.nodes_weights(n)
    g = fl.legendre_nodes_weights(n)
    s = np.sin(g.theta)
    assert np.all(np.abs(g.theta - th) <= 4 * EPS / s + 2 * EPS)
    # the reference's weights carry ~N/18 eps of recurrence rounding in the interior
    assert np.all(np.abs(g.weights - w) <= (8 / s ** 2 + n / 16 + 16) * EPS * w)


def test_quadrature_exactness():  # acceptance.cpp:127-141, test_quadrature.cpp:130-141
    for n in (5, 20, 50):
        g = fl.legendre_nodes_weights(n)
        for m in range(2 * n):
            exact = 0.0 if m % 2 else 2.0 / (m + 1)
            assert abs(np.sum(g.weights * g.x ** m) - exact) <= 1e-13


def test_node_proximity_bounds():  # acceptance.cpp:102-123
    for n in (10, 100, 1000, 10000):
        g = fl.legendre_nodes_weights(n)
        ms = np.max(np.abs(fl.reference_grid(g, fl.GridKind.chebstar).delta_theta))
        m1 = np.max(np.abs(fl.reference_grid(g, fl.GridKind.cheb1).delta_theta))
        bs, b1 = 1 / (6 * math.pi * n), 0.83845 / n
        assert ms <= bs and m1 <= b1
        if n >= 100:
            assert ms >= bs / 3 and m1 >= b1 / 3


@pytest.mark.parametrize("kind", [CHEB1, CHEBSTAR])
def test_reference_grid_bitexact(kind):  # test_quadrature.cpp:143-157
    for n in (1, 7, 256, 4097):
        g = fl.legendre_nodes_weights(n)
        r = fl.reference_grid(g, K[kind])
        ts, d = np.empty(n), np.empty(n)
        O._refg(n, kind, g.theta, ts, d)
        assert np.array_equal(r.theta_star, ts) and np.array_equal(r.delta_theta, d)
        for k in range(min(n, 50)):
            assert r.theta_star[k] == fl.reference_angle(n, K[kind], k)


def test_lambda_table():  # conversion.hpp:25-30; test_conversion.cpp:27-35
    for m in (0, 1, 63, 64, 1000, 70000):
        c = fl.LambdaCache(m)
        ref = O.lambda_table(m)
        assert np.all(np.abs(c.table - ref) <= 2e-15 * np.maximum(1, np.sqrt(np.arange(m + 1))) * ref)
        z = np.arange(m)
        ratio = c.table[1:] / c.table[:-1]
        assert np.all(np.abs(ratio - (z + 0.5) / (z + 1.0)) <= 4 * EPS)


# --------------------------------------------------------------------------- DCT/DST engine

def test_trig_known_answers():  # test_trig.cpp:86-114
    for kind in (fl.GridKind.cheb1, fl.GridKind.chebstar):
        e0 = np.zeros(6)
        e0[0] = 1.0
        assert np.all(np.abs(fl.dct_iii(e0, kind) - 1.0) <= 4 * EPS)
        assert np.all(fl.dst_iii(e0, kind) == 0.0)
    e1 = np.zeros(4)
    e1[1] = 1.0
    a = (np.arange(4) + 0.5) * math.pi / 4
    assert np.all(np.abs(fl.dct_iii(e1, fl.GridKind.cheb1) - np.cos(a)) <= 8 * EPS)
    assert np.all(np.abs(fl.dst_iii(e1, fl.GridKind.cheb1) - np.sin(a)) <= 8 * EPS)
    e0 = np.array([1.0, 0.0, 0.0])
    out = fl.dct_iii_transpose(e0, fl.GridKind.cheb1)
    assert np.all(np.abs(out - [1.0, math.cos(math.pi / 6), math.cos(2 * math.pi / 6)]) <= 4 * EPS)


def test_trig_every_size_up_to_128():  # test_trig.cpp:131-155
    ops = (fl.dct_iii, fl.dst_iii, fl.dct_iii_transpose, fl.dst_iii_transpose)
    for n in range(1, 129):
        c = np.random.default_rng(1000 + n).uniform(-1, 1, n)
        tol = 100 * EPS * n * np.abs(c).sum()
        for kind in (CHEB1, CHEBSTAR):
            th = angles(kind, n)
            k = np.arange(n)
            Cm, Sm = np.cos(np.outer(th, k)), np.sin(np.outer(th, k))
            for op, ref in enumerate((Cm @ c, Sm @ c, Cm.T @ c, Sm.T @ c)):
                got = ops[op](c, K[kind])
                assert np.max(np.abs(got - ref)) <= tol, (n, kind, op)
                assert np.max(np.abs(got - O.trig(op, c, kind))) <= tol, (n, kind, op)


def test_trig_adjoint_and_linearity():  # test_trig.cpp:157-184
    for n in range(1, 65):
        rng = np.random.default_rng(2 * n)
        c, g = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        tol = 1e-12 * np.linalg.norm(c) * np.linalg.norm(g)
        for kind in K.values():
            assert abs(fl.dct_iii(c, kind) @ g - c @ fl.dct_iii_transpose(g, kind)) <= tol
            assert abs(fl.dst_iii(c, kind) @ g - c @ fl.dst_iii_transpose(g, kind)) <= tol
    c, d = np.random.default_rng(5).uniform(-1, 1, (2, 24))
    for kind in K.values():
        lhs = fl.dct_iii(0.37 * c - 1.25 * d, kind)
        rhs = 0.37 * fl.dct_iii(c, kind) - 1.25 * fl.dct_iii(d, kind)
        assert np.max(np.abs(lhs - rhs)) <= 100 * EPS


@pytest.mark.parametrize("n", [1000, 4096, 8192, 65536])
def test_trig_batched_large(n):
    rng = np.random.default_rng(n)
    c = rng.standard_normal((3, n))
    for kind in (CHEB1, CHEBSTAR):
        for op, f in enumerate((fl.dct_iii, fl.dst_iii, fl.dct_iii_transpose, fl.dst_iii_transpose)):
            got = f(c, K[kind])
            for j in range(3):
                ref = O.trig(op, c[j], kind)
                assert rel_err(got[j], ref, np.abs(c[j]).sum()) <= tol_n(n), (kind, op, j)


@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_trig_streaming_pass_device(op):
    """The persistent streaming passes (device columns, even stride, 16-byte
    aligned): DCT-III / DST-III (N = 4096: outputs stored straight from the
    mirrored last-pass butterflies) and their transposes (the next column
    bulk-copied while the current one is transformed, de-interleaved in
    shared memory) against the oracle on sampled columns and against the
    per-column kernel (odd stride) on all of them."""
    import ctypes as C
    import torch
    from paper_1505_00354_b200 import _lib
    n, batch = 4096, 1000
    x = torch.randn(batch, n, dtype=torch.float64, device="cuda")
    y = torch.full_like(x, 3.0)
    _lib.check(_lib.LIB.fl_trig(op, 0, n, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), batch, n, None))
    xs = torch.zeros(batch, n + 1, dtype=torch.float64, device="cuda")
    xs[:, :n] = x
    ys = torch.zeros_like(xs)
    _lib.check(_lib.LIB.fl_trig(op, 0, n, C.c_void_p(xs.data_ptr()), C.c_void_p(ys.data_ptr()), batch, n + 1,
                                None))
    yh, xh, ysh = y.cpu().numpy(), x.cpu().numpy(), ys[:, :n].cpu().numpy()
    scale = np.abs(xh).sum(axis=1)
    assert np.max(np.abs(yh - ysh).max(axis=1) / scale) <= 1e-15
    for j in (0, 1, 517, batch - 1):
        assert rel_err(yh[j], O.trig(op, xh[j], CHEB1), scale[j]) <= tol_n(n), j


def test_trig_golden(ref_vectors):
    """Reference outputs (compiled reference headers) on its own inputs."""
    for t in ref_vectors["trig"]:
        c = unhex(t["in"])
        got = (fl.dct_iii, fl.dst_iii, fl.dct_iii_transpose, fl.dst_iii_transpose)[t["op"]](c, K[t["kind"]])
        n = t["n"]
        assert np.max(np.abs(got - unhex(t["out"]))) <= 100 * EPS * n * np.abs(c).sum()


# --------------------------------------------------------------------------- NDCT

def _plan(n, kind, tol, grid=None):
    grid = grid or fl.legendre_nodes_weights(n)
    return grid, fl.plan_ndct(grid, K[kind], tol)


@pytest.mark.parametrize("n", [8, 13, 64, 256, 1024, 4096])
def test_ndct_parity(n):
    rng = np.random.default_rng(n)
    for kind in (CHEB1, CHEBSTAR):
        for tol in (2.0 ** -23, 2.0 ** -52):
            grid, plan = _plan(n, kind, tol)
            assert plan.num_terms == O.min_taylor_terms(kind, tol)
            delta = O.reference_delta(n, kind, grid.theta)
            assert np.array_equal(np.asarray(plan.reference.delta_theta), delta)
            c = rng.standard_normal(n)
            f = fl.ndct_apply(plan, c)
            assert rel_err(f, O.ndct(c, kind, plan.num_terms, delta), np.abs(c).sum()) <= tol_n(n)
            t = fl.ndct_apply_transpose(plan, c)
            assert rel_err(t, O.ndct(c, kind, plan.num_terms, delta, True), np.abs(c).sum()) <= tol_n(n)


def test_ndct_golden(ref_vectors):
    for t in ref_vectors["ndct"]:
        n, kind = t["n"], t["kind"]
        plan = fl.TaylorPlan(n, K[kind], t["tol"], t["L"],
                             fl.ReferenceGrid(n, K[kind], angles(kind, n), unhex(t["delta"])))
        c = unhex(t["in"])
        assert rel_err(fl.ndct_apply(plan, c), unhex(t["fwd"]), np.abs(c).sum()) <= tol_n(n)
        assert rel_err(fl.ndct_apply_transpose(plan, c), unhex(t["tr"]), np.abs(c).sum()) <= tol_n(n)


def test_ndct_known_answers():  # test_ndct.cpp:59-73
    for kind in K.values():
        plan = fl.plan_ndct(13, kind, fl.default_tolerance)
        e0 = np.zeros(13)
        e0[0] = 1.0
        assert np.all(np.abs(fl.ndct_apply(plan, e0) - 1.0) <= 4 * EPS)
    grid = fl.legendre_nodes_weights(8)
    plan = fl.plan_ndct(grid, fl.GridKind.chebstar, 1e-14)
    e1 = np.zeros(8)
    e1[1] = 1.0
    assert np.all(np.abs(fl.ndct_apply(plan, e1) - grid.x) <= 1e-13)


def test_ndct_zero_perturbation_bitexact():  # test_ndct.cpp:112-125
    n = 21
    plan = fl.plan_ndct(n, fl.GridKind.cheb1, fl.default_tolerance)
    plan.reference.delta_theta = np.zeros(n)
    c = fl.random_decaying(n, 0.5, 99)
    assert np.array_equal(fl.ndct_apply(plan, c), fl.dct_iii(c, fl.GridKind.cheb1))
    plan.num_terms = 1
    assert np.array_equal(fl.ndct_apply_transpose(plan, c), fl.dct_iii_transpose(c, fl.GridKind.cheb1))


def test_ndct_adjoint_and_matrix():  # test_ndct.cpp:87-110, acceptance.cpp:215-241
    for n in (1, 2, 7, 32, 129):
        grid = fl.legendre_nodes_weights(n)
        rng = np.random.default_rng(n)
        for kind in K.values():
            plan = fl.plan_ndct(grid, kind, fl.default_tolerance)
            for _ in range(5):
                v, w = rng.standard_normal((2, n))
                lhs, rhs = fl.ndct_apply(plan, v) @ w, v @ fl.ndct_apply_transpose(plan, w)
                assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(v) * np.linalg.norm(w)
    n = 8
    plan = fl.plan_ndct(n, fl.GridKind.cheb1, fl.default_tolerance)
    I = np.eye(n)
    Mf = fl.ndct_apply(plan, I)          # row j = ndct(e_j)
    Mt = fl.ndct_apply_transpose(plan, I)
    assert np.max(np.abs(Mt - Mf.T)) <= 1e-14


def test_ndct_vs_direct_bound():  # test_ndct.cpp:75-85, acceptance.cpp:145-168
    for n in (64, 256, 1024):
        grid = fl.legendre_nodes_weights(n)
        c = fl.random_decaying(n, 1.0, 3)
        exact = O.eval_chebyshev_direct(c, grid.x)
        for kind in K.values():
            for tol in (2.0 ** -23, 2.0 ** -52):
                plan = fl.plan_ndct(grid, kind, tol)
                err = np.max(np.abs(fl.ndct_apply(plan, c) - exact))
                assert err <= fl.ndct_error_bound(plan, c) + 1e-11 * np.abs(c).sum()


def test_ndct_error_bound_values():  # test_ndct.cpp:127-155
    star = fl.plan_ndct(16, fl.GridKind.chebstar, 2.0 ** -52)
    unit = np.zeros(16)
    unit[5] = 1.0
    b = fl.ndct_error_bound(star, unit)
    assert 0.0 < b <= 9.2e-18
    assert fl.ndct_error_bound(star, np.zeros(16)) == 0.0
    delta = np.asarray(star.reference.delta_theta)
    assert b == O.ndct_error_bound(unit, CHEBSTAR, 9, delta)


def test_ndct_validation():  # test_ndct.cpp:185-195
    plan = fl.plan_ndct(8, fl.GridKind.chebstar, fl.default_tolerance)
    with pytest.raises(fl.InvalidArgument, match="input size"):
        fl.ndct_apply(plan, np.zeros(9))
    with pytest.raises(fl.InvalidArgument, match="input size"):
        fl.ndct_apply_transpose(plan, np.zeros(9))
    for bad in (np.nan, np.inf):
        v = np.zeros(8)
        v[3] = bad
        with pytest.raises(fl.InvalidArgument, match="ndct_apply: non-finite input"):
            fl.ndct_apply(plan, v)
        with pytest.raises(fl.InvalidArgument, match="ndct_apply_transpose: non-finite input"):
            fl.ndct_apply_transpose(plan, v)


# --------------------------------------------------------------------------- leg2cheb

@pytest.mark.parametrize("n", [1, 2, 3, 16, 33, 128, 1000, 4096])
def test_leg2cheb_parity(n):
    rng = np.random.default_rng(n)
    c = rng.standard_normal((4, n))
    f = fl.leg2cheb_apply(fl.legendre_coefficients(c)).values
    t = fl.leg2cheb_apply_transpose(c)
    for j in range(4):
        assert rel_err(f[j], O.leg2cheb(c[j]), np.abs(c[j]).sum()) <= tol_n(n)
        assert rel_err(t[j], O.leg2cheb(c[j], True), np.abs(c[j]).sum()) <= tol_n(n)


def test_leg2cheb_golden_and_entries(ref_vectors):
    for t in ref_vectors["leg2cheb"]:
        c = unhex(t["in"])
        n = t["n"]
        assert rel_err(fl.leg2cheb_apply(fl.legendre_coefficients(c)).values, unhex(t["fwd"]),
                       np.abs(c).sum()) <= tol_n(n)
        assert rel_err(fl.leg2cheb_apply_transpose(c), unhex(t["tr"]), np.abs(c).sum()) <= tol_n(n)
    cache = fl.LambdaCache(64)  # acceptance.cpp:245-257
    worst = 0.0
    for n in range(33):
        orc = O.cheb_coeffs_of_legendre(n, 80)
        for k in range(n + 1):
            worst = max(worst, abs(fl.leg2cheb_entry(k, n, cache) - orc[k]))
    assert worst <= 1e-13
    # P_2 = 1/4 T_0 + 3/4 T_2 (test_conversion.cpp:106-109)
    out = fl.leg2cheb_apply(fl.legendre_coefficients([0.0, 0.0, 1.0])).values
    assert np.all(np.abs(out - [0.25, 0.0, 0.75]) <= 4 * EPS)


def test_leg2cheb_adjoint():
    for n in (1, 2, 7, 32, 129):
        rng = np.random.default_rng(n)
        cache = fl.LambdaCache(n)
        for _ in range(10):
            v, w = rng.standard_normal((2, n))
            lhs = fl.leg2cheb_apply(fl.legendre_coefficients(v), cache).values @ w
            rhs = v @ fl.leg2cheb_apply_transpose(w, cache)
            assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(v) * np.linalg.norm(w)


# --------------------------------------------------------------------------- DLT / IDLT

@pytest.mark.parametrize("n", [1, 2, 3, 8, 64, 256, 1024, 4096])
@pytest.mark.parametrize("mode", [fl.NDCT_LITERAL, fl.NDCT_FAST])
def test_dlt_idlt_parity_injected_grid(n, mode):
    """SURVEY.md 8c protocol 1: the GPU grid injected into the reference."""
    for kind in (CHEB1, CHEBSTAR):
        cfg = fl.TransformConfig(n, fl.default_tolerance, K[kind], ndct_mode=mode)
        g = cfg.grid()
        c = fl.random_decaying(n, 0.5, 1, batch=3)
        f = fl.dlt(c, cfg)
        back = fl.idlt(f, cfg).values
        for j in range(3):
            ref_f = O.dlt_grid(c[j], kind, fl.default_tolerance, g.theta, g.x, g.weights)
            assert rel_err(f[j], ref_f, np.abs(c[j]).sum()) <= tol_n(n), (kind, j)
            ref_b = O.idlt_grid(f[j], kind, fl.default_tolerance, g.theta, g.x, g.weights)
            assert rel_err(back[j], ref_b, np.abs(f[j]).sum()) <= tol_n(n), (kind, j)
            assert np.max(np.abs(back[j] - c[j])) <= 1e-10 * np.max(np.abs(c[j]))


def test_transforms_golden(ref_vectors):
    """Reference DLT/IDLT outputs on the reference's own (Newton) grid, injected."""
    for t in ref_vectors["transforms"]:
        n, kind = t["n"], t["kind"]
        grid = fl.LegendreGrid(n, unhex(t["theta"]), unhex(t["x"]), unhex(t["w"]))
        cfg = fl.TransformConfig(n, fl.default_tolerance, K[kind], grid=grid, ndct_mode=fl.NDCT_LITERAL)
        c = unhex(t["c"])
        f = fl.dlt(fl.legendre_coefficients(c), cfg)
        assert rel_err(f, unhex(t["f"]), np.abs(c).sum()) <= tol_n(n)
        back = fl.idlt(unhex(t["f"]), cfg).values
        assert rel_err(back, unhex(t["back"]), np.abs(unhex(t["f"])).sum()) <= tol_n(n)


def test_dlt_vs_direct_and_round_trip():  # acceptance.cpp:172-211
    for n in (8, 64, 512, 2048):
        cfg = fl.TransformConfig(n)
        assert cfg.plan().num_terms == 9
        for decay in (0.0, 0.5, 1.0, 1.5):
            c = fl.random_decaying(n, decay, 55 + n)
            err = np.max(np.abs(fl.dlt(fl.legendre_coefficients(c), cfg) - O.eval_legendre_direct(c, cfg.grid().x)))
            rel = 1e-8 if (decay == 0.0 and n == 2048) else 1e-10
            assert err <= rel * np.abs(c).sum()
        for seed in range(1, 6):
            c = fl.random_decaying(n, 1.0, seed)
            back = fl.idlt(fl.dlt(fl.legendre_coefficients(c), cfg), cfg).values
            assert np.max(np.abs(back - c)) / np.max(np.abs(c)) <= 1e-10


def test_degenerate_sizes_exact():  # acceptance.cpp:295-334
    x2, s32 = 0.57735026918962576451, 0.86602540378443864676
    worst = 0.0
    rng = np.random.default_rng(10)
    for kind in K.values():
        one = fl.TransformConfig(1, fl.default_tolerance, kind)
        two = fl.TransformConfig(2, fl.default_tolerance, kind)
        for trial in range(20):
            c0 = 1.0 if trial == 0 else rng.standard_normal()
            s1 = max(1.0, abs(c0))
            worst = max(worst, abs(fl.dlt(fl.legendre_coefficients([c0]), one)[0] - c0) / s1,
                        abs(fl.idlt([c0], one).values[0] - c0) / s1)
            u, v = rng.standard_normal(2)
            if trial == 0:
                u, v = 1.0, 0.0
            if trial == 1:
                u, v = 0.0, 1.0
            f2 = fl.dlt(fl.legendre_coefficients([u, v]), two)
            s2 = max(1.0, abs(u) + abs(v))
            worst = max(worst, abs(f2[0] - (u + v * x2)) / s2, abs(f2[1] - (u - v * x2)) / s2)
            b2 = fl.idlt([u, v], two).values
            worst = max(worst, abs(b2[0] - 0.5 * (u + v)) / s2, abs(b2[1] - s32 * (u - v)) / s2)
    assert worst <= 4 * EPS, worst / EPS


def test_transforms_validation():  # test_transforms.cpp:145-152
    cfg = fl.TransformConfig(8)
    with pytest.raises(fl.InvalidArgument, match="dlt: expected Legendre"):
        fl.dlt(fl.chebyshev_coefficients(np.zeros(8)), cfg)
    with pytest.raises(fl.InvalidArgument, match="dlt: coefficient size"):
        fl.dlt(fl.legendre_coefficients(np.zeros(9)), cfg)
    with pytest.raises(fl.InvalidArgument, match="idlt: value size"):
        fl.idlt(np.zeros(7), cfg)
    bad = np.zeros(8)
    bad[2] = np.nan
    with pytest.raises(fl.InvalidArgument, match="non-finite"):
        fl.dlt(fl.legendre_coefficients(bad), cfg)
    with pytest.raises(fl.InvalidArgument):
        fl.TransformConfig(0)
    with pytest.raises(fl.InvalidArgument):
        fl.TransformConfig(8, 0.0)


def test_device_resident_batched_matches_host():
    import torch
    n, b = 1024, 8
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4000, batch=b)
    f_host = fl.dlt(c, cfg)
    f_dev = fl.dlt(torch.from_numpy(c).cuda(), cfg)
    assert isinstance(f_dev, torch.Tensor) and f_dev.is_cuda
    assert np.array_equal(f_dev.cpu().numpy(), f_host)
    for j in range(b):
        assert np.array_equal(fl.dlt(c[j], cfg), f_host[j])


@pytest.mark.parametrize("batch,extra", [(17, 2), (17, 1), (300, 2), (3, 5)])
def test_dlt_idlt_strided_device_columns(batch, extra):
    """Device columns with ld > n (even and odd strides; more than 16 columns
    take the split-int8 conversion, whose kernels read and write one stride):
    results equal the contiguous call bit for bit, the padding is untouched
    and the IDLT round trip holds."""
    import ctypes as C
    import torch
    from paper_1505_00354_b200 import _lib
    n = 4096
    ld = n + extra
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4200 + batch, batch=batch)
    x = torch.zeros(batch, ld, dtype=torch.float64, device="cuda")
    x[:, :n] = torch.from_numpy(c).cuda()
    f = torch.full_like(x, 7.0)
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(f.data_ptr()), batch, ld, None))
    b = torch.full_like(x, 5.0)
    _lib.check(_lib.LIB.fl_idlt(cfg.handle, C.c_void_p(f.data_ptr()), C.c_void_p(b.data_ptr()), batch, ld, None))
    fh, bh = f.cpu().numpy(), b.cpu().numpy()
    assert np.all(fh[:, n:] == 7.0) and np.all(bh[:, n:] == 5.0)
    f_ref = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
    assert np.array_equal(fh[:, :n], f_ref)
    b_ref = fl.idlt(torch.from_numpy(f_ref).cuda(), cfg).values.cpu().numpy()
    assert np.array_equal(bh[:, :n], b_ref)
    assert np.max(np.abs(bh[:, :n] - c)) <= 1e-10


def test_dlt_idlt_4096_batch_invariance():
    """N = 4096 (the TMEM-resident Chebyshev NDCT kernels, split GEMM): a
    column's DLT / IDLT does not depend on the batch it is computed in
    (17 vs 300 columns, bit-identical) and matches the oracle."""
    import torch
    n = 4096
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4100, batch=300)
    dev = torch.from_numpy(c).cuda()
    f_all = fl.dlt(dev, cfg).cpu().numpy()
    f_17 = fl.dlt(dev[:17].contiguous(), cfg).cpu().numpy()
    assert np.array_equal(f_17, f_all[:17])
    b_all = fl.idlt(torch.from_numpy(f_all).cuda(), cfg).values.cpu().numpy()
    b_17 = fl.idlt(torch.from_numpy(f_all[:17]).cuda(), cfg).values.cpu().numpy()
    assert np.array_equal(b_17, b_all[:17])
    g = cfg.grid()
    for j in (0, 16, 299):
        ref = O.dlt_grid(c[j], CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        assert rel_err(f_all[j], ref, np.abs(c[j]).sum()) <= tol_n(n), j
        assert np.max(np.abs(b_all[j] - c[j])) <= 1e-10 * np.max(np.abs(c[j])), j


@pytest.mark.parametrize("n", [64, 100, 1024, 4096])
def test_leg2cheb_tensor_core_path(n):
    """> 16 columns: the DMMA (fp64 mma.sync) GEMM kernel; odd N / unaligned
    strides take the FMA-tiled kernel. Both against the oracle."""
    rng = np.random.default_rng(n)
    c = rng.uniform(-1, 1, (40, n))
    f = fl.leg2cheb_apply(fl.legendre_coefficients(c)).values
    t = fl.leg2cheb_apply_transpose(c)
    for j in (0, 17, 39):
        assert rel_err(f[j], O.leg2cheb(c[j]), np.abs(c[j]).sum()) <= tol_n(n)
        assert rel_err(t[j], O.leg2cheb(c[j], True), np.abs(c[j]).sum()) <= tol_n(n)


@pytest.mark.parametrize("n", [1 << 14, 1 << 16])
def test_leg2cheb_single_vector_large(n):
    c = fl.random_decaying(n, 1.0, 3)
    f = fl.leg2cheb_apply(fl.legendre_coefficients(c)).values
    t = fl.leg2cheb_apply_transpose(c)
    assert rel_err(f, O.leg2cheb(c), np.abs(c).sum()) <= tol_n(n)
    assert rel_err(t, O.leg2cheb(c, True), np.abs(c).sum()) <= tol_n(n)


@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 5, (1 << 24) - 3])
def test_leg2cheb_sampled_rows(n):
    """N = 2^20 (C3 size; the O(N^2) CPU loop is minutes) and the two-pass
    FFT sizes whose Toeplitz-Hankel sweep folds the accumulation into the last
    inverse pass (L = 2^23, 2^24): sampled rows of conversion.hpp:106-111 /
    :126-133 restated in numpy, O(N) each."""
    c = fl.random_decaying(n, 1.0, 3)
    f = fl.leg2cheb_apply(fl.legendre_coefficients(c)).values
    t = fl.leg2cheb_apply_transpose(c)
    lam = O.lambda_table(n - 1)
    s = lam / lam[0]
    for k in (0, 1, 2, 777, n // 2, n - 2, n - 1):
        j = np.arange((n - k + 1) // 2)
        ref = (1.0 if k == 0 else 2.0) * np.sum(s[j] * s[k + j] * c[k + 2 * j])
        assert abs(f[k] - ref) <= tol_n(n) * np.abs(c).sum()
        m = k
        j = np.arange((m + 1) // 2) if m % 2 else np.arange(m // 2)
        reft = 2.0 * np.sum(s[j] * s[m - j] * c[m - 2 * j])
        if m % 2 == 0:
            reft += s[m // 2] * s[m - m // 2] * c[0]
        assert abs(t[m] - reft) <= tol_n(n) * np.abs(c).sum()


@pytest.mark.parametrize("n", [16384, 65536])
def test_ndct_multipass_power_of_two(n):
    """N > 8192: the multi-pass fast NDCT (cheb1 packing + six-step FFT)."""
    grid = fl.legendre_nodes_weights(n)
    c = np.random.default_rng(n).standard_normal((2, n))
    for tol in (2.0 ** -23, 2.0 ** -52):
        plan = fl.plan_ndct(grid, fl.GridKind.cheb1, tol)
        delta = np.asarray(plan.reference.delta_theta)
        f = fl.ndct_apply(plan, c)
        t = fl.ndct_apply_transpose(plan, c)
        for j in range(2):
            s = np.abs(c[j]).sum()
            assert rel_err(f[j], O.ndct(c[j], CHEB1, plan.num_terms, delta), s) <= tol_n(n)
            assert rel_err(t[j], O.ndct(c[j], CHEB1, plan.num_terms, delta, True), s) <= tol_n(n)
    for op, fn in enumerate((fl.dct_iii, fl.dst_iii, fl.dct_iii_transpose, fl.dst_iii_transpose)):
        got = fn(c[0], fl.GridKind.cheb1)
        assert rel_err(got, O.trig(op, c[0], CHEB1), np.abs(c[0]).sum()) <= tol_n(n)


@pytest.mark.parametrize("n", [1 << 15, (1 << 16) + 3])
def test_leg2cheb_fast_toeplitz_hankel_vs_direct(n):
    """The Toeplitz-Hankel conversion inside dlt/idlt against the direct
    triangular product (same plan, mode switch) and the CPU oracle."""
    cfg = fl.TransformConfig(n)
    k0, k1 = cfg.leg2cheb_rank(0), cfg.leg2cheb_rank(1)
    assert 10 < k0 < 100 and 10 < k1 < 100, (k0, k1)
    c = fl.random_decaying(n, 0.5, 11, batch=2)
    f_fast = fl.dlt(c, cfg)
    b_fast = fl.idlt(f_fast, cfg).values
    cfg.set_leg2cheb_mode(fl.LEG2CHEB_DIRECT)
    f_dir = fl.dlt(c, cfg)
    b_dir = fl.idlt(f_fast, cfg).values
    for j in range(2):
        assert rel_err(f_fast[j], f_dir[j], np.abs(c[j]).sum()) <= tol_n(n)
        assert rel_err(b_fast[j], b_dir[j], np.abs(f_fast[j]).sum()) <= tol_n(n)
    v = c[0]
    g = cfg.grid()
    ref = O.leg2cheb(v)
    lam = fl.LambdaCache(n - 1)
    got = fl.leg2cheb_apply(fl.legendre_coefficients(v), lam).values  # free function (direct < 2^17)
    assert rel_err(got, ref, np.abs(v).sum()) <= tol_n(n)
