"""GPU parity across the north star's size range (N = 2^9 .. 2^26), through
the C ABI, against the CPU oracle on the same injected grid (SURVEY.md 8c
protocol 1). The tolerance is the north star's:
    DLT / NDCT / conversion: ||gpu - oracle||_inf / ||input||_1 <= 1e-13 log2 N
    IDLT:                    ||gpu - oracle||_inf / ||f||_1     <= 1e-13 log2 N

* Sweep: every power of two 2^9 .. 2^18 x {cheb1, chebstar} x {fast, literal}
  x batch {1, 40}. The default code paths change across this range (fused
  on-chip NDCT up to 8192 with per-size kernel configurations, the multi-pass
  NDCT above; the int8-split tensor-core conversion for > 16 columns up to
  16384, the fp64 DMMA product above; the matrix-vector conversion for one
  column, Toeplitz-Hankel from 2^15), so every size is checked end to end
  against the oracle's full DLT / IDLT (oracle/fastleg_oracle.c, pinned bit
  for bit to the compiled reference in tests/test_oracle_pins.py).
* C2 exactly: NDCT and NDCT^T of 65536 x 64 iid N(0,1) columns, every
  column, both grids (the free functions ndct_apply / _transpose).
* C3 (2^20) and C5 (2^26): both stages of the default (fast) DLT and IDLT:
  the conversion (full O(N^2) oracle at 2^20; 96 sampled rows incl. the first
  and last ones at 2^26) and the NDCT / NDCT^T of the transform's own
  conversion output (the full O(N log N) oracle, oracle/ndct_np.py), plus the
  full DLT / IDLT at 2^20 against the composed oracle.
* The compiled reference itself (oracle/_ref) against the GPU at N = 4096.
"""
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import CHEB1, CHEBSTAR, ORACLE as O, REF
from oracle import ndct_np as NP
import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu
K = {CHEB1: fl.GridKind.cheb1, CHEBSTAR: fl.GridKind.chebstar}
TOL = fl.default_tolerance
POOL = ThreadPoolExecutor(os.cpu_count() or 4)  # the oracle's ctypes calls release the GIL


def tol_n(n):
    return 1e-13 * max(math.log2(n), 1.0)


def rel(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / (scale if scale > 0 else 1.0)


SWEEP = [1 << k for k in range(9, 19)]
COLS = (0, 17, 39)


@pytest.mark.parametrize("n", SWEEP)
@pytest.mark.parametrize("kind", [CHEB1, CHEBSTAR])
def test_dlt_idlt_sweep(n, kind):
    # the default plan (for N <= 8192 the direct method: the int8 tensor-core
    # product for 40 columns, the fp64 table product for one) and the
    # factored path (conversion + NDCT) in both NDCT modes
    dflt = fl.TransformConfig(n, TOL, K[kind])
    g = dflt.grid()
    fast = fl.TransformConfig(n, TOL, K[kind], grid=g, ndct_mode=fl.NDCT_FAST)
    fast.set_dlt_method(fl.DLT_FACTORED)
    lit = fl.TransformConfig(n, TOL, K[kind], grid=g, ndct_mode=fl.NDCT_LITERAL)
    lit.set_dlt_method(fl.DLT_FACTORED)
    c = fl.random_decaying(n, 0.5, 900 + n, batch=40)
    v = fl.random_decaying(n, 0.0, 5000 + n, batch=40)  # values at the nodes for the IDLT
    jobs_f = {j: POOL.submit(O.dlt_grid, c[j], kind, TOL, g.theta, g.x, g.weights) for j in COLS}
    jobs_b = {j: POOL.submit(O.idlt_grid, v[j], kind, TOL, g.theta, g.x, g.weights) for j in COLS}
    got = {}
    for name, cfg in (("default", dflt), ("factored fast", fast), ("factored literal", lit)):
        got[name] = (fl.dlt(c, cfg), fl.idlt(v, cfg).values, fl.dlt(c[0], cfg), fl.idlt(v[0], cfg).values)
    ref_f = {j: jobs_f[j].result() for j in COLS}
    ref_b = {j: jobs_b[j].result() for j in COLS}
    t = tol_n(n)
    for name, (f40, b40, f1, b1) in got.items():
        for j in COLS:
            assert rel(f40[j], ref_f[j], np.abs(c[j]).sum()) <= t, (name, "dlt", j)
            assert rel(b40[j], ref_b[j], np.abs(v[j]).sum()) <= t, (name, "idlt", j)
        assert rel(f1, ref_f[0], np.abs(c[0]).sum()) <= t, (name, "dlt batch 1")
        assert rel(b1, ref_b[0], np.abs(v[0]).sum()) <= t, (name, "idlt batch 1")


@pytest.mark.parametrize("kind", [CHEB1, CHEBSTAR])
def test_c2_ndct_65536_x_64_every_column(kind):
    """BASELINE config C2 exactly: the node kernel's grid, the plan's own
    kind and 2^-52 terms, 64 columns of iid N(0,1) (seeds 1000 + j)."""
    n, cols = 65536, 64
    c = fl.random_decaying(n, 0.0, 1000, batch=cols)
    grid = fl.legendre_nodes_weights(n)
    plan = fl.plan_ndct(grid, K[kind], TOL)
    delta = np.asarray(plan.reference.delta_theta)
    L = plan.num_terms
    jf = [POOL.submit(O.ndct, c[j], kind, L, delta) for j in range(cols)]
    jt = [POOL.submit(O.ndct, c[j], kind, L, delta, True) for j in range(cols)]
    f = fl.ndct_apply(plan, c)
    tr = fl.ndct_apply_transpose(plan, c)
    t = tol_n(n)
    for j in range(cols):
        s = np.abs(c[j]).sum()
        assert rel(f[j], jf[j].result(), s) <= t, ("ndct", j)
        assert rel(tr[j], jt[j].result(), s) <= t, ("ndct^T", j)


def test_c3_2_20_full_dlt_idlt_and_stages():
    """N = 2^20 (C3), default config (chebstar, fast mode, Toeplitz-Hankel
    conversion). Oracle: the C restatement's O(N^2) conversion (row-parallel,
    bit-identical to the serial loop) composed with the NumPy NDCT
    restatement on the injected grid."""
    n = 1 << 20
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    plan = cfg.plan()
    delta = np.asarray(plan.reference.delta_theta)
    c = fl.random_decaying(n, 1.0, 3)
    t = tol_n(n)
    # DLT: the conversion stage, the NDCT stage of its own output, the whole
    chat = cfg.convert(c)
    ref_chat = O.leg2cheb(c)
    assert rel(chat, ref_chat, np.abs(c).sum()) <= t
    f_stage = cfg.ndct(chat)
    assert rel(f_stage, NP.ndct_apply(chat, CHEBSTAR, plan.num_terms, delta), np.abs(chat).sum()) <= t
    f = fl.dlt(c, cfg)
    assert np.array_equal(f, f_stage)  # dlt = ndct(convert(c)) on the device
    assert rel(f, NP.ndct_apply(ref_chat, CHEBSTAR, plan.num_terms, delta), np.abs(c).sum()) <= t
    # IDLT: the weighted NDCT^T stage, the transposed conversion of its own
    # output, the whole against the composed oracle
    wf = g.weights * f
    vt = cfg.ndct(wf, transpose=True)
    ref_vt = NP.ndct_apply_transpose(wf, CHEBSTAR, plan.num_terms, delta)
    assert rel(vt, ref_vt, np.abs(wf).sum()) <= t
    m = np.arange(n) + 0.5
    back_stage = cfg.convert(vt, transpose=True)
    assert rel(back_stage, m * O.leg2cheb(vt, True), np.abs(vt).sum()) <= t
    back = fl.idlt(f, cfg).values
    assert rel(back, m * O.leg2cheb(ref_vt, True), np.abs(f).sum()) <= t
    assert np.max(np.abs(back - c)) <= 1e-7 * np.max(np.abs(c))


def _rows(n):
    rng = np.random.default_rng(n)
    inner = rng.integers(4, n - 4, 80)
    return sorted(set([0, 1, 2, 3, n // 2, n // 2 + 1, n - 4, n - 3, n - 2, n - 1] + list(inner)))


def test_c5_2_26_stages():
    """N = 2^26 (C5: c_n = g_n e^{-n/N}, 512 MiB), one GPU, default config.
    The conversion (Toeplitz-Hankel) at >= 90 sampled rows of the reference
    loop (conversion.hpp:106-111 / :126-133) incl. k = 0..3 and N-4..N-1; the
    NDCT / NDCT^T of the transform's own stage inputs against the full-length
    O(N log N) oracle (ndct.hpp:98-143). The reference's chebstar NDCT
    evaluates at theta*_k + delta_k (its exact grid angle plus the fp64
    offset); the oracle evaluates the same angles as cheb1 Taylor terms about
    theta0_k with the offsets re-based exactly, delta_k + (N - 2k - 1) pi /
    (2N(2N+1)) (|N delta'| <= 0.83845, the cheb1 bound, so L = 17 terms
    reach 2^-52): power-of-two transforms instead of length-(2N+1) ones,
    which do not fit the test's time at 2^26."""
    n = 1 << 26
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    assert np.all(np.diff(g.theta[:1000]) > 0) and g.theta[n - 1] == math.pi - g.theta[0]
    c = fl.random_decaying(n, 0.0, 5) * np.exp(-np.arange(n) / n)
    t = tol_n(n)
    lam = cfg.lambda_().table
    s = lam / lam[0]
    rows = _rows(n)
    sc = np.abs(c).sum()
    chat = cfg.convert(c)
    rows_pool = ThreadPoolExecutor(4)  # 2^25-element temporaries per row
    ref = list(rows_pool.map(lambda k: NP.leg2cheb_rows(c, s, [k])[0], rows))
    assert np.max(np.abs(chat[rows] - ref)) <= t * sc
    plan = cfg.plan()
    k = np.arange(n, dtype=np.float64)
    d1 = np.asarray(plan.reference.delta_theta) + (n - 2.0 * k - 1.0) * (math.pi / (2.0 * n * (2.0 * n + 1.0)))
    L1 = O.min_taylor_terms(CHEB1, TOL)
    assert np.max(np.abs(d1)) * n <= 0.83845
    f = cfg.ndct(chat)
    assert rel(f, NP.ndct_apply(chat, CHEB1, L1, d1), np.abs(chat).sum()) <= t
    wf = g.weights * f
    vt = cfg.ndct(wf, transpose=True)
    assert rel(vt, NP.ndct_apply_transpose(wf, CHEB1, L1, d1), np.abs(wf).sum()) <= t
    back = cfg.convert(vt, transpose=True)
    ref_t = list(rows_pool.map(lambda k: (k + 0.5) * NP.leg2cheb_transpose_rows(vt, s, [k])[0], rows))
    assert np.max(np.abs(back[rows] - ref_t)) <= t * np.abs(vt).sum()
    assert np.max(np.abs(back - c)) <= 1e-5 * np.max(np.abs(c))  # round trip: a sanity bound only


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built")
def test_gpu_vs_compiled_reference_4096():
    """The unmodified reference headers (oracle/_ref) against the GPU on one
    injected grid, both kinds: DLT, IDLT, NDCT, NDCT^T, conversion."""
    n = 4096
    for kind in (CHEB1, CHEBSTAR):
        cfg = fl.TransformConfig(n, TOL, K[kind])
        g = cfg.grid()
        c = fl.random_decaying(n, 0.5, 77, batch=20)
        f = fl.dlt(c, cfg)
        b = fl.idlt(f, cfg).values
        plan = fl.plan_ndct(g, K[kind], TOL)
        delta = np.asarray(plan.reference.delta_theta)
        nd, ndt = fl.ndct_apply(plan, c[3]), fl.ndct_apply_transpose(plan, c[3])
        l2c, l2ct = fl.leg2cheb_apply(fl.legendre_coefficients(c[3])).values, fl.leg2cheb_apply_transpose(c[3])
        for j in (0, 19):
            assert rel(f[j], REF.dlt_grid(c[j], kind, TOL, g.theta, g.x, g.weights), np.abs(c[j]).sum()) <= tol_n(n)
            assert rel(b[j], REF.idlt_grid(f[j], kind, TOL, g.theta, g.x, g.weights), np.abs(f[j]).sum()) <= tol_n(n)
        s = np.abs(c[3]).sum()
        assert rel(nd, REF.ndct(c[3], kind, plan.num_terms, delta), s) <= tol_n(n)
        assert rel(ndt, REF.ndct(c[3], kind, plan.num_terms, delta, True), s) <= tol_n(n)
        assert rel(l2c, REF.leg2cheb(c[3]), s) <= tol_n(n)
        assert rel(l2ct, REF.leg2cheb(c[3], True), s) <= tol_n(n)


@pytest.mark.parametrize("n", [512, 4096, 8192, 16384, 65536])
def test_free_functions_fast_vs_literal_vs_oracle(n):
    """The free functions at power-of-two N: ndct_apply / _transpose (both
    kinds) and the chebstar dct_iii / dst_iii / transposes run the Chebyshev
    expansion about cheb1 by default (fl_set_free_ndct_mode FAST) and the
    plan's literal Taylor terms / length-(2N+1) transforms as the ablation;
    both against the oracle, and the fast path takes fewer launches than the
    chebstar chirp-z path."""
    grid = fl.legendre_nodes_weights(n)
    c = fl.random_decaying(n, 0.0, 31 + n, batch=3)
    t = tol_n(n)
    trig = (fl.dct_iii, fl.dst_iii, fl.dct_iii_transpose, fl.dst_iii_transpose)
    refs = {}
    for kind in (CHEB1, CHEBSTAR):
        plan = fl.plan_ndct(grid, K[kind], TOL)
        d = np.asarray(plan.reference.delta_theta)
        refs[kind] = [(POOL.submit(O.ndct, c[j], kind, plan.num_terms, d),
                       POOL.submit(O.ndct, c[j], kind, plan.num_terms, d, True)) for j in range(3)]
    trig_refs = [[POOL.submit(O.trig, op, c[j], CHEBSTAR) for j in range(3)] for op in range(4)]
    launches = {}
    try:
        for mode in (fl.NDCT_FAST, fl.NDCT_LITERAL):
            fl.set_free_ndct_mode(mode)
            for kind in (CHEB1, CHEBSTAR):
                plan = fl.plan_ndct(grid, K[kind], TOL)
                l0 = fl.launch_count()
                f = fl.ndct_apply(plan, c)
                launches[(mode, kind)] = fl.launch_count() - l0
                tr = fl.ndct_apply_transpose(plan, c)
                for j in range(3):
                    s = np.abs(c[j]).sum()
                    assert rel(f[j], refs[kind][j][0].result(), s) <= t, (mode, kind, "ndct", j)
                    assert rel(tr[j], refs[kind][j][1].result(), s) <= t, (mode, kind, "ndct^T", j)
            for op in range(4):
                got = trig[op](c, fl.GridKind.chebstar)
                for j in range(3):
                    assert rel(got[j], trig_refs[op][j].result(), np.abs(c[j]).sum()) <= t, (mode, op, j)
    finally:
        fl.set_free_ndct_mode(fl.NDCT_FAST)
    assert launches[(fl.NDCT_FAST, CHEBSTAR)] < launches[(fl.NDCT_LITERAL, CHEBSTAR)], launches


def test_free_ndct_literal_when_truncation_is_visible():
    """A reduced tolerance (2^-23: L = 5 chebstar / 10 cheb1 Taylor terms)
    leaves a truncation error far above rounding: the free function keeps the
    literal evaluation (so it equals the reference to 1e-13 log2 N, not just
    to the 2^-23 bound), as does an all-zero offset vector."""
    n = 4096
    grid = fl.legendre_nodes_weights(n)
    c = fl.random_decaying(n, 0.0, 8)
    for kind in (CHEB1, CHEBSTAR):
        plan = fl.plan_ndct(grid, K[kind], 2.0 ** -23)
        d = np.asarray(plan.reference.delta_theta)
        assert rel(fl.ndct_apply(plan, c), O.ndct(c, kind, plan.num_terms, d), np.abs(c).sum()) <= tol_n(n)
        assert rel(fl.ndct_apply_transpose(plan, c), O.ndct(c, kind, plan.num_terms, d, True),
                   np.abs(c).sum()) <= tol_n(n)
    plan = fl.plan_ndct(n, fl.GridKind.cheb1, TOL)
    plan.reference.delta_theta = np.zeros(n)
    assert np.array_equal(fl.ndct_apply(plan, c), fl.dct_iii(c, fl.GridKind.cheb1))


@pytest.mark.parametrize("n", [1024, 4096, 65536])
def test_reduced_tolerance_dlt_idlt(n):
    """SURVEY.md 8f row f4, tolerance 2^-23 (L = 5 chebstar / 10 cheb1 Taylor
    terms in the reference). The literal factored path (FL_NDCT_LITERAL)
    reproduces the reference's truncated evaluation to 1e-13 log2 N; the
    defaults (the direct product for batches, the Chebyshev expansion to
    2^-23 otherwise) stay within the two certified bounds of it
    (test_ndct.cpp:173-183): |f - f_ref| <= (tol + C(L)) ||chat||_1 +
    1e-13 log2 N ||c||_1, C(L) the reference's bound, tol the plan's."""
    tol = 2.0 ** -23
    for kind in (CHEB1, CHEBSTAR):
        cfg = fl.TransformConfig(n, tol, K[kind])
        g = cfg.grid()
        c = fl.random_decaying(n, 0.5, 300 + n, batch=20)
        refs = [O.dlt_grid(c[j], kind, tol, g.theta, g.x, g.weights) for j in (0, 19)]
        bound = O.taylor_term_bound(kind, O.min_taylor_terms(kind, tol))
        f_def = fl.dlt(c, cfg)
        lit = fl.TransformConfig(n, tol, K[kind], grid=g, ndct_mode=fl.NDCT_LITERAL)
        lit.set_dlt_method(fl.DLT_FACTORED)
        f_lit = fl.dlt(c, lit)
        for j, ref in zip((0, 19), refs):
            chat = O.leg2cheb(c[j])
            assert rel(f_lit[j], ref, np.abs(c[j]).sum()) <= tol_n(n), (kind, "literal", j)
            lim = (tol + bound) * np.abs(chat).sum() + tol_n(n) * np.abs(c[j]).sum()
            assert np.max(np.abs(f_def[j] - ref)) <= lim, (kind, "default", j)
        b_lit = fl.idlt(f_lit, lit).values
        refb = O.idlt_grid(f_lit[0], kind, tol, g.theta, g.x, g.weights)
        assert rel(b_lit[0], refb, np.abs(f_lit[0]).sum()) <= tol_n(n), (kind, "literal idlt")
