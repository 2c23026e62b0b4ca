"""CPU: pin the oracle (C restatement) against the reference's own known
answers and against the reference itself (golden vectors produced by the
unmodified reference headers, tests/golden/make_golden.py)."""
import math

import numpy as np
import pytest

from conftest import EPS, unhex
from oracle import CHEB1, CHEBSTAR, ORACLE as O, REF
import oracle


def test_restatement_matches_reference_golden_bitwise(ref_vectors):
    for n, d in ref_vectors["nodes"].items():
        th, x, w = O.nodes_weights(int(n))
        assert np.array_equal(th, unhex(d["theta"]))
        assert np.array_equal(x, unhex(d["x"]))
        assert np.array_equal(w, unhex(d["w"]))
    for t in ref_vectors["trig"]:
        assert np.array_equal(O.trig(t["op"], unhex(t["in"]), t["kind"]), unhex(t["out"])), t["n"]
    for t in ref_vectors["ndct"]:
        c, delta = unhex(t["in"]), unhex(t["delta"])
        assert np.array_equal(O.ndct(c, t["kind"], t["L"], delta), unhex(t["fwd"]))
        assert np.array_equal(O.ndct(c, t["kind"], t["L"], delta, True), unhex(t["tr"]))
    for t in ref_vectors["leg2cheb"]:
        c = unhex(t["in"])
        assert np.array_equal(O.leg2cheb(c), unhex(t["fwd"]))
        assert np.array_equal(O.leg2cheb(c, True), unhex(t["tr"]))
    assert np.array_equal(O.lambda_table(64), unhex(ref_vectors["lambda"]))
    for t in ref_vectors["transforms"]:
        th, x, w, c = (unhex(t[k]) for k in ("theta", "x", "w", "c"))
        f = O.dlt_grid(c, t["kind"], EPS, th, x, w)
        assert np.array_equal(f, unhex(t["f"]))
        assert np.array_equal(O.idlt_grid(f, t["kind"], EPS, th, x, w), unhex(t["back"]))


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built")
def test_restatement_matches_compiled_reference_random():
    rng = np.random.default_rng(0)
    for n in (3, 31, 200):
        th, x, w = REF.nodes_weights(n)
        assert np.array_equal(np.array(O.nodes_weights(n)), np.array((th, x, w)))
        c = rng.standard_normal(n)
        for kind in (CHEB1, CHEBSTAR):
            assert np.array_equal(O.dlt_grid(c, kind, EPS, th, x, w), REF.dlt_grid(c, kind, EPS, th, x, w))
            assert np.array_equal(O.idlt_grid(c, kind, EPS, th, x, w), REF.idlt_grid(c, kind, EPS, th, x, w))


def test_closed_form_rules():  # test_quadrature.cpp:59-85
    th, x, w = O.nodes_weights(1)
    assert th[0] == math.pi / 2 and x[0] == 0.0 and w[0] == 2.0
    th, x, w = O.nodes_weights(2)
    assert abs(x[0] - 1 / math.sqrt(3)) <= 4 * EPS and abs(x[1] + 1 / math.sqrt(3)) <= 4 * EPS
    assert np.all(np.abs(w - 1.0) <= 4 * EPS)
    th, x, w = O.nodes_weights(3)
    assert abs(x[0] - math.sqrt(0.6)) <= 8 * EPS and x[1] == 0.0
    assert abs(w[0] - 5 / 9) <= 8 * EPS and abs(w[1] - 8 / 9) <= 8 * EPS
    with pytest.raises(oracle.OracleError):
        O.nodes_weights(0)


def test_node_invariants():  # test_quadrature.cpp:99-128
    for n in (1, 2, 5, 16, 17, 64, 257):
        th, x, w = O.nodes_weights(n)
        assert np.all(np.diff(th) > 0) and np.all(np.diff(x) < 0)
        assert np.array_equal(w, w[::-1])
        assert abs(w.sum() - 2.0) <= 16 * EPS * n


def test_known_answers():
    # Lambda values, test_conversion.cpp:29, :39-56
    t = O.lambda_table(64)
    assert t[0] == pytest.approx(1.77245385090551603, abs=4 * EPS)
    assert t[1] == pytest.approx(0.886226925452758014, abs=4 * EPS)
    assert t[50] == pytest.approx(0.141068250297538267, rel=1e-14)
    assert oracle.lambda_ratio(0.5, 64) == pytest.approx(1.12837916709551257, rel=1e-14)
    assert oracle.lambda_ratio(10.25, 64) == pytest.approx(0.308563027939506361, rel=1e-14)
    assert oracle.lambda_ratio(35.5, 64) == pytest.approx(0.16724635756231336, rel=1e-14)
    with pytest.raises(oracle.OracleError):
        oracle.lambda_ratio(-1.0, 64)
    # M entries, test_conversion.cpp:61-68
    assert O.leg2cheb_entry(0, 0, 8) == pytest.approx(1.0, abs=4 * EPS)
    assert O.leg2cheb_entry(0, 2, 8) == pytest.approx(0.25, abs=4 * EPS)
    assert O.leg2cheb_entry(2, 2, 8) == pytest.approx(0.75, abs=4 * EPS)
    assert O.leg2cheb_entry(1, 2, 8) == 0.0 and O.leg2cheb_entry(3, 2, 8) == 0.0
    # P_3(0.3) = -0.3825, test_oracle.cpp:27-29
    assert O.eval_legendre_direct([0, 0, 0, 1], [0.3])[0] == pytest.approx(-0.3825, abs=1e-15)
    # term counts, test_ndct.cpp:40-43
    assert O.min_taylor_terms(CHEBSTAR, 2.0 ** -52) == 9
    assert O.min_taylor_terms(CHEB1, 2.0 ** -52) == 17
    assert O.min_taylor_terms(CHEBSTAR, 2.0 ** -23) == 5
    assert O.min_taylor_terms(CHEB1, 2.0 ** -23) == 10
    # Table 1, acceptance.cpp:64-69 (two significant figures)
    row1 = [8.4e-1, 3.5e-1, 9.8e-2, 2.1e-2, 3.5e-3, 4.8e-4, 5.8e-5, 6.1e-6, 5.6e-7, 4.7e-8, 3.6e-9,
            2.5e-10, 1.6e-11, 9.7e-13, 5.4e-14, 2.9e-15, 1.4e-16, 6.6e-18]
    for l, v in enumerate(row1, 1):
        assert abs(O.taylor_term_bound(CHEB1, l) - v) <= 10 ** (math.floor(math.log10(v)) - 1)
    # std::mt19937_64: the 10000th output for the default seed (C++ standard)
    assert O.mt19937_64_nth(5489, 10000) == 9981545732273789042


def test_oracle_trig_direct_sums():  # test_trig.cpp:131-155
    for n in range(1, 65):
        c = np.random.default_rng(n).uniform(-1, 1, n)
        for kind in (CHEB1, CHEBSTAR):
            k = np.arange(n)
            th = (k + 0.5) * np.pi / n if kind == CHEB1 else (k + 0.75) * np.pi / (n + 0.5)
            Cm, Sm = np.cos(np.outer(th, k)), np.sin(np.outer(th, k))
            tol = 100 * EPS * n * np.abs(c).sum()
            for op, ref in enumerate((Cm @ c, Sm @ c, Cm.T @ c, Sm.T @ c)):
                assert np.max(np.abs(O.trig(op, c, kind) - ref)) <= tol


def test_oracle_nodes_vs_truth(nodes_truth):
    """The reference's Newton nodes against 40-digit truth: the error model
    |dtheta| <= 4 eps / sin(theta)."""
    for n, rows in nodes_truth["nodes"].items():
        th, x, w = O.nodes_weights(int(n))
        for r in rows:
            t = float(r["theta"])
            assert abs(th[r["k"]] - t) <= 4 * EPS / math.sin(t) + 2 * EPS
            assert abs(w[r["k"]] - float(r["w"])) <= (8 / math.sin(t) ** 2 + int(n) / 64 + 16) * EPS * float(r["w"])


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("n", [1024, 4096, 16384])
def test_restatement_matches_compiled_reference_transforms_large(n):
    """The pins above stop at N = 256; the GPU parity sweep runs to 2^18. The
    restatement's DLT / IDLT on an injected grid equal the compiled
    reference's bit for bit at the sweep's sizes where the reference's O(N^2)
    conversion still runs in well under a second (both kinds)."""
    th, x, w = O.nodes_weights(n)
    rng = np.random.default_rng(n + 7)
    c = rng.standard_normal(n) / np.sqrt(np.arange(n) + 1.0)
    for kind in (CHEB1, CHEBSTAR):
        f = O.dlt_grid(c, kind, EPS, th, x, w)
        assert np.array_equal(f, REF.dlt_grid(c, kind, EPS, th, x, w)), kind
        assert np.array_equal(O.idlt_grid(f, kind, EPS, th, x, w), REF.idlt_grid(f, kind, EPS, th, x, w)), kind


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built")
def test_restatement_matches_compiled_reference_ndct_65536():
    """C2's size: the restatement's NDCT / NDCT^T equal the compiled
    reference's bit for bit on a perturbed grid, both kinds."""
    n = 65536
    th = (np.arange(n) + 0.5) * np.pi / n + 0.3 / n * np.sin(np.arange(n))
    c = np.random.default_rng(3).standard_normal(n)
    for kind, L in ((CHEB1, 17), (CHEBSTAR, 9)):
        d = O.reference_delta(n, kind, th)
        assert np.array_equal(O.ndct(c, kind, L, d), REF.ndct(c, kind, L, d)), kind
        assert np.array_equal(O.ndct(c, kind, L, d, True), REF.ndct(c, kind, L, d, True)), kind


@pytest.mark.parametrize("n", [1, 2, 7, 1000, 4096, 65536])
def test_numpy_restatement_matches_c_oracle(n):
    """oracle/ndct_np.py (the large-N NDCT oracle: pocketfft at the FFT
    boundary) against the C restatement: the r2r passes and the NDCT / NDCT^T
    agree to FFT rounding (<= 1e-15 ||c||_1), both kinds."""
    from oracle import ndct_np as NP
    rng = np.random.default_rng(n)
    c = rng.standard_normal(n)
    th = (np.arange(n) + 0.5) * np.pi / n + 0.3 / n * np.sin(np.arange(n) + 1.0)
    s = np.abs(c).sum()
    fns = (NP.dct_iii, NP.dst_iii, NP.dct_iii_transpose, NP.dst_iii_transpose)
    for kind, L in ((CHEB1, 17), (CHEBSTAR, 9)):
        for op in range(4):
            assert np.max(np.abs(O.trig(op, c, kind) - fns[op](c, kind))) <= 1e-15 * s, (kind, op)
        d = O.reference_delta(n, kind, th)
        assert np.max(np.abs(O.ndct(c, kind, L, d) - NP.ndct_apply(c, kind, L, d))) <= 1e-15 * s
        assert np.max(np.abs(O.ndct(c, kind, L, d, True) - NP.ndct_apply_transpose(c, kind, L, d))) <= 1e-15 * s


def test_numpy_leg2cheb_rows_match_c_oracle():
    n = 3001
    c = np.random.default_rng(5).standard_normal(n)
    lam = O.lambda_table(n - 1)
    s = lam / lam[0]
    from oracle import ndct_np as NP
    rows = [0, 1, 2, 3, 100, 1500, n - 2, n - 1]
    full, full_t = O.leg2cheb(c), O.leg2cheb(c, True)
    assert np.max(np.abs(NP.leg2cheb_rows(c, s, rows) - full[rows])) <= 1e-15 * np.abs(c).sum()
    assert np.max(np.abs(NP.leg2cheb_transpose_rows(c, s, rows) - full_t[rows])) <= 1e-15 * np.abs(c).sum()
