"""GPU: the direct O(N^2) evaluations of oracle.hpp as device kernels
 against the CPU oracle, and used as an independent check
of the fast DLT at a size where the CPU oracle would be slow."""
import math

import numpy as np
import pytest

from conftest import EPS
from oracle import ORACLE as O
import oracle
import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu


def test_eval_direct_known_answers():  # test_oracle.cpp:22-56
    P2 = fl.legendre_coefficients([0.0, 0.0, 1.0])
    v = fl.eval_legendre_direct(P2, [1.0, 0.0])
    assert abs(v[0] - 1.0) <= 4 * EPS and abs(v[1] + 0.5) <= 4 * EPS
    P3 = fl.legendre_coefficients([0.0, 0.0, 0.0, 1.0])
    assert abs(fl.eval_legendre_direct(P3, [0.3])[0] + 0.3825) <= 1e-15
    T2 = fl.chebyshev_coefficients([0.0, 0.0, 1.0])
    assert abs(fl.eval_chebyshev_direct(T2, [1.0, 0.0])[1] + 1.0) <= 4 * EPS
    with pytest.raises(fl.DomainError):
        fl.eval_legendre_direct(P2, [1.5])
    with pytest.raises(fl.DomainError):
        fl.eval_chebyshev_direct(T2, [-1.0000001])
    with pytest.raises(fl.InvalidArgument):
        fl.eval_legendre_direct(T2, [0.0])


@pytest.mark.parametrize("n", [1, 2, 17, 256, 1000])
def test_eval_direct_vs_oracle(n):
    rng = np.random.default_rng(n)
    c = rng.standard_normal(n)
    xs = np.cos(rng.uniform(0, np.pi, 300))
    scale = np.abs(c).sum()
    assert np.max(np.abs(fl.eval_legendre_direct(fl.legendre_coefficients(c), xs)
                         - O.eval_legendre_direct(c, xs))) <= 1e-13 * scale
    assert np.max(np.abs(fl.eval_chebyshev_direct(fl.chebyshev_coefficients(c), xs)
                         - O.eval_chebyshev_direct(c, xs))) <= 1e-13 * scale


@pytest.mark.parametrize("n", [1, 2, 8, 300, 1024])
def test_idlt_direct_vs_oracle(n):
    g = fl.legendre_nodes_weights(n)
    f = np.random.default_rng(n).standard_normal(n)
    got = fl.idlt_direct(f, g).values
    ref = oracle.idlt_direct(f, g.x, g.weights)
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(math.log2(n), 1) * np.abs(f).sum()


def test_cheb_coeffs_of_legendre():  # test_oracle.cpp:112-129, acceptance.cpp:245-257
    for n in (0, 1, 2, 7, 32):
        got = fl.cheb_coeffs_of_legendre(n, 80)
        assert np.max(np.abs(got - O.cheb_coeffs_of_legendre(n, 80))) <= 1e-14
    cache = fl.LambdaCache(64)
    for n in range(20):
        got = fl.cheb_coeffs_of_legendre(n, 80)
        for k in range(n + 1):
            assert abs(fl.leg2cheb_entry(k, n, cache) - got[k]) <= 1e-13
    with pytest.raises(fl.InvalidArgument):
        fl.cheb_coeffs_of_legendre(5, 5)


def test_fast_dlt_against_device_direct_large():
    """N = 2^16: the fast DLT against the device's own O(N^2) evaluation at all
    nodes, and the fast IDLT against idlt_direct (independent code paths)."""
    n = 1 << 16
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    c = fl.random_decaying(n, 1.0, 3)
    f = fl.dlt(fl.legendre_coefficients(c), cfg)
    direct = fl.eval_legendre_direct(fl.legendre_coefficients(c), g.x)
    assert np.max(np.abs(f - direct)) <= 1e-10 * np.abs(c).sum()
    back = fl.idlt(f, cfg).values
    back_direct = fl.idlt_direct(f, g).values
    assert np.max(np.abs(back - back_direct)) <= 1e-10 * np.abs(f).sum()
    assert np.max(np.abs(back - c)) <= 1e-9 * np.max(np.abs(c))
