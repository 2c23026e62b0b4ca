"""The cluster-fused forward NDCT (N = 2^14, 2^15, cluster_ndct_fwd_kernel:
one column per thread-block cluster of N/8192 CTAs, the N/2-point FFT of each
Chebyshev-expansion term as a four-step over the cluster with the exchange
through distributed shared memory). It runs for batches whose packed rows
(terms x columns) exceed the multi-pass path's 8 GiB scratch; checked against
the oracle and against the multi-pass path (a few columns of the same block)
at the north star's tolerance."""
import math

import numpy as np
import pytest

from oracle import CHEBSTAR, ORACLE as O
import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,cols", [(16384, 2400), (32768, 1200)])
def test_cluster_ndct_vs_oracle_and_multipass(n, cols):
    import torch
    grid = fl.legendre_nodes_weights(n)
    plan = fl.plan_ndct(grid, fl.GridKind.chebstar, fl.default_tolerance)
    delta = np.asarray(plan.reference.delta_theta)
    c = fl.random_decaying(n, 0.0, 77, batch=cols)
    f = fl.ndct_apply(plan, torch.from_numpy(c).cuda()).cpu().numpy()   # cluster kernel
    few = fl.ndct_apply(plan, c[:3])                                     # multi-pass
    tol = 1e-13 * math.log2(n)
    for j in (0, 1, 2):
        s = np.abs(c[j]).sum()
        assert np.max(np.abs(f[j] - few[j])) <= tol * s, j
    for j in (0, cols // 2, cols - 1):
        ref = O.ndct(c[j], CHEBSTAR, plan.num_terms, delta)
        assert np.max(np.abs(f[j] - ref)) <= tol * np.abs(c[j]).sum(), j
    # bit-reproducible and batch-invariant (per-column arithmetic)
    f2 = fl.ndct_apply(plan, torch.from_numpy(c).cuda()).cpu().numpy()
    assert np.array_equal(f, f2)


def test_cluster_dlt_batched_65536():
    """The factored DLT of a 2^16 batch (multi-pass NDCT, direct conversion)."""
    n, cols = 65536, 128
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    c = fl.random_decaying(n, 1.0, 5, batch=cols)
    f = fl.dlt(c, cfg)
    for j in (0, cols - 1):
        ref = O.dlt_grid(c[j], CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        assert np.max(np.abs(f[j] - ref)) <= 1e-13 * 16 * np.abs(c[j]).sum(), j
