"""Host-buffer dlt/idlt (>= 64 MiB of host columns): the column chunks are
pipelined over H2D | compute | D2H streams inside the call. Results must be
bit-identical to the device-resident call (per-column arithmetic does not
depend on the chunking), strided host blocks must be honoured and a
non-finite value in any chunk must still raise invalid_argument.
"""
import ctypes as C

import numpy as np
import pytest

import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib

pytestmark = pytest.mark.gpu


def _call(fn, cfg, x, y, batch, ld):
    _lib.check(fn(cfg.handle, C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data), batch, ld, None))


@pytest.mark.parametrize("inverse", [False, True])
def test_pipelined_host_matches_device(inverse):
    import torch
    n, batch = 4096, 2100  # 66 MiB of columns: pipelined, last chunk ragged
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 31, batch=batch)
    dev = torch.from_numpy(c).cuda()
    if inverse:
        ref = fl.idlt(dev, cfg).values.cpu().numpy()
        got = fl.idlt(c, cfg).values
    else:
        ref = fl.dlt(dev, cfg).cpu().numpy()
        got = fl.dlt(c, cfg)
    assert np.array_equal(got, ref)


def test_pipelined_host_strided():
    n, batch, ld = 4096, 2048, 4096 + 24
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 8, batch=batch)
    x = np.zeros((batch, ld))
    x[:, :n] = c
    y = np.full((batch, ld), 5.0)
    _call(_lib.LIB.fl_dlt, cfg, x, y, batch, ld)
    assert np.array_equal(y[:, :n], fl.dlt(c, cfg))
    assert np.all(y[:, n:] == 5.0)


def test_pipelined_nonfinite_in_last_chunk():
    n, batch = 4096, 2048
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4, batch=batch)
    c[batch - 1, 17] = np.nan
    with pytest.raises(fl.InvalidArgument):
        fl.dlt(c, cfg)
    c[batch - 1, 17] = -np.inf
    with pytest.raises(fl.InvalidArgument):
        fl.idlt(c, cfg)
