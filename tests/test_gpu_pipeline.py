"""Host-buffer dlt/idlt (>= 64 MiB of PINNED host columns): the column chunks
are pipelined over H2D | compute | D2H streams inside the call (pageable
buffers take one copy each way instead; both give the same bits). Results must be
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


def pinned(a):
    """A page-locked copy of a (numpy view of a pinned torch tensor)."""
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    v = t.numpy()  # the array's base keeps the pinned storage alive
    v[...] = a
    return v


def _call(fn, cfg, x, y, batch, ld):
    _lib.check(fn(cfg.handle, C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data), batch, ld, None))


@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("pin", [True, False])
def test_pipelined_host_matches_device(inverse, pin):
    import torch
    n, batch = 4096, 2100  # 66 MiB of columns: pipelined, last chunk ragged
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 31, batch=batch)
    dev = torch.from_numpy(c).cuda()
    x = pinned(c) if pin else c
    y = pinned(np.zeros_like(c)) if pin else np.zeros_like(c)
    fn = _lib.LIB.fl_idlt if inverse else _lib.LIB.fl_dlt
    ref = (fl.idlt(dev, cfg).values if inverse else fl.dlt(dev, cfg)).cpu().numpy()
    _call(fn, cfg, x, y, batch, n)
    assert np.array_equal(y, ref)


def test_pipelined_host_strided():
    n, batch, ld = 4096, 2048, 4096 + 24
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 8, batch=batch)
    x = np.zeros((batch, ld))
    x[:, :n] = c
    x = pinned(x)
    y = pinned(np.full((batch, ld), 5.0))
    _call(_lib.LIB.fl_dlt, cfg, x, y, batch, ld)
    assert np.array_equal(y[:, :n], fl.dlt(c, cfg))
    assert np.all(y[:, n:] == 5.0)


def test_pipelined_nonfinite_in_last_chunk():
    n, batch = 4096, 2048
    cfg = fl.TransformConfig(n)
    c = fl.random_uniform_pm1(n, 4, batch=batch)
    c = pinned(c)
    y = pinned(np.zeros_like(c))
    c[batch - 1, 17] = np.nan
    with pytest.raises(fl.InvalidArgument):
        _call(_lib.LIB.fl_dlt, cfg, c, y, batch, n)
    c[batch - 1, 17] = -np.inf
    with pytest.raises(fl.InvalidArgument):
        _call(_lib.LIB.fl_idlt, cfg, c, y, batch, n)
