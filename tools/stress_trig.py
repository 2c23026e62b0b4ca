"""Stride / batch sweep of fl_trig (the four DCT/DST passes, both grids) and
fl_ndct on the GPU (development tool): strided against contiguous calls
(equal, or within 1e-15 ||x||_1 where a different kernel runs), sampled
columns against the CPU oracle, untouched padding."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from oracle import CHEB1, CHEBSTAR, ORACLE as O  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p
rng = np.random.default_rng(5)
for n in (64, 1000, 4096, 8192, 16384):
    for batch in (1, 5, 300):
        c = rng.standard_normal((batch, n))
        xc = torch.from_numpy(c).cuda()
        for kind, ok in ((0, CHEB1), (1, CHEBSTAR)):
            for op in range(4):
                yc = torch.empty_like(xc)
                _lib.check(_lib.LIB.fl_trig(op, kind, n, vp(xc.data_ptr()), vp(yc.data_ptr()), batch, n, None))
                ych = yc.cpu().numpy()
                j = batch - 1
                ref = O.trig(op, c[j], ok)
                e = np.max(np.abs(ych[j] - ref)) / np.abs(c[j]).sum()
                assert e <= 1e-13 * max(np.log2(n), 1), (n, batch, kind, op, e)
                for extra in (1, 2):
                    ld = n + extra
                    x = torch.zeros(batch, ld, dtype=torch.float64, device="cuda")
                    x[:, :n] = xc
                    y = torch.full_like(x, 9.0)
                    _lib.check(_lib.LIB.fl_trig(op, kind, n, vp(x.data_ptr()), vp(y.data_ptr()), batch, ld, None))
                    yh = y.cpu().numpy()
                    if batch > 1:
                        assert np.all(yh[:, n:] == 9.0), (n, batch, kind, op, ld)
                    d = np.max(np.abs(yh[:, :n] - ych) / np.abs(c).sum(axis=1, keepdims=True))
                    assert d <= 1e-15, (n, batch, kind, op, ld, d)
        print(f"n={n} batch={batch} trig ok", flush=True)
print("trig sweep ok")
