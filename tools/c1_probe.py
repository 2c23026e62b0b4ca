"""C1 (N = 1024, one column) DLT / IDLT latency with a launch breakdown
(development tool): python tools/c1_probe.py [n]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = fl.TransformConfig(n)
x = torch.rand(1, n, dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty_like(x)
xh = x.cpu().numpy().copy()
yh = np.empty_like(xh)
vp = C.c_void_p


def dev():
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, None))


def host():
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(xh.ctypes.data), vp(yh.ctypes.data), 1, n, None))


for f in (dev, host):
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        f()
    torch.cuda.synchronize()
    print(f"{f.__name__}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per DLT (N={n}, 1 column)")
