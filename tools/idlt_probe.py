"""Device-resident batched IDLT (N = 4096) for an ncu capture of the NDCT^T
kernel (development tool): python tools/idlt_probe.py [cols]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

n = 4096
cols = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = torch.rand(cols, n, dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty_like(x)
cfg = fl.TransformConfig(n)
for _ in range(2):
    _lib.check(_lib.LIB.fl_idlt(cfg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), cols, n, None))
torch.cuda.synchronize()
