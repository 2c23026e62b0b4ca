"""One C5 DLT (N = 2^26) for a launch-list profile (development tool)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
cfg = fl.TransformConfig(n)
c = torch.from_numpy(fl.random_decaying(n, 0.0, 5) * np.exp(-np.arange(n) / n)).cuda()
y = torch.empty_like(c)
_lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(c.data_ptr()), C.c_void_p(y.data_ptr()), 1, n, None))
torch.cuda.synchronize()
