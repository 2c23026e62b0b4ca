import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib
n, cols = int(sys.argv[1]), int(sys.argv[2])
c = (torch.rand(cols, n, dtype=torch.float64, device="cuda") * 2 - 1)
y = torch.empty_like(c)
cfg = fl.TransformConfig(n)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(c.data_ptr()), C.c_void_p(y.data_ptr()), cols, n, sp))
torch.cuda.synchronize()
