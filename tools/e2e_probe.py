"""e2e probe (development): host-pinned fl_dlt at C4 and raw PCIe copy rates."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib
n, cols = 4096, 65536
xh = (torch.rand(cols, n, dtype=torch.float64) * 2 - 1).pin_memory()
yh = torch.empty_like(xh).pin_memory()
cfg = fl.TransformConfig(n)
vp = C.c_void_p
def step():
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(xh.data_ptr()), vp(yh.data_ptr()), cols, n, None))
step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(3): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
xd = torch.empty(cols, n, dtype=torch.float64, device="cuda")
def t(f):
    f(); torch.cuda.synchronize(); e0.record(); f(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
h2d = t(lambda: xd.copy_(xh, non_blocking=True))
d2h = t(lambda: yh.copy_(xd, non_blocking=True))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2): yh.copy_(xd[:], non_blocking=True)
    torch.cuda.synchronize()
import time
both(); t0 = time.perf_counter(); both(); dual = (time.perf_counter() - t0) * 1e3
print(f"{os.environ.get('FLB_LIB_PATH','default')}: e2e {ms:.1f} ms ({n*cols/ms/1e6:.2f} Gcoef/s); H2D {2*2**30/h2d/1e6:.1f} GB/s, D2H {2*2**30/d2h/1e6:.1f} GB/s, both-directions {dual:.1f} ms")
