"""e2e A/B (development): host-pinned fl_dlt at C4, repeated, with the PCIe
duplex floor measured between repetitions; min / median in ms."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

n, cols = 4096, 65536
xh = (torch.rand(cols, n, dtype=torch.float64) * 2 - 1).pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = torch.empty(cols, n, dtype=torch.float64, device="cuda")
cfg = fl.TransformConfig(n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def dlt():
    _lib.check(_lib.LIB.fl_dlt(cfg.handle, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), cols, n, None))


def duplex():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(xd, non_blocking=True)
    torch.cuda.synchronize()


dlt()
duplex()
e, d = [], []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    t0 = time.perf_counter(); dlt(); torch.cuda.synchronize(); e.append((time.perf_counter() - t0) * 1e3)
    t0 = time.perf_counter(); duplex(); d.append((time.perf_counter() - t0) * 1e3)
print(f"ramp={os.environ.get('FLB_PIPE_RAMP', '1')}: e2e min {min(e):.1f} med {statistics.median(e):.1f} ms;"
      f" duplex floor min {min(d):.1f} med {statistics.median(d):.1f} ms")
