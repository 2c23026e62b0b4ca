"""Batched plain DCT-III pass (N = 4096 x 65536 columns, device-resident) for
an ncu capture of the streaming DCT kernel (development tool)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1505_00354_b200 import _lib  # noqa: E402

n = 4096
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
op = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # fl_trig_op: 0 DCT-III, 1 DST-III, 2/3 transposes
x = torch.rand(batch, n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    _lib.check(_lib.LIB.fl_trig(op, 0, n, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), batch, n, None))
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    _lib.check(_lib.LIB.fl_trig(op, 0, n, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), batch, n, None))
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"trig op {op} {n} x {batch}: {ms:.3f} ms, {2 * 8 * n * batch / ms / 1e6:.0f} GB/s")
