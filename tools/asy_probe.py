"""One asymptotic conversion (forward and transposed) per size, for ncu
launch lists (development tool).

  python tools/asy_probe.py LOG2N [LOG2N ...]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    cfg = fl.TransformConfig(n)
    cfg.set_leg2cheb_mode(fl.LEG2CHEB_ASYMPTOTIC)
    x = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
    y = torch.empty_like(x)
    s = vp(torch.cuda.current_stream().cuda_stream)
    for t in (0, 1):
        _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, t, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, s))
    torch.cuda.synchronize()
    print(lg, cfg.leg2cheb_asy_info(), flush=True)
