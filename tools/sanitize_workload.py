"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
each hot kernel once at a small batch.

  compute-sanitizer --tool racecheck python tools/sanitize_workload.py [which]

which: all (default) | ndct | ndct_t | dct | gemm | big
  ndct   : fast_ndct_fwd_kernel<12,1> (fl_plan_ndct, N = 4096, 4 columns)
  ndct_t : fast_ndct_tr_kernel<12,1>  (the transpose)
  dct    : fast_dct_stream_fwd_kernel<12> + fast_dct_plain_tr_kernel (fl_trig)
  gemm   : oz_split_b_kernel + oz_gemm2_kernel (fl_plan_leg2cheb, 64 columns)
  big    : the multi-pass NDCT (N = 16384, 2 columns)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p


def main(which: str) -> None:
    n = 4096
    cfg = fl.TransformConfig(n)
    x = torch.from_numpy(fl.random_uniform_pm1(n, 4000, batch=64)).cuda()
    y = torch.empty_like(x)
    s = vp(torch.cuda.current_stream().cuda_stream)
    if which in ("all", "ndct"):
        _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), 4, n, s))
    if which in ("all", "ndct_t"):
        _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), 4, n, s))
    if which in ("all", "dct"):
        _lib.check(_lib.LIB.fl_trig(0, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), 64, n, s))
        _lib.check(_lib.LIB.fl_trig(2, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), 8, n, s))
    if which in ("all", "gemm"):
        _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), 64, n, s))
        _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), 64, n, s))
    if which in ("all", "big"):
        m = 16384
        big = fl.TransformConfig(m)
        xb = torch.from_numpy(fl.random_uniform_pm1(m, 5, batch=2)).cuda()
        yb = torch.empty_like(xb)
        _lib.check(_lib.LIB.fl_plan_ndct(big.handle, 0, vp(xb.data_ptr()), vp(yb.data_ptr()), 2, m, s))
        _lib.check(_lib.LIB.fl_plan_ndct(big.handle, 1, vp(xb.data_ptr()), vp(yb.data_ptr()), 2, m, s))
    torch.cuda.synchronize()
    print("sanitize workload done:", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
