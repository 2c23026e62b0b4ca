"""One hot-path stage on device-resident columns, for ncu captures (the
profiled process must exit 0 without ncu first; timings under ncu are not
bench numbers).

  python tools/kernel_probe.py STAGE N COLS [REPS]

STAGE: dlt | idlt | ndct | ndct_t | conv | conv_t | dct | dct_t | ndct_free
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p


def main() -> None:
    stage, n, cols = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    cfg = fl.TransformConfig(n)
    x = torch.from_numpy(fl.random_uniform_pm1(n, 4000, batch=cols)).cuda()
    y = torch.empty_like(x)
    s = vp(torch.cuda.current_stream().cuda_stream)
    L = _lib.LIB
    plan = fl.plan_ndct(cfg.grid(), fl.GridKind.chebstar, fl.default_tolerance)
    d = torch.from_numpy(__import__("numpy").asarray(plan.reference.delta_theta)).cuda()
    calls = {
        "dlt": lambda: L.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "idlt": lambda: L.fl_idlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "ndct": lambda: L.fl_plan_ndct(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "ndct_t": lambda: L.fl_plan_ndct(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "conv": lambda: L.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "conv_t": lambda: L.fl_plan_leg2cheb(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "dct": lambda: L.fl_trig(0, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "dct_t": lambda: L.fl_trig(2, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "ndct_free": lambda: L.fl_ndct(0, 1, n, plan.num_terms, vp(d.data_ptr()), vp(x.data_ptr()),
                                       vp(y.data_ptr()), cols, n, s),
    }
    for _ in range(reps):
        _lib.check(calls[stage]())
    torch.cuda.synchronize()
    print("probe done", stage, n, cols, reps)


if __name__ == "__main__":
    main()
