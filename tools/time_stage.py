"""CUDA-event timing of one hot-path stage (development tool; the library is
the one FLB_LIB_PATH names, so experiment builds can be compared).

  python tools/time_stage.py STAGE N COLS [REPS]     (stages as tools/kernel_probe.py)
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
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    cfg = fl.TransformConfig(n)
    x = torch.from_numpy(fl.random_uniform_pm1(n, 4000, batch=cols)).cuda()
    y = torch.empty_like(x)
    st = torch.cuda.current_stream()
    s = vp(st.cuda_stream)
    L = _lib.LIB
    f = {
        "dlt": lambda: L.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "idlt": lambda: L.fl_idlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "ndct": lambda: L.fl_plan_ndct(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "ndct_t": lambda: L.fl_plan_ndct(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "conv": lambda: L.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "conv_t": lambda: L.fl_plan_leg2cheb(cfg.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "dct": lambda: L.fl_trig(0, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
        "dct_t": lambda: L.fl_trig(2, 0, n, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, s),
    }[stage]
    for _ in range(2):
        _lib.check(f())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        _lib.check(f())
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{stage} N={n} cols={cols}: {ms:.3f} ms  ({n * cols / ms / 1e6:.2f} G coef/s)"
          f"  lib={os.path.basename(_lib.LIB_PATH)}")


if __name__ == "__main__":
    main()
