"""CUDA-event timing of the Legendre -> Chebyshev conversion by the
asymptotic expansion against the Toeplitz-Hankel form, single vectors
(development tool).

  python tools/time_asy.py [LOG2N ...]     (default 14 16 18 20 22 24 26)
  FLB_ASY_M / FLB_ASY_R / FLB_ASY_LEVELS select the expansion's shape.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p


def timed(f, reps):
    st = torch.cuda.current_stream()
    for _ in range(1):
        _lib.check(f())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        _lib.check(f())
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main() -> None:
    logs = [int(a) for a in sys.argv[1:]] or [14, 16, 18, 20, 22, 24, 26]
    for lg in logs:
        n = 1 << lg
        cfg = fl.TransformConfig(n)
        x = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
        y = torch.empty_like(x)
        s = vp(torch.cuda.current_stream().cuda_stream)
        L = _lib.LIB
        reps = 5 if lg <= 22 else 2
        row = {}
        for mode, name in ((fl.LEG2CHEB_TOEPLITZ, "th"), (fl.LEG2CHEB_ASYMPTOTIC, "asy")):
            cfg.set_leg2cheb_mode(mode)
            for t in (0, 1):
                row[f"{name}{'_t' if t else ''}"] = min(timed(
                    lambda: L.fl_plan_leg2cheb(cfg.handle, t, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, s),
                    reps) for _ in range(3))
        info = cfg.leg2cheb_asy_info()
        print(f"2^{lg}: " + "  ".join(f"{k} {v:.3f} ms" for k, v in row.items()) + f"  {info}", flush=True)


if __name__ == "__main__":
    main()
