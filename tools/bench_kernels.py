"""Per-kernel timing of the hot path at the C4 shape (development tool).

  python tools/bench_kernels.py [--n 4096] [--cols 65536] [--reps 5]

Times, with CUDA events on the launching stream, device-resident:
  dct    : one power-of-two cheb1 DCT-III pass (fl_trig)        -> GB/s vs HBM
  ndct   : fused Taylor NDCT, cheb1, L = 17 (fl_ndct)            -> TFLOP/s
  ndctT  : its transpose
  l2c    : leg2cheb direct (fl_leg2cheb)                         -> TFLOP/s
  l2cT   : its transpose
  dlt    : fl_dlt (chebstar plan, fast mode)
  idlt   : fl_idlt
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    n, cols = a.n, a.cols
    vp = C.c_void_p
    s = torch.cuda.current_stream()
    sp = vp(s.cuda_stream)
    x = torch.rand(cols, n, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    cfg = fl.TransformConfig(n)
    th = torch.from_numpy(cfg.grid().theta).cuda()
    d1 = torch.empty_like(th)
    _lib.check(_lib.LIB.fl_reference_grid(n, 0, vp(th.data_ptr()), None, vp(d1.data_ptr()), sp))
    lam = torch.from_numpy(cfg.lambda_().table).cuda()
    L1 = fl.min_taylor_terms(fl.GridKind.cheb1, 2.0 ** -52)

    def t(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    X, Y = vp(x.data_ptr()), vp(y.data_ptr())
    coef = n * cols
    ndct_fl = coef * L1 * (2.5 * math.log2(n) + 3)
    l2c_fl = coef * n / 2.0
    ops = {
        "dct": (lambda: _lib.check(_lib.LIB.fl_trig(0, 0, n, X, Y, cols, n, sp)), 16.0 * coef, "GB/s"),
        "dctT": (lambda: _lib.check(_lib.LIB.fl_trig(2, 0, n, X, Y, cols, n, sp)), 16.0 * coef, "GB/s"),
        "ndct": (lambda: _lib.check(_lib.LIB.fl_ndct(0, 0, n, L1, vp(d1.data_ptr()), X, Y, cols, n, sp)), ndct_fl, "TFLOP/s"),
        "ndctT": (lambda: _lib.check(_lib.LIB.fl_ndct(1, 0, n, L1, vp(d1.data_ptr()), X, Y, cols, n, sp)), ndct_fl, "TFLOP/s"),
        "l2c": (lambda: _lib.check(_lib.LIB.fl_leg2cheb(0, n, vp(lam.data_ptr()), n, X, Y, cols, n, sp)), l2c_fl, "TFLOP/s"),
        "l2cT": (lambda: _lib.check(_lib.LIB.fl_leg2cheb(1, n, vp(lam.data_ptr()), n, X, Y, cols, n, sp)), l2c_fl, "TFLOP/s"),
        "dlt": (lambda: _lib.check(_lib.LIB.fl_dlt(cfg.handle, X, Y, cols, n, sp)), 16.0 * coef, "GB/s"),
        "idlt": (lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, X, Y, cols, n, sp)), 16.0 * coef, "GB/s"),
    }
    res = {}
    for name, (fn, work, unit) in ops.items():
        if a.only and name not in a.only.split(","):
            continue
        ms = t(fn)
        rate = work / (ms / 1e3) / (1e9 if unit == "GB/s" else 1e12)
        res[name] = {"ms": round(ms, 3), unit: round(rate, 2), "Gcoef/s": round(coef / ms / 1e6, 3)}
        print(f"{name:6s} {ms:9.3f} ms  {rate:9.2f} {unit}  {coef / ms / 1e6:8.3f} Gcoef/s", flush=True)
    print(json.dumps({"n": n, "cols": cols, **res}))


if __name__ == "__main__":
    main()
