"""Timings of the BASELINE.json parity configurations besides the C4 headline
(bench.py): device-resident inputs, CUDA events, plan construction timed
separately. Prints one JSON line per config.

  C1: DLT + IDLT, N = 1024, c_n = g_n/(n+1)^0.5 (seed 1)
  C2: NDCT only, N = 65536 x 64 columns, iid N(0,1) (seeds 1000+j), cheb1 plan
  C3: DLT + IDLT, N = 2^20, c_n = g_n/(n+1) (seed 3)
  C5: DLT + IDLT, N = 2^26, c_n = g_n e^{-n/N} (seed 5), one GPU

  python tools/bench_configs.py [--only c1,c2,c3,c5] [--reps 5]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run(name, reps):
    sp = vp(torch.cuda.current_stream().cuda_stream)
    if name == "c2":
        n, cols = 65536, 64
        c = np.stack([fl.random_decaying(n, 0.0, 1000 + j) for j in range(cols)])
        t0 = time.perf_counter()
        grid = fl.legendre_nodes_weights(n)
        plan = fl.plan_ndct(grid, fl.GridKind.cheb1, fl.default_tolerance)
        t_plan = time.perf_counter() - t0
        x = torch.from_numpy(c).cuda()
        y = torch.empty_like(x)
        d = torch.from_numpy(np.asarray(plan.reference.delta_theta)).cuda()
        fwd = timed(lambda: _lib.check(_lib.LIB.fl_ndct(0, 0, n, plan.num_terms, vp(d.data_ptr()), vp(x.data_ptr()),
                                                        vp(y.data_ptr()), cols, n, sp)), reps)
        tr = timed(lambda: _lib.check(_lib.LIB.fl_ndct(1, 0, n, plan.num_terms, vp(d.data_ptr()), vp(x.data_ptr()),
                                                       vp(y.data_ptr()), cols, n, sp)), reps)
        return {"config": "C2 NDCT N=65536 x 64, iid N(0,1), cheb1 plan (L=17)", "plan_s": t_plan,
                "ndct_ms": fwd, "ndct_T_ms": tr, "ndct_coeffs_per_s": n * cols / fwd * 1e3,
                "ndct_T_coeffs_per_s": n * cols / tr * 1e3}
    spec = {"c1": (1024, 0.5, 1, "C1 DLT/IDLT N=1024"), "c3": (1 << 20, 1.0, 3, "C3 DLT/IDLT N=2^20"),
            "c5": (1 << 26, 0.0, 5, "C5 DLT/IDLT N=2^26 (one GPU)")}[name]
    n, decay, seed, desc = spec
    c = fl.random_decaying(n, decay, seed)
    if name == "c5":
        c = c * np.exp(-np.arange(n) / n)
    t0 = time.perf_counter()
    cfg = fl.TransformConfig(n)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t0
    x = torch.from_numpy(c).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    dlt = timed(lambda: _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, sp)), reps)
    idlt = timed(lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(y.data_ptr()), vp(z.data_ptr()), 1, n, sp)), reps)
    rt = float((z - x).abs().max() / x.abs().max())
    return {"config": desc, "plan_s": t_plan, "dlt_ms": dlt, "idlt_ms": idlt,
            "dlt_coeffs_per_s": n / dlt * 1e3, "idlt_coeffs_per_s": n / idlt * 1e3,
            "leg2cheb": ("asymptotic expansion " + json.dumps(cfg.leg2cheb_asy_info())
                         if n >= (1 << 16) and n & (n - 1) == 0
                         else "toeplitz-hankel" if cfg.leg2cheb_rank(0) else "direct"),
            "round_trip_rel": rt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,c5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for name in a.only.split(","):
        print(json.dumps(run(name, a.reps if name != "c5" else 2)), flush=True)


if __name__ == "__main__":
    main()
