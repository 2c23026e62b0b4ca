"""Split-int8 conversion product vs the fp64 (DMMA) one inside dlt/idlt
(development check): max difference relative to ||input||_1 and timings."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib

def run(n, cols, reps=3):
    torch.manual_seed(0)
    c = (torch.rand(cols, n, dtype=torch.float64, device="cuda") * 2 - 1).contiguous()
    cfg = fl.TransformConfig(n)
    out = {}
    for mode in (fl.GEMM_FP64, fl.GEMM_INT8_SPLIT):
        cfg.set_gemm_mode(mode)
        outs = []
        sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for inv in (False, True):
            y = torch.empty_like(c)
            call = _lib.LIB.fl_idlt if inv else _lib.LIB.fl_dlt
            fn = lambda call=call, y=y: _lib.check(call(cfg.handle, C.c_void_p(c.data_ptr()),
                                                        C.c_void_p(y.data_ptr()), cols, n, sp))
            fn(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record(); torch.cuda.synchronize()
            outs.append((y.clone(), e0.elapsed_time(e1) / reps))
        out[mode] = outs
    for k, name in enumerate(("dlt", "idlt")):
        a, ta = out[fl.GEMM_FP64][k]
        b, tb = out[fl.GEMM_INT8_SPLIT][k]
        l1 = c.abs().sum(dim=1)
        rel = ((a - b).abs().max(dim=1).values / l1).max().item()
        print(f"n={n} cols={cols} {name}: fp64 {ta:.3f} ms  int8split {tb:.3f} ms  max|diff|/||c||_1 = {rel:.3e}", flush=True)

for n, cols in ((512, 64), (1024, 100), (4096, 256), (4096, 65536)):
    run(n, cols)
