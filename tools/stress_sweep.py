"""Stride / batch / size sweep of dlt, idlt and fl_plan_leg2cheb on the GPU
(development tool): every case against the contiguous call (bit-identical),
sampled columns against the CPU oracle, the IDLT round trip, untouched
padding. python tools/stress_sweep.py [sizes...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from oracle import CHEBSTAR, ORACLE as O  # noqa: E402
from paper_1505_00354_b200 import _lib  # noqa: E402

vp = C.c_void_p
sizes = [int(a) for a in sys.argv[1:]] or [512, 1000, 1024, 2048, 4097, 8192, 16384]
rng = np.random.default_rng(11)
for n in sizes:
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    tol = 1e-13 * max(np.log2(n), 1.0)
    for batch in (1, 3, 17, 70):
        c = rng.uniform(-1, 1, (batch, n))
        f_ref = fl.dlt(torch.from_numpy(c).cuda(), cfg).cpu().numpy()
        b_ref = fl.idlt(torch.from_numpy(f_ref).cuda(), cfg).values.cpu().numpy()
        for j in {0, batch - 1}:
            ref = O.dlt_grid(c[j], CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
            e = np.max(np.abs(f_ref[j] - ref)) / np.abs(c[j]).sum()
            assert e <= tol, (n, batch, j, e)
        rt = np.max(np.abs(b_ref - c))
        assert rt <= 1e-10 * (n / 2048) * np.log2(n) / 11 + 1e-11, (n, batch, rt)
        for extra in (1, 2, 7):
            ld = n + extra
            x = torch.zeros(batch, ld, dtype=torch.float64, device="cuda")
            x[:, :n] = torch.from_numpy(c).cuda()
            f = torch.full_like(x, 7.0)
            _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(f.data_ptr()), batch, ld, None))
            b = torch.full_like(x, 5.0)
            _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(f.data_ptr()), vp(b.data_ptr()), batch, ld, None))
            m = torch.full_like(x, 3.0)
            _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()), vp(m.data_ptr()), batch, ld, None))
            mc = torch.empty(batch, n, dtype=torch.float64, device="cuda")
            xc = torch.from_numpy(c).cuda()
            _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 0, vp(xc.data_ptr()), vp(mc.data_ptr()), batch, n, None))
            fh, bh, mh = f.cpu().numpy(), b.cpu().numpy(), m.cpu().numpy()
            if batch > 1:
                assert np.all(fh[:, n:] == 7.0) and np.all(bh[:, n:] == 5.0) and np.all(mh[:, n:] == 3.0), (n, batch, ld)
            assert np.array_equal(fh[:, :n], f_ref), (n, batch, ld, "dlt")
            assert np.array_equal(bh[:, :n], b_ref), (n, batch, ld, "idlt")
            assert np.array_equal(mh[:, :n], mc.cpu().numpy()), (n, batch, ld, "leg2cheb")
        print(f"n={n} batch={batch} ok (round trip {rt:.1e})", flush=True)
print("sweep ok")
