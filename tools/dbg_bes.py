"""Fast-mode NDCT accuracy (development check): DLT / IDLT error against the
oracle on the injected grid, relative to ||input||_1, for whichever library
FLB_LIB_PATH selects (Bessel or Taylor expansion about cheb1)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1505_00354_b200 as fl
from oracle import ORACLE as O
for n in (1024, 4096, 8192):
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    for name, c in (("uniform", fl.random_uniform_pm1(n, 11, batch=4)), ("decay", fl.random_decaying(n, 1.0, 12, batch=4))):
        f = fl.dlt(c, cfg)
        b = fl.idlt(f, cfg).values
        ef = max(np.max(np.abs(f[j] - O.dlt_grid(c[j], 1, fl.default_tolerance, g.theta, g.x, g.weights))) / np.abs(c[j]).sum() for j in range(4))
        eb = max(np.max(np.abs(b[j] - O.idlt_grid(f[j], 1, fl.default_tolerance, g.theta, g.x, g.weights))) / np.abs(f[j]).sum() for j in range(4))
        print(f"{os.environ.get('FLB_LIB_PATH','bessel')} n={n} {name}: dlt {ef:.2e} idlt {eb:.2e}")
