import numpy as np, sys
sys.path.insert(0, '.')
import paper_1505_00354_b200 as fl
n = 1 << 14
cfg = fl.TransformConfig(n); g = cfg.grid()
c = fl.random_decaying(n, 1.0, 3)
f_a = fl.dlt(fl.legendre_coefficients(c), cfg); f_b = fl.dlt(fl.legendre_coefficients(c), cfg)
print("dlt twice", np.max(np.abs(f_a - f_b)))
l_a = fl.leg2cheb_apply(fl.legendre_coefficients(c), cfg.lambda_()).values
l_b = fl.leg2cheb_apply(fl.legendre_coefficients(c)).values
print("l2c twice", np.max(np.abs(l_a - l_b)))
plan1 = fl.plan_ndct(g, fl.GridKind.cheb1, fl.default_tolerance)
n_a = fl.ndct_apply(plan1, l_a); n_b = fl.ndct_apply(plan1, l_a)
print("ndct twice", np.max(np.abs(n_a - n_b)), "vs dlt", np.max(np.abs(n_a - f_a)))
cfg.set_ndct_mode(fl.NDCT_LITERAL)
f_lit = fl.dlt(fl.legendre_coefficients(c), cfg)
print("dlt literal vs fast", np.max(np.abs(f_lit - f_a)))
th = fl.api._Arr(g.theta)
ref1 = fl.reference_grid(g, fl.GridKind.cheb1).delta_theta
print("delta equal", np.array_equal(ref1, plan1.reference.delta_theta))
