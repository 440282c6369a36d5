import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd
from oracle.oracle import Oracle
c = Oracle("c")
d = np.load("tests/golden/solvers.npz")
for i in (4, 10):
    y, h, xs = d[f"pg_y{i}"], d[f"pg_h{i}"], tuple(int(v) for v in d[f"pg_xs{i}"])
    s_ref = c.estimate_step(h, xs, 30)
    s_gpu = nd.estimate_step(h, xs, 30)
    x0 = np.maximum(c.adjoint_apply(y, h, xs), 0)
    print(i, xs, h.shape, "step", s_ref, s_gpu)
    print("  adj", np.abs(nd.adjoint_apply(y, h, xs) - c.adjoint_apply(y, h, xs)).max(),
          "conv", np.abs(nd.conv_full(x0, h) - c.conv_full(x0, h)).max(),
          "grad", np.abs(nd.normal_gradient(x0, y, h) - c.normal_gradient(x0, y, h)).max())
    r1 = nd.deconv_pg(y, h, xs, nd.DeconvConfig(max_iters=1, tol_rel_objective=0.0, initial_step=s_ref))
    o1 = c.deconv_pg(y, h, xs, max_iters=1, tol_rel_objective=0.0, initial_step=s_ref)
    print("  1 iter f", r1.objective_trace, o1.objective_trace, "x diff", np.abs(r1.estimate - o1.estimate).max())
    print("  x gpu", r1.estimate.ravel()[:8], "\n  x ref", o1.estimate.ravel()[:8])
