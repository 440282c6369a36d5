import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd
d = np.load("tests/golden/solvers.npz")
i = 18
cfg = d[f"pg_cfg{i}"]
rep = nd.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], (32, 32), nd.DeconvConfig(max_iters=500, tol_rel_objective=0.0, initial_step=8.0))
a, b = rep.objective_trace, d[f"pg_obj{i}"]
rel = np.abs(a - b) / np.abs(b)
for k in list(range(0, 60, 3)) + list(range(60, 501, 40)):
    print(k, a[k], b[k], rel[k])
