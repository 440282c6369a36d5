"""Where do the device and reference PG trajectories part in the backtracking regime?"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd
d = np.load("tests/golden/solvers.npz")
for i in range(int(d["npg"])):
    cfg = d[f"pg_cfg{i}"]
    kw = dict(max_iters=int(cfg[0]), tol_rel_objective=float(cfg[1]))
    if cfg[2] > 0:
        kw["initial_step"] = float(cfg[2])
    rep = nd.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], tuple(int(v) for v in d[f"pg_xs{i}"]), nd.DeconvConfig(**kw))
    a, b = rep.objective_trace, d[f"pg_obj{i}"]
    n = min(len(a), len(b))
    rel = np.abs(a[:n] - b[:n]) / np.maximum(np.abs(b[:n]), 1e-300)
    first = int(np.argmax(rel > 1e-4)) if np.any(rel > 1e-4) else -1
    x = rep.estimate; xr = d[f"pg_x{i}"]
    print(i, rep.stop_reason, str(d[f"pg_stop{i}"]), rep.iterations_run, int(d[f"pg_it{i}"]), "bt", rep.extra["backtracks"],
          "first>1e-4 at", first, "f there", (a[first], b[first], b[0]) if first >= 0 else None,
          "relL2 x", np.linalg.norm(x - xr) / max(np.linalg.norm(xr), 1e-300))
