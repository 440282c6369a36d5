"""Phase breakdown of the end-to-end config-2 solve through the plan API."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd, synth
x, y, h = synth.make("c2")
y64 = np.ascontiguousarray(y, np.float64)
for rep in range(2):
    t = [time.perf_counter()]
    p = nd.Plan(x.shape[1:], h, batch=16); t.append(time.perf_counter())
    p.set_observation(y64); t.append(time.perf_counter())
    p.pg_begin(nd.DeconvConfig(max_iters=100, tol_rel_objective=0.0)); t.append(time.perf_counter())
    p.pg_iterate(100); t.append(time.perf_counter())
    p.pg_end(); t.append(time.perf_counter())
    est = p.estimate(); t.append(time.perf_counter())
    p.close(); t.append(time.perf_counter())
    names = ["create", "H2D+pack", "begin(step,x0,f)", "100 iters", "end(kkt)", "D2H+unpack", "destroy"]
    print(" ".join(f"{n}={1e3*(b-a):.1f}ms" for n, a, b in zip(names, t, t[1:])), f"total={1e3*(t[-1]-t[0]):.1f}ms")
