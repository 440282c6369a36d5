"""Phase breakdown of an end-to-end solve through the plan API (output buffer reused,
as a caller streaming many solves would).  usage: python tools/e2e_phases.py [c2|c2s]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1711_11224_b200 import _native as N, ndconv as nd, synth  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
x, y, h = synth.make(cfg_name)
y64 = np.ascontiguousarray(y, np.float64)
out = np.empty(x.shape, np.float64)
out.fill(0.0)  # touch the pages once
for rep in range(3):
    t = [time.perf_counter()]
    p = nd.Plan(x.shape[1:], h, batch=x.shape[0]); t.append(time.perf_counter())
    p.set_observation(y64); t.append(time.perf_counter())
    p.pg_begin(nd.DeconvConfig(max_iters=100, tol_rel_objective=0.0)); t.append(time.perf_counter())
    p.pg_iterate(100); t.append(time.perf_counter())
    p.pg_end(); t.append(time.perf_counter())
    N.lib().ndc_plan_get_estimate_f64(p.handle, out.ctypes.data_as(N.dbl_p)); t.append(time.perf_counter())
    p.close(); t.append(time.perf_counter())
    names = ["create", "H2D+pack", "begin(step,x0,f)", "100 iters", "end(kkt)", "D2H+unpack", "destroy"]
    print(cfg_name, " ".join(f"{n}={1e3*(b-a):.1f}ms" for n, a, b in zip(names, t, t[1:])),
          f"total={1e3*(t[-1]-t[0]):.1f}ms", flush=True)
