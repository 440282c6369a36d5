"""Two forward + adjoint passes of a BASELINE-shaped plan on zero inputs, for ncu captures of a
single launch (`ncu --set full --import-source on -k regex:correlate -s N -c 1 python
tools/ncu_run_cfg.py c4s`, then tools/ncu_lines.py on the report)."""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd, synth
name = sys.argv[1]
SH = {"c4s": (1, (64, 1024, 1024)), "c3": (1, (128, 256, 256)), "c5s": (1, (16, 2048, 2048)), "c2": (16, (2048, 2048))}
B, xs = SH[name]
h = synth.psf_for(name[:2])
ys = tuple(s + k - 1 for s, k in zip(xs, h.shape))
p = nd.Plan(xs, h, batch=B)
p.set_observation(np.zeros((B,) + ys, np.float32))
for _ in range(2):
    p.forward(); p.adjoint()
p.close()
