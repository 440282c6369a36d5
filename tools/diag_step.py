import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd
from oracle.oracle import Oracle
c = Oracle("c")
g = np.random.Generator(np.random.PCG64(1))
cases = [((2, 1), (5, 1)), ((4, 5), (3, 1)), ((5,), (3,)), ((8,), (5,)), ((2, 3), (5, 1)), ((6, 6), (3, 3)),
         ((2, 1), (1, 1)), ((3, 4), (1, 3)), ((4,), (1,)), ((1, 4), (3, 3)), ((2, 2, 2), (3, 1, 1)), ((2, 2, 2), (1, 3, 1))]
for xs, hs in cases:
    h = g.uniform(-1, 1, hs)
    out = []
    for it in (1, 2, 30):
        out.append((round(c.estimate_step(h, xs, it), 6), round(nd.estimate_step(h, xs, it), 6)))
    v = np.ones(xs) / np.sqrt(np.prod(xs))
    w_ref = c.adjoint_apply(c.conv_full(v, h), h, xs)
    w_gpu = nd.adjoint_apply(nd.conv_full(v, h), h, xs)
    print(xs, hs, out, "opsdiff", np.abs(w_ref - w_gpu).max())
