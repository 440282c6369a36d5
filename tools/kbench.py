"""Kernel micro-benchmark: device time of the forward / adjoint correlation passes on a
BASELINE config shape (inputs are zeros -- FFMA time does not depend on values)."""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["c2"])
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
SHAPES = {"c2": (16, (2048, 2048)), "c3": (1, (128, 256, 256)), "c4": (1, (512, 1024, 1024)),
          "c4s": (1, (64, 1024, 1024)), "c5s": (1, (16, 2048, 2048)), "c1": (1, (256, 256)),
          "c2k5": (16, (2048, 2048)), "c2k9": (16, (2048, 2048)), "c2k3": (16, (2048, 2048))}
for name in a.configs:
    B, xs = SHAPES[name]
    h = synth.gaussian_psf((int(name[3:]),) * 2, 1.0) if name.startswith("c2k") else synth.psf_for(name[:2])
    K = int(np.prod(h.shape))
    ys = tuple(s + k - 1 for s, k in zip(xs, h.shape))
    p = nd.Plan(xs, h, batch=B)
    p.set_observation(np.zeros((B,) + ys, np.float32))
    p.forward(); p.adjoint()
    p.reset_stats(); p.set_timing(True)
    for _ in range(a.reps):
        p.forward(); p.adjoint()
    nf, msf = p.stats(0)
    na, msa = p.stats(1)
    flops = 2.0 * K * B * int(np.prod(xs))
    f_ms, a_ms = msf / a.reps, msa / a.reps
    nbytes = 4.0 * B * (int(np.prod(xs)) + int(np.prod(ys)))  # read one volume, write the other
    print(f"{name}: x {xs} x{B} K={K}  fwd {f_ms:.3f} ms ({flops / f_ms / 1e9:.1f} TF, "
          f"{nbytes / f_ms / 1e6:.0f} GB/s)  adj {a_ms:.3f} ms ({flops / a_ms / 1e9:.1f} TF, "
          f"{nbytes / a_ms / 1e6:.0f} GB/s)  launches/pass {nf // a.reps}", flush=True)
    p.close()
