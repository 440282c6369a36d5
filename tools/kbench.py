"""Kernel micro-benchmark: device time of the PG forward (residual epilogue) / adjoint (PG
epilogue) correlation passes on a BASELINE config shape (inputs are zeros -- FFMA time
does not depend on values); GB/s are the passes' algorithmic bytes."""
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
          "c4s": (1, (64, 1024, 1024)), "c5s": (1, (16, 2048, 2048)),
          "c5": (1, (256, 2048, 2048)), "c5m": (1, (64, 2048, 2048)), "c1": (1, (256, 256)),
          "c2k1": (16, (2048, 2048)), "c2k3": (16, (2048, 2048)), "c2k5": (16, (2048, 2048)),
          "c2k9": (16, (2048, 2048)), "c2k11": (16, (2048, 2048)), "c2k13": (16, (2048, 2048)),
          "c2k15": (16, (2048, 2048)), "c2k17": (16, (2048, 2048)), "c2k21": (16, (2048, 2048)),
          "c2k25": (16, (2048, 2048)), "c2k33": (16, (2048, 2048))}
for name in a.configs:
    B, xs = SHAPES[name] if name in SHAPES else (16, (2048, 2048))  # c2k<N>: N x N Gaussian
    if name.startswith("c2b"):  # c2b<N>: config 2 with a batch of N images (wave-tail sizing)
        B, name = int(name[3:]), "c2"
    if name.startswith("c3k"):  # c3k<N>: N x N x N Gaussian on a 256 x 512 x 512 volume
        B, xs = 1, (256, 512, 512)
        h = synth.gaussian_psf((int(name[3:]),) * 3, 1.0)
    elif name == "c2k1":
        h = np.ones((1, 1))
    elif name.startswith("c2k"):
        h = synth.gaussian_psf((int(name[3:]),) * 2, 1.0)
    else:
        h = synth.psf_for(name[:2])
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
    # algorithmic bytes of the PG passes (Plan::bench_forward / bench_adjoint):
    # forward reads x and Y, writes r; adjoint reads r and x, writes trial and g
    nx, ny = B * int(np.prod(xs)), B * int(np.prod(ys))
    fb, ab = 4.0 * (nx + 2 * ny), 4.0 * (ny + 3 * nx)
    print(f"{name}: x {xs} x{B} K={K}  fwd {f_ms:.3f} ms ({flops / f_ms / 1e9:.1f} TF, "
          f"{fb / f_ms / 1e6:.0f} GB/s)  adj {a_ms:.3f} ms ({flops / a_ms / 1e9:.1f} TF, "
          f"{ab / a_ms / 1e6:.0f} GB/s)  launches/pass {nf // a.reps}", flush=True)
    p.close()
