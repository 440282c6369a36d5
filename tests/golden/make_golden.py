"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libndconv_ref.so,
i.e. /root/reference/proj/include compiled unmodified behind oracle/ref_shim.cpp).

Run in the build container (the only place /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are committed; tests on the GPU box only read them.

Cases (reference test each restates, file:line under /root/reference/proj/tests/):
  kat_*        test_convolution.cpp:11-19, 40-45, 104-108; test_solvers.cpp:12-22, 24-40
  rand_conv    random family ndim<=3, extents<=5, radii<=2 (verification.hpp:54-60)
  pg_*         test_solvers.cpp:62-112 (identity, sparse, negative data, monotone family)
  pg_accept6   acceptance.cpp:171-206 (32x32 sparse, 5x5 sigma 1, step 8, 500 iterations)
  pg_c1        BASELINE config 1 (256x256, 15x15 sigma 2, 50 iterations) incl. estimate_step
  rl_*         test_solvers.cpp:191-278 (flux conservation family)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1711_11224_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rand_family(g, n, max_ndim=3, max_ext=5, max_rad=2):
    cases = []
    for _ in range(n):
        nd = int(g.integers(1, max_ndim + 1))
        xs = tuple(int(v) for v in g.integers(1, max_ext + 1, nd))
        hs = tuple(int(2 * v + 1) for v in g.integers(0, max_rad + 1, nd))
        cases.append((g.uniform(-1, 1, xs), g.uniform(-1, 1, hs)))
    return cases


BIG = [((96, 97), (5, 5)), ((200, 130), (15, 31)), ((9, 40, 37), (5, 7, 9)),
       ((6, 40, 36), (13, 3, 33)), ((3, 5, 300), (3, 1, 1)), ((1000,), (33,))]


def big_inputs(i):
    """Deterministic inputs of BIG[i] (numpy PCG64 is platform-independent)."""
    xs, hs = BIG[i]
    g = np.random.Generator(np.random.PCG64(7000 + i))
    x = g.uniform(-1, 1, xs)
    h = g.uniform(-1, 1, hs)
    r = g.uniform(-1, 1, tuple(a + b - 1 for a, b in zip(xs, hs)))
    return x, h, r


def main():
    ref = Oracle("ref")
    ref.set_threads(os.cpu_count() or 1)
    g = np.random.Generator(np.random.PCG64(20240915))

    # --- operators -------------------------------------------------------------------
    d = {}
    cases = rand_family(g, 40)
    d["n"] = len(cases)
    for i, (x, h) in enumerate(cases):
        y = ref.conv_full(x, h)
        r = g.uniform(-1, 1, y.shape)
        d[f"x{i}"], d[f"h{i}"], d[f"y{i}"] = x, h, y
        d[f"r{i}"], d[f"atr{i}"] = r, ref.adjoint_apply(r, h, x.shape)
    # larger 2-D / 3-D instances (device tiling, halos, tap chunking paths); inputs are
    # regenerated from big_inputs(i) so only the reference outputs are stored
    d["nbig"] = len(BIG)
    for i in range(len(BIG)):
        x, h, r = big_inputs(i)
        d[f"by{i}"] = ref.conv_full(x, h)
        d[f"batr{i}"] = ref.adjoint_apply(r, h, x.shape)
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **d)

    # --- solver fixtures ---------------------------------------------------------------
    d = {}
    # estimate_step KATs and a random family
    d["step_h1"] = ref.estimate_step(np.array([1.0]), (5,), 10)
    d["step_h2"] = ref.estimate_step(np.array([2.0]), (5,), 10)
    d["step_box"] = ref.estimate_step(np.ones(3), (8,), 30)
    pg_cases = []
    for i, (x, h) in enumerate(rand_family(np.random.Generator(np.random.PCG64(41)), 15, 2, 6, 2)):
        if not np.any(h != 0):
            continue
        y = np.random.Generator(np.random.PCG64(100 + i)).uniform(-1, 1, ref.conv_full(x, h).shape)
        pg_cases.append((y, h, x.shape, dict(max_iters=40, tol_rel_objective=0.0)))
    # test_solvers.cpp:62-93
    pg_cases.append((np.array([3.0, -2.0, 0.0, 5.0]), np.array([1.0]), (4,), dict(max_iters=50)))
    pg_cases.append((ref.conv_full(np.array([0.0, 4.0, 0.0]), np.array([0.0, 1.0, 0.0])),
                     np.array([0.0, 1.0, 0.0]), (3,), dict(max_iters=200, tol_rel_objective=0.0)))
    pg_cases.append((np.full(6, -2.0), np.array([0.2, 0.5, 0.3]), (4,), dict(max_iters=100)))
    # acceptance.cpp:171-206 (backtracking regime)
    truth = np.zeros((32, 32))
    ag = np.random.Generator(np.random.PCG64(1006))
    for rr in range(4, 32, 9):
        for cc in range(4, 32, 9):
            truth[rr, cc] = ag.uniform(0.5, 2.0)
    psf = synth.gaussian_psf((5, 5), 1.0)
    pg_cases.append((ref.conv_full(truth, psf), psf, (32, 32),
                     dict(max_iters=500, tol_rel_objective=0.0, initial_step=8.0)))
    # BASELINE config 1, auto step (power iteration) and default tolerance off
    x1, y1, h1 = synth.make("c1")
    pg_cases.append((y1, h1, x1.shape, dict(max_iters=50, tol_rel_objective=0.0)))
    d["c1_step"] = ref.estimate_step(h1, x1.shape, 30)
    d["npg"] = len(pg_cases)
    for i, (y, h, xs, kw) in enumerate(pg_cases):
        rep = ref.deconv_pg(y, h, xs, **kw)
        d[f"pg_y{i}"], d[f"pg_h{i}"], d[f"pg_xs{i}"] = y, h, np.array(xs)
        d[f"pg_cfg{i}"] = np.array([kw.get("max_iters", 500), kw.get("tol_rel_objective", 1e-6),
                                    kw.get("initial_step", 0.0) or 0.0])
        d[f"pg_x{i}"], d[f"pg_obj{i}"], d[f"pg_kkt{i}"] = rep.estimate, rep.objective_trace, rep.kkt_trace
        d[f"pg_it{i}"] = rep.iterations_run
        d[f"pg_stop{i}"] = np.array(rep.stop_reason)
    # Richardson-Lucy flux family (test_solvers.cpp:191-220)
    rg = np.random.Generator(np.random.PCG64(43))
    rl = []
    for _ in range(8):
        nd = int(rg.integers(1, 3))
        xs = tuple(int(v) for v in rg.integers(1, 6, nd))
        hs = tuple(int(2 * v + 1) for v in rg.integers(0, 2, nd))
        h = rg.uniform(0.05, 1.0, hs)
        x = rg.uniform(0.05, 1.0, xs)
        rl.append((ref.conv_full(x, h), h, xs))
    rl.append((np.array([1.0, -0.5, 2.0, -0.1, 3.0, 0.0]), np.array([0.25, 0.5, 0.25]), (4,)))
    d["nrl"] = len(rl)
    for i, (y, h, xs) in enumerate(rl):
        rep = ref.deconv_rl(y, h, xs, max_iters=7, tol_rel_change=0.0)
        d[f"rl_y{i}"], d[f"rl_h{i}"], d[f"rl_xs{i}"] = y, h, np.array(xs)
        d[f"rl_x{i}"], d[f"rl_obj{i}"], d[f"rl_kkt{i}"] = rep.estimate, rep.objective_trace, rep.kkt_trace
        d[f"rl_clamped{i}"] = rep.extra["negative_pixels_clamped"]
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **d)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
