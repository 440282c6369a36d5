"""Helper for tests/test_gpu_guards.py, run with NDC_GUARD_BANDS=1: exercises the device
paths with the riskiest addressing (tap chunks through scratch, edge tiles, packed
widths, deep z-chunks, speculation with staggered stops, backtracking, RL, z-slab ranks,
power iterations, tensor-file streaming, device noise) twice each, checks that every run
is bit-identical to its repeat (a data race would show up as run-to-run differences), and
prints the process-wide count of changed guard bytes as JSON."""
import json
import os
import sys
import tempfile
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_11224_b200 import ndconv as nd, synth  # noqa: E402


def cases():
    rng = np.random.default_rng(9)
    out = []
    for xs, hs in [((37, 50), (3, 35)), ((60, 90), (37, 71)), ((50, 40), (201, 3)), ((9, 30, 70), (3, 5, 67)),
                   ((124, 100), (15, 15)), ((231, 90), (31, 31)), ((6, 64, 64), (5, 15, 15)),
                   ((12, 40, 50), (9, 33, 33)), ((70, 20, 36), (65, 33, 33)), ((140, 140), (11, 11)),
                   ((130, 150), (3, 3)), ((4, 64, 64), (3, 7, 7))]:
        x = rng.uniform(0, 1, xs)
        h = rng.uniform(0, 1, hs)
        out.append((x, h / h.sum()))
    return out


def run_all():
    res = []
    for x, h in cases():
        y = nd.conv_full(x, h)
        res.append(y)
        res.append(nd.adjoint_apply(y, h, x.shape))
        rep = nd.deconv_pg(y + 1e-3, h, x.shape, nd.DeconvConfig(max_iters=3, tol_rel_objective=0.0, initial_step=1.0))
        res.append(rep.estimate)
    # staggered stops with speculation, backtracking
    xs4, y4, h4 = synth.make("c1", batch=4, shape=(40, 36), n_objects=8)
    y4 = np.stack([y4[0], y4[2], y4[3], -np.abs(y4[1]) - 0.1])
    for r in nd.deconv_pg_batch(y4, h4, (40, 36), nd.DeconvConfig(max_iters=80, tol_rel_objective=2e-3)):
        res.append(r.estimate)
    d = np.load(os.path.join(ROOT, "tests", "golden", "solvers.npz"))
    i = int(d["npg"]) - 2
    res.append(nd.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], (32, 32),
                            nd.DeconvConfig(max_iters=100, tol_rel_objective=0.0, initial_step=8.0)).estimate)
    # plan: RL, guards checked while the plan is alive
    bad = 0
    with nd.Plan((40, 36), h4, batch=2) as p:
        p.set_observation(y4[:2])
        p.rl_run(nd.RlConfig(max_iters=5))
        res.append(p.estimate())
        p.pg_run(nd.DeconvConfig(max_iters=5, tol_rel_objective=0.0))
        res.append(p.estimate())
        with tempfile.TemporaryDirectory() as td:
            p.save_estimate(os.path.join(td, "x.ndt"))
            res.append(nd.read_tensor(os.path.join(td, "x.ndt")))
        p.add_gaussian_noise(0.0, 0.01, 5)
        res.append(p.observation())
        bad += p.check_guards()
    # step estimates: float64 device path, float32 device path (non-separable, > 2^28)
    hh = np.outer(np.hanning(15)[1:-1] + 0.1, np.hanning(7)[1:-1] + 0.2)[:, :5]
    hh[0, 0] += 0.05
    res.append(np.array([nd.estimate_step(hh, (96, 80), 30), nd.estimate_step(hh, (2048, 2048), 30)]))
    # z-slab ranks over the in-process transport
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    for world in (2, 3):
        group = nd.LocalGroup(world)
        plans = [nd.Plan.local(group, r, x.shape, h) for r in range(world)]
        outs = [None] * world

        def rank_main(r):
            pl = plans[r]
            ya, yb = pl.y_range
            pl.set_observation(y[ya:yb])
            pl.pg_run(nd.DeconvConfig(max_iters=6, tol_rel_objective=0.0))
            outs[r] = pl.estimate()[0]

        th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for pl in plans:
            bad += pl.check_guards()
            pl.close()
        group.close()
        res.append(np.concatenate(outs, axis=0))
    return res, bad


a, bad_a = run_all()
b, bad_b = run_all()
same = all(np.array_equal(u, v) for u, v in zip(a, b)) and len(a) == len(b)
print(json.dumps({"arrays": len(a), "repeat_bit_identical": bool(same), "live_plan_bad": int(bad_a + bad_b),
                  "total_guard_violations": int(nd.guard_violations())}))
