"""GPU: the z-slab sharded driver run as W in-process ranks on one GPU
(ndc_local_group: host-thread barrier + device-to-device halo copies -- no kernel ever
waits on another, so ranks can share a device).  The same Plan code drives the NCCL
transport across processes; only the Transport differs.

Checks: slab ownership covers both volumes, halos make every rank's convolutions equal
to the unsharded ones, the rank-order scalar combine keeps every rank's decisions
identical, and the assembled estimate matches the unsharded run and the oracle."""
import threading

import numpy as np
import pytest

from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def run_sharded(nd, world, y, h, x_shape, cfg):
    group = nd.LocalGroup(world)
    plans = [nd.Plan.local(group, r, x_shape, h) for r in range(world)]
    out = [None] * world
    errs = []

    def rank_main(r):
        try:
            p = plans[r]
            ya, yb = p.y_range
            p.set_observation(y[ya:yb])
            p.pg_begin(cfg)
            p.pg_iterate(cfg.max_iters)
            p.pg_end()
            out[r] = (p.estimate()[0], p.report(0, cfg.max_iters + 1), p.x_range)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for p in plans:
        p.close()
    group.close()
    x = np.concatenate([o[0] for o in sorted(out, key=lambda o: o[2][0])], axis=0)
    return x, [o[1] for o in out]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pg_matches_unsharded(nd, oracle_c, world):
    from paper_1711_11224_b200 import synth
    # config-4 PSF (21x9x9, p_z = 10) on a reduced volume: slabs of >= 10 planes
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0)
    xs, reps = run_sharded(nd, world, y, h, x.shape, cfg)
    full = nd.deconv_pg(y, h, x.shape, cfg)
    ref = oracle_c.deconv_pg(y, h, x.shape, max_iters=12, tol_rel_objective=0.0)
    assert xs.shape == x.shape
    # every rank took the same decisions (identical traces, iterations, stop reason)
    for r in reps[1:]:
        assert np.array_equal(r.objective_trace, reps[0].objective_trace)
        assert r.iterations_run == reps[0].iterations_run and r.stop_reason == reps[0].stop_reason
    assert reps[0].iterations_run == full.iterations_run == ref.iterations_run
    assert rel_l2(xs, full.estimate) <= 1e-5
    assert rel_l2(xs, ref.estimate) <= 1e-4
    np.testing.assert_allclose(reps[0].objective_trace, ref.objective_trace, rtol=1e-4)
    assert abs(reps[0].extra["step0"] - full.extra["step0"]) <= 1e-6 * full.extra["step0"]


def test_sharded_rejects_thin_slabs(nd):
    h = np.ones((21, 3, 3)) / 189.0
    group = nd.LocalGroup(4)
    with pytest.raises(nd.UnsupportedError):
        nd.Plan.local(group, 0, (20, 8, 8), h)  # 5-plane slabs < p_z = 10
    group.close()


def _run_env(tmp_path, world, step, **env):
    import os
    import subprocess
    import sys
    out = tmp_path / f"run_{world}_{step}_{'_'.join(f'{k}{v}' for k, v in env.items())}.npz"
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, os.path.join(root, "tests", "_sharded_run.py"), str(out), str(world),
                    str(step)], check=True, env=e, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("world,step", [(2, 0.0), (3, 0.0), (2, 8.0), (3, 8.0)])
def test_sharded_overlap_and_speculation_are_exact(nd, tmp_path, world, step):
    """The halo exchange overlapped with the interior planes (comm stream, per-buffer
    events) and the speculative next adjoint change only WHEN things run, never what is
    computed: estimates and traces are bit-identical to the serialised schedule.  World 3
    on 36 planes gives 12-plane slabs < 2 p_z = 20, where every plane of the middle rank
    is a boundary plane; initial_step = 8 forces backtracking (acceptance criterion 6's
    regime), which discards speculative passes."""
    base = _run_env(tmp_path, world, step, NDC_HALO_OVERLAP=0, NDC_SPECULATE=0)
    fast = _run_env(tmp_path, world, step)
    assert np.array_equal(base["x"], fast["x"])
    assert np.array_equal(base["obj"], fast["obj"]) and np.array_equal(base["kkt"], fast["kkt"])
    assert int(base["iters"]) == int(fast["iters"]) and str(base["reason"]) == str(fast["reason"])
    assert int(base["backtracks"]) == int(fast["backtracks"])
    if step == 8.0:
        assert int(fast["backtracks"]) > 0  # the backtracking path ran


def test_sharded_backtracking_matches_unsharded(nd):
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=8.0)
    xs, reps = run_sharded(nd, 2, y, h, x.shape, cfg)
    full = nd.deconv_pg(y, h, x.shape, cfg)
    assert reps[0].extra["backtracks"] == full.extra["backtracks"] > 0
    assert reps[0].iterations_run == full.iterations_run
    assert rel_l2(xs, full.estimate) <= 1e-5
    np.testing.assert_allclose(reps[0].objective_trace, full.objective_trace, rtol=1e-5)
