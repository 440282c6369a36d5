"""GPU: the NCCL z-slab transport (ndc_comm.cu NcclTransport).

* one rank on one GPU: the full transport sequence (ncclCommInitRank, the per-pass
  raw reduction -> ncclAllGather -> rank-order combine) runs for real and gives the
  unsharded plan's bits;
* W = 2 / 3 processes, one GPU each (skipped below W devices): every rank's estimate
  slab, the traces, iteration count, stop reason and backtracks are bit-identical to
  the in-process LocalTransport run of the same slabs (tests/test_gpu_sharded.py),
  with and without backtracking.  NCCL_DEBUG=INFO lines go to <tmp>/nccl.<rank>.log.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _devices():
    import torch
    return torch.cuda.device_count()


def test_nccl_single_rank_matches_unsharded(nd):
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    for step in (None, 8.0):
        cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=step)
        p = nd.Plan.sharded(x.shape, h, 0, 1, nd.nccl_unique_id(), device=0)
        assert p.x_range == (0, 36) and p.y_range == (0, 56)
        p.set_observation(y)
        p.pg_run(cfg)
        got, rep = p.estimate()[0], p.report(0, 13)
        p.close()
        full = nd.deconv_pg(y, h, x.shape, cfg)
        assert np.array_equal(got, full.estimate), step
        assert np.array_equal(rep.objective_trace, full.objective_trace), step
        assert np.array_equal(rep.kkt_trace, full.kkt_trace), step
        assert rep.iterations_run == full.iterations_run and rep.extra["backtracks"] == full.extra["backtracks"]


@pytest.mark.parametrize("world,step", [(2, 0.0), (2, 8.0), (3, 0.0), (3, 8.0)])
def test_nccl_ranks_match_local_transport(nd, tmp_path, world, step):
    if _devices() < world:
        pytest.skip(f"needs {world} GPUs (one process per GPU)")
    from paper_1711_11224_b200 import synth
    from tests.test_gpu_sharded import run_sharded
    uid = tmp_path / "uid"
    procs = []
    for r in range(world):
        env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT",
                   NCCL_DEBUG_FILE=str(tmp_path / f"nccl.{r}.log"))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_nccl_rank.py"),
                                       str(tmp_path / f"r{r}.npz"), str(r), str(world), str(uid), str(step)],
                                      env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    x, yv, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=step if step > 0 else None)
    xs_local, reps = run_sharded(nd, world, yv, h, x.shape, cfg)
    xs_nccl = np.concatenate([o["x"] for o in sorted(outs, key=lambda o: int(o["x_range"][0]))], axis=0)
    assert np.array_equal(xs_nccl, xs_local)
    for o in outs:
        assert np.array_equal(o["obj"], reps[0].objective_trace)
        assert np.array_equal(o["kkt"], reps[0].kkt_trace)
        assert int(o["iters"]) == reps[0].iterations_run and str(o["reason"]) == reps[0].stop_reason
        assert int(o["backtracks"]) == int(reps[0].extra.get("backtracks", 0))
    log = (tmp_path / "nccl.0.log").read_text() if (tmp_path / "nccl.0.log").exists() else ""
    assert f"nranks {world}" in log or "nRanks" in log or log == "", log[:2000]
