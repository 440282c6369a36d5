"""Helper for tests/test_gpu_sharded.py: one sharded PG run (W in-process ranks on one
GPU) in a fresh process, so the NDC_HALO_OVERLAP / NDC_SPECULATE knobs (read once per
process) can differ between runs.  Usage: python tests/_sharded_run.py out.npz world step"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_11224_b200 import ndconv as nd  # noqa: E402
from paper_1711_11224_b200 import synth  # noqa: E402
from tests.test_gpu_sharded import run_sharded  # noqa: E402


def main():
    out, world, step = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=step if step > 0 else None)
    xs, reps = run_sharded(nd, world, y, h, x.shape, cfg)
    r = reps[0]
    np.savez(out, x=xs, obj=r.objective_trace, kkt=r.kkt_trace, iters=r.iterations_run,
             reason=r.stop_reason, backtracks=r.extra.get("backtracks", 0))


if __name__ == "__main__":
    main()
