"""Helper for tests/test_gpu_nccl.py: ONE z-slab rank of a multi-process NCCL run (one
process per GPU, device = rank).  Rank 0 writes the NCCL unique id to `uid_file`; the
others wait for it.  Usage:
    python tests/_nccl_rank.py out.npz rank world uid_file step"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_11224_b200 import ndconv as nd  # noqa: E402
from paper_1711_11224_b200 import synth  # noqa: E402


def main():
    out, rank, world, uid_file, step = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], float(sys.argv[5])
    if rank == 0:
        tmp = uid_file + ".tmp"
        with open(tmp, "wb") as f:
            f.write(nd.nccl_unique_id())
        os.replace(tmp, uid_file)
    t_end = time.time() + 120
    while not os.path.exists(uid_file):
        if time.time() > t_end:
            raise SystemExit("no NCCL id")
        time.sleep(0.05)
    uid = open(uid_file, "rb").read()
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=60)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=step if step > 0 else None)
    p = nd.Plan.sharded(x.shape, h, rank, world, uid, device=rank)
    ya, yb = p.y_range
    p.set_observation(y[ya:yb])
    p.pg_run(cfg)
    r = p.report(0, cfg.max_iters + 1)
    np.savez(out, x=p.estimate()[0], x_range=np.array(p.x_range), obj=r.objective_trace, kkt=r.kkt_trace,
             iters=r.iterations_run, reason=r.stop_reason, backtracks=r.extra.get("backtracks", 0),
             step0=r.extra["step0"])
    p.close()


if __name__ == "__main__":
    main()
