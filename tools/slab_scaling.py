"""Projected z-slab scaling for the sharded 3-D configs (c4, c5) from ONE GPU.

Only one B200 is available here, and ranks whose kernels wait on one another must not
share a GPU (B200_PROFILING.md), so the multi-GPU run is projected, not measured:

* compute: for W = 1, 2, 4, 8 the per-rank forward + adjoint passes are timed at the
  exact slab geometry each rank of a W-way run holds (Plan.local for that rank alone --
  the bench hooks run only the correlation passes, no exchange), CUDA events on the
  plan's stream.  Ranks 0, 1 and W-1 cover the three slab shapes (first, interior, last).
* communication: per iteration each rank exchanges p_z planes of x and of r with each
  neighbour (bytes printed), and runs two 2-double all-gathers.  The halo exchange
  overlaps the next pass's interior planes (ndc_plan.cu correlate()); only what exceeds
  that interior time is exposed.  NVLink 5 is taken at 900 GB/s per direction and an
  all-gather at 20 us (assumptions, stated in the output).

T_W = max_r (fwd_r + adj_r) + exposed halo + 2 all-gathers; efficiency = T_1 / (W T_W).
Usage: python tools/slab_scaling.py [c4] [c5] [--reps N]
"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd, synth  # noqa: E402

NVLINK_GBS = 900.0
ALLGATHER_US = 20.0
SHAPES = {"c4": (512, 1024, 1024), "c5": (256, 2048, 2048)}


def _time(p, reps):
    p.forward()
    p.adjoint()
    p.reset_stats()
    p.set_timing(True)
    for _ in range(reps):
        p.forward()
        p.adjoint()
    _, f = p.stats(0)
    _, a = p.stats(1)
    p.set_timing(False)
    xa, xb = p.x_range
    return f / reps, a / reps, xb - xa


def time_ranks(shape, h, world, ranks, reps):
    """{rank: (fwd ms, adj ms, owned planes)}.  All W slab plans are created (loading the
    observation exchanges halos, which needs every rank), then the requested ranks' passes
    are timed one rank at a time, alone on the GPU."""
    import threading
    if world == 1:
        p = nd.Plan(shape, h)
        p.set_observation(np.zeros((1,) + p.owned_y_shape(), np.float32))
        out = {0: _time(p, reps)}
        p.close()
        return out
    group = nd.LocalGroup(world)
    plans = [nd.Plan.local(group, r, shape, h) for r in range(world)]
    th = [threading.Thread(target=lambda p=p: p.set_observation(np.zeros((1,) + p.owned_y_shape(), np.float32)))
          for p in plans]
    for t in th:
        t.start()
    for t in th:
        t.join()
    out = {r: _time(plans[r], reps) for r in ranks}
    for p in plans:
        p.close()
    group.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4", "c5"])
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    out = {}
    for cfg in a.configs:
        shape = SHAPES[cfg]
        h = synth.psf_for(cfg)
        pz = (h.shape[0] - 1) // 2
        mz, my, mx = shape
        K = int(np.prod(h.shape))
        reps = a.reps if cfg == "c4" else 1
        rows = []
        t1 = None
        for W in (1, 2, 4, 8):
            ranks = sorted({0, min(1, W - 1), W - 1})
            per = {}
            for r, (f, ad, n) in time_ranks(shape, h, W, ranks, reps).items():
                per[r] = {"fwd_ms": f, "adj_ms": ad, "planes": n}
                print(f"{cfg} W={W} rank {r}: {n} planes  fwd {f:.2f} ms  adj {ad:.2f} ms", flush=True)
            worst = max(v["fwd_ms"] + v["adj_ms"] for v in per.values())
            # halo bytes per iteration per interior rank: p_z planes of x (after the
            # adjoint) and of r (after the forward) to each of the two neighbours, sent
            # and received at once (NVLink per direction)
            x_plane = my * mx * 4
            y_plane = (my + 2 * ((h.shape[1] - 1) // 2)) * (mx + 2 * ((h.shape[2] - 1) // 2)) * 4
            halo_b = 0 if W == 1 else 2 * pz * (x_plane + y_plane)
            t_hx = 2 * pz * x_plane / (NVLINK_GBS * 1e9) * 1e3
            t_hy = 2 * pz * y_plane / (NVLINK_GBS * 1e9) * 1e3
            t_halo = t_hx + t_hy if W > 1 else 0.0
            n_min = min(v["planes"] for v in per.values())
            interior = max(0, n_min - 2 * pz) / max(n_min, 1)
            exposed = 0.0
            if W > 1:
                # x halo overlaps the forward's interior planes, r halo the adjoint's
                fwd = max(v["fwd_ms"] for v in per.values())
                adj = max(v["adj_ms"] for v in per.values())
                exposed = max(0.0, t_hx - interior * fwd) + max(0.0, t_hy - interior * adj)
                exposed += 2 * ALLGATHER_US / 1e3
            t = worst + exposed
            if W == 1:
                t1 = t
            eff = t1 / (W * t)
            vox_it = mz * my * mx / (t / 1e3)
            rows.append({"W": W, "ranks": per, "compute_ms": worst, "halo_bytes_per_iter": halo_b,
                         "halo_ms_at_nvlink": t_halo, "interior_fraction": interior,
                         "exposed_comm_ms": exposed, "iter_ms": t, "voxel_it_per_s": vox_it,
                         "efficiency": eff, "fp32_tflops_per_gpu": 4.0 * K * mz * my * mx / (t / 1e3) / W / 1e12})
            print(f"{cfg} W={W}: iter {t:.2f} ms (compute {worst:.2f}, exposed comm {exposed:.3f})  "
                  f"{vox_it:.3e} voxel-it/s  efficiency {eff:.3f}", flush=True)
        out[cfg] = {"shape": list(shape), "psf": list(h.shape), "rows": rows,
                    "assumptions": {"nvlink_gbs_per_direction": NVLINK_GBS, "allgather_us": ALLGATHER_US,
                                    "basis": "per-rank pass times measured on one B200 at each rank's slab "
                                             "geometry; communication modelled (one GPU available)"}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
