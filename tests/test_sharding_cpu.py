"""CPU, world size 2 over gloo: the z-slab decomposition the sharded driver uses
(ndc_slab_range ownership, p_z-plane halos per pass, rank-order scalar combine),
exercised end to end with the CPU oracle as the per-slab compute.  Each rank holds only
its x planes [a-p, b+p) / y planes [a, b+2p), exchanges p_z-plane halos with its
neighbours over torch.distributed, and produces its owned planes; rank 0 checks the
assembled forward / adjoint / objective against the unsharded oracle bitwise (the
per-voxel sum order does not depend on the slab)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(rank, world, send_lo, send_hi, shape_lo, shape_hi):
    """Send send_lo to rank-1 and send_hi to rank+1; receive the neighbours' planes."""
    recv_lo = torch.zeros(shape_lo, dtype=torch.float64) if rank > 0 else None
    recv_hi = torch.zeros(shape_hi, dtype=torch.float64) if rank < world - 1 else None
    ops = []
    if rank > 0:
        ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(send_lo)), rank - 1),
                dist.P2POp(dist.irecv, recv_lo, rank - 1)]
    if rank < world - 1:
        ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(send_hi)), rank + 1),
                dist.P2POp(dist.irecv, recv_hi, rank + 1)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return (None if recv_lo is None else recv_lo.numpy()), (None if recv_hi is None else recv_hi.numpy())


def boundary_counts(rank, world, pz):
    """Planes at the start / end of a pass's computed planes that read the input's halo
    (ndc_plan.cu correlate(): lo = p_z unless rank 0, hi = p_z unless the last rank)."""
    return (pz if rank > 0 else 0), (pz if rank < world - 1 else 0)


def test_boundary_planes_are_the_halo_planes():
    """For every slab layout: the computed planes outside the first lo / last hi read only
    owned input planes (so they may run before the halo exchange), and the planes each
    neighbour receives as its halo are all among the first lo / last hi (so the exchange
    can start once those are done) -- forward (x -> y) and adjoint (y -> x)."""
    from paper_1711_11224_b200 import ndconv as nd
    for mz in range(1, 41):
        for pz in range(0, 8):
            for world in range(1, 6):
                if world > 1 and mz // world < max(pz, 1):
                    continue
                for rank in range(world):
                    a, b, ya, yb = nd.slab_range(mz, pz, rank, world)
                    nlo, nhi = boundary_counts(rank, world, pz)
                    if world == 1:
                        nlo = nhi = 0
                    own_y = set(range(ya, yb))
                    # forward: output plane o reads x planes [o-2p, o] within [0, mz)
                    for k, o in enumerate(range(ya, yb)):
                        reads = {z for z in range(o - 2 * pz, o + 1) if 0 <= z < mz}
                        if nlo <= k < (yb - ya) - nhi:
                            assert reads <= set(range(a, b)), (mz, pz, world, rank, o)
                    # adjoint: output x plane o reads y planes [o, o+2p]
                    for k, o in enumerate(range(a, b)):
                        reads = set(range(o, o + 2 * pz + 1))
                        if nlo <= k < (b - a) - nhi:
                            assert reads <= own_y, (mz, pz, world, rank, o)
                    # what the neighbours pull: x planes [a, a+p) / [b-p, b), y planes
                    # [a+p, a+2p) / [b, b+p)
                    if rank > 0:
                        assert set(range(a, a + pz)) <= set(range(a, a + nlo))
                        assert set(range(a + pz, a + 2 * pz)) <= set(range(ya, ya + nlo))
                    if rank < world - 1:
                        assert set(range(b - pz, b)) <= set(range(b - nhi, b))
                        assert set(range(b, b + pz)) <= set(range(yb - nhi, yb))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_1711_11224_b200 import ndconv as nd
        orc = Oracle("c")
        g = np.random.Generator(np.random.PCG64(11))
        mz, my, mx = 13, 9, 8
        h = g.uniform(-1, 1, (5, 3, 3))
        pz = 2
        x = g.uniform(-1, 1, (mz, my, mx))
        y = g.uniform(-1, 1, (mz + 4, my + 2, mx + 2))
        a, b, ya, yb = nd.slab_range(mz, pz, rank, world)
        # overlapped schedule (ndc_plan.cu correlate()): the planes that need no halo are
        # computed from the owned planes alone BEFORE the exchange
        nlo, nhi = boundary_counts(rank, world, pz)
        interior_fwd = orc.conv_full(x[a:b], h)[ya + nlo - a: yb - nhi - a]
        # forward: hold x planes [max(0,a-p), min(mz,b+p)) via halos
        lo, hi = _exchange(rank, world, x[a:a + pz], x[b - pz:b], (pz, my, mx), (pz, my, mx))
        parts = [p for p in (lo, x[a:b], hi) if p is not None]
        xl = np.concatenate(parts, axis=0)
        x0 = a - (pz if lo is not None else 0)
        yl = orc.conv_full(xl, h)                      # local full conv of the slab
        own_fwd = yl[ya - x0: yb - x0]                  # owned y planes
        assert np.array_equal(own_fwd[nlo:own_fwd.shape[0] - nhi], interior_fwd)
        # adjoint: hold y planes [a, b+2p): own [ya, yb) + halos from neighbours
        lo, hi = _exchange(rank, world, y[a + pz:a + 2 * pz], y[b:b + pz], (pz,) + y.shape[1:],
                           (pz,) + y.shape[1:])
        yloc = np.concatenate([p for p in (lo, y[ya:yb], hi) if p is not None], axis=0)
        assert yloc.shape[0] == (b - a) + 2 * pz
        own_adj = orc.adjoint_apply(yloc, h, (b - a, my, mx))
        # scalar combine in rank order: per-rank partial of 0.5||Ax - y||^2 over owned y
        part = torch.tensor([0.5 * float(np.sum((own_fwd - y[ya:yb]) ** 2))], dtype=torch.float64)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, part)
        f = sum(float(t) for t in gathered)
        objs = [None] * world
        dist.all_gather_object(objs, (ya, yb, own_fwd, a, b, own_adj, f))
        if rank == 0:
            yf = np.concatenate([o[2] for o in sorted(objs, key=lambda o: o[0])], axis=0)
            xa = np.concatenate([o[5] for o in sorted(objs, key=lambda o: o[3])], axis=0)
            ok = (np.array_equal(yf, orc.conv_full(x, h)) and
                  np.array_equal(xa, orc.adjoint_apply(y, h, x.shape)) and
                  abs(f - orc.objective(x, y, h)) <= 1e-12 * abs(f) and
                  all(o[6] == f for o in objs))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_halo_decomposition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=10) is True


def _gen_worker(rank, world, port, q):
    """bench.py's per-rank observation generation (inputs_volume over gloo: the volume
    maximum all-reduced, noise seeded per plane) -- each rank only its own y planes."""
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"], os.environ["LOCAL_RANK"] = str(rank), str(world), str(rank)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_1711_11224_b200 import ndconv as nd
    d = bench.Dist("gloo")
    try:
        shape, nobj = (40, 30, 34), 60
        for cfg in ("c4", "c5"):
            kz = {"c4": 21, "c5": 65}[cfg]
            if cfg == "c5":
                shape = (72, 20, 22)
            _, _, ya, yb = nd.slab_range(shape[0], (kz - 1) // 2, rank, world)
            mine = bench.inputs_volume(cfg, ya, yb, d, None, shape=shape, n_objects=nobj)[0]
            objs = [None] * world
            dist.all_gather_object(objs, (ya, mine))
            if rank == 0:
                got = np.concatenate([o[1] for o in sorted(objs, key=lambda o: o[0])], axis=0)
                d1 = bench.Dist.__new__(bench.Dist)
                d1.world = 1
                whole = bench.inputs_volume(cfg, 0, shape[0] + kz - 1, d1, None, shape=shape, n_objects=nobj)[0]
                q.put((cfg, got.shape == whole.shape and np.array_equal(got, whole)))
    finally:
        dist.destroy_process_group()


def test_bench_per_rank_inputs_gloo():
    """Two ranks' generated observation planes assemble to the single-rank volume bit for
    bit (configs 4 and 5 generators, Poisson noise on the host fallback)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gen_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {"c4": True, "c5": True}, res
