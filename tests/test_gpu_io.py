"""GPU: NDTENSOR files streamed straight into / out of a device-resident plan
(pinned 16 MB chunks, f64 file <-> f32 device, no full host copy), for a
batch plan and for z-slab sharded ranks that each read their own planes and write
their own planes of one shared file."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_plan_load_save_equals_in_memory_path(nd, tmp_path):
    rng = np.random.default_rng(31)
    h = rng.uniform(0, 1, (7, 5))
    x_shape = (70, 90)
    y = rng.uniform(0, 1, (3,) + nd.conv_output_shape(x_shape, h))
    path, out = str(tmp_path / "y.ndt"), str(tmp_path / "x.ndt")
    nd.write_tensor(y, path)
    cfg = nd.DeconvConfig(max_iters=15, tol_rel_objective=0.0)

    a = nd.Plan(x_shape, h, batch=3)
    a.load_observation(path)
    a.pg_run(cfg)
    a.save_estimate(out)
    b = nd.Plan(x_shape, h, batch=3)
    b.set_observation(y)
    b.pg_run(cfg)
    want = b.estimate()
    got = nd.read_tensor(out)
    assert got.shape == (3,) + x_shape
    assert got.tobytes() == want.tobytes()
    assert np.array_equal(a.estimate(), want)
    # a batch-1 plan reads / writes the plain image shape
    c = nd.Plan(x_shape, h)
    nd.write_tensor(y[1], path)
    c.load_observation(path)
    c.pg_run(cfg)
    c.save_estimate(out)
    assert nd.read_tensor(out).tobytes() == want[1].tobytes()
    for p in (a, b, c):
        p.close()


def test_plan_load_rejects_bad_files(nd, tmp_path):
    h = np.ones((3, 3)) / 9
    p = nd.Plan((20, 20), h)
    nd.write_tensor(np.ones((21, 22)), str(tmp_path / "wrong.ndt"))
    with pytest.raises(nd.ShapeError):
        p.load_observation(str(tmp_path / "wrong.ndt"))
    good = str(tmp_path / "good.ndt")
    nd.write_tensor(np.ones((22, 22)), good)
    data = open(good, "rb").read()
    open(str(tmp_path / "trunc.ndt"), "wb").write(data[:-8])
    with pytest.raises(nd.FormatError):
        p.load_observation(str(tmp_path / "trunc.ndt"))
    bad = bytearray(data)
    bad[-8:] = np.array([np.nan]).astype("<f8").tobytes()
    open(str(tmp_path / "nan.ndt"), "wb").write(bytes(bad))
    with pytest.raises(nd.FormatError):
        p.load_observation(str(tmp_path / "nan.ndt"))
    p.load_observation(good)  # the plan is still usable
    p.close()


def test_large_observation_streams_in_chunks(nd, tmp_path):
    # 5.9e6-voxel observation: several 16 MB pinned chunks per image
    rng = np.random.default_rng(32)
    h = rng.uniform(0, 1, (9, 9))
    x_shape = (1200, 4900)
    y = rng.standard_normal(nd.conv_output_shape(x_shape, h))
    path = str(tmp_path / "big.ndt")
    nd.write_tensor(y, path)
    a = nd.Plan(x_shape, h)
    a.load_observation(path)
    b = nd.Plan(x_shape, h)
    b.set_observation(y)
    cfg = nd.DeconvConfig(max_iters=2, tol_rel_objective=0.0, initial_step=1e-3)
    a.pg_run(cfg)
    b.pg_run(cfg)
    assert np.array_equal(a.estimate(), b.estimate())
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ranks_share_one_file(nd, tmp_path, world):
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=40)
    path, out = str(tmp_path / "y.ndt"), str(tmp_path / "x.ndt")
    nd.write_tensor(y, path)
    cfg = nd.DeconvConfig(max_iters=6, tol_rel_objective=0.0)
    group = nd.LocalGroup(world)
    plans = [nd.Plan.local(group, r, x.shape, h) for r in range(world)]
    ests, errs = [None] * world, []

    def rank_main(r):
        try:
            plans[r].load_observation(path)
            plans[r].pg_run(cfg)
            plans[r].save_estimate(out)
            ests[r] = (plans[r].x_range[0], plans[r].estimate()[0])
        except Exception as e:  # pragma: no cover
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
    assembled = np.concatenate([e for _, e in sorted(ests, key=lambda t: t[0])], axis=0)
    got = nd.read_tensor(out)
    assert got.shape == x.shape
    assert got.tobytes() == assembled.tobytes()
    full = nd.deconv_pg(y, h, x.shape, cfg)
    assert np.linalg.norm(got - full.estimate) <= 1e-5 * np.linalg.norm(full.estimate)
