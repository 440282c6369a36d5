"""Simulation generators (reference simulation.hpp), pinned against the
reference compiled in oracle/_ref (ref_shim.cpp ref_sim_* / ref_mt19937_64) and
restating tests/test_simulation.cpp.

CPU: the kernel-sized host generators (gaussian / delta PSF) bit for bit, and the
reference's argument validation (raised before any device work).  GPU: phantoms bit
for bit, the device mt19937_64 stream bit for bit at arbitrary offsets, Box-Muller
noise within a few ulp, the plan's in-place noise (batch and z-slab sharded) and the
CLI `simulate` subcommand.
"""
from __future__ import annotations

import os
import subprocess
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_1711_11224_b200 import build as B
from paper_1711_11224_b200 import ndconv as ndm

needs_ref = pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    return O.Oracle("ref")


# --- CPU ---------------------------------------------------------------------------------
@needs_ref
@pytest.mark.parametrize("ext,sigma", [((5, 5), 1.0), ((3,), 0.5), ((7, 3), 2.5), ((3, 5, 7), 1.3), ((1, 9), 0.7)])
def test_gaussian_psf_bitwise(ref, ext, sigma):
    assert ndm.gaussian_psf(ext, sigma).tobytes() == ref.gaussian_psf(ext, sigma).tobytes()


def test_gaussian_psf_matches_closed_form():
    h = ndm.gaussian_psf((5, 5), 1.0)
    i = np.arange(5) - 2
    g = np.exp(-(i[:, None] ** 2 + i[None, :] ** 2) / 2.0)
    np.testing.assert_allclose(h, g / g.sum(), rtol=1e-14)
    assert abs(h.sum() - 1.0) < 1e-14


@needs_ref
def test_delta_psf_is_centred_unit_impulse(ref):
    for ext in [(3, 3), (5,), (1, 7), (3, 5, 3)]:
        d = ndm.delta_psf(ext)
        assert d.tobytes() == ref.delta_psf(ext).tobytes()
        assert d.sum() == 1.0 and d[tuple(e // 2 for e in ext)] == 1.0


def test_generator_argument_errors():
    with pytest.raises(ndm.ShapeError):
        ndm.gaussian_psf((4, 5), 1.0)
    with pytest.raises(ndm.NumericError):
        ndm.gaussian_psf((5, 5), 0.0)
    with pytest.raises(ndm.NumericError):
        ndm.gaussian_psf((5, 5), float("nan"))
    with pytest.raises(ndm.ShapeError):
        ndm.delta_psf((2,))
    with pytest.raises(ndm.ShapeError):
        ndm.phantom_lines(2, 10, 3, 1.0)
    with pytest.raises(ndm.Error):
        ndm.phantom_lines(10, 10, 0, 1.0)
    with pytest.raises(ndm.ShapeError):
        ndm.phantom_texture(10, 2)
    with pytest.raises(ndm.NumericError):
        ndm.add_gaussian_noise(np.zeros(4), 0.0, -1.0, 1)


@pytest.mark.skipif(ndm.device_count() > 0, reason="checks the no-device path")
def test_device_generators_fail_loudly_without_a_gpu():
    with pytest.raises(ndm.DeviceError):
        ndm.phantom_lines(8, 8, 2, 1.0)
    with pytest.raises(ndm.DeviceError):
        ndm.add_gaussian_noise(np.zeros(4), 0.0, 1.0, 1)
    with pytest.raises(ndm.DeviceError):
        ndm.mt19937_64(1, 4)


def test_snr_db_definition():
    assert ndm.snr_db([3.0, 4.0], [3.0, 3.0]) == pytest.approx(10 * np.log10(25.0), rel=1e-15)
    assert ndm.snr_db([1.0, 2.0], [1.0, 2.0]) == float("inf")
    with pytest.raises(ndm.NumericError):
        ndm.snr_db([0.0, 0.0], [1.0, 2.0])
    with pytest.raises(ndm.ShapeError):
        ndm.snr_db([1.0, 2.0], [1.0])


# --- GPU ---------------------------------------------------------------------------------
@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("rows,cols,n", [(128, 128, 9), (3, 3, 1), (24, 24, 3), (37, 91, 7), (200, 50, 16),
                                         (1025, 513, 33)])
def test_phantom_lines_bitwise(nd, ref, rows, cols, n):
    got = nd.phantom_lines(rows, cols, n, 255.0)
    assert got.tobytes() == ref.phantom_lines(rows, cols, n, 255.0).tobytes()
    assert set(np.unique(got)) <= {0.0, 255.0}


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("rows,cols", [(128, 128), (3, 3), (64, 200), (333, 97), (2048, 2048)])
def test_phantom_texture_bitwise(nd, ref, rows, cols):
    got = nd.phantom_texture(rows, cols)
    assert got.tobytes() == ref.phantom_texture(rows, cols).tobytes()
    assert got.min() >= 0.0 and got.max() <= 255.0


@pytest.mark.gpu
@needs_ref
def test_mt19937_64_stream_bitwise(nd, ref):
    for seed in (1, 5489, 2**64 - 1, 20240915):
        for skip, n in [(0, 1), (0, 1000), (311, 5), (312, 624), (1000, 3000), (123457, 10)]:
            assert np.array_equal(nd.mt19937_64(seed, n, skip), ref.mt19937_64(seed, n, skip)), (seed, skip, n)
    assert int(nd.mt19937_64(5489, 1)[0]) == 14514284786278117030  # the engine's published first word


def _ulp_close(a, b, scale, ulps=8):
    """|a - b| within `ulps` ulp of the magnitudes that were summed (cancellation-safe)."""
    return np.all(np.abs(a - b) <= ulps * np.finfo(np.float64).eps * scale)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n", [1, 2, 7, 312, 625, 100_003])
def test_gaussian_noise_matches_reference(nd, ref, n):
    rng = np.random.default_rng(n)
    t = rng.uniform(0, 100, n)
    got = nd.add_gaussian_noise(t, 1.5, 5.0, 42)
    want = ref.add_gaussian_noise(t, 1.5, 5.0, 42)
    # noise-only comparison: the draws agree to a few ulp (device vs glibc log/sin/cos)
    z_got, z_want = got - (t + 1.5), want - (t + 1.5)
    assert np.max(np.abs(z_got - z_want)) <= 1e-12 * 5.0
    assert _ulp_close(got, want, np.abs(t + 1.5) + np.abs(z_want), ulps=16)
    assert np.mean(got == want) > 0.5  # most draws are bit-identical


@pytest.mark.gpu
def test_noise_is_reproducible_and_signal_independent(nd):
    a = nd.add_gaussian_noise(np.zeros(5000), 0.0, 1.0, 7)
    b = nd.add_gaussian_noise(np.zeros(5000), 0.0, 1.0, 7)
    c = nd.add_gaussian_noise(np.zeros(5000), 0.0, 1.0, 8)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    s = nd.add_gaussian_noise(np.full(5000, 3.0), 0.0, 1.0, 7)
    np.testing.assert_allclose(s - 3.0, a, atol=1e-14)
    big = nd.add_gaussian_noise(np.zeros(400_000), 2.0, 3.0, 11)
    assert abs(big.mean() - 2.0) < 0.03 and abs(big.std() - 3.0) < 0.03
    z = nd.add_gaussian_noise(np.arange(6.0), 0.5, 0.0, 3)
    assert np.array_equal(z, np.arange(6.0) + 0.5)


@pytest.mark.gpu
@needs_ref
def test_plan_noise_in_place_batch(nd, ref):
    rng = np.random.default_rng(3)
    h = nd.gaussian_psf((5, 7), 1.2)
    x_shape = (90, 70)
    y = rng.uniform(0, 50, (3,) + nd.conv_output_shape(x_shape, h)).astype(np.float32).astype(np.float64)
    p = nd.Plan(x_shape, h, batch=3)
    p.set_observation(y)
    p.add_gaussian_noise(0.25, 2.0, 99)
    want = ref.add_gaussian_noise(y.ravel(), 0.25, 2.0, 99).reshape(y.shape).astype(np.float32)
    got = p.observation().astype(np.float32)
    # identical up to f32 rounding of f64 values that differ by a few ulp
    assert np.mean(got == want) > 0.9999
    np.testing.assert_allclose(got, want, rtol=2e-7, atol=1e-6)
    p.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_plan_noise_sharded_equals_unsharded(nd, world):
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c4", shape=(36, 40, 44), n_objects=30)
    full = nd.Plan(x.shape, h)
    full.set_observation(y)
    full.add_gaussian_noise(0.0, 0.5, 1234)
    want = full.observation()[0]
    full.close()
    group = nd.LocalGroup(world)
    plans = [nd.Plan.local(group, r, x.shape, h) for r in range(world)]
    parts, errs = [None] * world, []

    def rank_main(r):
        try:
            ya, yb = plans[r].y_range
            plans[r].set_observation(y[ya:yb])
            plans[r].add_gaussian_noise(0.0, 0.5, 1234)
            parts[r] = (ya, plans[r].observation()[0])
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
    got = np.concatenate([o for _, o in sorted(parts, key=lambda t: t[0])], axis=0)
    assert np.array_equal(got, want)


# --- CLI simulate (test_cli.cpp:130-159, 212-230) -----------------------------------------
def _cli():
    if not os.path.exists(B.CLI):
        B.build()
    return B.CLI


def _run(args, cwd):
    p = subprocess.run([_cli(), *args], cwd=cwd, capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def test_simulate_usage_errors(tmp_path):
    assert _run(["simulate"], tmp_path)[0] == 2                                    # --outdir required
    assert _run(["simulate", "--outdir", "o", "--size", "1,2,3"], tmp_path)[0] == 2  # at most 2 values
    assert _run(["simulate", "--outdir", "o", "--lines", "0"], tmp_path)[0] == 2
    assert _run(["simulate", "--outdir", "o", "--seed", "-1"], tmp_path)[0] == 2
    assert _run(["simulate", "--outdir", "o", "--size", "2"], tmp_path)[0] == 4     # phantom < 3x3
    # a PGM phantom keeps the truth on the host, so the PSF checks run without a device
    ndm.write_pgm(np.full((8, 8), 9.0), str(tmp_path / "p.pgm"))
    pgm = ["--phantom", "p.pgm"]
    assert _run(["simulate", "--outdir", "o", "--psf-size", "4", *pgm], tmp_path)[0] == 4  # even psf
    assert _run(["simulate", "--outdir", "o", "--sigma", "-1", *pgm], tmp_path)[0] == 5
    assert _run(["simulate", "--outdir", "o", "--psf", "airy", *pgm], tmp_path)[0] == 1
    assert _run(["simulate", "--outdir", "o", "--phantom", "/nonexistent.pgm"], tmp_path)[0] == 3


@pytest.mark.gpu
def test_simulate_is_seed_reproducible(nd, tmp_path):
    base = ["simulate", "--phantom", "lines", "--size", "48", "--lines", "5", "--psf", "gaussian", "--psf-size",
            "5", "--sigma", "1.0", "--noise-std", "2"]
    for d, seed in (("a", "1"), ("b", "1"), ("c", "2")):
        rc, _, err = _run(base + ["--seed", seed, "--outdir", str(tmp_path / d)], tmp_path)
        assert rc == 0, err
    oa, ob, oc = (nd.read_tensor(str(tmp_path / d / "observed.ndt")) for d in "abc")
    assert np.array_equal(oa, ob) and not np.array_equal(oa, oc)
    ta, tc = (nd.read_tensor(str(tmp_path / d / "truth.ndt")) for d in "ac")
    assert np.array_equal(ta, tc)
    m = dict(line.rstrip("\n").split("=", 1) for line in open(tmp_path / "a" / "manifest.txt"))
    assert m["subcommand"] == "simulate" and m["seed"] == "1" and m["observed_shape"] == "52,52"
    assert list(m) == ["subcommand", "version", "phantom", "size", "lines", "psf", "psf_size", "sigma", "noise_mean",
                       "noise_std", "seed", "outdir", "truth", "psf_file", "observed", "observed_shape"]
    for name in ("truth.ndt", "truth.pgm", "psf.ndt", "observed.ndt", "observed.pgm", "manifest.txt"):
        assert (tmp_path / "a" / name).exists()


@pytest.mark.gpu
@needs_ref
def test_simulate_matches_reference_pipeline(nd, ref, tmp_path):
    rc, _, err = _run(["simulate", "--phantom", "texture", "--size", "64,80", "--psf-size", "7,5", "--sigma", "1.5",
                       "--noise-mean", "0.5", "--noise-std", "3", "--seed", "77", "--outdir", str(tmp_path / "s")],
                      tmp_path)
    assert rc == 0, err
    truth = ref.phantom_texture(64, 80)
    psf = ref.gaussian_psf((7, 5), 1.5)
    assert nd.read_tensor(str(tmp_path / "s" / "truth.ndt")).tobytes() == truth.tobytes()
    assert nd.read_tensor(str(tmp_path / "s" / "psf.ndt")).tobytes() == psf.tobytes()
    blurred = ref.conv_full(truth, psf)
    want = ref.add_gaussian_noise(blurred.ravel(), 0.5, 3.0, 77).reshape(blurred.shape)
    got = nd.read_tensor(str(tmp_path / "s" / "observed.ndt"))
    # the blur runs in float32 on the device (<= 1e-5 rel-L2 per convolution)
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(blurred)


@pytest.mark.gpu
def test_deconv_rl_on_simulated_clean_data_conserves_flux(nd, tmp_path):
    rc, _, err = _run(["simulate", "--phantom", "lines", "--size", "24", "--lines", "3", "--psf", "gaussian",
                       "--psf-size", "5", "--sigma", "1.0", "--noise-std", "0", "--seed", "4", "--outdir",
                       str(tmp_path / "sim")], tmp_path)
    assert rc == 0, err
    rc, _, err = _run(["deconv", "--observed", str(tmp_path / "sim" / "observed.ndt"), "--kernel",
                       str(tmp_path / "sim" / "psf.ndt"), "--shape", "24,24", "--method", "rl", "--max-iters", "40",
                       "--tol", "0", "--output", str(tmp_path / "est.ndt")], tmp_path)
    assert rc == 0, err
    est = nd.read_tensor(str(tmp_path / "est.ndt"))
    obs = nd.read_tensor(str(tmp_path / "sim" / "observed.ndt"))
    assert abs(est.sum() - obs.sum()) <= 1e-5 * abs(obs.sum())  # fp32 (reference f64: 1e-8)
    m = dict(line.rstrip("\n").split("=", 1) for line in open(str(tmp_path / "est.ndt") + ".manifest"))
    assert m["negative_pixels_clamped"] == "0"
