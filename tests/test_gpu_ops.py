"""GPU parity of the operators (convolution.hpp / solvers.hpp scalar functions) through
the C-ABI against the reference's golden outputs and the CPU oracle.

Tolerance (BASELINE.json north_star): relative L2 <= 1e-5 per convolution.  Integer
known-answer tests are exact in float32 and are checked for exact equality.
"""
import numpy as np
import pytest

from tests.conftest import rel_l2
from tests.golden.make_golden import big_inputs

pytestmark = pytest.mark.gpu
TOL_CONV = 1e-5


def test_kat_conv_full_exact(nd):
    # test_convolution.cpp:11-19, 40-45
    assert np.array_equal(nd.conv_full([1.0, 2.0], [1.0, 1.0, 1.0]), [1, 3, 3, 2])
    assert np.array_equal(nd.conv_full([1.0, 2.0, 3.0], [0.0, 1.0, 0.0]), [0, 1, 2, 3, 0])
    assert np.array_equal(nd.conv_full([3.0], [1.0, 2.0, 4.0, 2.0, 1.0]), [3, 6, 12, 6, 3])


def test_kat_adjoint_impulse_exact(nd):
    # test_convolution.cpp:104-108
    assert np.array_equal(nd.adjoint_apply([1.0, 0, 0, 0], [1.0, 2.0, 3.0], (2,)), [1.0, 0.0])


def test_kat_flip_crop(nd):
    # test_convolution.cpp:61-82: flip reverses every axis, is an involution
    h = np.arange(1.0, 10.0).reshape(3, 3)
    f = nd.flip(h)
    assert np.array_equal(f, h[::-1, ::-1]) and np.array_equal(nd.flip(f), h)


def test_golden_small_family(nd, golden_ops):
    d = golden_ops
    for i in range(int(d["n"])):
        x, h = d[f"x{i}"], d[f"h{i}"]
        y = nd.conv_full(x, h)
        assert y.shape == d[f"y{i}"].shape
        assert rel_l2(y, d[f"y{i}"]) <= TOL_CONV, i
        a = nd.adjoint_apply(d[f"r{i}"], h, x.shape)
        assert rel_l2(a, d[f"atr{i}"]) <= TOL_CONV, i


def test_golden_large(nd, golden_ops):
    d = golden_ops
    for i in range(int(d["nbig"])):
        x, h, r = big_inputs(i)
        assert rel_l2(nd.conv_full(x, h), d[f"by{i}"]) <= TOL_CONV, i
        assert rel_l2(nd.adjoint_apply(r, h, x.shape), d[f"batr{i}"]) <= TOL_CONV, i


def test_linearity_and_adjoint_identity(nd):
    # test_convolution.cpp:47-59 and 110-122 at float32 tolerance
    g = np.random.Generator(np.random.PCG64(24))
    for _ in range(10):
        ndim = int(g.integers(1, 4))
        xs = tuple(int(v) for v in g.integers(1, 9, ndim))
        hs = tuple(int(2 * v + 1) for v in g.integers(0, 3, ndim))
        h = g.uniform(-1, 1, hs)
        a, b = g.uniform(-1, 1, xs), g.uniform(-1, 1, xs)
        lhs = nd.conv_full(2.5 * a - 1.25 * b, h)
        rhs = 2.5 * nd.conv_full(a, h) - 1.25 * nd.conv_full(b, h)
        assert rel_l2(lhs, rhs) <= 1e-5
        y = g.uniform(-1, 1, lhs.shape)
        l = float(np.sum(nd.conv_full(a, h) * y))
        r = float(np.sum(a * nd.adjoint_apply(y, h, xs)))
        assert abs(l - r) / max(1.0, abs(l), abs(r)) <= 1e-5


def test_missing_flip_would_be_caught(nd):
    # test_convolution.cpp:124-136: the device adjoint must pass, a flip-less one fails
    h = np.array([1.0, 0.0, -2.0])
    x = np.array([1.0, -1.0, 2.0, 0.5])
    y = np.array([0.5, 1.0, -2.0, 0.0, 1.5, -1.0])
    good = float(np.dot(x, nd.adjoint_apply(y, h, (4,))))
    assert abs(float(np.dot(nd.conv_full(x, h), y)) - good) <= 1e-6


def test_normal_gradient_and_scalars(nd, oracle_c):
    g = np.random.Generator(np.random.PCG64(25))
    for _ in range(5):
        h = g.uniform(-1, 1, (3, 5))
        x = g.uniform(-1, 1, (17, 23))
        y = g.uniform(-1, 1, (19, 27))
        assert rel_l2(nd.normal_gradient(x, y, h), oracle_c.normal_gradient(x, y, h)) <= 1e-5
        f_ref = oracle_c.objective(x, y, h)
        assert abs(nd.objective(x, y, h) - f_ref) <= 1e-5 * abs(f_ref)
        k_ref = oracle_c.kkt_residual(x, y, h)
        assert abs(nd.kkt_residual(x, y, h) - k_ref) <= 1e-5 * max(1.0, abs(k_ref))


def test_kat_objective_kkt(nd):
    # test_solvers.cpp:12-22, 42-60
    assert nd.objective([1.0], [3.0], [1.0]) == 2.0
    box = np.array([0.5, 1.0, -0.25])
    x = np.array([1.0, -2.0, 0.5])
    assert abs(nd.objective(x, nd.conv_full(x, box), box)) <= 1e-12
    h = np.array([0.5, 1.0, 0.25])
    truth = np.array([0.0, 2.0, 0.0, 1.0])
    assert nd.kkt_residual(truth, nd.conv_full(truth, h), h) <= 1e-6
    assert nd.kkt_residual(np.zeros(4), np.full(6, -1.0), h) == 0.0


def test_estimate_step_kats(nd, golden_solvers):
    # test_solvers.cpp:24-40 at the reference's own 1e-12 (small problems run the power
    # iteration in float64 on the device)
    assert abs(nd.estimate_step([1.0], (5,), 10) - 1.0) <= 1e-12
    assert abs(nd.estimate_step([2.0], (5,), 10) - 0.25) <= 1e-12
    s = nd.estimate_step([1.0, 1.0, 1.0], (8,), 30)
    assert 1 / 9 <= s <= 1.0 and abs(s - float(golden_solvers["step_box"])) <= 1e-12 * s
    with pytest.raises(nd.NumericError):
        nd.estimate_step([0.0, 0.0, 0.0], (4,), 5)


def test_error_classes(nd):
    # test_convolution.cpp:33-38, kernel.hpp:18-22, test_solvers.cpp:168-189
    with pytest.raises(nd.ShapeError):
        nd.conv_full(np.ones((2, 2)), np.ones(3))
    with pytest.raises(nd.ShapeError):
        nd.adjoint_apply(np.ones((2, 2)), np.ones(3), (2, 2))
    with pytest.raises(nd.ShapeError):
        nd.conv_full(np.ones(4), np.ones(2))
    with pytest.raises(nd.NumericError):
        nd.conv_full(np.ones(4), np.array([1.0, np.nan, 1.0]))
    with pytest.raises(nd.ShapeError):
        nd.deconv_pg(np.zeros(6), [0.1, 0.8, 0.1], (5,))
    with pytest.raises(nd.NumericError):
        nd.deconv_pg(np.zeros(6), [0.0, 0.0, 0.0], (4,))
    with pytest.raises(nd.Error):
        nd.deconv_pg(np.zeros(6), [0.1, 0.8, 0.1], (4,), nd.DeconvConfig(backtrack_factor=1.0))
    with pytest.raises(nd.Error):
        nd.deconv_pg(np.zeros(6), [0.1, 0.8, 0.1], (4,), nd.DeconvConfig(max_iters=0))
    with pytest.raises(nd.UnsupportedError):
        nd.conv_full(np.ones((1,) * 9), np.ones((1,) * 9))  # at most 8 dimensions


@pytest.mark.parametrize("xs,hs", [((37, 50), (3, 35)), ((60, 90), (37, 71)), ((50, 40), (201, 3)),
                                   ((9, 30, 70), (3, 5, 67)), ((140,), (99,)), ((30, 260), (5, 129))])
def test_large_psfs_chunked(nd, oracle_c, xs, hs):
    """PSFs beyond one launch's tap block (more than 33 columns, more rows than one TMA box
    holds) run as several chunk launches accumulated on the device; forward, adjoint and
    a short PG run against the oracle."""
    rng = np.random.default_rng(sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    assert rel_l2(nd.conv_full(x, h), oracle_c.conv_full(x, h)) <= 1e-5
    y = oracle_c.conv_full(x, h) + rng.uniform(0, 1e-3, nd.conv_output_shape(xs, h))
    assert rel_l2(nd.adjoint_apply(y, h, xs), oracle_c.adjoint_apply(y, h, xs)) <= 1e-5
    cfg = nd.DeconvConfig(max_iters=5, tol_rel_objective=0.0, initial_step=1.0)
    got = nd.deconv_pg(y, h, xs, cfg)
    want = oracle_c.deconv_pg(y, h, xs, max_iters=5, tol_rel_objective=0.0, initial_step=1.0)
    assert got.iterations_run == want.iterations_run
    assert rel_l2(got.estimate, want.estimate) <= 1e-4


def test_config_shapes_sampled(nd, oracle_c):
    """BASELINE config 3 / 4 / 5 PSFs on reduced volumes, checked at sampled voxels
    through the reference's per-voxel routine."""
    from paper_1711_11224_b200 import synth
    g = np.random.Generator(np.random.PCG64(31))
    for name, shape in (("c3", (20, 40, 48)), ("c4", (24, 36, 40)), ("c5", (6, 40, 44))):
        h = synth.psf_for(name)
        x = synth.fp32_exact(g.uniform(0, 1, shape))
        y = nd.conv_full(x, h)
        idx = g.integers(0, y.size, 3000)
        ref = oracle_c.conv_full_sample(x, h, idx)
        assert rel_l2(y.ravel()[idx], ref) <= TOL_CONV, name
        r = synth.fp32_exact(g.uniform(-1, 1, y.shape))
        a = nd.adjoint_apply(r, h, shape)
        idx = g.integers(0, a.size, 3000)
        ref = oracle_c.adjoint_sample(r, h, shape, idx)
        assert rel_l2(a.ravel()[idx], ref) <= TOL_CONV, name


def test_batched_float32_operators(nd, oracle_c):
    """ndc_conv_full_batch_f32 / ndc_adjoint_apply_batch_f32: every image of the batch as
    the f64 single-image operator (float32 in and out)."""
    rng = np.random.default_rng(77)
    for xs, hs in (((3, 70, 90), (7, 9)), ((2, 12, 30, 40), (5, 3, 7)), ((4, 500), (41,))):
        x = rng.uniform(0, 1, xs).astype(np.float32)
        h = rng.uniform(0, 1, hs)
        y = nd.conv_full_batch(x, h)
        assert y.dtype == np.float32 and y.shape == (xs[0],) + nd.conv_output_shape(xs[1:], h)
        for b in range(xs[0]):
            assert rel_l2(y[b], oracle_c.conv_full(x[b].astype(np.float64), h)) <= 1e-5
        r = rng.uniform(-1, 1, y.shape).astype(np.float32)
        g = nd.adjoint_apply_batch(r, h, xs[1:])
        for b in range(xs[0]):
            assert rel_l2(g[b], oracle_c.adjoint_apply(r[b].astype(np.float64), h, xs[1:])) <= 1e-5


@pytest.mark.parametrize("xs,hs", [((124, 100), (15, 15)), ((231, 90), (31, 31)), ((125, 200), (9, 9)),
                                   ((6, 64, 64), (5, 15, 15)), ((6, 128, 100), (5, 9, 9)),
                                   ((3, 50, 64), (3, 15, 7))])
def test_edge_tiles_few_rows(nd, oracle_c, xs, hs):
    """Output extents that leave 1-16 rows in the last tile row (config 3's 270-row and
    config 4's 1032-row forward outputs are of this kind) run the edge kernel's compact
    lane mapping (8 or 16 rows x 4 or 2 strips per warp); every element of forward and
    adjoint, and a short PG run (fused epilogues + reductions), against the oracle."""
    rng = np.random.default_rng(sum(xs) + sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    y_ref = oracle_c.conv_full(x, h)
    y = nd.conv_full(x, h)
    assert np.max(np.abs(y - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
    r = rng.uniform(-1, 1, y_ref.shape)
    a_ref = oracle_c.adjoint_apply(r, h, xs)
    assert np.max(np.abs(nd.adjoint_apply(r, h, xs) - a_ref)) <= 1e-5 * np.max(np.abs(a_ref))
    yo = y_ref + rng.uniform(0, 1e-3, y_ref.shape)
    cfg = nd.DeconvConfig(max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    got = nd.deconv_pg(yo, h, xs, cfg)
    want = oracle_c.deconv_pg(yo, h, xs, max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    assert got.iterations_run == want.iterations_run
    assert rel_l2(got.estimate, want.estimate) <= 1e-4
    np.testing.assert_allclose(got.objective_trace, want.objective_trace, rtol=1e-4)


@pytest.mark.parametrize("xs,hs", [((13, 140, 70), (5, 9, 9)), ((6, 130, 130), (3, 7, 7)), ((7, 260, 70), (4 * 2 + 1, 9, 7)),
                                   ((13, 140, 70), (31, 31, 9)), ((1, 130, 70), (3, 9, 9)), ((2, 130, 70), (21, 9, 9))])
def test_two_planes_per_cta(nd, oracle_c, xs, hs):
    """Narrow 3-D PSFs (x-extent 7 or 9) on 128-row tiles run their full tiles two output planes
    per CTA (ndc_correlate_pair.cuh): odd and even plane counts, PSFs deeper than the volume
    (most staged planes meet only one of the two planes), a PSF of two tap chunks (31 x 31 x 9:
    24 + 7 slices accumulated through the scratch volume), and a single-plane volume whose
    adjoint falls back to the general kernel; every element of forward and adjoint and a short
    PG run against the oracle."""
    rng = np.random.default_rng(sum(xs) + 7 * sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    y_ref = oracle_c.conv_full(x, h)
    y = nd.conv_full(x, h)
    assert np.max(np.abs(y - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
    r = rng.uniform(-1, 1, y_ref.shape)
    a_ref = oracle_c.adjoint_apply(r, h, xs)
    assert np.max(np.abs(nd.adjoint_apply(r, h, xs) - a_ref)) <= 1e-5 * np.max(np.abs(a_ref))
    yo = y_ref + rng.uniform(0, 1e-3, y_ref.shape)
    cfg = nd.DeconvConfig(max_iters=3, tol_rel_objective=0.0, initial_step=1.0)
    got = nd.deconv_pg(yo, h, xs, cfg)
    want = oracle_c.deconv_pg(yo, h, xs, max_iters=3, tol_rel_objective=0.0, initial_step=1.0)
    assert got.iterations_run == want.iterations_run
    assert rel_l2(got.estimate, want.estimate) <= 1e-4
    np.testing.assert_allclose(got.objective_trace, want.objective_trace, rtol=1e-4)


@pytest.mark.parametrize("xs,hs", [((130, 150), (7, 7)), ((150, 130), (9, 9)), ((140, 140), (11, 11)),
                                   ((129, 200), (13, 13)), ((200, 129), (17, 17)), ((150, 160), (21, 21)),
                                   ((5, 70, 90), (3, 9, 9)), ((5, 70, 90), (3, 11, 19)), ((4, 64, 64), (3, 7, 7))])
def test_packed_ffma2_widths(nd, oracle_c, xs, hs):
    """PSF widths whose tap loop runs packed FFMA2 (11..21 always, 7 / 9 for single-slice
    launches) and their scalar 3-D counterparts: every element of forward and adjoint
    (full and edge tiles) and a short PG run against the oracle."""
    rng = np.random.default_rng(sum(xs) * 7 + sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    y_ref = oracle_c.conv_full(x, h)
    assert rel_l2(nd.conv_full(x, h), y_ref) <= TOL_CONV
    assert np.max(np.abs(nd.conv_full(x, h) - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
    r = rng.uniform(-1, 1, y_ref.shape)
    a_ref = oracle_c.adjoint_apply(r, h, xs)
    assert np.max(np.abs(nd.adjoint_apply(r, h, xs) - a_ref)) <= 1e-5 * np.max(np.abs(a_ref))
    yo = y_ref + rng.uniform(0, 1e-3, y_ref.shape)
    cfg = nd.DeconvConfig(max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    got = nd.deconv_pg(yo, h, xs, cfg)
    want = oracle_c.deconv_pg(yo, h, xs, max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    assert got.iterations_run == want.iterations_run
    assert rel_l2(got.estimate, want.estimate) <= 1e-4


@pytest.mark.parametrize("xs,hs", [((12, 40, 50), (9, 33, 33)), ((40, 37, 45), (31, 31, 31)),
                                   ((70, 20, 36), (65, 33, 33)), ((30, 64, 70), (101, 21, 21)),
                                   ((20, 30, 30), (41, 25, 27)), ((16, 20, 70), (47, 19, 13))])
def test_deep_psfs_z_chunks(nd, xs, hs):
    """3-D PSFs with more z-slices than one kernel-parameter tap block holds (config 5's
    65x33x33 and others: 2..16 z-chunk launches accumulated through the scratch volume,
    packed and scalar widths, edge tiles, out-of-range planes skipped): forward and adjoint
    against the float64 oracle over the whole tensor (rel-L2; a float32 sum of up to
    70,785 positive terms is only good to ~sqrt(K) ulp per element), and a short PG run."""
    from oracle.oracle import Oracle
    import os
    fast = Oracle("fast")
    fast.set_threads(os.cpu_count() or 1)
    rng = np.random.default_rng(sum(xs) * 3 + sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    y_ref = fast.conv_full(x, h)
    y = nd.conv_full(x, h)
    assert rel_l2(y, y_ref) <= TOL_CONV
    r = rng.uniform(-1, 1, y_ref.shape)
    a_ref = fast.adjoint_apply(r, h, xs)
    a = nd.adjoint_apply(r, h, xs)
    assert rel_l2(a, a_ref) <= TOL_CONV
    yo = y_ref + rng.uniform(0, 1e-3, y_ref.shape)
    cfg = nd.DeconvConfig(max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    got = nd.deconv_pg(yo, h, xs, cfg)
    want = fast.deconv_pg(yo, h, xs, max_iters=4, tol_rel_objective=0.0, initial_step=1.0)
    assert got.iterations_run == want.iterations_run
    assert rel_l2(got.estimate, want.estimate) <= 1e-4
    np.testing.assert_allclose(got.objective_trace, want.objective_trace, rtol=1e-4)


ND_CASES = [((3, 4, 10, 12), (3, 1, 3, 5)), ((2, 3, 2, 8, 9), (1, 3, 3, 3, 5)), ((2, 3, 6, 7), (5, 3, 3, 3)),
            ((2, 2, 2, 2, 5, 6), (3, 1, 3, 1, 3, 3)), ((4, 5, 33, 40), (3, 3, 7, 9))]


@pytest.mark.parametrize("xs,hs", ND_CASES)
def test_more_than_three_dims(nd, xs, hs):
    """Tensors with 4-6 dimensions (the reference recurses over any ndim,
    convolution.hpp:55-74): the leading dimensions merge into the plane axis with the
    observation's strides (zero planes / zero tap slices in between).  Against the
    reference compiled from its sources (oracle/_ref; the C restatement where it is not
    built): every element of forward and adjoint, a PG run with backtracking, and the
    step estimate."""
    from oracle.oracle import Oracle, available
    ref = Oracle("ref" if available("ref") else "c")
    rng = np.random.default_rng(sum(xs) + 10 * sum(hs))
    x = rng.uniform(0, 1, xs)
    h = rng.uniform(0, 1, hs)
    h /= h.sum()
    y_ref = ref.conv_full(x, h)
    y = nd.conv_full(x, h)
    assert y.shape == y_ref.shape
    assert np.max(np.abs(y - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
    r = rng.uniform(-1, 1, y_ref.shape)
    a_ref = ref.adjoint_apply(r, h, xs)
    assert np.max(np.abs(nd.adjoint_apply(r, h, xs) - a_ref)) <= 1e-5 * np.max(np.abs(a_ref))
    yo = y_ref + rng.uniform(0, 1e-3, y_ref.shape)
    for step in (1.0, 8.0):
        cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0, initial_step=step)
        got = nd.deconv_pg(yo, h, xs, cfg)
        want = ref.deconv_pg(yo, h, xs, max_iters=12, tol_rel_objective=0.0, initial_step=step)
        assert got.estimate.shape == tuple(xs)
        assert got.iterations_run == want.iterations_run and got.stop_reason == want.stop_reason
        assert rel_l2(got.estimate, want.estimate) <= 1e-4, step
        np.testing.assert_allclose(got.objective_trace, want.objective_trace, rtol=1e-4)
    s_ref = ref.estimate_step(h, xs, 30)
    assert abs(nd.estimate_step(h, xs, 30) - s_ref) <= 1e-5 * s_ref
    # the plan keeps the caller's shapes
    with nd.Plan(xs, h) as p:
        p.set_observation(yo)
        assert np.array_equal(p.observation()[0], yo.astype(np.float32).astype(np.float64))
        p.pg_run(nd.DeconvConfig(max_iters=3, tol_rel_objective=0.0, initial_step=1.0))
        assert p.estimate()[0].shape == tuple(xs)
