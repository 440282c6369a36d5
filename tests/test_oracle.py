"""CPU: pin the oracle (oracle/ndconv_oracle.c) against the reference.

* golden fixtures produced by the compiled reference (tests/golden/make_golden.py) --
  bitwise equality, since the restatement keeps the reference's summation order;
* the reference's own known-answer tests, restated (file:line under
  /root/reference/proj/tests/);
* when oracle/_ref/libndconv_ref.so is present, random cross-checks against it.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, available
from tests.golden.make_golden import big_inputs


def test_golden_operators_bitwise(oracle_c, golden_ops):
    d = golden_ops
    for i in range(int(d["n"])):
        x, h = d[f"x{i}"], d[f"h{i}"]
        assert np.array_equal(oracle_c.conv_full(x, h), d[f"y{i}"]), i
        assert np.array_equal(oracle_c.adjoint_apply(d[f"r{i}"], h, x.shape), d[f"atr{i}"]), i
    for i in range(int(d["nbig"])):
        x, h, r = big_inputs(i)
        assert np.array_equal(oracle_c.conv_full(x, h), d[f"by{i}"]), i
        assert np.array_equal(oracle_c.adjoint_apply(r, h, x.shape), d[f"batr{i}"]), i


def _pg_kwargs(cfg):
    kw = dict(max_iters=int(cfg[0]), tol_rel_objective=float(cfg[1]))
    if cfg[2] > 0:
        kw["initial_step"] = float(cfg[2])
    return kw


def test_golden_pg_bitwise(oracle_c, golden_solvers):
    d = golden_solvers
    for i in range(int(d["npg"])):
        rep = oracle_c.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], tuple(d[f"pg_xs{i}"]),
                                 **_pg_kwargs(d[f"pg_cfg{i}"]))
        assert np.array_equal(rep.estimate, d[f"pg_x{i}"]), i
        assert np.array_equal(rep.objective_trace, d[f"pg_obj{i}"]), i
        assert np.array_equal(rep.kkt_trace, d[f"pg_kkt{i}"]), i
        assert rep.iterations_run == int(d[f"pg_it{i}"])
        assert rep.stop_reason == str(d[f"pg_stop{i}"])


def test_golden_steps(oracle_c, golden_solvers):
    d = golden_solvers
    assert oracle_c.estimate_step(np.array([1.0]), (5,), 10) == d["step_h1"]
    assert oracle_c.estimate_step(np.array([2.0]), (5,), 10) == d["step_h2"]
    assert oracle_c.estimate_step(np.ones(3), (8,), 30) == d["step_box"]


def test_golden_rl_bitwise(oracle_c, golden_solvers):
    d = golden_solvers
    for i in range(int(d["nrl"])):
        rep = oracle_c.deconv_rl(d[f"rl_y{i}"], d[f"rl_h{i}"], tuple(d[f"rl_xs{i}"]), max_iters=7)
        assert np.array_equal(rep.estimate, d[f"rl_x{i}"]), i
        assert np.array_equal(rep.objective_trace, d[f"rl_obj{i}"]), i
        assert np.array_equal(rep.kkt_trace, d[f"rl_kkt{i}"]), i
        assert rep.extra["negative_pixels_clamped"] == int(d[f"rl_clamped{i}"])


# --- the reference's KATs, restated -----------------------------------------------------

def test_kat_conv_full(oracle_c):
    # test_convolution.cpp:11-19, 40-45
    assert np.array_equal(oracle_c.conv_full([1.0, 2.0], [1.0, 1.0, 1.0]), [1, 3, 3, 2])
    assert np.array_equal(oracle_c.conv_full([1.0, 2.0, 3.0], [0.0, 1.0, 0.0]), [0, 1, 2, 3, 0])
    assert np.array_equal(oracle_c.conv_full([3.0], [1.0, 2.0, 4.0, 2.0, 1.0]), [3, 6, 12, 6, 3])


def test_kat_adjoint_impulse(oracle_c):
    # test_convolution.cpp:104-108
    assert np.array_equal(oracle_c.adjoint_apply([1.0, 0, 0, 0], [1.0, 2.0, 3.0], (2,)), [1.0, 0.0])


def test_kat_objective_and_steps(oracle_c):
    # test_solvers.cpp:12-40
    assert oracle_c.objective([1.0], [3.0], [1.0]) == 2.0
    assert abs(oracle_c.estimate_step([1.0], (5,), 10) - 1.0) <= 1e-12
    assert abs(oracle_c.estimate_step([2.0], (5,), 10) - 0.25) <= 1e-12
    s = oracle_c.estimate_step([1.0, 1.0, 1.0], (8,), 30)
    assert 1 / 9 <= s <= 1.0
    with pytest.raises(OracleError) as e:
        oracle_c.estimate_step([0.0, 0.0, 0.0], (4,), 5)
    assert e.value.kind == "NumericError"


def test_kat_solver_edges(oracle_c):
    # test_solvers.cpp:62-93
    rep = oracle_c.deconv_pg(np.array([3.0, -2.0, 0.0, 5.0]), [1.0], (4,), max_iters=50)
    assert np.array_equal(rep.estimate, [3.0, 0.0, 0.0, 5.0])
    assert rep.stop_reason == "converged" and rep.iterations_run <= 2
    rep = oracle_c.deconv_pg(np.full(6, -2.0), [0.2, 0.5, 0.3], (4,), max_iters=100)
    assert np.array_equal(rep.estimate, np.zeros(4)) and rep.kkt_trace[-1] == 0.0


def test_error_kinds(oracle_c):
    # test_convolution.cpp:33-38, test_solvers.cpp:168-189
    with pytest.raises(OracleError) as e:
        oracle_c.deconv_pg(np.zeros(6), [0.1, 0.8, 0.1], (5,))
    assert e.value.kind == "ShapeError"
    with pytest.raises(OracleError) as e:
        oracle_c.deconv_pg(np.zeros(6), [0.0, 0.0, 0.0], (4,))
    assert e.value.kind == "NumericError"
    with pytest.raises(OracleError) as e:
        oracle_c.deconv_pg(np.zeros(6), [0.1, 0.8, 0.1], (4,), backtrack_factor=1.0)
    assert e.value.kind == "Error"


def test_sampled_equals_full(oracle_c):
    g = np.random.Generator(np.random.PCG64(5))
    x = g.uniform(-1, 1, (7, 9, 11))
    h = g.uniform(-1, 1, (3, 5, 7))
    y = oracle_c.conv_full(x, h)
    idx = g.integers(0, y.size, 50)
    assert np.array_equal(oracle_c.conv_full_sample(x, h, idx), y.ravel()[idx])
    r = g.uniform(-1, 1, y.shape)
    a = oracle_c.adjoint_apply(r, h, x.shape)
    idx = g.integers(0, a.size, 50)
    assert np.array_equal(oracle_c.adjoint_sample(r, h, x.shape, idx), a.ravel()[idx])


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
def test_c_restatement_matches_reference_random():
    c, r = Oracle("c"), Oracle("ref")
    g = np.random.Generator(np.random.PCG64(99))
    for _ in range(60):
        nd = int(g.integers(1, 4))
        xs = tuple(int(v) for v in g.integers(1, 6, nd))
        hs = tuple(int(2 * v + 1) for v in g.integers(0, 3, nd))
        x, h = g.uniform(-1, 1, xs), g.uniform(-1, 1, hs)
        y = r.conv_full(x, h)
        assert np.array_equal(c.conv_full(x, h), y)
        yy = g.uniform(-1, 1, y.shape)
        assert np.array_equal(c.adjoint_apply(yy, h, xs), r.adjoint_apply(yy, h, xs))
        if np.any(h != 0):
            a = c.deconv_pg(yy, h, xs, max_iters=15, tol_rel_objective=0.0)
            b = r.deconv_pg(yy, h, xs, max_iters=15, tol_rel_objective=0.0)
            assert np.array_equal(a.estimate, b.estimate)
            assert np.array_equal(a.objective_trace, b.objective_trace)


# --- the threaded float64 oracle (oracle/ndconv_fast.c) used for config-scale parity ----

@pytest.fixture(scope="module")
def oracle_fast():
    import os
    o = Oracle("fast")
    o.set_threads(os.cpu_count() or 1)
    return o


def _rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - b).ravel()) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def test_fast_oracle_operators(oracle_c, oracle_fast, golden_ops):
    """Same sums in another order: every golden operator case and random 1-3-d shapes
    (kernels larger than the input included) to 1e-13 relative."""
    d = golden_ops
    for i in range(int(d["n"])):
        x, h = d[f"x{i}"], d[f"h{i}"]
        if x.ndim > 3:
            continue
        assert _rel(oracle_fast.conv_full(x, h), d[f"y{i}"]) <= 1e-13, i
        assert _rel(oracle_fast.adjoint_apply(d[f"r{i}"], h, x.shape), d[f"atr{i}"]) <= 1e-13, i
    g = np.random.Generator(np.random.PCG64(2024))
    for _ in range(60):
        nd_ = int(g.integers(1, 4))
        xs = tuple(int(v) for v in g.integers(1, 40 if nd_ < 3 else 12, nd_))
        hs = tuple(int(2 * v + 1) for v in g.integers(0, 9 if nd_ < 3 else 4, nd_))
        x, h = g.uniform(-1, 1, xs), g.uniform(-1, 1, hs)
        y = oracle_c.conv_full(x, h)
        assert _rel(oracle_fast.conv_full(x, h), y) <= 1e-13, (xs, hs)
        r = g.uniform(-1, 1, y.shape)
        assert _rel(oracle_fast.adjoint_apply(r, h, xs), oracle_c.adjoint_apply(r, h, xs)) <= 1e-13, (xs, hs)


def test_fast_oracle_steps_and_pg(oracle_c, oracle_fast, golden_solvers):
    """estimate_step and whole PG runs (golden family, config 1 with the auto step, the
    KATs) against the bitwise oracle: steps to 1e-12, estimates / traces to 1e-10, same
    iteration counts and stop reasons."""
    d = golden_solvers
    assert oracle_fast.estimate_step(np.array([2.0]), (5,), 10) == pytest.approx(float(d["step_h2"]), rel=1e-14)
    assert oracle_fast.estimate_step(np.ones(3), (8,), 30) == pytest.approx(float(d["step_box"]), rel=1e-12)
    n = int(d["npg"])
    for i in list(range(n - 5)) + [n - 5, n - 4, n - 3, n - 1]:
        kw = _pg_kwargs(d[f"pg_cfg{i}"])
        xs = tuple(int(v) for v in d[f"pg_xs{i}"])
        rep = oracle_fast.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], xs, **kw)
        assert rep.stop_reason == str(d[f"pg_stop{i}"]), i
        n_it = int(d[f"pg_it{i}"])
        tol = 1e-10 if rep.iterations_run == n_it else 1e-8
        assert _rel(rep.estimate, d[f"pg_x{i}"]) <= tol or np.max(np.abs(rep.estimate - d[f"pg_x{i}"])) <= 1e-12, i
        if rep.iterations_run != n_it:
            # the bitwise fixed-point test trial == x (solvers.hpp:191) near a stalled
            # optimum: a reordered sum may accept one more (or one fewer) tiny step
            assert rep.stop_reason == "converged" and abs(rep.iterations_run - n_it) <= 2, i
            m = min(rep.iterations_run, n_it) + 1
            np.testing.assert_allclose(rep.objective_trace[:m], d[f"pg_obj{i}"][:m], rtol=1e-10)
        else:
            np.testing.assert_allclose(rep.objective_trace, d[f"pg_obj{i}"], rtol=1e-10, atol=1e-300)
    assert rep.extra["step0"] == pytest.approx(float(d["c1_step"]), rel=1e-12)


def test_fast_oracle_3d_pg(oracle_c, oracle_fast):
    """A 3-D run with the config-3 PSF shape (31x15x15) on a small volume: whole PG run
    equal to the bitwise oracle to 1e-10."""
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c3", shape=(12, 16, 14), n_objects=6)
    a = oracle_c.deconv_pg(y, h, x.shape, max_iters=8, tol_rel_objective=0.0)
    b = oracle_fast.deconv_pg(y, h, x.shape, max_iters=8, tol_rel_objective=0.0)
    assert a.iterations_run == b.iterations_run == 8
    assert _rel(b.estimate, a.estimate) <= 1e-10
    np.testing.assert_allclose(b.objective_trace, a.objective_trace, rtol=1e-10)
    np.testing.assert_allclose(b.kkt_trace, a.kkt_trace, rtol=1e-8)


def test_f64_sensitivity_of_the_golden_family(oracle_c, golden_solvers):
    """The bar the GPU PG tests hold the random family to (1e-4) is not looser than the
    reference's own conditioning: rerun on inputs perturbed at float32 rounding level
    (relative 2^-24 per entry), the f64 reference's estimates move by <= 1e-6 on every
    golden PG case except acceptance criterion 6's marginally contractive step-8 run
    (measured 1e-7 .. 9e-7), which tests/test_gpu_pg.py holds to the envelope of such
    perturbed runs instead."""
    d = golden_solvers
    n = int(d["npg"])
    for i in range(n):
        if i == n - 2 or i == n - 1:  # acceptance 6 (envelope test) and config 1 (slow here)
            continue
        y, h, xs = d[f"pg_y{i}"], d[f"pg_h{i}"], tuple(int(v) for v in d[f"pg_xs{i}"])
        g = np.random.Generator(np.random.PCG64(i))
        for _ in range(3):
            yp = y * (1 + g.uniform(-1, 1, y.shape) * 2.0 ** -24)
            hp = h * (1 + g.uniform(-1, 1, h.shape) * 2.0 ** -24)
            r = oracle_c.deconv_pg(yp, hp, xs, **_pg_kwargs(d[f"pg_cfg{i}"]))
            assert _rel(r.estimate, d[f"pg_x{i}"]) <= 1e-6, i


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
def test_oracle_more_than_three_dims_bitwise():
    """4-6-d tensors: the C restatement equals the compiled reference bit for bit
    (conv_full, adjoint_apply, a short PG run) -- the reference recurses over any ndim
    (convolution.hpp:55-74)."""
    ref, orc = Oracle("ref"), Oracle("c")
    g = np.random.Generator(np.random.PCG64(41))
    for xs, hs in (((3, 4, 10, 12), (3, 1, 3, 5)), ((2, 3, 2, 8, 9), (1, 3, 3, 3, 5)),
                   ((2, 3, 6, 7), (5, 3, 3, 3)), ((2, 2, 2, 2, 5, 6), (3, 1, 3, 1, 3, 3))):
        x, h = g.uniform(0, 1, xs), g.uniform(-1, 1, hs)
        y = ref.conv_full(x, h)
        assert np.array_equal(orc.conv_full(x, h), y)
        assert np.array_equal(orc.adjoint_apply(y, h, xs), ref.adjoint_apply(y, h, xs))
        a = ref.deconv_pg(y, np.abs(h), xs, max_iters=5, tol_rel_objective=0.0, initial_step=1.0)
        b = orc.deconv_pg(y, np.abs(h), xs, max_iters=5, tol_rel_objective=0.0, initial_step=1.0)
        assert np.array_equal(a.estimate, b.estimate) and np.array_equal(a.objective_trace, b.objective_trace)


def test_f32_restatement_tracks_the_reference(oracle_c, golden_solvers):
    """oracle/pg_f32.py (deconv_pg in float32, the GPU tests' measure of what float32 can
    resolve) follows the f64 reference on the golden random family to <= 2e-4, with the
    same stop reasons, and reproduces the identity-kernel KATs exactly."""
    from oracle.pg_f32 import deconv_pg_f32
    d = golden_solvers
    n = int(d["npg"])
    for i in list(range(n - 5)) + [n - 5, n - 4, n - 3]:
        cfg = d[f"pg_cfg{i}"]
        xs = tuple(int(v) for v in d[f"pg_xs{i}"])
        step = float(cfg[2]) if cfg[2] > 0 else oracle_c.estimate_step(d[f"pg_h{i}"], xs, 30)
        x, tr, it, reason = deconv_pg_f32(d[f"pg_y{i}"], d[f"pg_h{i}"], xs, step, int(cfg[0]), float(cfg[1]))
        assert reason == str(d[f"pg_stop{i}"]), i
        assert _rel(x, d[f"pg_x{i}"]) <= 2e-4 or np.max(np.abs(x - d[f"pg_x{i}"])) <= 1e-6, i
