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
