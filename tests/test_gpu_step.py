"""estimate_step (solvers.hpp:127-143) for separable PSFs: the power iteration as the
product of 1-D power iterations (Kronecker structure, Plan::estimate_step_separable)
against the reference oracle and against the device power iteration."""
import os

import numpy as np
import pytest

from paper_1711_11224_b200 import synth

pytestmark = pytest.mark.gpu


def _sep(shape, sig, seed):
    # separable by construction: outer product of 1-D profiles
    g = np.random.default_rng(seed)
    fs = [np.exp(-0.5 * ((np.arange(k) - k // 2) / s) ** 2) * g.uniform(0.9, 1.1) for k, s in zip(shape, sig)]
    h = fs[0]
    for f in fs[1:]:
        h = np.multiply.outer(h, f)
    return h / h.sum()


@pytest.fixture
def env():
    old = os.environ.get("NDC_SEPARABLE_STEP")
    yield os.environ
    if old is None:
        os.environ.pop("NDC_SEPARABLE_STEP", None)
    else:
        os.environ["NDC_SEPARABLE_STEP"] = old


@pytest.mark.parametrize("xs,hs", [((40,), (7,)), ((30, 44), (9, 5)), ((12, 20, 26), (5, 7, 3)),
                                   ((6, 9, 11), (1, 3, 5)), ((2, 1), (5, 1))])
def test_separable_step_matches_reference(nd, oracle_c, env, xs, hs):
    """Forced onto the separable path even for small problems: the reference's step to
    1e-12 (its own estimate_step KAT tolerance), including the symmetric tiny case whose
    all-ones start is a non-dominant eigenvector."""
    h = _sep(hs, [max(1.0, k / 3) for k in hs], sum(xs))
    env["NDC_SEPARABLE_STEP"] = "2"
    got = nd.estimate_step(h, xs, 30)
    want = oracle_c.estimate_step(h, xs, 30)
    assert abs(got - want) <= 1e-12 * abs(want)


def test_nonseparable_falls_back(nd, oracle_c, env):
    g = np.random.default_rng(5)
    h = g.uniform(0, 1, (5, 7))
    h /= h.sum()
    env["NDC_SEPARABLE_STEP"] = "2"
    got = nd.estimate_step(h, (30, 40), 30)
    assert abs(got - oracle_c.estimate_step(h, (30, 40), 30)) <= 1e-12 * got


def test_fp32_rounded_separable_psf(nd, oracle_c, env):
    """A separable Gaussian rounded to float32 (how the BASELINE PSFs are fed) is rank-1
    only to ~1e-7 per entry: the separable path's step stays within 2e-6 of the
    reference's (the float32 device iteration it replaces: ~1e-5)."""
    h = synth.gaussian_psf((9, 7, 5), (2.0, 1.5, 1.2)).astype(np.float32).astype(np.float64)
    env["NDC_SEPARABLE_STEP"] = "2"
    got = nd.estimate_step(h, (14, 22, 30), 30)
    want = oracle_c.estimate_step(h, (14, 22, 30), 30)
    assert abs(got - want) <= 2e-6 * want


@pytest.mark.parametrize("name,shape", [("c2", (2048, 2048)), ("c3", (128, 256, 256)), ("c4", (64, 256, 256))])
def test_separable_step_config_psfs(nd, env, name, shape):
    """BASELINE PSFs (float32-rounded Gaussians, separable to ~1e-7 per tap) at sizes
    that use the float32 device power iteration otherwise: both paths agree to float32
    accuracy."""
    h = synth.psf_for(name)
    env["NDC_SEPARABLE_STEP"] = "1"
    sep = nd.estimate_step(h, shape, 30)
    env["NDC_SEPARABLE_STEP"] = "0"
    dev = nd.estimate_step(h, shape, 30)
    assert abs(sep - dev) <= 2e-5 * dev
