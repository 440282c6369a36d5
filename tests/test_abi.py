"""CPU: the C-ABI library loads, exports exactly what include/ndconv_b200.h declares,
and fails loudly (no CPU fallback) when no B200 is present."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1711_11224_b200 import _native as N
from paper_1711_11224_b200 import ndconv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ndconv_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ndc_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(N.EXPORTED)


def test_library_exports_every_header_symbol():
    lib = N.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(header_functions())


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_defaults():
    assert b"sm_100a" in N.lib().ndc_version()
    c = N.DeconvConfig()
    N.lib().ndc_deconv_config_default(c)
    # solvers.hpp:20-28
    assert (c.max_iters, c.tol_rel_objective, c.has_initial_step, c.backtrack_factor,
            c.max_backtracks, c.power_iters) == (500, 1e-6, 0, 0.5, 50, 30)
    assert N.lib().ndc_stop_reason_name(2) == b"stalled"


def test_shape_rules_without_device():
    # convolution.hpp:30-38 and kernel.hpp:18-22 are checked before any device work
    assert ndconv.conv_output_shape((4, 5), np.ones((3, 5))) == (6, 9)
    with pytest.raises(ndconv.ShapeError):
        ndconv.conv_output_shape((4, 5), np.ones((2, 5)))
    with pytest.raises(ndconv.ShapeError):
        ndconv.conv_output_shape((4,), np.ones((3, 3)))
    ndconv.set_max_threads(4)
    assert ndconv.max_threads() == 4
    ndconv.set_max_threads(0)
    assert ndconv.max_threads() == 1


@pytest.mark.skipif(ndconv.device_count() > 0, reason="checks the no-device error path")
def test_no_cpu_fallback():
    with pytest.raises(ndconv.DeviceError):
        ndconv.conv_full(np.ones(4), np.ones(3))
    with pytest.raises(ndconv.DeviceError):
        ndconv.deconv_pg(np.ones(6), np.ones(3), (4,))


def slab_py(mz, pz, rank, world):
    base, rem = divmod(mz, world)
    a = rank * base + min(rank, rem)
    b = a + base + (1 if rank < rem else 0)
    ya = 0 if rank == 0 else a + pz
    yb = mz + 2 * pz if rank == world - 1 else b + pz
    return a, b, ya, yb


@pytest.mark.parametrize("mz,pz,world", [(512, 10, 8), (256, 32, 8), (100, 3, 3), (7, 0, 7), (9, 1, 2)])
def test_slab_ranges_partition_both_volumes(mz, pz, world):
    xs, ys = [], []
    for r in range(world):
        got = ndconv.slab_range(mz, pz, r, world)
        assert got == slab_py(mz, pz, r, world)
        xs.append(got[:2])
        ys.append(got[2:])
    assert xs[0][0] == 0 and xs[-1][1] == mz and ys[0][0] == 0 and ys[-1][1] == mz + 2 * pz
    for r in range(1, world):
        assert xs[r][0] == xs[r - 1][1] and ys[r][0] == ys[r - 1][1]
