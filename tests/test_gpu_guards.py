"""GPU memory-safety and race evidence without compute-sanitizer (closed on the GPU
pool): the library's guard-band mode (NDC_GUARD_BANDS=1 puts 1 MB of a fill pattern
before and after every plan allocation and checks it on demand and at plan destruction)
over the device paths with the riskiest addressing, each run twice -- no guard byte may
change (no out-of-bounds device write) and every result must repeat bit for bit (no
data race between warps, CTAs, the edge-tile side stream, the halo comm stream or the
speculative pass).  See tests/_guard_run.py for the cases."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_and_repeatability(nd):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_guard_run.py")], capture_output=True,
                       text=True, timeout=900, env=dict(os.environ, NDC_GUARD_BANDS="1"))
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["arrays"] > 40
    assert r["live_plan_bad"] == 0 and r["total_guard_violations"] == 0, r
    assert r["repeat_bit_identical"], r


def test_guard_bands_detect_a_corruption(nd):
    """The checker itself: 16 bytes written just past the observation buffer (the debug
    entry ndc_plan_debug_corrupt_guard) are reported, live and at destruction."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from paper_1711_11224_b200 import ndconv as nd, _native as N\n"
        "p = nd.Plan((64, 64), np.ones((3, 3)) / 9, batch=1)\n"
        "p.set_observation(np.zeros((66, 66)))\n"
        "p.pg_run(nd.DeconvConfig(max_iters=2))\n"
        "assert p.check_guards() == 0\n"
        "assert N.lib().ndc_plan_debug_corrupt_guard(p.handle) == 0\n"
        "assert p.check_guards() == 16\n"
        "p.close()\n"
        "assert nd.guard_violations() == 32\n"
        "print('ok')\n" % ROOT)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, NDC_GUARD_BANDS="1"))
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-3000:]
