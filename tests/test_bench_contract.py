"""bench.py's driver contract, checked on CPU: the reference arm's JSON line (the
reference's own CPU implementation, oracle/_ref) and the product arm failing loudly
when no B200 is visible (no CPU fallback behind the headline number)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libndconv_ref.so")


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_reference_arm_line():
    p = _run("--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference"
    assert d["metric"] == base["metric"]
    assert d["unit"] == "voxel-iterations/s" and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["workload"].startswith("c2:")


def test_product_arm_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    p = _run("--steps", "1", "--warmup", "3", timeout=300)
    assert p.returncode != 0
    assert not [l for l in p.stdout.splitlines() if l.startswith("{") and '"value"' in l]


def test_default_workload_is_config5_at_every_n():
    """north_star's scaling target is config 5 (the largest 3-D volume): the default
    workload for every N, z-slab sharded when N > 1 (BENCH N=1 == SCALE N=1)."""
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse([])
    assert a.config == "c5" and a.gpus == 1 and a.warmup >= 3
    assert bench.WORK["c5"]["e2e_iters"] == 20 and "c5" in bench.VOLUME
