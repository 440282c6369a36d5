"""SASS guard for the tap loop (CPU-only: reads the built library with cuobjdump).

The correlation kernels keep their tap operand on the uniform datapath (`LDCU` into a
uniform register, `FFMA R, R, UR` / `FFMA2 R, R, UR.F32, R`), which is what holds the
issue rate of the loop at ~96 % FFMA ("Kernels").  ptxas decides this per
instantiation and small unrelated source edits can flip it: a build whose config-3
kernel had 113 of 565 FFMA2 on uniform taps ran config 3's forward 10 % slower
(profiles/r01m_kbench_z_fast.txt, lib_zf0).  This test fails such a build before it
reaches the GPU.
"""
import os
import re
import shutil
import subprocess

import pytest

from paper_1711_11224_b200 import _native as N

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

# (KX, RY, PK) of the full-tile kernels the BASELINE configs run, and the minimum share
# of their FFMA / FFMA2 instructions whose tap operand is a uniform register.  RY = 1
# kernels keep ~15 % of their FMAs in the epilogue-side NR = 1 path on registers.
EXPECT = {
    (31, 2, 0): 1.0,   # c2 (31x31)
    (15, 2, 1): 1.0,   # c3 (15x15 in-plane, packed FFMA2)
    (9, 2, 0): 1.0,    # c4 (9x9 in-plane)
    (33, 2, 0): 1.0,   # c5 (33x33 in-plane, 128-row tiles on one stage)
    (33, 1, 0): 0.80,  # 33-wide PSFs too tall for a 128-row TMA box (64-row tiles)
    (5, 2, 0): 1.0,    # c2s (5x5)
}

EPILOGUE_FMAS = 48


def _scan():
    out = subprocess.run([CUOBJDUMP, "-sass", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    stats, key = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : \S*correlate_kernelILi(\d+)ELi(\d)ELi(\d)ELb(\d)ELb(\d)E", line)
        if m:
            kx, sh, ry, edge, pk = map(int, m.groups())
            key = (kx, sh, ry, edge, pk)
            stats[key] = [0, 0]
            continue
        m = re.search(r"Function : \S*correlate_pair_kernelILi(\d+)ELi(\d)ELi(\d)E", line)
        if m:  # two output planes per CTA (config 4's full tiles): key edge = -1
            kx, sh, ry = map(int, m.groups())
            key = (kx, sh, ry, -1, 0)
            stats[key] = [0, 0]
            continue
        if "Function :" in line:
            key = None
            continue
        if key is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?FFMA2?\b([^;]*);", line)
        if m:
            stats[key][0] += 1
            if re.search(r"\bUR\d+\b", m.group(1)):
                stats[key][1] += 1
    return stats


@pytest.mark.skipif(not os.path.exists(N.LIB_PATH), reason="library not built")
def test_tap_operands_on_uniform_datapath():
    if not (os.path.exists(CUOBJDUMP) or shutil.which("cuobjdump")):
        pytest.skip("cuobjdump not available")
    stats = _scan()
    bad = []
    for (kx, ry, pk), need in EXPECT.items():
        for sh in (0, 2):
            t, u = stats.get((kx, sh, ry, 0, pk), (0, 0))
            assert t > 0, f"correlate_kernel<{kx},{sh},{ry},0,{pk}> not found in {N.LIB_PATH}"
            # (up to EPILOGUE_FMAS register-operand FMAs are the epilogue's own: the Newton
            # steps of the Richardson-Lucy ratio's divisions, inlined or not as ptxas decides)
            if (u + min(t - u, EPILOGUE_FMAS)) / t < need:
                bad.append(f"<{kx},{sh},{ry},0,{pk}>: {u}/{t} FMAs on uniform taps (need {need:.0%})")
    for sh in (0, 2):  # config 4's two-planes kernel
        t, u = stats.get((9, sh, 2, -1, 0), (0, 0))
        assert t > 0, f"correlate_pair_kernel<9,{sh},2> not found in {N.LIB_PATH}"
        if (u + min(t - u, EPILOGUE_FMAS)) / t < 1.0:
            bad.append(f"pair<9,{sh},2>: {u}/{t} FMAs on uniform taps")
    assert not bad, "tap loop left the uniform datapath: " + "; ".join(bad)
