"""Bring-up probe: run the conv_full KAT under NDC_DEBUG flag combinations in subprocesses."""
import os, subprocess, sys
code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
from paper_1711_11224_b200 import ndconv as nd
try:
    print("conv", nd.conv_full([1.0, 2.0], [1.0, 1.0, 1.0]).tolist())
    print("conv2d", nd.conv_full(np.ones((5,6)), np.ones((3,3))).sum())
except Exception as e:
    print("ERR", type(e).__name__, e)
'''
for flags in [1, 2, 4, 10, 5, 6, 3]:
    env = dict(os.environ, NDC_DEBUG=str(flags))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    print(flags, (p.stdout + p.stderr).strip().replace("\n", " | ")[-300:], flush=True)
