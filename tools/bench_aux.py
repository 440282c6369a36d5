"""Throughput of the §8f rows around the PG path (tensor files <-> HBM, device noise and
phantoms) against the reference's CPU code on the same data (oracle/_ref), one JSON line.

    python tools/bench_aux.py [--out profiles/r01_aux.json]

Files are written to /tmp first, so the streamed load reads from the page cache: the
number is the host->HBM path (parse, validate, f64->f32, pinned H2D), not the disk.
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402
from paper_1711_11224_b200 import ndconv as nd, synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ref = Oracle("ref")
    res = {}
    h = synth.psf_for("c2")
    B, xs = 16, (2048, 2048)
    ys = nd.conv_output_shape(xs, h)
    rng = np.random.default_rng(0)
    y = rng.uniform(0, 1000, (B,) + ys)
    tmp = tempfile.mkdtemp(dir="/tmp")
    path, out = os.path.join(tmp, "y.ndt"), os.path.join(tmp, "x.ndt")
    nd.write_tensor(y, path)
    fbytes = os.path.getsize(path)
    p = nd.Plan(xs, h, batch=B)
    t_load = timed(lambda: p.load_observation(path))
    t_set = timed(lambda: p.set_observation(y))
    t_save = timed(lambda: p.save_estimate(out))
    img = y[0]
    img_bytes = b"NDTENSOR 2 %d %d\n" % img.shape + img.astype("<f8").tobytes()
    t_ref_parse = timed(lambda: ref.parse_tensor(img_bytes), reps=2)
    res["ndtensor_load"] = {"workload": f"c2 observation {B}x{ys[0]}x{ys[1]} f64 ({fbytes / 1e9:.2f} GB file)",
                            "s": t_load, "GB_per_s": fbytes / t_load / 1e9,
                            "in_memory_set_observation_GB_per_s": y.nbytes / t_set / 1e9,
                            "reference_read_tensor_GB_per_s": len(img_bytes) / t_ref_parse / 1e9,
                            "reference_sample": "io::read_tensor(std::istream) on one image, bytes in memory"}
    xb = B * xs[0] * xs[1] * 8
    res["ndtensor_save"] = {"s": t_save, "GB_per_s": xb / t_save / 1e9}

    n = y.size
    t_noise = timed(lambda: p.add_gaussian_noise(0.0, 5.0, 1))
    t_ref_noise = timed(lambda: ref.add_gaussian_noise(img.ravel(), 0.0, 5.0, 1), reps=2)
    res["gaussian_noise"] = {"workload": f"{n} samples in place on the resident observation",
                             "s": t_noise, "samples_per_s": n / t_noise,
                             "reference_samples_per_s": img.size / t_ref_noise,
                             "reference_sample": "sim::add_gaussian_noise on one 2078^2 image, 1 thread"}
    t_mt = timed(lambda: nd.mt19937_64(1, 50_000_000))
    res["mt19937_64_raw"] = {"words": 50_000_000, "s": t_mt, "words_per_s": 5e7 / t_mt,
                             "note": "includes the 400 MB D2H"}
    t_tex = timed(lambda: nd.phantom_texture(4096, 4096))
    t_ref_tex = timed(lambda: ref.phantom_texture(4096, 4096), reps=1)
    res["phantom_texture"] = {"pixels": 4096 * 4096, "s": t_tex, "reference_s": t_ref_tex}
    p.close()
    os.remove(path)
    os.remove(out)
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
