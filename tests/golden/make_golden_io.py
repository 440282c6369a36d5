"""Write tests/golden/io/: tensor and graymap files produced by the REFERENCE writer
(imageio.hpp via oracle/_ref ref_io_serialize_*), plus fixtures.npz with the values
the reference reader returns for each file.  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden_io.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle.oracle import Oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "io")


def main():
    ref = Oracle("ref")
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2024)
    files = {
        "t_1d.ndt": ref.serialize_tensor(rng.standard_normal(9)),
        "t_2d.ndt": ref.serialize_tensor(rng.standard_normal((5, 6)) * 1e5),
        "t_3d.ndt": ref.serialize_tensor(rng.uniform(0, 1, (3, 4, 5))),
        "g_8bit.pgm": ref.serialize_pgm(rng.integers(0, 256, (6, 9)).astype(np.float64), False),
        "g_round.pgm": ref.serialize_pgm(np.array([[0.5, 1.5, 2.5, 3.49, 254.5, 255.0]]), False),
        # inputs only (not re-written bit-exactly: P2 / 16-bit are read-only forms)
        "in_ascii.pgm": b"P2\n# comment\n3 2\n1000\n0 500 1000\n7 8 9\n",
        "in_wide.pgm": b"P5 3 1 4095\n" + bytes([0, 1, 15, 255, 0, 0]),
    }
    values = {}
    for name, data in files.items():
        with open(os.path.join(OUT, name), "wb") as f:
            f.write(data)
        stem, ext = os.path.splitext(name)
        values[stem] = ref.parse_pgm(data) if ext == ".pgm" else ref.parse_tensor(data)
    np.savez(os.path.join(OUT, "fixtures.npz"), **values)
    print("wrote", sorted(files))


if __name__ == "__main__":
    main()
