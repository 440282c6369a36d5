"""The C++ drop-in header (include/ndconv_b200/ndconv.hpp): the reference's own test
cases restated in C++ compile against it (CPU) and pass on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
PKG = os.path.join(ROOT, "paper_1711_11224_b200")


def build_binary(out):
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           "-L", PKG, "-lndconv_b200", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_dropin_compiles(tmp_path):
    exe = build_binary(str(tmp_path / "test_dropin"))
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_dropin_reference_cases_pass(tmp_path):
    exe = build_binary(str(tmp_path / "test_dropin"))
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
