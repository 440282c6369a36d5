"""Build recipe for libndconv_b200.so (sm_100a) -- in-tree, no JIT cache.

    python -m paper_1711_11224_b200.build          # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  The CUDA runtime is linked
statically and only the ndc_* C-ABI is exported (exports.map), so the library never
interposes on the torch-bundled CUDA runtime or libstdc++ in the same process.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libndconv_b200.so")
CLI = os.path.join(PKG, "ndconv")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
SOURCES = ["ndc_corr_sh0_ry1.cu", "ndc_corr_sh0_ry2.cu", "ndc_corr_sh2_ry1.cu", "ndc_corr_sh2_ry2.cu", "ndc_corr_pair.cu",
           "ndc_kernels.cu", "ndc_plan.cu", "ndc_capi.cu", "ndc_comm.cu", "ndc_io.cu", "ndc_sim.cu",
           "ndc_probe.cu"]
HEADERS = ["ndc_internal.h", "ndc_plan.h", "ndc_correlate.cuh", "ndc_correlate_pair.cuh", "ndc_io.h", "ndc_sim.h", os.path.join("..", "..", "include", "ndconv_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                "-Xptxas", "-v", "-I", os.path.join(PKG, "..", "include")]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    log = ""
    if _newer(obj, deps):
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        log = p.stdout + p.stderr
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{log}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(log)
    return obj, log


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [r[0] for r in results]
    if verbose:
        for _, log in results:
            sys.stdout.write(log)
    mapfile = os.path.join(CSRC, "exports.map")
    if _newer(LIB, objs + [mapfile]):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
               "-Xlinker", f"--version-script={mapfile}", "-ldl", "-lpthread"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}{p.stderr}")
    build_cli()
    return LIB


def build_cli() -> str:
    """The `ndconv` command-line drop-in (tools/main.cpp), linked against the library."""
    src = os.path.join(CSRC, "ndconv_cli.cpp")
    inc = os.path.join(PKG, "..", "include")
    deps = [src, LIB, os.path.join(inc, "ndconv_b200.h"), os.path.join(inc, "ndconv_b200", "ndconv.hpp")]
    if _newer(CLI, deps):
        cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", inc, src, "-o", CLI, f"-L{PKG}", "-l:libndconv_b200.so",
               "-Wl,-rpath,$ORIGIN"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"ndconv CLI build failed:\n{p.stdout}{p.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
