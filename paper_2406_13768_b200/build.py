"""Build libfastpersist.so in-tree with nvcc for sm_100a.

    python -m paper_2406_13768_b200.build [--force]

The library is plain C++ + CUDA behind the C-ABI in include/fastpersist.h;
the Python binding loads it with ctypes (no torch extension).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libfastpersist.so")
BUILD = os.path.join(ROOT, "build")

SOURCES = ["layout.cpp", "io.cpp", "crc32.cpp", "runtime.cpp", "load.cpp", "gds.cpp", "pack.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _newest_input():
    paths = [os.path.join(CSRC, s) for s in SOURCES]
    paths += [os.path.join(CSRC, "fp_internal.h"), os.path.join(CSRC, "ctx.h"), os.path.join(INCLUDE, "fastpersist.h"),
              os.path.abspath(__file__)]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall", "-I", INCLUDE, "-I", CSRC]
    common += os.environ.get("FP_NVCC_FLAGS", "").split()  # experiments (e.g. -DFP_BC_SKIP_CRC)

    def compile_one(src):
        obj = os.path.join(BUILD, src + ".o")
        cmd = [NVCC, *common, *ARCH, "-lineinfo", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if src.endswith(".cu"):
            with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
                f.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
