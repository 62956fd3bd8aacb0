"""Builds libgempe_b200.so in-tree: nvcc for the sm_100a kernels, g++ for the host C++ behind the C-ABI.

    python -m paper_2011_03479_b200.build [--force]

The library links cudart statically and exports exactly the symbols of include/gempe.h.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(OUT_DIR, "libgempe_b200.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

CU_SOURCES = ["kernels.cu"]
CXX_SOURCES = ["hostmath.cpp", "context.cpp", "engine.cpp", "group.cpp", "formats.cpp", "hostcopy.cpp"]
HEADERS = ["kernels.hpp", "context.hpp", "hostmath.hpp", "device_fns.cuh", os.path.join(ROOT, "include", "gempe.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"] + os.environ.get("GEMPE_NVCC_EXTRA", "").split()
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", f"-I{CUDA_HOME}/include"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    tag = os.path.join(OUT_DIR, ".flags")  # built with other flags (GEMPE_NVCC_EXTRA A/B builds)
    if os.path.exists(tag) and open(tag).read() != " ".join(NVCC_FLAGS + CXX_FLAGS):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in CU_SOURCES + CXX_SOURCES] + \
           [h if os.path.isabs(h) else os.path.join(CSRC, h) for h in HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [h if os.path.isabs(h) else os.path.join(CSRC, h) for h in HEADERS] + [os.path.abspath(__file__)]
    flags_tag = os.path.join(OUT_DIR, ".flags")
    flags_now = " ".join(NVCC_FLAGS + CXX_FLAGS)
    flags_same = os.path.exists(flags_tag) and open(flags_tag).read() == flags_now

    def fresh(obj, source):  # the object is newer than its source and every header, and the flags did not change
        return (not force and flags_same and os.path.exists(obj) and
                all(os.path.getmtime(obj) > os.path.getmtime(d) for d in [source] + headers))

    objs = []
    for s in CU_SOURCES:
        o = os.path.join(OUT_DIR, s + ".o")
        if not fresh(o, os.path.join(CSRC, s)):
            cmd = [NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, s), "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.check_call(cmd)
        objs.append(o)
    for s in CXX_SOURCES:
        o = os.path.join(OUT_DIR, s + ".o")
        if not fresh(o, os.path.join(CSRC, s)):
            subprocess.check_call(["g++", *CXX_FLAGS, "-c", os.path.join(CSRC, s), "-o", o])
        objs.append(o)
    with open(flags_tag, "w") as f:
        f.write(flags_now)
    subprocess.check_call([NVCC, "-shared", "-o", LIB, *objs, "-cudart", "static",
                           "-Xlinker", "--exclude-libs=ALL"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
