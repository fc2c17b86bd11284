"""Builds libsg2v.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2009_11665_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsg2v.so")
SOURCES = ["api.cpp", "planner.cpp", "kernels.cu", "akernels.cu"]
HEADERS = ["sg2v_internal.h", "kcommon.cuh", os.path.join("..", "..", "include", "sg2v.h")]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cuda_lib = "/usr/local/cuda/lib64"
    cmd = [nvcc(), "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-cudart", "shared", "-Xlinker", f"-rpath,{cuda_lib}", "-ldl",
           "-I", os.path.join(ROOT, "include"),
           "-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
