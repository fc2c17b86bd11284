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
CHECK_LIB = os.path.join(LIBDIR, "libsg2v_check.so")  # device bounds checks (SG2V_DASSERT), tests only
SOURCES = ["api.cpp", "planner.cpp", "kernels.cu", "akernels.cu"]
HEADERS = ["sg2v_internal.h", "kcommon.cuh", os.path.join("..", "..", "include", "sg2v.h")]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """sha256 (16 hex) of the library sources: stamps profiles (ncu traffic) so a bench
    line only quotes DRAM traffic measured on the code it runs."""
    import hashlib
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, check: bool = False) -> str:
    """check=True builds lib/libsg2v_check.so with the device bounds checks compiled in
    (-DSG2V_CHECK); select it with SG2V_LIB for a test run."""
    out = CHECK_LIB if check else LIB
    if not force and not _stale(out):
        return out
    os.makedirs(LIBDIR, exist_ok=True)
    cuda_lib = "/usr/local/cuda/lib64"
    common = [nvcc(), "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-I", os.path.join(ROOT, "include")] + (["-DSG2V_CHECK"] if check else [])
    if verbose:
        common.insert(1, "-Xptxas=-v")
    objdir = os.path.join(LIBDIR, "obj_check" if check else "obj")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for s in SOURCES:  # one nvcc per translation unit, in parallel
        o = os.path.join(objdir, s + ".o")
        objs.append(o)
        cmd = common + ["-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "shared",
            "-Xlinker", f"-rpath,{cuda_lib}", "-ldl", "-o", out] + objs
    subprocess.check_call(link)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, check="--check" in sys.argv))
