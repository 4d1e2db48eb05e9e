"""Build libcmn.so in-tree: sm_100a kernels + host runtime behind include/cmn.h.

    python -m paper_1908_00213_b200.build

nvcc cross-compiles for sm_100a without a GPU.  IEEE fp32 semantics are
required for bitwise parity with the oracle, so the flags never include
--use_fast_math / -ftz / -prec-div=false.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcmn.so")
SOURCES = ["cmn_kernels.cu", "cmn_core.cpp", "cmn_schedules.cpp", "cmn_api.cpp", "cmn_nvls.cpp"]
HEADERS = ["cmn_internal.h", "cmn_device.cuh", "cmn_nvls.h", "cmn_comm.h", os.path.join("..", "..", "include", "cmn.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true"]


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
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        extra = os.environ.get("CMN_EXTRA_NVFLAGS", "").split()   # measurement builds only
        cmd = [nvcc(), *ARCH, *NVFLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
