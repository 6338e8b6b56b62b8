"""Compiles the sm_100a library (nvcc, in-tree) — used by __graft_entry__.build() and the loader."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libfastblend.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
DEPS = SOURCES + sorted(glob.glob(os.path.join(PKG, "csrc", "*.h"))) + sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) \
    + [os.path.join(ROOT, "include", "fb.h")]

# -fmad=false: no implicit FMA contraction anywhere (the arithmetic contract, DESIGN.md §3 D20);
# no --use_fast_math (IEEE division / rounding are part of the contract).
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-fmad=false",
              "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build_library(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, *SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
