"""Build libipls.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so travels with the repo."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libipls.so")
SOURCES = [os.path.join(HERE, "csrc", "ipls_api.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu*")) +
              [os.path.join(ROOT, "include", "ipls.h")])

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # the model is written with __dmul_rn/__dadd_rn anyway (R7)
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if c == "nvcc" or os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB, *SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
