"""Build recipe for the in-tree sm_100a library (libtt_b200.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs anywhere the
CUDA 12.9 toolkit is present; the .so is built in-tree so that it travels to
the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtt_b200.so")

SOURCES = ["tt_kernels.cu", "tt_context.cpp", "tt_device_api.cpp", "tt_host.cpp", "tt_jit.cpp"]
HEADERS = ["tt_kernels.cuh", "tt_jit.h", "tt_context_impl.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "tt_b200.h"),
                                                                 __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libtt_b200.so (or a variant with extra -D flags into `out`, for experiments)."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    cmd = ["nvcc", "-ccbin", "g++", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off", *ARCH, "-O3",
           "-lineinfo", "-std=c++17", "-I" + os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines],
           *[os.path.join(CSRC, f) for f in SOURCES], "-ldl", "-o", target + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
