"""Build recipe for the in-tree sm_100a library (libtt_b200.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs anywhere the
CUDA 12.9 toolkit is present; the .so is built in-tree so that it travels to
the GPU box with the repo snapshot.  Each source compiles to its own object
(build/obj, in parallel; only sources newer than their object, or whose
headers changed, are recompiled), then one link.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtt_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

SOURCES = ["tt_kernels.cu", "tt_context.cpp", "tt_device_api.cpp", "tt_host.cpp", "tt_jit.cpp"]
HEADERS = ["tt_kernels.cuh", "tt_jit.h", "tt_context_impl.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-ccbin", "g++", "-Xcompiler", "-fPIC,-ffp-contract=off", *ARCH, "-O3", "-lineinfo", "-std=c++17"]


def _deps():
    return [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(ROOT, "include", "tt_b200.h"), __file__]


def _stale(target: str, srcs) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in srcs)


def _compile(src: str, obj: str, defines, verbose: bool) -> None:
    cmd = ["nvcc", *FLAGS, "-I" + os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines], "-c",
           os.path.join(CSRC, src), "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(obj + ".tmp", obj)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libtt_b200.so (or a variant with extra -D flags into `out`, for experiments)."""
    target = out or LIB
    tag = "" if not defines else "_" + "_".join(d.replace("=", "-") for d in defines)
    objdir = OBJ + tag
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s + ".o") for s in SOURCES]
    todo = [(s, o) for s, o in zip(SOURCES, objs)
            if force or _stale(o, [os.path.join(CSRC, s)] + _deps())]
    if not todo and out is None and not _stale(LIB, objs):
        return LIB
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for f in [ex.submit(_compile, s, o, defines, verbose) for s, o in todo]:
            f.result()
    cmd = ["nvcc", *FLAGS, "-shared", *objs, "-ldl", "-o", target + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
