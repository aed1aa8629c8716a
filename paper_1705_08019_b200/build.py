"""Build the in-tree C-ABI library libparaexp.so for sm_100a (nvcc cross-compiles without
a GPU).  Usage: python paper_1705_08019_b200/build.py [--force] [--verbose] [--debug]

--debug builds libparaexp_debug.so instead: the same sources with -DPARAEXP_DEBUG_CHECKS
(device-side bounds checks on the fused kernels' global stores and shared-memory indices, and
a trap on an mbarrier wait that never completes; compute-sanitizer is closed on this GPU
pool).  Load it with PARAEXP_LIBRARY_VARIANT=debug."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libparaexp.so")
OBJ_DEBUG = os.path.join(HERE, "build_debug")
LIB_DEBUG = os.path.join(HERE, "libparaexp_debug.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
                  "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("PARAEXP_PTXAS_V") else "-O3",
                  "-I" + os.path.join(HERE, "..", "include")]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-I/usr/local/cuda/include",
            "-I" + os.path.join(HERE, "..", "include")]
SOURCES = ["kernels.cu", "fused.cu", "small.cu", "mid.cu", "grid.cpp", "plan.cpp", "api.cpp"]
HEADERS = ["internal.h", "kernels_common.cuh", "../../include/paraexp.h"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    obj_dir, lib = (OBJ_DEBUG, LIB_DEBUG) if debug else (OBJ, LIB)
    extra = ["-DPARAEXP_DEBUG_CHECKS"] if debug else []
    os.makedirs(obj_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(obj_dir, src + ".o")
        objs.append(obj)
        if not force and not _newer(obj, [path] + hdrs):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC] + CUFLAGS + extra + ["-c", path, "-o", obj]
        else:
            cmd = ["g++"] + CXXFLAGS + extra + ["-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    if force or _newer(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv)
