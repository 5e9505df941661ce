"""Builds paper_2309_08125_b200/liboobleck_plan.so in-tree (sm_100a, no GPU needed).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false for the CUDA DP engine;
g++ -ffp-contract=off for the host planner; cudart linked statically.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "liboobleck_plan.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")


def _nccl_dir() -> str:
    """NCCL shipped with the torch wheel (site-packages/nvidia/nccl): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (site-packages/nvidia/nccl)")


NCCL = _nccl_dir()

CU_SOURCES = ["oob_dp.cu", "oob_exact.cu"]
CPP_SOURCES = ["oob_host.cpp", "oob_geometry.cpp", "oob_instantiate.cpp", "oob_dist.cpp", "oob_reconfig.cpp"]
HEADERS = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".h", ".cuh"))] + \
    [os.path.join(INC, "oobleck_plan.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", INC, "-I", CSRC]
if os.environ.get("OOB_FLUSH_STATS"):          # diagnostic build (scripts/flush_stats.py)
    NVCC_FLAGS += ["-DOOB_FLUSH_STATS"]
for _d in os.environ.get("OOB_NVCC_DEFS", "").split():   # diagnostic builds: OOB_NVCC_DEFS="X=1 Y"
    NVCC_FLAGS += ["-D" + _d]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
             "-I", INC, "-I", CSRC, "-I", os.path.join(CUDA, "include"), "-I", os.path.join(NCCL, "include")]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + HEADERS)


def _run(cmd, log):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if log is not None:
        log.append(r.stdout)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("build failed: " + " ".join(cmd))


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    log: list[str] = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, s):
            _run([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o], log)
        objs.append(o)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, s):
            _run(["g++"] + CXX_FLAGS + ["-c", s, "-o", o], log)
        objs.append(o)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        nlib = os.path.join(NCCL, "lib")
        _run([NVCC, "-shared", "-o", LIB] + objs + ["-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                                                     "-L", nlib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nlib, "-lpthread"], log)
    if verbose:
        print("\n".join(x for x in log if x.strip()))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
