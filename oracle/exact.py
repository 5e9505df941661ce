"""ORACLE (test infrastructure only) — ctypes loader for oracle/c/oob_exact.c: the exact
minimum of the 1F1B objective over every GPU-stage mapping of one template (parametric DP
over the bottleneck stage time; derivation in the C file's header).

Used to measure the paper heuristic's gap (scripts/heuristic_gap.py) and pinned
against oracle/brute.py (tests/test_oracle_exact.py).  The returned total is recomputed with
`dp.closed_form` from the stage times, so it is comparable bit for bit with the recursion's.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .dp import closed_form, stage_time

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "oob_exact.c")
LIB = os.path.join(HERE, "c", "liboob_exact.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fopenmp",
                               "-fPIC", "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        f = lib.oob_exact_template
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)]
        _lib = lib
    return _lib


def exact_template(fwd, bwd, M: int, n: int, ub: float = 0.0):
    """Optimal mapping of L layers onto n nodes x M GPUs: dict(stages=[(u, v, d, node)], S,
    total, T1, T2, T3, kstar, dp_value), or None if no mapping exists (n > L).  ub > 0: a known
    total (e.g. the recursion's) that restricts the bottleneck values searched (see the C file);
    the result is then the optimum provided it is <= ub, which it is when ub is attained."""
    lib = _load()
    fwd = np.ascontiguousarray(fwd, dtype=np.float64)
    bwd = np.ascontiguousarray(bwd, dtype=np.float64)
    L = fwd.shape[0]
    if n > L:
        return None
    st = np.zeros((L, 4), np.int32)
    S = ctypes.c_int32(0)
    v = ctypes.c_double(0.0)
    rc = lib.oob_exact_template(L, M, fwd.ctypes.data, bwd.ctypes.data, n, float(ub), st.ctypes.data, ctypes.byref(S),
                                ctypes.byref(v))
    if rc == 2:
        raise ValueError("bad arguments")
    if rc != 0:
        return None
    stages = [tuple(int(x) for x in st[i]) for i in range(S.value)]
    times = [float(stage_time(fwd, bwd, u, w, d)) for (u, w, d, _) in stages]
    total, T1, T2, T3, k = closed_form(times)
    return {"stages": stages, "S": S.value, "total": total, "T1": T1, "T2": T2, "T3": T3, "kstar": k,
            "dp_value": v.value}
