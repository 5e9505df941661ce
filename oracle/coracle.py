"""ORACLE (test infrastructure only) — ctypes loader for oracle/c/oob_oracle.c.

`build()` compiles it with gcc -O2 -ffp-contract=off (no FMA, no fast-math).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "oob_oracle.c")
LIB = os.path.join(HERE, "c", "liboob_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", LIB, SRC])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        f = lib.oob_oracle_template_set
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong),
                      ctypes.POINTER(ctypes.c_longlong)]
        g = lib.oob_oracle_template_set_masked
        g.restype = ctypes.c_int
        g.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                      ctypes.c_int, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong),
                      ctypes.POINTER(ctypes.c_longlong)]
        _lib = lib
    return _lib


def template_set(fwd, bwd, M: int, n_lo: int, n_hi: int, pow2_tp: bool = False, stage_bytes=None,
                 mem_cap=None):
    """Templates for sizes n_lo..n_hi; same dict format as oracle.dp.TemplateDP.template
    (None for a size without a feasible mapping: stage masks, reading R31).  Also returns
    (cells, splits) the oracle evaluated."""
    lib = _load()
    fwd = np.ascontiguousarray(fwd, dtype=np.float64)
    bwd = np.ascontiguousarray(bwd, dtype=np.float64)
    L = fwd.shape[0]
    p = n_hi - n_lo + 1
    S = np.zeros(p, np.int32)
    ks = np.zeros(p, np.int32)
    costs = np.zeros((p, 6), np.float64)
    stages = np.zeros((p, L, 5), np.int32)
    cells = ctypes.c_longlong(0)
    splits = ctypes.c_longlong(0)
    sb = None if stage_bytes is None else np.ascontiguousarray(stage_bytes, dtype=np.float64)
    rc = lib.oob_oracle_template_set_masked(L, M, fwd.ctypes.data, bwd.ctypes.data, n_lo, n_hi,
                                            1 if pow2_tp else 0, None if sb is None else sb.ctypes.data,
                                            float(mem_cap) if mem_cap is not None else 0.0,
                                            S.ctypes.data, ks.ctypes.data, costs.ctypes.data,
                                            stages.ctypes.data, ctypes.byref(cells), ctypes.byref(splits))
    if rc == 2:
        raise ValueError("bad arguments")
    out = []
    for i in range(p):
        if S[i] == 0:
            out.append(None)
            continue
        st = [tuple(int(x) for x in stages[i, j]) for j in range(S[i])]
        out.append({"nodes": n_lo + i, "S": int(S[i]), "stages": st,
                    "T1": float(costs[i, 0]), "T2": float(costs[i, 1]), "T3": float(costs[i, 2]),
                    "kstar": int(ks[i]), "tstar": float(costs[i, 3]), "total": float(costs[i, 4])})
    return out, (cells.value, splits.value)
