"""Test helpers: golden-file loading and packing oracle templates into the C ABI's packed
format (so host-side C++ steps can be tested on CPU with oracle-made template sets)."""
import json
import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(key: str, mode: str = "real"):
    path = os.path.join(GOLDEN, f"{key}_{mode}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        rec = json.load(fh)
    for p in rec["profiles"]:
        for t in p["templates"]:
            for k in ("T1", "T2", "T3", "tstar", "total"):
                t[k] = float.fromhex(t[k])
            t["stages"] = [tuple(s) for s in t["stages"]]
    return rec


def pack_templates(templates_per_profile, L: int, M: int, n_lo: int, n_hi: int):
    """Packed layout of include/oobleck_plan.h (oob_dp_run): 64-byte header
    {int32 nodes, S, kstar, status; double T1, T2, T3, tstar, iter; pad} + L x 5 int32,
    padded to a multiple of 64 bytes."""
    tpl_bytes = (64 + L * 20 + 63) // 64 * 64
    p = n_hi - n_lo + 1
    buf = bytearray(tpl_bytes * p * len(templates_per_profile))
    for pi, tpls in enumerate(templates_per_profile):
        for i, t in enumerate(tpls):
            o = (pi * p + i) * tpl_bytes
            if t is None:       # infeasible size (stage masks): S = 0, status 3, costs +inf
                inf = float("inf")
                struct.pack_into("<iiiidddddd", buf, o, n_lo + i, 0, 0, 3, inf, inf, inf, inf, inf, 0.0)
                continue
            struct.pack_into("<iiiidddddd", buf, o, t["nodes"], t["S"], t["kstar"], 0, t["T1"], t["T2"],
                             t["T3"], t["tstar"], t["total"], 0.0)
            for j, s in enumerate(t["stages"]):
                struct.pack_into("<iiiii", buf, o + 64 + 20 * j, *s)
    info = dict(L=L, M=M, n_lo=n_lo, n_hi=n_hi, num_profiles=len(templates_per_profile),
                packed_template_bytes=tpl_bytes, packed_profile_bytes=tpl_bytes * p,
                packed_bytes=tpl_bytes * p * len(templates_per_profile))
    return np.frombuffer(bytes(buf), dtype=np.uint8), info


def count_universe(L: int, M: int, n_hi: int):
    """Independent count of DP cells and feasible splits straight from the cell/split
    definitions (enumerating every cell and every (k, device split, s)); small L only."""
    def allocs(l):
        Q = n_hi if l == L else max(1, n_hi - 1)
        out = [("I", r) for r in range(1, M)] + [("W", q) for q in range(1, Q + 1)]
        return out

    def lo(a):
        return a[1] if a[0] == "W" else 1

    def hi(a, l):
        return min(l, a[1] * M if a[0] == "W" else a[1])

    def dsplits(a):
        k, n = a
        if k == "W" and n >= 2:
            return [(("W", j), ("W", n - j)) for j in range(1, n)]
        if k == "W":
            return [(("I", m), ("I", M - m)) for m in range(1, M)]
        return [(("I", m), ("I", n - m)) for m in range(1, n)]

    cells = splits = 0
    for l in range(1, L + 1):
        for u in range(0, L - l + 1):
            for a in allocs(l):
                for Sp in range(lo(a), hi(a, l) + 1):
                    cells += 1
                    if Sp < 2:
                        continue
                    for l1 in range(1, l):
                        l2 = l - l1
                        for a1, a2 in dsplits(a):
                            for s in range(1, Sp):
                                if lo(a1) <= s <= hi(a1, l1) and lo(a2) <= Sp - s <= hi(a2, l2):
                                    splits += 1
    return cells, splits
