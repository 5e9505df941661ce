"""Diagnostic: run the reference thread-per-cell kernel (v1) and the W kernel on the same
profile and report the first cells whose ARG / values differ, with the exact totals and the
filter's binary32 lower bounds of both splits (python scripts/dbg_table.py cfg4 [mode])."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from paper_2309_08125_b200._lib import _lib as lib  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
mode = sys.argv[2] if len(sys.argv) > 2 else "real"
cfg = CONFIGS[key]
M = cfg.M
prof = config_profiles(cfg, mode)[0]
fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device="cuda")
bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device="cuda")


def run(kernel):
    if kernel:
        os.environ["OOB_DP_KERNEL"] = kernel
    else:
        os.environ.pop("OOB_DP_KERNEL", None)
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
    info = plan.info
    ws = torch.zeros(info.workspace_bytes, dtype=torch.uint8, device="cuda")
    packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    o = (ctypes.c_ulonglong * 7)()
    lib.oob_dbg_offsets.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.oob_dbg_offsets(plan._h, o)
    C = info.cells_per_profile
    A = int(o[6])
    wsn = ws.cpu().numpy()
    cell = wsn[o[0]:o[0] + 32 * C].view(np.float64).reshape(C, 4)
    sh = wsn[o[1]:o[1] + 16 * C].view(np.float32).reshape(C, 4)
    arg = wsn[o[2]:o[2] + 4 * C].view(np.uint32)
    base = wsn[o[3]:o[3] + 8 * (cfg.L + 2)].view(np.int64)
    cells = wsn[o[4]:o[4] + 4 * (cfg.L + 1)].view(np.int32)
    off = wsn[o[5]:o[5] + 4 * (cfg.L + 1) * A].view(np.int32).reshape(cfg.L + 1, A)
    return cell, sh, arg, base, cells, off, A


c1, s1, a1, base, cells, off, A = run("v1")
c2, s2, a2, _, _, _, _ = run(None)
bad = np.nonzero((a1 != a2) | np.any(c1.view(np.uint64) != c2.view(np.uint64), axis=1))[0]
print(f"{key} {mode}: {len(bad)} of {len(a1)} cells differ; shadows differ at {np.sum(np.any(s1.view(np.uint32) != s2.view(np.uint32), axis=1))}")


def lo(a):
    return a - (M - 1) + 1 if a >= M - 1 else 1


def cidx(Sp, u, l, a):
    return int(base[l] + u * cells[l] + off[l, a] + (Sp - lo(a)))


def locate(i):
    l = int(np.searchsorted(base, i, side="right")) - 1
    u, r = divmod(int(i - base[l]), int(cells[l]))
    a = max(aa for aa in range(A) if 0 <= off[l, aa] <= r)
    return l, u, a, lo(a) + r - off[l, a]


def rd32(x):
    f = np.float32(x)
    if float(f) > x:
        f = np.nextafter(f, np.float32(-np.inf))
    return f


def fadd_rd(a, b):
    return rd32(float(np.float64(a) + np.float64(b)))  # exact in fp64 for fp32 inputs, then round down


def ffma_rd(a, b, c):
    from fractions import Fraction as F
    x = F(float(a)) * F(float(b)) + F(float(c))
    d = float(x)
    if F(d) > x:
        d = np.nextafter(d, -np.inf)
    return rd32(d)


for i in bad[:6]:
    l, u, a, Sp = locate(i)
    q = a - (M - 1) + 1
    print(f"cell {i}: l={l} u={u} W({q}) S'={Sp}  value {c1[i]}")
    for name, arg in (("v1", a1[i]), ("w", a2[i])):
        l1 = int(arg & 1023) + 1
        j = int((arg >> 10) & 1023) + 1
        s = int(arg >> 20)
        aX, aY = (M - 1) + j - 1, (M - 1) + (q - j) - 1
        X, Y = c1[cidx(s, u, l1, aX)], c1[cidx(Sp - s, u + l1, l - l1, aY)]
        sX, sY = s1[cidx(s, u, l1, aX)], s1[cidx(Sp - s, u + l1, l - l1, aY)]
        left = X[2] >= Y[2]
        c = (X[3] + 3.0 * (Sp - s)) if left else (Y[3] + 4.0 * s)
        ts = X[2] if left else Y[2]
        T3 = (X[1] + Y[0]) if left else Y[1]
        tot = ((X[0] + Y[0]) + c * ts) + T3
        tl = fadd_rd(ffma_rd(np.float32(3 * (Sp - s)), sX[2], sX[0]), sY[3])
        tr = ffma_rd(np.float32(4 * s), sY[2], fadd_rd(sY[0], sX[1]))
        lb = tl if sX[2] >= sY[2] else tr
        print(f"   {name}: l1={l1} j={j} s={s} total={tot!r} lb={float(lb)!r} lb/total-1={float(lb)/tot-1:.3g} "
              f"shadowX={sX} X={X} shadowY={sY} Y={Y}")
