"""Diagnostic (build with OOB_NVCC_DEFS=OOB_DBG_FILTER): run cfg4 once and print the
filter violations recorded by k_wave_w (python scripts/dbg_filter.py)."""
import ctypes
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from paper_2309_08125_b200._lib import _lib as lib  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

cfg = CONFIGS["cfg4"]
prof = config_profiles(cfg, "real")[0]
fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device="cuda")
bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device="cuda")
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
ws = torch.zeros(plan.info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(plan.info.packed_bytes, dtype=torch.uint8, device="cuda")
buf = (ctypes.c_ulonglong * 256)()
lib.oob_dbg_filter(buf)
plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), 0)
torch.cuda.synchronize()
lib.oob_dbg_filter(buf)
print("violations:", buf[0])
d = lambda b: struct.unpack("<d", struct.pack("<Q", b))[0]
f = lambda b: struct.unpack("<f", struct.pack("<I", b & 0xFFFFFFFF))[0]
for n in range(min(7, buf[0])):
    r = buf[1 + 9 * n: 10 + 9 * n]
    print(f"tot={d(r[0])!r} acc={d(r[1])!r} key={r[2] & 0xFFFFFFFF:#x} acckey={r[2] >> 32:#x} mn={f(r[3])!r} "
          f"filt={f(r[3] >> 32)!r} t={r[4] & 0xFFFF} e={(r[4] >> 16) & 0xFFFF} Ep={r[4] >> 32} LT={r[5] & 0xFF} "
          f"TE={(r[5] >> 8) & 0xFF} rl={(r[5] >> 16) & 0xFFFF} ncell={r[5] >> 32} idx={r[6] & 0xFFFFFFFF} "
          f"S0={r[6] >> 32} rs={r[7] & 0xFFFF} nb_ok={(r[7] >> 16) & 0xFFFF} nb_iss={(r[7] >> 32) & 0xFFFF} rb={r[7] >> 48} lane={r[8]}")
fl = np.frombuffer(bytes(buf), dtype=np.float32)
for n in range(min(3, buf[0])):
    q = fl[2 * (100 + 8 * n): 2 * (100 + 8 * n) + 16]
    print("  fast tile (TA,TB,TS,TC) =", q[0:4], " ring x =", q[4:8])
    print("  global SH of the streamed cell =", q[8:12], " shadow(stream fp64) =", q[12:16])
