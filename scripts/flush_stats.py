"""Flush-test pass statistics of k_wave_w for one template set (diagnostic; needs an
OOB_FLUSH_STATS=1 build):  python scripts/flush_stats.py cfg5 [profiles]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from paper_2309_08125_b200._lib import lib  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = CONFIGS[key]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
profs = config_profiles(cfg, "real", count=P)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
info = plan.info
fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
f = lib.oob_dbg_flush_stats
f.argtypes = [ctypes.c_int, ctypes.c_void_p]
out = (ctypes.c_ulonglong * 4)()
f(1, None)
plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
f(0, out)
print(f"{key}: filter passes {out[0]}, CAS successes {out[1] & 0xFFFFFFFF}, exact ties {out[2]} (same split {out[1] >> 32}), exact worse {out[3]}, "
      f"feasible splits {info.splits_per_profile * P} ({100 * out[0] / (info.splits_per_profile * P):.3f}% pass)")
