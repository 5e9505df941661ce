"""Run one device-resident template-set DP (for profiling): python scripts/dp_once.py cfg4 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nprof = int(sys.argv[3]) if len(sys.argv) > 3 else (64 if key == "cfg5" else 1)
cfg = CONFIGS[key]
profs = config_profiles(cfg, "real", count=nprof)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
info = plan.info
fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", key, reps, info.kernel_launches)
