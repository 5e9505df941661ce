"""Time the device-resident DP (oob_dp_run) for a config (diagnostic):
    python scripts/dp_time.py cfg4 [reps] [profiles]   (3 untimed sets first; cfg5 default 64 profiles)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[key]
nprof = int(sys.argv[3]) if len(sys.argv) > 3 else (64 if key == "cfg5" else 1)
profs = config_profiles(cfg, "real", count=nprof)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
info = plan.info
fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), s)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), s)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"{key}: {ms:.3f} ms per template set, {info.splits_per_profile * len(profs) * 7 / (ms * 1e-3) / 18.61248e12:.3f} of FP64 roofline")
