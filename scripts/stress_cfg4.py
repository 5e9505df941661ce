"""Stress check: the cfg4 template set N times (device-resident plan, same workspace) vs the
golden oracle output each time (python scripts/stress_cfg4.py [N] [mode])."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from tests.helpers import load_golden  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
mode = sys.argv[2] if len(sys.argv) > 2 else "real"
cfg = CONFIGS["cfg4"]
prof = config_profiles(cfg, mode)[0]
want = load_golden("cfg4", mode)["profiles"][0]["templates"]
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
info = plan.info
fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device="cuda")
bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
bad = 0
for i in range(n):
    packed = torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda")
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = plan.template_set(packed.cpu().numpy()).templates(0)
    ok = all((g["S"], g["kstar"], g["stages"], g["total"]) == (w["S"], w["kstar"], w["stages"], w["total"])
             for g, w in zip(got, want)) and len(got) == len(want)
    bad += not ok
print(f"cfg4 {mode}: {n} runs, {bad} mismatching")
