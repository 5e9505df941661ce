"""Time the exact-optimum solver (oob_exact_run) on device-resident inputs after the
recursion (oob_dp_run) whose templates bound it (diagnostic):
    python scripts/exact_time.py cfg4 [reps] [profiles]
Prints the recursion's and the exact solver's ms per set, the (profile, tau) tasks solved,
and how many sizes the exact optimum improves (and by how much)."""
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[key]
nprof = int(sys.argv[3]) if len(sys.argv) > 3 else (64 if key == "cfg5" else 1)
profs = config_profiles(cfg, "real", count=nprof)
P = len(profs)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
info = plan.info
fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
heur = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
out = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
xb = planner.exact_workspace_bytes(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
xws = torch.empty(xb, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def dp():
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), heur.data_ptr(), s)


def ex():
    planner.exact_run(cfg.L, cfg.M, cfg.n0, cfg.n_max, P, fwd.data_ptr(), bwd.data_ptr(), heur.data_ptr(),
                      xws.data_ptr(), xb, out.data_ptr(), s)


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dp()
ex()
t_dp = timed(dp)
t_ex = timed(ex)
tasks = int(xws[:8].cpu().numpy().view(np.uint64)[0])
H, X = heur.cpu().numpy().tobytes(), out.cpu().numpy().tobytes()
nsz = cfg.n_max - cfg.n0 + 1
better, gaps = 0, []
for i in range(P * nsz):
    o = i * info.packed_template_bytes
    h = struct.unpack_from("<iiiidddddd", H, o)
    x = struct.unpack_from("<iiiidddddd", X, o)
    assert x[3] == 0, ("status", i, x)
    if x[8] < h[8] * (1 - 1e-12):
        better += 1
        gaps.append(h[8] / x[8] - 1)
print(f"{key}: {P} profiles x {nsz} sizes, workspace {xb / 2**20:.1f} MiB: recursion {t_dp:.3f} ms, "
      f"exact {t_ex:.3f} ms ({tasks} tasks); exact better on {better} of {P * nsz} templates"
      + (f", recursion above the optimum by max {100 * max(gaps):.3f}% / mean {100 * np.mean(gaps):.3f}%"
         if gaps else ""))
