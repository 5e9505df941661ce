"""Per-wavefront timeline of one device-resident template set (diagnostic; needs a build with
OOB_NVCC_DEFS=OOB_TIMELINE):  python scripts/timeline.py cfg4 [reps]

For each wave l: main-CTA start, first CTA past its prologue waits, last CTA done with its
units, last CTA done (finalize), aux blocks (next wave's seeds + in-node cells) start/end,
last seed block / last in-node block done —
relative to the first wave's start, in microseconds, taken from %globaltimer inside k_wave_w.
"""
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
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[key]
profs = config_profiles(cfg, "real", count=1 if key != "cfg5" else 1024)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
info = plan.info
fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
f = lib.oob_dbg_timeline
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((cfg.L + 1, 8), dtype=np.uint64)
for r in range(reps + 1):
    assert f(None, cfg.L + 1) == 0, "library built without OOB_TIMELINE"
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert f(buf.ctypes.data, cfg.L + 1) == 0
t0 = min(int(buf[l, 0]) for l in range(2, cfg.L + 1) if buf[l, 0] != np.uint64(2**64 - 1))
print(f"{key}: waves 2..{cfg.L}, us since wave 2's first CTA; pipelined={info.pipelined}")
print("   l   start  ready  units   done | aux_s  aux_e seeds_e innode_e | span")
for l in range(2, cfg.L + 1):
    v = [int(x) for x in buf[l]]
    def us(x):
        return (x - t0) / 1e3 if 0 < x < 2**63 else float("nan")
    print(f"{l:4d} {us(v[0]):7.1f} {us(v[1]):6.1f} {us(v[2]):6.1f} {us(v[3]):6.1f} | {us(v[4]):6.1f} {us(v[5]):6.1f}"
          f" {us(v[6]):7.1f} {us(v[7]):7.1f} |"
          f" {(v[3] - v[0]) / 1e3:6.1f}")
