"""Per-wavefront timeline of single-profile sharding (diagnostic; torchrun, N GPUs; needs a
build with OOB_NVCC_DEFS=OOB_TIMELINE):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/timeline_shard.py cfg4
Rank 0 prints its own waves (us since its wave 2 start): start / ready / units done / done;
`done - units` is the exchange wait + finalize (the partials of every rank are in)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from paper_2309_08125_b200._lib import lib  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = CONFIGS[key]
prof = config_profiles(cfg, "real")[0]
comm = planner.NcclComm(world, rank, local)
plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
plan.set_comm(comm)
info = plan.info
fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device="cuda")
bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device="cuda")
ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
f = lib.oob_dbg_timeline
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((cfg.L + 1, 8), dtype=np.uint64)
for r in range(4):
    assert f(None, cfg.L + 1) == 0, "library built without OOB_TIMELINE"
    dist.barrier()
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert f(buf.ctypes.data, cfg.L + 1) == 0
if rank == 0:
    t0 = min(int(buf[l, 0]) for l in range(2, cfg.L + 1) if buf[l, 0] != np.uint64(2**64 - 1))
    print(f"{key}: world {world}, pipelined={info.pipelined}, exchange={info.exchange}")
    print("   l   start  ready  units   done | span  xwait")
    tot_x = 0.0
    for l in range(2, cfg.L + 1):
        v = [int(x) for x in buf[l]]

        def us(x):
            return (x - t0) / 1e3 if 0 < x < 2**63 else float("nan")
        xw = (v[3] - v[2]) / 1e3 if 0 < v[2] < 2**63 and 0 < v[3] < 2**63 else 0.0
        tot_x += xw
        print(f"{l:4d} {us(v[0]):7.1f} {us(v[1]):6.1f} {us(v[2]):6.1f} {us(v[3]):6.1f} | {(v[3] - v[0]) / 1e3:6.1f} {xw:6.1f}")
    print(f"sum of (done - units): {tot_x:.1f} us")
dist.barrier()
dist.destroy_process_group()
