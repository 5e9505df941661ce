"""Single-profile wavefront sharding check (torchrun, N GPUs): every rank plans the same cfg4
profile with the work split across ranks; the packed output must equal the stored oracle set
(tests/golden/cfg4_real.json) on every rank; prints the per-step time (max over ranks).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/shard_check.py [cfg4] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2309_08125_b200 import planner  # noqa: E402
from tests.helpers import load_golden  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
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
packed = torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), s)
torch.cuda.synchronize()
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), s)
b.record()
torch.cuda.synchronize()
ms = torch.tensor([a.elapsed_time(b) / steps], device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
ts = plan.template_set(packed.cpu().numpy())
got = ts.templates(0)
rec = load_golden(key, "real")
ok = rec is not None and got == rec["profiles"][0]["templates"]
oks = [None] * world
dist.all_gather_object(oks, ok)
if rank == 0:
    print(json.dumps({"workload": key, "world": world, "ms_per_template_set": float(ms), "identical_to_oracle": oks,
                      "pipelined": info.pipelined, "exchange": info.exchange, "fused": info.fused}))
dist.barrier()
dist.destroy_process_group()
