"""Measure a GPT-shaped layer profile on this B200 (paper_2309_08125_b200/profiler.py) and plan
templates from it:  python scripts/profile_b200.py [out.json] [--hidden 12288 --heads 96
--layers 96 --seq 2048 --mb 1 --M 8 --nodes 512 --f 4 --n0 3]

Under torchrun (WORLD_SIZE = W >= 2) the tensor-parallel all-reduces are measured with NCCL
over groups of d <= W GPUs; larger d use the ring model fitted to the measured bus bandwidth.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2309_08125_b200 import profiler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out", nargs="?", default="gpurun_out/profile_b200.json")
ap.add_argument("--hidden", type=int, default=12288)
ap.add_argument("--heads", type=int, default=96)
ap.add_argument("--layers", type=int, default=96)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--mb", type=int, default=1)
ap.add_argument("--M", type=int, default=8)
ap.add_argument("--nodes", type=int, default=512)
ap.add_argument("--f", type=int, default=4)
ap.add_argument("--n0", type=int, default=3)
ap.add_argument("--busbw", type=float, default=0.0, help="GB/s for the ring model (0: measure / fit)")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
measured = {}
nbytes = a.mb * a.seq * a.hidden * 2
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
    for d in range(2, min(world, a.M) + 1):
        g = dist.new_group(list(range(d)))
        if rank < d:
            measured[d] = profiler.measure_allreduce(nbytes, g)
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        sys.exit(0)
busbw = a.busbw
if measured and not busbw:    # fit: busbw = 2 (d-1)/d bytes / t for the largest measured d
    d = max(measured)
    busbw = 2 * (d - 1) / d * nbytes / (measured[d] * 1e-3) / 1e9
if not busbw:
    busbw = 600.0             # no measurement: a stated assumption, recorded in the JSON

def ar(nb, d):
    return measured[d] if d in measured else profiler.allreduce_model_ms(nb, d, busbw)

t0 = time.time()
doc = profiler.profile_gpt(a.hidden, a.heads, a.layers, a.seq, a.mb, a.M, allreduce_ms=ar)
doc["allreduce"] = {"bytes": nbytes, "measured_ms": measured, "busbw_gbps_model": busbw}
doc["profiling_s"] = time.time() - t0
os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
profiler.write_profile(doc, a.out)
from paper_2309_08125_b200 import planner  # noqa: E402
prof = planner.load_profile(a.out)
t0 = time.perf_counter()
ts = planner.generate_templates([prof], nodes=a.nodes, gpus_per_node=a.M, f=a.f, n0=a.n0, device=0)
ms = (time.perf_counter() - t0) * 1e3
tpl = ts.templates(0)
print(json.dumps({"profile": a.out, "fwd_ms_block": doc["layers"][1]["fwd_ms"], "bwd_ms_block": doc["layers"][1]["bwd_ms"],
                  "allreduce": doc["allreduce"], "templates": len(tpl), "plan_ms_first_call": ms,
                  "smallest": {k: tpl[0][k] for k in ("nodes", "S", "total", "tstar")},
                  "largest": {k: tpl[-1][k] for k in ("nodes", "S", "total", "tstar")}}))
