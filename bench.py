"""Benchmark: Oobleck pipeline-template generation on B200 (BASELINE.json metric
"template-DP cells/s and full-plan latency at 1/2/4/8 B200; % of roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

One step = one full template set (every size n0..min(N - f n0, L)) of the workload's
profile(s): base cells, all DP wavefronts, template extraction (all SURVEY §8(a) rows),
inputs already resident in HBM.  With N > 1 GPUs (torchrun, one rank per GPU, NCCL) each
rank plans its own seeded profile of the same shape (independent template DPs, "weak"
scaling) and one NCCL all-gather assembles the packed template sets.
Rank 0 prints one JSON line.  L2 is flushed (256 MiB write) before every timed step.

`--impl reference` times the oracle (oracle/c, the plain C recursion) on the host cores
on a bounded sample of the same workload (rank 0 only); see DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import CONFIGS, config_profiles  # noqa: E402

FP64_PER_SPLIT = 7          # algorithmic FP64 instructions per split
SCREEN_INSTR_PER_SPLIT = 6  # k_wave_w's binary32 screen: FFMA, FADD, FADD, FSETP, FFMA, FMNMX
SMS = 148
FP64_LANES_PER_SM = 64      # B200 FP64 (non-tensor) FMA lanes per SM per clock
METRIC = "template-DP cells/s"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._proc = None
        self._thr = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return self

        def pump():
            for line in self._proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
        self._thr = threading.Thread(target=pump, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thr:
            self._thr.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def cpu_oracle_sample(cfg, prof, n_hi_sample: int):
    """Time the C oracle on templates n0..n_hi_sample of the workload profile (a bounded
    sample: the full cfg4 set takes ~5 min single-threaded).  Returns a dict in cells/s of
    the FULL workload, projected from the oracle's measured split rate (splits are the
    per-unit cost of the recursion), plus the raw sample numbers."""
    from oracle import coracle
    t0 = time.perf_counter()
    _, (cells, splits) = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, n_hi_sample)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "cells": cells, "splits": splits, "splits_per_s": splits / dt}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2309_08125_b200.planner import dp_info  # geometry counts only (no GPU work)
    info = dp_info(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
    prof = config_profiles(cfg, "real")[0]
    n_s = min(cfg.n_max, cfg.n0 + args.ref_sample_sizes - 1)
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, prof, n_s)
    rates, secs = [], []
    last = None
    for _ in range(args.steps):
        last = cpu_oracle_sample(cfg, prof, n_s)
        rates.append(last["splits_per_s"])
        secs.append(last["seconds"])
    sps = statistics.median(rates)
    full_s = info.splits_per_profile / sps
    value = info.cells_per_profile / full_s
    sample = (f"C oracle (oracle/c, 1 thread) on {cfg.key} templates n={cfg.n0}..{n_s} "
              f"({last['cells']} cells, {last['splits']} splits, {statistics.median(secs):.2f} s/step); "
              f"cells/s of the full set projected from the measured split rate")
    line = {"metric": METRIC, "value": value, "unit": "cells/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.key, "label": cfg.label, "L": cfg.L, "M": cfg.M, "N": cfg.N,
                       "f": cfg.f, "n0": cfg.n0, "sizes": [cfg.n0, cfg.n_max]},
            "cpu_baseline": {"value": value, "unit": "cells/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_set_seconds_projected": full_s}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--profiles-per-rank", type=int, default=0,
                    help="profiles per rank (default: 1; cfg5: 1024/N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard-profile", action="store_true",
                    help="N > 1: all ranks plan ONE profile, wavefronts split across GPUs (strong scaling)")
    ap.add_argument("--ref-sample-sizes", type=int, default=5,
                    help="reference arm / cpu_baseline: number of template sizes in the sample")
    args = ap.parse_args()
    cfg = CONFIGS[args.workload]
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2309_08125_b200 import planner

    from paper_2309_08125_b200 import dist as odist
    if cfg.key == "cfg5":
        # the 1024-profile sweep sharded in contiguous blocks (weak scaling: --profiles-per-rank)
        from workloads import random_profile
        if args.profiles_per_rank:
            first, P = rank * args.profiles_per_rank, args.profiles_per_rank
        else:
            first, P = odist.shard(cfg.num_profiles, world, rank)
        profs = [random_profile(cfg.seed + first + i, cfg.L, cfg.M, "lognormal") for i in range(P)]
    else:
        P = args.profiles_per_rank or 1
        from workloads import gpt_profile
        seed_rank = 0 if args.shard_profile else rank
        profs = [gpt_profile(cfg, cfg.seed + 1000 * (seed_rank * P + i)) for i in range(P)]

    shard = args.shard_profile and world > 1 and cfg.key != "cfg5"
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
    comm = None
    if shard:   # single-profile wavefront sharding: NCCL all-gather of partial argmins per wavefront
        comm = planner.NcclComm(world, rank, local)
        plan.set_comm(comm)
    info = plan.info
    dev = torch.device("cuda", local)
    fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device=dev)
    bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device=dev)
    ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device=dev)
    packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), sptr)
        if world > 1 and not shard:   # one NCCL all-gather assembles every rank's packed template sets
            odist.allgather_packed(packed, info.packed_bytes)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.kernel_time(reset=True)
    plan.set_timing(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                  # L2 flush between timed steps
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    plan.set_timing(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    kern_ms, kern_launches = plan.kernel_time(reset=True)
    t = torch.tensor([total_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_ms_max = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    units = P * (1 if shard else world)       # profiles planned per step by the whole job
    cells_step = info.cells_per_profile * units
    # cfg5 default: the fixed 1024-profile sweep is split across ranks (strong scaling);
    # --shard-profile: one profile split across ranks (strong); otherwise every rank plans
    # its own profile(s) of the workload's shape (weak scaling)
    scaling = "strong" if ((cfg.key == "cfg5" and not args.profiles_per_rank) or shard) else "weak"
    splits_step = info.splits_per_profile * units
    value = cells_step / (ms_per_step / 1e3)

    # roofline of the dominant kernel (the wavefront DP kernel): FP64 pipe
    clocks = clk.summary()
    sm_max = clocks.get("sm_max_mhz") or _peaks().get("sm_max_mhz", 1965.0)
    kern_ms_per_step = kern_ms / args.steps
    # per-rank algorithmic work (sharded: ~1/world of the splits; short wavefronts are
    # replicated, so this slightly under-counts the rank's work)
    rank_splits = info.splits_per_profile * P / (world if shard else 1)
    achieved = rank_splits * FP64_PER_SPLIT / (kern_ms_per_step / 1e3) / 1e12
    peak = SMS * FP64_LANES_PER_SM * sm_max * 1e6 / 1e12
    traffic = None
    try:   # DRAM bytes per launch of the dominant kernel, from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.key}.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        traffic = None
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFP64inst/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes/launch (ncu, k_wave_w)",
                "kernel": "k_wave_w (W-cell wavefront DP)", "kernel_ms_per_step": kern_ms_per_step,
                "kernel_share_of_step": kern_ms_per_step / (total_ms / args.steps) if world == 1 else None,
                "peak_basis": f"148 SMs x 64 FP64 lanes x {sm_max:.0f} MHz (max clock)",
                "work_basis": "7 algorithmic FP64 instructions per feasible split (the method's binary64 "
                              "Eq.1-3 combine); the kernel screens splits with a binary32 round-down lower "
                              "bound (6 FMA/ALU instructions) and re-evaluates candidates in binary64",
                # the kernel's own limit: instruction issue (1 warp-instruction per scheduler per
                # clock) at the 6 instructions per split of its binary32 screen
                "issue_roofline": {"achieved_splits_per_s": rank_splits / (kern_ms_per_step / 1e3),
                                   "peak_splits_per_s": SMS * 4 * 32 * sm_max * 1e6 / SCREEN_INSTR_PER_SPLIT,
                                   "frac": rank_splits / (kern_ms_per_step / 1e3) /
                                   (SMS * 4 * 32 * sm_max * 1e6 / SCREEN_INSTR_PER_SPLIT),
                                   "basis": "148 SMs x 4 schedulers x 32 lanes x max clock / 6 instructions"},
                "frac_at_observed_clock": (achieved / (SMS * FP64_LANES_PER_SM * clocks["sm_mhz"] * 1e6 / 1e12))
                if clocks.get("sm_mhz") else None}

    # e2e: through the public C ABI with host buffers (H2D of the profiles, D2H + host
    # template-set build inside the timed region), workspace preallocated by torch.
    hprofs = [planner.Profile.from_arrays(p.fwd_ms, p.bwd_ms) for p in profs]
    e2e_ws = torch.empty(info.workspace_bytes + (4 << 20) + info.packed_bytes + 2 * 8 * cfg.L * cfg.M * P + (1 << 20),
                         dtype=torch.uint8, device=dev)

    h_fwd = torch.from_numpy(np.stack([p.fwd_ms for p in profs])).pin_memory()
    h_bwd = torch.from_numpy(np.stack([p.bwd_ms for p in profs])).pin_memory()

    def e2e_step():
        if shard:   # public DPPlan API: pinned H2D, sharded DP, D2H + host template set
            fwd.copy_(h_fwd, non_blocking=True)
            bwd.copy_(h_bwd, non_blocking=True)
            plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(), sptr)
            return plan.template_set(packed.cpu().numpy())
        ts = planner.generate_templates(hprofs, nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f, n0=cfg.n0,
                                        device=local, stream=sptr, workspace=e2e_ws.data_ptr(),
                                        workspace_bytes=e2e_ws.numel())
        return ts

    for _ in range(2):
        e2e_step()
    e2e_times = []
    for _ in range(max(3, min(args.steps, 10))):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ts = e2e_step()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s[0])
    e2e = {"value": cells_step / e2e_s, "unit": "cells/s",
           "h2d_bytes_per_step": 2 * 8 * cfg.L * cfg.M * P, "d2h_bytes_per_step": int(info.packed_bytes),
           "planning_latency_ms": e2e_s * 1e3}
    # full-plan latency: template set (e2e) + instantiation/batch distribution at N
    t0 = time.perf_counter()
    try:
        inst = planner.instantiate(ts, 0, cfg.N, cfg.f, global_batch=1024, microbatch=1, max_enumerated=10000)
        inst_ok = {"counts_nonzero": {str(cfg.n0 + i): c for i, c in enumerate(inst["counts"]) if c},
                   "num_feasible": inst["num_feasible"], "capped": inst["capped"]}
    except Exception as exc:  # report, never hide
        inst_ok = {"error": str(exc)}
    inst_ms = (time.perf_counter() - t0) * 1e3

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            n_s = min(cfg.n_max, cfg.n0 + args.ref_sample_sizes - 1)
            r = cpu_oracle_sample(cfg, profs[0], n_s)
            full_s = info.splits_per_profile / r["splits_per_s"]
            cpu = {"value": info.cells_per_profile / full_s, "unit": "cells/s", "cores": 1, "kind": "oracle",
                   "sample": (f"C oracle, 1 thread, {cfg.key} profile 0 templates n={cfg.n0}..{n_s}: "
                              f"{r['cells']} cells / {r['splits']} splits in {r['seconds']:.2f} s; "
                              f"full-set cells/s projected from the split rate"),
                   "host_cpu": _cpu_model(), "host_cores": os.cpu_count()}
        line = {"metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg.key, "label": cfg.label, "L": cfg.L, "M": cfg.M, "N": cfg.N,
                           "f": cfg.f, "n0": cfg.n0, "sizes": [cfg.n0, cfg.n_max], "profiles_per_rank": P,
                           "cells_per_step": cells_step, "splits_per_step": splits_step,
                           "l2": "flushed (256 MiB write) before every timed step",
                           "parallelism": (f"one profile, wavefronts sharded over {world} GPUs (NCCL all-gather of "
                                           f"partial argmins per wavefront)") if shard else
                                          f"independent template DPs, {P} profile(s) per rank x {world} rank(s)"
                                          + (", NCCL all-gather of packed template sets" if world > 1 and not shard
                                             else "")},
                "splits_per_s": splits_step / (ms_per_step / 1e3),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "full_plan_latency_ms": {"templates_e2e": e2e_s * 1e3, "instantiate_N_capped_1e4": inst_ms,
                                         "instantiate": inst_ok},
                "gpu_launches": int(info.kernel_launches) * args.steps,
                "clocks": clocks, "step_ms": {"min": min(step_ms), "max": max(step_ms)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


if __name__ == "__main__":
    main()
