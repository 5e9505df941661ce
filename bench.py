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
    """SM clock + clock-event (throttle) reasons of this rank's GPU, sampled DURING the timed
    region: NVML polled every ~2 ms from a thread (nvidia-smi -lms as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.device = device
        self.samples = []          # (sm_mhz, reasons bitmask)
        self.sm_max = None
        self._stop = threading.Event()
        self._thr = None
        self._h = None
        self._nvml = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        self._nvml = pynvml
        try:   # the physical GPU behind torch's device index (CUDA_VISIBLE_DEVICES remaps)
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            return pynvml.nvmlDeviceGetHandleByIndex(idx)

    def __enter__(self):
        try:
            self._h = self._handle()
            nv = self._nvml
            self.sm_max = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))

            def poll():
                while not self._stop.is_set():
                    try:
                        mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                        self.samples.append((float(mhz), int(rs)))
                    except Exception:
                        pass
                    time.sleep(0.002)
        except Exception:
            self._h = None

            def poll():   # fallback: nvidia-smi every 20 ms
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")
                try:
                    proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                             "--format=csv,noheader,nounits", "-lms", "20"],
                                            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                except OSError:
                    return
                for line in proc.stdout:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 3 and parts[0].replace(".", "").isdigit():
                        self.sm_max = float(parts[1])
                        self.samples.append((float(parts[0]), int(parts[2], 16)))
                    if self._stop.is_set():
                        break
                proc.terminate()
        self._thr = threading.Thread(target=poll, daemon=True)
        self._thr.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.sm_max,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._h is not None else "nvidia-smi"}


def cpu_oracle_sample(cfg, prof, n_hi_sample: int):
    """Time the C oracle (oracle/c, one thread, as it stands) on templates n0..n_hi_sample of
    the workload profile: a bounded sample of the workload (the full cfg4 set takes minutes
    single-threaded).  Returns the raw sample numbers and the oracle's split rate."""
    from oracle import coracle
    t0 = time.perf_counter()
    _, (cells, splits) = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, n_hi_sample)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "cells": cells, "splits": splits, "splits_per_s": splits / dt}


def run_reference(args, cfg):
    """The reference arm: the oracle (the only reference this paper-only tier has) timed on
    the host cores, on rank 0 only; it loads nothing from paper_2309_08125_b200/."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.count import universe
    from workloads import config_profiles
    cells_full, splits_full = universe(cfg.L, cfg.M, cfg.n_max)
    prof = config_profiles(cfg, "real")[0]
    n_s = cfg.n_max if args.ref_full else min(cfg.n_max, cfg.n0 + args.ref_sample_sizes - 1)
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, prof, n_s)
    rates, secs = [], []
    last = None
    for _ in range(args.steps):
        last = cpu_oracle_sample(cfg, prof, n_s)
        rates.append(last["splits_per_s"])
        secs.append(last["seconds"])
    sps = statistics.median(rates)
    full = n_s == cfg.n_max
    full_s = statistics.median(secs) if full else splits_full / sps
    value = cells_full / full_s
    if full:
        sample = (f"C oracle (oracle/c, 1 thread) on the FULL {cfg.key} template set n={cfg.n0}..{cfg.n_max} "
                  f"({last['cells']} cells, {last['splits']} splits, {statistics.median(secs):.2f} s/step)")
    else:
        sample = (f"C oracle (oracle/c, 1 thread) on the bounded sample {cfg.key} templates n={cfg.n0}..{n_s} "
                  f"({last['cells']} cells, {last['splits']} splits, {statistics.median(secs):.2f} s/step); "
                  f"value = cells/s of the full set PROJECTED from the sample's split rate "
                  f"({splits_full} splits, oracle/count.py)")
    line = {"metric": METRIC, "value": value, "unit": "cells/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.key, "label": cfg.label, "L": cfg.L, "M": cfg.M, "N": cfg.N,
                       "f": cfg.f, "n0": cfg.n0, "sizes": [cfg.n0, cfg.n_max]},
            "cpu_baseline": {"value": value, "unit": "cells/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "projected": not full, "host_cpu": _cpu_model(), "host_cores": os.cpu_count()},
            "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_set_seconds" + ("" if full else "_projected"): full_s}
    print(json.dumps(line), flush=True)


def run_planning_grid(args):
    """Context runs: the 36 points of tab:planning_latency —
    ONE template of n nodes x M GPUs for L layers — on this GPU, beside the paper's seconds
    (its Python planner on unstated hardware: context, not a target).  Device-resident GPU
    time (CUDA events, median of --steps runs after --warmup) and the e2e latency through
    oob_generate_templates with host buffers; points up to 5e7 splits are checked against
    the C oracle."""
    import torch
    from paper_2309_08125_b200 import planner
    from workloads import (PLANNING_GRID_GPUS, PLANNING_GRID_LAYERS, PLANNING_GRID_NODES, PLANNING_GRID_PAPER_S,
                           gpt_profile, planning_grid_config)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    pts = []
    for nodes in PLANNING_GRID_NODES:
        for M in PLANNING_GRID_GPUS:
            for li, L in enumerate(sorted(PLANNING_GRID_LAYERS)):
                cfg = planning_grid_config(L, nodes, M)
                prof = gpt_profile(cfg)
                plan = planner.DPPlan(L, M, nodes, nodes, 1)
                info = plan.info
                fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device=dev)
                bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device=dev)
                ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device=dev)
                packed = torch.empty(info.packed_bytes, dtype=torch.uint8, device=dev)

                def run():
                    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
                             stream.cuda_stream)
                for _ in range(max(2, args.warmup)):
                    run()
                ms = []
                for _ in range(max(3, args.steps)):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    run()
                    b.record(stream)
                    torch.cuda.synchronize()
                    ms.append(a.elapsed_time(b))
                hp = planner.Profile.from_arrays(prof.fwd_ms, prof.bwd_ms)
                e2e = []
                for _ in range(4):         # first call: plan creation + geometry upload (not timed)
                    t0 = time.perf_counter()
                    ts = planner.generate_templates([hp], nodes=nodes, gpus_per_node=M, f=0, n0=nodes, device=0)
                    e2e.append((time.perf_counter() - t0) * 1e3)
                e2e_ms = statistics.median(e2e[1:])
                first_ms = e2e[0]
                checked = None
                if info.splits_per_profile <= 5e7:
                    from oracle import coracle
                    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, nodes, nodes)
                    checked = ts.templates(0) == want
                paper_s = PLANNING_GRID_PAPER_S[(nodes, M)][li]
                gpu_ms = statistics.median(ms)
                pts.append({"layers": L, "nodes": nodes, "gpus_per_node": M, "cells": info.cells_per_profile,
                            "splits": info.splits_per_profile, "gpu_ms": gpu_ms, "e2e_ms": e2e_ms,
                            "first_call_ms": first_ms,
                            "paper_s": paper_s, "paper_over_e2e": paper_s * 1e3 / e2e_ms,
                            "oracle_match": checked, "iter_ms": ts.templates(0)[0]["total"]})
    line = {"metric": "planning latency grid (tab:planning_latency, one template)", "unit": "ms",
            "workload": "planning_grid", "data": "synthetic GPT-shaped profiles (hidden 1024/2560/8192/12288)",
            "paper_context": "PAPER P:817-836, Python planner, hardware unstated (seconds)",
            "clocks_note": "context run, not the bench contract", "points": pts}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(CONFIGS) + ["planning_grid"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--profiles-per-rank", type=int, default=0,
                    help="profiles per rank (default: 1; cfg5: 1024/N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-optimum context run (1 GPU only)")
    ap.add_argument("--shard-profile", action="store_true",
                    help="N > 1: all ranks plan ONE profile, wavefronts split across GPUs (strong scaling)")
    ap.add_argument("--ref-sample-sizes", type=int, default=5,
                    help="reference arm / cpu_baseline: number of template sizes in the sample")
    ap.add_argument("--ref-full", action="store_true",
                    help="reference arm: time the oracle on the full template set (minutes for cfg4)")
    args = ap.parse_args()
    if args.workload == "planning_grid":
        run_planning_grid(args)
        return
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
    # the library's own NCCL communicator (torch.distributed only bootstraps its unique id):
    # per-wavefront partial argmins (--shard-profile) or the packed template sets (batched)
    comm = planner.NcclComm(world, rank, local) if world > 1 else None
    if shard:   # single-profile wavefront sharding: NCCL all-gather of partial argmins per wavefront
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
            odist.allgather_packed(packed, info.packed_bytes, comm=comm, stream=sptr)

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
        if world > 1:
            # device-side start line: every rank's stream leaves this all-reduce together, so
            # the first timed step does not absorb the ranks' host skew after the barrier
            dist.all_reduce(torch.zeros(1, device=dev))
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
    e2e_ws = torch.empty(info.workspace_bytes + (world + 2) * info.packed_bytes + 2 * 8 * cfg.L * cfg.M * P * world +
                         (8 << 20), dtype=torch.uint8, device=dev)

    # the e2e call: every rank passes the job's profiles (all ranks' blocks, or the one
    # sharded profile) and the library's communicator; each rank plans its share and gets
    # the whole template set
    if world > 1 and not shard:
        if cfg.key == "cfg5":
            all_profs = [random_profile(cfg.seed + i, cfg.L, cfg.M, "lognormal")
                         for i in range(P * world if args.profiles_per_rank else cfg.num_profiles)]
        else:
            from workloads import gpt_profile
            all_profs = [gpt_profile(cfg, cfg.seed + 1000 * i) for i in range(P * world)]
        e2e_profs = [planner.Profile.from_arrays(p.fwd_ms, p.bwd_ms) for p in all_profs]
    else:
        e2e_profs = hprofs

    def e2e_step():
        return planner.generate_templates(e2e_profs, nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f, n0=cfg.n0,
                                          device=local, stream=sptr, workspace=e2e_ws.data_ptr(),
                                          workspace_bytes=e2e_ws.numel(), comm=comm)

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
           "h2d_bytes_per_step": 2 * 8 * cfg.L * cfg.M * P,
           "d2h_bytes_per_step": int(info.packed_bytes) * (world if world > 1 and not shard else 1),
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
    # plans for EVERY surviving node count N' in [(f+1) n0, N] in one call (certified bounds)
    t0 = time.perf_counter()
    try:
        allp = planner.instantiate_all(ts, 0, (cfg.f + 1) * cfg.n0, cfg.N, cfg.f, global_batch=1024, microbatch=1,
                                       max_enumerated=10000)
        ok = [r for r in allp if r["status"] == 0]
        gaps = [r["upper_bound"] / r["throughput"] - 1.0 for r in ok]
        all_ok = {"node_counts": len(allp), "planned": len(ok), "exact": sum(r["exact"] for r in ok),
                  "max_certified_gap": max(gaps) if gaps else None,
                  "median_certified_gap": statistics.median(gaps) if gaps else None}
    except Exception as exc:  # report, never hide
        all_ok = {"error": str(exc)}
    inst_all_ms = (time.perf_counter() - t0) * 1e3
    # dynamic reconfiguration (PAPER §5) of the plan at N after f simultaneous node failures
    # spread over the job (reinstantiate / borrow / merge, batch redistribution, copy plan)
    t0 = time.perf_counter()
    try:
        ex = planner.ExecState(ts, 0, cfg.f, 1024, 1, counts=inst["counts"], node_ids=range(cfg.N))
        failed = {(i * cfg.N) // max(1, cfg.f) + 1 for i in range(max(1, cfg.f))}
        acts, xfers = ex.fail(failed)
        reconf = {"failed_nodes": len(failed), "actions": len(acts), "transfers": len(xfers),
                  "pipelines_after": len(ex.pipelines())}
    except Exception as exc:  # report, never hide
        reconf = {"error": str(exc)}
    reconf_ms = (time.perf_counter() - t0) * 1e3
    # context (outside the timed region): the exact optimum of the same objective on the same
    # device-resident inputs, bounded by the recursion's templates of the last timed step
    exact = None
    if world == 1 and not args.no_exact:
        try:
            exact = exact_context(planner, cfg, P, fwd, bwd, packed, info, sptr)
        except Exception as exc:  # report, never hide
            exact = {"error": str(exc)}

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
                           "parallelism": (f"one profile, wavefronts sharded over {world} GPUs (partial argmins "
                                           + ("exchanged inside k_wave_w over NVLink peer memory" if plan.info.exchange == 1
                                              else "all-gathered by NCCL per wavefront") + ")") if shard else
                                          f"independent template DPs, {P} profile(s) per rank x {world} rank(s)"
                                          + (", NCCL all-gather of packed template sets" if world > 1 and not shard
                                             else "")},
                "splits_per_s": splits_step / (ms_per_step / 1e3),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "full_plan_latency_ms": {"templates_e2e": e2e_s * 1e3, "instantiate_N_capped_1e4": inst_ms,
                                         "instantiate": inst_ok,
                                         "instantiate_every_surviving_N": inst_all_ms,
                                         "instantiate_every_surviving_N_detail": all_ok,
                                         "reconfigure_after_f_failures": reconf_ms,
                                         "reconfigure_detail": reconf,
                                         "total": e2e_s * 1e3 + inst_ms + inst_all_ms + reconf_ms},
                "exact_optimum": exact,
                "gpu_launches": int(info.kernel_launches) * args.steps,
                "clocks": clocks, "step_ms": {"min": min(step_ms), "max": max(step_ms), "median": statistics.median(step_ms),
                            "all": [round(x, 4) for x in step_ms]}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def exact_context(planner, cfg, P, fwd, bwd, packed, info, sptr):
    """oob_exact_run on the timed step's inputs, bounded by its packed templates: ms per set
    (CUDA events, after one warm-up run), tasks, and how far the recursion is from the optimum."""
    import torch
    xb = planner.exact_workspace_bytes(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
    xws = torch.empty(xb, dtype=torch.uint8, device=fwd.device)
    out = torch.empty_like(packed)

    def run():
        planner.exact_run(cfg.L, cfg.M, cfg.n0, cfg.n_max, P, fwd.data_ptr(), bwd.data_ptr(), packed.data_ptr(),
                          xws.data_ptr(), xb, out.data_ptr(), sptr)
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    tb = int(info.packed_template_bytes)
    n = P * (cfg.n_max - cfg.n0 + 1)
    hh = packed.cpu().numpy()[: n * tb].reshape(n, tb)
    xx = out.cpu().numpy()[: n * tb].reshape(n, tb)
    h_iter = hh[:, 48:56].copy().view(np.float64)[:, 0]
    x_iter = xx[:, 48:56].copy().view(np.float64)[:, 0]
    x_stat = xx[:, 12:16].copy().view(np.int32)[:, 0]
    gap = h_iter / x_iter - 1.0
    better = gap > 1e-12
    return {"ms_per_set": a.elapsed_time(b), "tasks": int(xws[:8].cpu().numpy().view(np.uint64)[0]),
            "templates": n, "status_ok": int((x_stat == 0).sum()), "recursion_above_optimum": int(better.sum()),
            "max_gap": float(gap.max()), "mean_gap_where_above": float(gap[better].mean()) if better.any() else 0.0,
            "workspace_bytes": xb, "kernel": "oob_exact_run (k_ex_*), see DESIGN.md section 12"}


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
