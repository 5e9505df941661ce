"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (north star): stage boundaries, GPU counts, nodes, S and k* bit-exact; costs equal
under the shared operation order — asserted bit-exact here (stricter than the north
star's rel 1e-12, which `_close` would allow), on seeded synthetic inputs.
"""
import random

import numpy as np
import pytest

from oracle import coracle
from tests.helpers import load_golden
from workloads import CONFIGS, config_profiles, random_profile

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2309_08125_b200 import planner as p
    return p


def _gpu_set(planner, profs, cfg_like):
    L, M, N, f, n0 = cfg_like
    return planner.generate_templates([(p.fwd_ms, p.bwd_ms) for p in profs], nodes=N,
                                      gpus_per_node=M, f=f, n0=n0, device=0)


def _assert_same(got, want, ctx=""):
    assert len(got) == len(want), ctx
    for g, w in zip(got, want):
        assert g["nodes"] == w["nodes"], ctx
        assert (g["S"], g["kstar"], g["stages"]) == (w["S"], w["kstar"], w["stages"]), (ctx, g["nodes"])
        for k in ("T1", "T2", "T3", "tstar", "total"):
            assert g[k] == w[k], (ctx, g["nodes"], k, g[k], w[k])


@pytest.mark.parametrize("key", ["cfg1", "cfg2", "cfg3"])
@pytest.mark.parametrize("mode", ["real", "dyadic"])
def test_configs_vs_oracle(planner, key, mode):
    cfg = CONFIGS[key]
    prof = config_profiles(cfg, mode)[0]
    ts = _gpu_set(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
    _assert_same(ts.templates(0), want, key)


def test_random_small_vs_oracle(planner):
    """Many shapes (several tiles, ragged tails, ties): L 1..40, M 1..8, every kind."""
    rng = random.Random(2024)
    for i in range(150):
        L = rng.choice([1, 2, 3, 5, 7, 9, 12, 16, 20, 24, 31, 40])
        M = rng.choice([1, 2, 3, 4, 5, 8])
        kind = rng.choice(["integer", "uniform", "lognormal", "spiky", "constant"])
        mode = rng.choice(["real", "dyadic"])
        prof = random_profile(7000 + i, L, M, kind, mode)
        n0 = rng.randint(1, max(1, min(L, 3)))
        f = rng.randint(0, 3)
        N = (f + 1) * n0 + rng.randint(0, 2 * L)
        n_hi = min(N - f * n0, L)
        ts = _gpu_set(planner, [prof], (L, M, N, f, n0))
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, n0, n_hi)
        _assert_same(ts.templates(0), want, f"case {i} L={L} M={M} {kind}")


@pytest.mark.parametrize("warpmax", ["default", "0", "100000"])
def test_batched_warp_mode_vs_oracle(planner, warpmax, monkeypatch):
    """Batched sweeps run their short waves one warp per (profile, range) and their in-node
    cells one warp per (profile, range) (OOB_DP_WARPMAX: 0 = never, large = every wave
    that fits); every setting gives the oracle's sets.  160 profiles: enough ranges for the
    warp modes; 6 of them are checked."""
    cfg = CONFIGS["cfg5"]
    P = 160
    base = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P).info
    if warpmax != "default":
        monkeypatch.setenv("OOB_DP_WARPMAX", warpmax)
    info = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P).info
    assert base.warp_waves > 0 and base.small_range > 0
    if warpmax == "0":
        assert info.warp_waves == 0
    if warpmax == "100000":
        assert info.warp_waves >= base.warp_waves
    profs = config_profiles(cfg, "real", count=P)
    ts = _gpu_set(planner, profs, (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    for i in (0, 1, 57, 101, 158, 159):
        p = profs[i]
        want, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        _assert_same(ts.templates(i), want, f"cfg5 profile {i} WARPMAX={warpmax}")


def test_batched_profiles_vs_oracle(planner):
    """Batched sweep (cfg5 shape): several profiles in one call, each vs the oracle."""
    cfg = CONFIGS["cfg5"]
    rec = load_golden("cfg5", "real")
    profs = config_profiles(cfg, "real", count=4 if rec else 2)
    ts = _gpu_set(planner, profs, (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    for i, p in enumerate(profs):
        want = rec["profiles"][i]["templates"] if rec else \
            coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)[0]
        _assert_same(ts.templates(i), want, f"cfg5 profile {i}")


CFG4_VARIANTS = {"default": ({}, {"pipelined": 1, "fused": 1}),
                 "fuse0": ({"OOB_DP_FUSE": "0"}, {"pipelined": 0, "fused": 0}),
                 "pipe0": ({"OOB_DP_PIPE": "0"}, {"pipelined": 0, "fused": 1})}


@pytest.mark.parametrize("variant", sorted(CFG4_VARIANTS))
@pytest.mark.parametrize("mode", ["real", "dyadic"])
def test_cfg4_full_vs_golden(planner, mode, variant, monkeypatch):
    """Full template set of the north-star config (96 layers, 512 x 8 GPUs, f=4, n0=3)
    vs the C oracle's output stored by scripts/make_golden.py: pipelined wavefronts with the
    finalize fused into k_wave_w (default), separate k_fin launches (fuse0), and fused
    without the wavefront pipeline (pipe0).  The plan's reported switches prove the variant
    ran (every OOB_DP_* variable is part of the plan-cache key)."""
    env, want_sw = CFG4_VARIANTS[variant]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rec = load_golden("cfg4", mode)
    if rec is None:
        pytest.skip(f"tests/golden/cfg4_{mode}.json not generated")
    cfg = CONFIGS["cfg4"]
    info = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1).info
    for k, v in want_sw.items():
        assert getattr(info, k) == v, (variant, k)
    prof = config_profiles(cfg, mode)[0]
    ts = _gpu_set(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    _assert_same(ts.templates(0), rec["profiles"][0]["templates"], "cfg4")


def test_pipeline_timeout_is_an_error(planner, monkeypatch):
    """A pipelined wait that times out (OOB_DP_PIPE_SPIN=0: give up after one poll) must
    surface as OOB_E_CUDA, never as a template set built from an incomplete table."""
    from paper_2309_08125_b200._lib import OOB_E_CUDA, OobError
    monkeypatch.setenv("OOB_DP_PIPE_SPIN", "0")
    cfg = CONFIGS["cfg4"]
    assert planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1).info.pipelined == 1
    prof = config_profiles(cfg, "real")[0]
    with pytest.raises(OobError) as e:
        _gpu_set(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    assert e.value.status == OOB_E_CUDA and "timed out" in str(e.value)


def test_long_rows_queue_fields(planner, monkeypatch):
    """L = 150, 20-node templates: streamed W rows of up to 131 cells and wide accumulators
    (the candidate-queue entry fields must not overflow).  The tiled W kernel must
    equal the thread-per-cell kernel (k_wave_v1) on every template, and the oracle on the
    smallest ones."""
    L, M, N, f, n0 = 150, 8, 21, 1, 1
    prof = random_profile(150150, L, M, "lognormal")
    assert planner.DPPlan(L, M, n0, 20, 1).info.kernel == 2
    got = _gpu_set(planner, [prof], (L, M, N, f, n0)).templates(0)
    monkeypatch.setenv("OOB_DP_KERNEL", "v1")
    assert planner.DPPlan(L, M, n0, 20, 1).info.kernel == 1
    ref = _gpu_set(planner, [prof], (L, M, N, f, n0)).templates(0)
    _assert_same(got, ref, "L=150 W kernel vs v1")
    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, n0, 2)
    _assert_same(got[:2], want, "L=150 small templates vs oracle")


def test_cfg4_sampled_templates_vs_oracle(planner):
    """Full-size config, fresh seed: the oracle recomputes the smallest templates one by one
    (cheap: they touch few cells) and they must match the GPU's full-set run."""
    cfg = CONFIGS["cfg4"]
    prof = config_profiles(cfg, "real", count=2)[1]
    ts = _gpu_set(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    got = ts.templates(0)
    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n0 + 5)
    _assert_same(got[:6], want, "cfg4 seed 2 small templates")


def test_device_resident_path_matches(planner):
    """oob_dp_run on device-resident inputs == oob_generate_templates; deterministic."""
    import torch
    cfg = CONFIGS["cfg3"]
    profs = config_profiles(cfg, "real", count=3)
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
    info = plan.info
    fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        packed = torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda")
        plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs.append(packed.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    ts = plan.template_set(outs[0])
    ref = _gpu_set(planner, profs, (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    for i in range(len(profs)):
        assert ts.templates(i) == ref.templates(i)


def test_edge_cases(planner):
    # single layer, single template; N exactly (f+1) n0; M = 1 with many nodes
    for (L, M, N, f, n0) in [(1, 1, 1, 0, 1), (1, 8, 2, 1, 1), (6, 1, 6, 1, 3), (10, 1, 30, 0, 1),
                             (4, 8, 5, 0, 1)]:
        prof = random_profile(31 + L + M, L, M, "uniform")
        ts = _gpu_set(planner, [prof], (L, M, N, f, n0))
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, n0, min(N - f * n0, L))
        _assert_same(ts.templates(0), want, f"edge L={L} M={M} N={N}")
    from paper_2309_08125_b200._lib import OOB_E_INFEASIBLE, OobError
    prof = random_profile(3, 4, 2, "uniform")
    with pytest.raises(OobError) as e:
        _gpu_set(planner, [prof], (4, 2, 3, 1, 2))
    assert e.value.status == OOB_E_INFEASIBLE


VARIANTS = [
    ({"OOB_DP_KERNEL": "v1"}, {"kernel": 1}),                  # thread-per-cell reference kernel
    ({"OOB_DP_FUSE": "0"}, {"fused": 0, "pipelined": 0}),      # separate k_fin launches
    ({"OOB_DP_FUSE": "1"}, {"fused": 1}),                      # finalize + next wave's in-node cells inside k_wave_w
    ({"OOB_DP_SEEDSPO": "1000"}, {}),                          # only waves with >= 1000 splits per output seeded
    ({"OOB_DP_SEEDINIT": "0"}, {"seeded": 0}),                 # no seeds
    ({"OOB_DP_SMALLPAIRS": "4"}, {"small_pairs": 4}),          # fewer threads per in-node cell
    ({"OOB_DP_PIPE": "0"}, {"pipelined": 0, "fused": 1}),      # plain kernel boundaries between wavefronts
    ({"OOB_DP_PIPE": "0", "OOB_DP_SEEDINIT": "0"}, {"pipelined": 0, "seeded": 0}),
    ({"OOB_DP_CHMAX": "24"}, {"chunk_max": 24}),               # short units: many per range, long queues
    ({"OOB_DP_REFRESH": "0"}, {"refresh": 0}),                 # no per-unit filter refresh
    ({"OOB_DP_SMALLRANGE": "0"}, {"small_range": 0}),          # in-node cells thread(s) per cell
    ({"OOB_DP_FINWAIT": "0"}, {}),                             # merged CTAs exit; last one finalizes alone
    ({"OOB_DP_FINWAIT": "1"}, {}),                             # every merged CTA waits and shares the finalize
    ({"OOB_DP_FINHELP": "64"}, {}),                            # many finalize helpers (default: nout / 512)
]


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: ",".join(f"{k}={x}" for k, x in v[0].items()))
@pytest.mark.parametrize("key", ["cfg2", "cfg3"])
def test_kernel_variants_match(planner, key, variant, monkeypatch):
    """Alternative kernels and finalize / seeding / pipeline modes (plan-time switches) all
    give the oracle's template sets.  The plan's reported switches prove each variant ran."""
    env, want_sw = variant
    cfg = CONFIGS[key]
    base = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1).info
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    info = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1).info
    for k, v in want_sw.items():
        assert getattr(info, k) == v, (env, k, getattr(info, k))
    if "OOB_DP_SEEDSPO" in env:
        assert info.seeded < base.seeded
    for mode in ("real", "dyadic"):
        prof = config_profiles(cfg, mode)[0]
        ts = _gpu_set(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        _assert_same(ts.templates(0), want, f"{key} {mode} {env}")


def test_cfg5_full_sweep_sampled(planner):
    """The full batched sweep at BASELINE size (1024 profiles of 48 layers, one DP launch
    sequence, as bench.py --workload cfg5 times it); profiles 0..3 vs the oracle's stored
    sets, and a fresh oracle recomputation of two more sampled profiles' small templates."""
    import torch
    cfg = CONFIGS["cfg5"]
    rec = load_golden("cfg5", "real")
    if rec is None:
        pytest.skip("tests/golden/cfg5_real.json not generated")
    profs = config_profiles(cfg, "real")                     # all 1024
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
    info = plan.info
    fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
    packed = torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda")
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ts = plan.template_set(packed.cpu().numpy())
    for i in range(4):
        _assert_same(ts.templates(i), rec["profiles"][i]["templates"], f"cfg5 profile {i}")
    for i in (517, 1023):
        p = profs[i]
        want, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n0 + 3)
        _assert_same(ts.templates(i)[:4], want, f"cfg5 profile {i} sizes 1..4")


def _virtual_run(planner, cfg, profs, world):
    """oob_dp_run_virtual with `world` virtual ranks: every rank's packed output."""
    import torch
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, len(profs))
    plan.set_virtual_shards(world)
    info = plan.info
    assert info.world == world and info.pipelined == 0 and (world == 1 or info.exchange == 3)
    import os
    if "OOB_DP_CHMAX" not in os.environ:        # waves re-sized for the ranks' unit shares
        assert info.chunk_max == (320 if world == 1 else 192 if world <= 3 else 96)
    fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    ws = [torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    pk = [torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    plan.run_virtual(fwd.data_ptr(), bwd.data_ptr(), [w.data_ptr() for w in ws], info.workspace_bytes,
                     [p.data_ptr() for p in pk], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return [plan.template_set(p.cpu().numpy()) for p in pk]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_virtual_shards_cfg3_every_wave(planner, world, monkeypatch):
    """Single-profile sharding checked on ONE GPU (SURVEY §4 "virtual shards"): every
    wavefront's W units split across `world` virtual ranks (OOB_DP_SHARDMIN=0: all waves),
    the partial argmins exchanged by device copies, every rank finalizing the whole wave —
    every rank's template set equals the oracle's."""
    monkeypatch.setenv("OOB_DP_SHARDMIN", "0")
    cfg = CONFIGS["cfg3"]
    prof = config_profiles(cfg, "real")[0]
    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
    for r, ts in enumerate(_virtual_run(planner, cfg, [prof], world)):
        _assert_same(ts.templates(0), want, f"cfg3 virtual rank {r}/{world}")


def test_virtual_shards_cfg4_golden(planner):
    """The launch configuration bench.py --shard-profile uses (large waves sharded, default
    threshold), 4 virtual ranks, full cfg4 set vs the oracle's stored output."""
    rec = load_golden("cfg4", "real")
    if rec is None:
        pytest.skip("tests/golden/cfg4_real.json not generated")
    cfg = CONFIGS["cfg4"]
    prof = config_profiles(cfg, "real")[0]
    for r, ts in enumerate(_virtual_run(planner, cfg, [prof], 4)):
        _assert_same(ts.templates(0), rec["profiles"][0]["templates"], f"cfg4 virtual rank {r}/4")


def _shard_worker(rank, world, port, q, xmode="peer"):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if xmode == "nccl":
        os.environ["OOB_DP_SHARDX"] = "nccl"
    os.environ["OOB_DP_SHARDMIN"] = "0"          # every wavefront sharded
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2309_08125_b200 import planner as pl
        cfg = CONFIGS["cfg3"]
        prof = config_profiles(cfg, "real")[0]
        comm = pl.NcclComm(world, rank, rank)
        plan = pl.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, 1)
        plan.set_comm(comm)
        info = plan.info
        assert info.world == world and info.pipelined == (1 if xmode == "peer" else 0)
        assert info.exchange == (1 if xmode == "peer" else 2)
        fwd = torch.tensor(prof.fwd_ms[None], dtype=torch.float64, device="cuda")
        bwd = torch.tensor(prof.bwd_ms[None], dtype=torch.float64, device="cuda")
        ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
        packed = torch.zeros(info.packed_bytes, dtype=torch.uint8, device="cuda")
        ok = True
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        for _ in range(3):                    # repeated runs: epoch-based peer counters
            packed.zero_()
            plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), packed.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ok = ok and plan.template_set(packed.cpu().numpy()).templates(0) == want
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("xmode", ["peer", "nccl"])
def test_single_profile_sharding_two_gpus(planner, xmode):
    """oob_dp_set_comm: one profile split across 2 GPUs, every wavefront sharded — partial
    argmins exchanged inside k_wave_w through NVLink peer memory (peer, pipelined) or by a
    per-wavefront ncclAllGather + k_fin (nccl) — gives the oracle's template set on both
    ranks, run after run (needs >= 2 GPUs)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q, xmode)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)]


def test_stage_masks_vs_oracle(planner):
    """Stage masks (reading R31: power-of-two GPU counts per stage, per-stage memory
    sum_l state_bytes / d <= cap): GPU == C oracle on random shapes, including sizes with no
    allowed mapping (None), through oob_generate_templates' tp_pow2 / stage_mem_bytes."""
    rng = random.Random(909)
    feasible_seen = infeasible_seen = 0
    for i in range(60):
        L = rng.choice([3, 5, 8, 12, 16, 24])
        M = rng.choice([2, 3, 4, 6, 8])
        prof = random_profile(9100 + i, L, M, rng.choice(["lognormal", "integer", "uniform"]))
        state = np.array([rng.randint(1, 50) for _ in range(L)], dtype=np.int64)
        pow2 = rng.random() < 0.6
        cap = float(state.max()) * rng.uniform(1.0, max(1.5, L / 2)) if rng.random() < 0.7 else 0.0
        n0 = rng.randint(1, max(1, min(L, 3)))
        f = rng.randint(0, 2)
        N = (f + 1) * n0 + rng.randint(0, L)
        n_hi = min(N - f * n0, L)
        hp = planner.Profile.from_arrays(prof.fwd_ms, prof.bwd_ms, state)
        ts = planner.generate_templates([hp], nodes=N, gpus_per_node=M, f=f, n0=n0, device=0, tp_pow2=pow2,
                                        stage_mem_bytes=cap)
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, n0, n_hi, pow2_tp=pow2,
                                       stage_bytes=state.astype(np.float64) if cap > 0 else None,
                                       mem_cap=cap if cap > 0 else None)
        got = ts.templates(0)
        assert len(got) == len(want)
        for g, w in zip(got, want):
            if w is None:
                assert g is None, (i, L, M)
                infeasible_seen += 1
                continue
            _assert_same([g], [w], f"masks case {i}")
            feasible_seen += 1
    assert feasible_seen > 50 and infeasible_seen > 0


def test_stage_masks_cfg4_pow2(planner):
    """The north-star shape with power-of-two TP: the smallest templates vs the oracle (they
    touch few cells) and every template's stages use 1, 2, 4 or 8 GPUs."""
    cfg = CONFIGS["cfg4"]
    prof = config_profiles(cfg, "real")[0]
    ts = planner.generate_templates([(prof.fwd_ms, prof.bwd_ms)], nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f,
                                    n0=cfg.n0, device=0, tp_pow2=True)
    got = ts.templates(0)
    for t in got:
        assert all(d in (1, 2, 4, 8) for (_, _, d, _, _) in t["stages"])
    want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n0 + 2, pow2_tp=True)
    _assert_same(got[:3], want, "cfg4 pow2 small templates")


def test_profiler_to_templates(planner, tmp_path):
    """Real profile ingestion: the B200 layer profiler writes the SPEC
    profile JSON, oob_load_profile reads it back exactly, per-layer costs fall with
    the tensor-parallel degree for a large block, and the measured profile plans on the GPU
    bit-identically to the oracle."""
    from paper_2309_08125_b200 import profiler
    doc = profiler.profile_gpt(hidden=2048, heads=16, layers=6, seq=1024, microbatch=2, gpus_per_node=4,
                               reps=5, busbw_gbps=600.0)
    path = str(tmp_path / "prof.json")
    profiler.write_profile(doc, path)
    prof = planner.load_profile(path)
    f, b, st = prof.costs()
    for l, ly in enumerate(doc["layers"]):
        assert [f[l, d - 1] for d in range(1, 5)] == [ly["fwd_ms"][str(d)] for d in range(1, 5)]
        assert st[l] == ly["state_bytes"]
    assert f[1, 0] > f[1, 1] > f[1, 3] > 0 and b[1, 0] > b[1, 3] > 0
    ts = planner.generate_templates([prof], nodes=5, gpus_per_node=4, f=1, n0=1, device=0)
    want, _ = coracle.template_set(f, b, 4, 1, 4)
    _assert_same(ts.templates(0), want, "measured profile")


def _comm_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2309_08125_b200 import planner as pl
        comm = pl.NcclComm(world, rank, rank)
        ok = True
        # one profile, wavefronts sharded (every wave: OOB_DP_SHARDMIN=0)
        os.environ["OOB_DP_SHARDMIN"] = "0"
        cfg = CONFIGS["cfg3"]
        prof = config_profiles(cfg, "real")[0]
        ts = pl.generate_templates([(prof.fwd_ms, prof.bwd_ms)], nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f,
                                   n0=cfg.n0, device=rank, comm=comm)
        want, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        ok = ok and ts.templates(0) == want
        del os.environ["OOB_DP_SHARDMIN"]
        # a batch of 5 profiles in contiguous blocks + one all-gather (every rank: all 5)
        cfg = CONFIGS["cfg5"]
        profs = config_profiles(cfg, "real", count=5)
        ts = pl.generate_templates([(p.fwd_ms, p.bwd_ms) for p in profs], nodes=cfg.N, gpus_per_node=cfg.M,
                                   f=cfg.f, n0=cfg.n0, device=rank, comm=comm)
        heur = []
        for i, p in enumerate(profs):
            want, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
            heur.append(want)
            ok = ok and ts.templates(i) == want
        # the same batch with the exact optimum (opts.exact): each rank's block, all-gathered
        from oracle.exact import exact_template
        ts = pl.generate_templates([(p.fwd_ms, p.bwd_ms) for p in profs], nodes=cfg.N, gpus_per_node=cfg.M,
                                   f=cfg.f, n0=cfg.n0, device=rank, comm=comm, exact=True)
        for i, p in enumerate(profs):
            for t in ts.templates(i)[::6]:
                e = exact_template(p.fwd_ms, p.bwd_ms, cfg.M, t["nodes"], ub=heur[i][t["nodes"] - cfg.n0]["total"])
                ok = ok and (t["S"], t["total"], [s[:4] for s in t["stages"]]) == \
                    (e["S"], e["total"], [tuple(s) for s in e["stages"]])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_generate_templates_with_communicator_two_gpus(planner):
    """oob_generate_templates with opts.comm (the headline API's multi-GPU path): one
    profile sharded per wavefront, and a batch split in blocks + NCCL all-gather (also with
    opts.exact); every rank receives the oracle's whole template set (needs >= 2 GPUs)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)]
