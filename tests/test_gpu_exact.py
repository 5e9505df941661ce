"""GPU parity of the exact-optimum solver (oob_exact_run / generate_templates(exact=True))
against the CPU exact oracle (oracle/exact.py, a separate per-n push-form DP pinned to brute
force in tests/test_oracle_exact.py): stages, S, k* and all costs bit-exact; never above the
paper's recursion."""
import random

import numpy as np
import pytest

from oracle import coracle
from oracle.exact import exact_template
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


def _with_offsets(stages, M):
    out, off, node = [], 0, -1
    for (u, v, d, nd) in stages:
        if nd != node:
            node, off = nd, 0
        out.append((u, v, d, nd, off))
        off += d
    return out


def _assert_exact(got, prof, M, n_lo, ctx, ub=None):
    for i, g in enumerate(got):
        n = n_lo + i
        e = exact_template(prof.fwd_ms, prof.bwd_ms, M, n, ub=0.0 if ub is None else ub[n])
        assert g["nodes"] == n, ctx
        assert (g["S"], g["kstar"]) == (e["S"], e["kstar"]), (ctx, n)
        assert g["stages"] == _with_offsets(e["stages"], M), (ctx, n)
        for k in ("T1", "T2", "T3", "total"):
            assert g[k] == e[k], (ctx, n, k, g[k], e[k])


def _gen(planner, profs, cfg_like, exact=True):
    L, M, N, f, n0 = cfg_like
    return planner.generate_templates([(p.fwd_ms, p.bwd_ms) for p in profs], nodes=N, gpus_per_node=M, f=f, n0=n0,
                                      device=0, exact=exact)


@pytest.mark.parametrize("key", ["cfg1", "cfg2", "cfg3"])
def test_exact_configs_vs_oracle(planner, key):
    cfg = CONFIGS[key]
    prof = config_profiles(cfg)[0]
    ts = _gen(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    _assert_exact(ts.templates(0), prof, cfg.M, cfg.n0, key)


def test_exact_random_small_vs_oracle(planner):
    """Shapes with ties and ragged node counts: L 1..24, M 1..8, every kind; the exact set is
    never above the recursion's (same profile, same sizes)."""
    rng = random.Random(77)
    for i in range(60):
        L = rng.choice([1, 2, 3, 5, 7, 9, 12, 16, 24])
        M = rng.choice([1, 2, 3, 4, 8])
        kind = rng.choice(["integer", "uniform", "lognormal", "spiky", "constant"])
        prof = random_profile(8100 + i, L, M, kind, rng.choice(["real", "dyadic"]))
        n0 = rng.randint(1, max(1, min(L, 3)))
        f = rng.randint(0, 2)
        N = (f + 1) * n0 + rng.randint(0, 2 * L)
        ts = _gen(planner, [prof], (L, M, N, f, n0))
        got = ts.templates(0)
        _assert_exact(got, prof, M, n0, f"case {i} L={L} M={M} {kind}")
        heur, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, n0, n0 + len(got) - 1)
        for g, h in zip(got, heur):
            assert g["total"] <= h["total"] * (1 + 1e-12), (i, g["nodes"])


def test_exact_batched_cfg5_profiles(planner):
    """cfg5-shaped random profiles (where the recursion misses the optimum by up to 15%),
    8 per batch: every profile's set equals the oracle's; at least one size improves."""
    cfg = CONFIGS["cfg5"]
    profs = config_profiles(cfg, count=8)
    ts = _gen(planner, profs, (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    improved = 0
    for p in (0, 1, 3, 6):
        got = ts.templates(p)
        heur, _ = coracle.template_set(profs[p].fwd_ms, profs[p].bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        _assert_exact(got, profs[p], cfg.M, cfg.n0, f"cfg5 profile {p}", ub={h["nodes"]: h["total"] for h in heur})
        improved += sum(1 for g, h in zip(got, heur) if g["total"] < h["total"] * (1 - 1e-9))
    assert improved > 0


def test_exact_unbounded_equals_bounded(planner):
    """d_packed_ub = NULL searches every stage time: same templates as the bounded run."""
    import torch
    cfg = CONFIGS["cfg2"]
    profs = config_profiles(cfg) + [random_profile(8400 + i, cfg.L, cfg.M, "spiky") for i in range(3)]
    P = len(profs)
    plan = planner.DPPlan(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
    info = plan.info
    fwd = torch.tensor(np.stack([p.fwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    bwd = torch.tensor(np.stack([p.bwd_ms for p in profs]), dtype=torch.float64, device="cuda")
    ws = torch.empty(info.workspace_bytes, dtype=torch.uint8, device="cuda")
    heur = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
    plan.run(fwd.data_ptr(), bwd.data_ptr(), ws.data_ptr(), ws.numel(), heur.data_ptr())
    xb = planner.exact_workspace_bytes(cfg.L, cfg.M, cfg.n0, cfg.n_max, P)
    xws = torch.empty(xb, dtype=torch.uint8, device="cuda")
    outs = []
    for ub in (heur.data_ptr(), 0):
        out = torch.empty(info.packed_bytes, dtype=torch.uint8, device="cuda")
        planner.exact_run(cfg.L, cfg.M, cfg.n0, cfg.n_max, P, fwd.data_ptr(), bwd.data_ptr(), ub, xws.data_ptr(),
                          xb, out.data_ptr())
        torch.cuda.synchronize()
        outs.append((out.cpu().numpy(), int(xws[:8].cpu().numpy().view(np.uint64)[0])))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert 0 < outs[0][1] <= outs[1][1]          # the bound prunes tasks (never adds)


def test_exact_cfg4_sampled_sizes(planner):
    """cfg4 at full size (96 layers, 512 x 8, f = 4): the whole exact set on the GPU; sizes
    3, 24, 60 and 96 checked against the oracle (each a CPU exact solve bounded by the
    golden recursion totals, which only prunes)."""
    cfg = CONFIGS["cfg4"]
    prof = config_profiles(cfg)[0]
    gold = load_golden("cfg4")
    ub = {t["nodes"]: t["total"] for t in gold["profiles"][0]["templates"]}
    ts = _gen(planner, [prof], (cfg.L, cfg.M, cfg.N, cfg.f, cfg.n0))
    got = ts.templates(0)
    assert len(got) == cfg.n_max - cfg.n0 + 1
    for n in (3, 24, 60, 96):
        _assert_exact([got[n - cfg.n0]], prof, cfg.M, n, f"cfg4 n={n}", ub=ub)


def test_exact_rejects_masks(planner):
    cfg = CONFIGS["cfg1"]
    prof = config_profiles(cfg)[0]
    with pytest.raises(Exception):
        planner.generate_templates([(prof.fwd_ms, prof.bwd_ms)], nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f,
                                   n0=cfg.n0, device=0, exact=True, tp_pow2=True)
