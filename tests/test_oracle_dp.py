"""Pins for the template-generation oracle (oracle/dp.py, oracle/c) against things other
than itself: SPEC/paper worked values, closed forms, brute force, invariants."""
import itertools
import random

import pytest

from oracle import coracle
from oracle.brute import brute_force
from oracle.dp import Cell, TemplateDP, closed_form, node_sizes, stage_time, template_set
from workloads import CONFIGS, config_profiles, costs_profile, random_profile, unif6


def _tpl(costs, M, n):
    p = costs_profile(costs, M)
    return TemplateDP(p.fwd_ms, p.bwd_ms, M).template(n)


# ------------------------------------------------------------------ SPEC worked examples
def test_unif6_single_stage_eq4():
    """UNIF6, n=1, M=1 -> T1=36, T2=72, T3=36, total 144 (Eq.4)."""
    p = unif6()
    t = TemplateDP(p.fwd_ms, p.bwd_ms, 1).template(1)
    assert (t["S"], t["T1"], t["T2"], t["T3"], t["total"]) == (1, 36.0, 72.0, 36.0, 144.0)
    assert t["stages"] == [(0, 6, 1, 0, 0)]


def test_unif6_two_nodes():
    """UNIF6 on 2 single-GPU nodes -> (3,3), T1=36, k*=0, T2=90, T3=36,
    total 162; the alternatives (4,2) and (2,4) cost 192 and 204."""
    p = unif6()
    t = TemplateDP(p.fwd_ms, p.bwd_ms, 1).template(2)
    assert t["S"] == 2
    assert [s[:2] for s in t["stages"]] == [(0, 3), (3, 6)]
    assert (t["T1"], t["kstar"], t["T2"], t["T3"], t["total"]) == (36.0, 0, 90.0, 36.0, 162.0)
    assert closed_form([24.0, 12.0])[0] == 192.0
    assert closed_form([12.0, 24.0])[0] == 204.0


def test_stage_cost_spec():
    """UNIF6 stage (0,3,1) -> F+B = 18 and (0,6,1) -> 36."""
    p = unif6()
    assert stage_time(p.fwd_ms, p.bwd_ms, 0, 3, 1) == 18.0
    assert stage_time(p.fwd_ms, p.bwd_ms, 0, 6, 1) == 36.0


def test_eq4_is_eq2_at_one_stage():
    """Eq.4 T2 = 2(F+B) must equal Eq.2 at S'=1 with N_b = 4S' and the
    0-based k* = 0 — pins N_b = 4S' and the k* base."""
    for t in (0.5, 3.0, 7.25, 1e-3):
        assert Cell(t, t, t, 0, None).T2(1) == 2.0 * t


# ------------------------------------------------------------------ closed form
def test_closed_form_kstar_tie_rule():
    """Reading R7: leftmost max.  Stage times (18,6,18): k*=0 -> 18+6+18 + (9-1)*18 + 42 = 228;
    the rightmost rule would give 240."""
    tot, T1, T2, T3, k = closed_form([18.0, 6.0, 18.0])
    assert (tot, T1, T2, T3, k) == (228.0, 42.0, 144.0, 42.0, 0)


def test_counterexample_heuristic_gap():
    """the paper's per-cell argmin is not the global optimum.
    c = [1,9,1,3,9,2], M=1, n=3: DP picks (2,2,2) with total 146 (stage times 10,4,11,
    k*=2, T2 = (9+2-1)*11 = 110); brute force finds (3,1,2) with total 138."""
    t = _tpl([1, 9, 1, 3, 9, 2], 1, 3)
    assert [s[:2] for s in t["stages"]] == [(0, 2), (2, 4), (4, 6)]
    assert (t["total"], t["kstar"], t["T2"]) == (146.0, 2, 110.0)
    p = costs_profile([1, 9, 1, 3, 9, 2], 1)
    best, arg = brute_force(p.fwd_ms, p.bwd_ms, 1, 3)
    assert best == 138.0
    assert [m[:2] for m in arg[0]] == [(0, 3), (3, 4), (4, 6)]


@pytest.mark.parametrize("costs,n,dp_total,stages,bf", [
    ([9, 4, 1, 7, 8, 6], 3, 189.0, [(0, 1), (1, 4), (4, 6)], 182.0),
    ([6, 8, 3, 1, 4, 7, 4], 4, 198.0, [(0, 1), (1, 2), (2, 5), (5, 7)], 192.0),
    ([8, 3, 2, 5, 5, 8, 3], 4, 199.0, [(0, 1), (1, 3), (3, 5), (5, 7)], 189.0),
])
def test_survey_gap_vectors(costs, n, dp_total, stages, bf):
    t = _tpl(costs, 1, n)
    assert t["total"] == dp_total
    assert [s[:2] for s in t["stages"]] == stages
    p = costs_profile(costs, 1)
    assert brute_force(p.fwd_ms, p.bwd_ms, 1, n)[0] == bf


def _small_instances(count, seed, Lmax=6, Mmax=2, nmax=3, kinds=("integer", "uniform", "spiky")):
    rng = random.Random(seed)
    for i in range(count):
        L = rng.randint(2, Lmax)
        M = rng.randint(1, Mmax)
        kind = rng.choice(kinds)
        p = random_profile(seed * 1000 + i, L, M, kind)
        n = rng.randint(1, min(nmax, L))
        yield p, M, n


def _check_template_invariants(t, L, M, n):
    st = t["stages"]
    assert n <= t["S"] <= min(L, n * M) and len(st) == t["S"]
    assert st[0][0] == 0 and st[-1][1] == L
    for a, b in zip(st, st[1:]):
        assert a[1] == b[0] and a[0] < a[1]
    assert sum(s[2] for s in st) == n * M
    per_node = {}
    for (_, _, d, node, off) in st:
        per_node.setdefault(node, []).append((off, d))
    assert sorted(per_node) == list(range(n))
    for node, lst in per_node.items():
        lst.sort()
        pos = 0
        for off, d in lst:
            assert off == pos
            pos += d
        assert pos == M


def test_dp_vs_brute_force_small():
    """P:421 objective on every mapping (brute force): DP total >= optimum; equality for
    S = 2 cells (optimal substructure holds for two stages); the DP total equals the closed
    form of its own partition (exact on integer costs)."""
    checked = 0
    for p, M, n in _small_instances(120, 7):
        dp = TemplateDP(p.fwd_ms, p.bwd_ms, M)
        t = dp.template(n)
        _check_template_invariants(t, p.L, M, n)
        best, _ = brute_force(p.fwd_ms, p.bwd_ms, M, n)
        assert t["total"] >= best - 1e-9 * abs(best)
        times = [stage_time(p.fwd_ms, p.bwd_ms, u, v, d) for (u, v, d, _, _) in t["stages"]]
        cf = closed_form(times)
        assert cf[0] == pytest.approx(t["total"], rel=1e-12)
        assert cf[4] == t["kstar"]
        if 2 >= n and 2 <= min(p.L, n * M):
            c2 = dp.T(2, 0, p.L, ("W", n))
            b2, _ = brute_force(p.fwd_ms, p.bwd_ms, M, n, S_only=2)
            assert c2.total(2) == pytest.approx(b2, rel=1e-12)
        checked += 1
    assert checked == 120


def test_dp_closed_form_exact_on_integers():
    for p, M, n in _small_instances(60, 11, Lmax=9, Mmax=3, nmax=4, kinds=("integer", "spiky")):
        t = TemplateDP(p.fwd_ms, p.bwd_ms, M).template(n)
        times = [stage_time(p.fwd_ms, p.bwd_ms, u, v, d) for (u, v, d, _, _) in t["stages"]]
        tot, T1, T2, T3, k = closed_form(times)
        assert (tot, T1, T2, T3, k) == (t["total"], t["T1"], t["T2"], t["T3"], t["kstar"])


def test_unmemoized_equals_memoized():
    """SPEC acceptance #1: memoized recursion = exhaustive recursion w/o memo."""
    for p, M, n in _small_instances(25, 3, Lmax=5, Mmax=2, nmax=2):
        a = TemplateDP(p.fwd_ms, p.bwd_ms, M, memo=True).template(n)
        b = TemplateDP(p.fwd_ms, p.bwd_ms, M, memo=False).template(n)
        assert a == b


def test_validity_iff_finite():
    """A cell (S',u,v,a) is finite iff lo(a) <= S' <= min(v-u, gpus(a)) —
    the fully literal Python recursion (no early exits) reaches exactly these."""
    for p, M, n in _small_instances(30, 5, Lmax=6, Mmax=3, nmax=3):
        dp = TemplateDP(p.fwd_ms, p.bwd_ms, M)
        dp.template(n)
        for (Sp, u, v, a), c in dp.memo.items():
            kind, q = a
            lo = q if kind == "W" else 1
            g = q * M if kind == "W" else q
            assert (c is not None) == (lo <= Sp <= min(v - u, g)), (Sp, u, v, a)


def test_memo_sharing_equals_independent():
    """P:473 / SPEC S:184: the shared-memo template set equals per-size runs."""
    p = random_profile(42, 8, 2, "uniform")
    sizes = node_sizes(7, 1, 2, L=8)
    ts = template_set(p.fwd_ms, p.bwd_ms, 2, sizes)
    for t in ts:
        assert TemplateDP(p.fwd_ms, p.bwd_ms, 2).template(t["nodes"]) == t


def test_scaling_metamorphic():
    """Scaling every cost by 2^k gives identical choices and exactly scaled costs."""
    p = random_profile(9, 7, 2, "uniform")
    base = template_set(p.fwd_ms, p.bwd_ms, 2, [1, 2, 3])
    for k in (-3, 5):
        s = 2.0 ** k
        sc = template_set(p.fwd_ms * s, p.bwd_ms * s, 2, [1, 2, 3])
        for a, b in zip(base, sc):
            assert a["stages"] == b["stages"] and a["S"] == b["S"]
            for key in ("T1", "T2", "T3", "total", "tstar"):
                assert b[key] == a[key] * s


# ------------------------------------------------------------------ C oracle = Python oracle
def test_c_oracle_matches_python_small():
    rng = random.Random(99)
    for i in range(60):
        L = rng.randint(1, 9)
        M = rng.randint(1, 4)
        kind = rng.choice(["integer", "uniform", "lognormal", "spiky", "constant"])
        p = random_profile(500 + i, L, M, kind)
        n_hi = rng.randint(1, L)
        n_lo = rng.randint(1, n_hi)
        py = template_set(p.fwd_ms, p.bwd_ms, M, range(n_lo, n_hi + 1))
        c, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, M, n_lo, n_hi)
        assert c == py


@pytest.mark.parametrize("key", ["cfg1", "cfg2"])
def test_c_oracle_matches_python_configs(key):
    cfg = CONFIGS[key]
    for mode in ("real", "dyadic"):
        p = config_profiles(cfg, mode)[0]
        py = template_set(p.fwd_ms, p.bwd_ms, cfg.M, range(cfg.n0, cfg.n_max + 1))
        c, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        assert c == py


def test_template_invariants_configs_c():
    for key in ("cfg2", "cfg3"):
        cfg = CONFIGS[key]
        p = config_profiles(cfg)[0]
        ts, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
        for t in ts:
            _check_template_invariants(t, cfg.L, cfg.M, t["nodes"])
            times = [stage_time(p.fwd_ms, p.bwd_ms, u, v, d) for (u, v, d, _, _) in t["stages"]]
            assert closed_form(times)[0] == pytest.approx(t["total"], rel=1e-12)


# ------------------------------------------------------------------ node specification
def test_node_sizes_spec():
    """SPEC S:150-152 and P:362-363 (n_max = N - f n0)."""
    assert node_sizes(13, 2, 2) == list(range(2, 10))
    assert node_sizes(7, 1, 2) == [2, 3, 4, 5]
    assert node_sizes(4, 1, 2) == [2]
    with pytest.raises(ValueError):
        node_sizes(3, 1, 2)
    assert node_sizes(512, 4, 3, L=96) == list(range(3, 97))    # reading R4 (cap at L)


# ------------------------------------------------------------------ tie-rule pins (readings R6, R8)
def _cd_profile(cd):
    """Profile with F+B = cd[l][d-1] exactly (F = B = c/2; dyadic values, exact sums)."""
    import numpy as np
    c = np.asarray(cd, dtype=np.float64)
    return c / 2.0, c / 2.0


def _both_oracles(fwd, bwd, M, n):
    py = TemplateDP(fwd, bwd, M).template(n)
    c, _ = coracle.template_set(fwd, bwd, M, n, n)
    assert c[0] == py
    return py


def test_s_tie_smaller_s_wins():
    """Reading R8 ("smaller S"): L=2, M=2, n=1, per-layer F+B on 1 GPU
    = 1 and on 2 GPUs = 1.125 (both layers).
      S=1: one stage (0,2) on 2 GPUs, t = 2.25: T1 = T3 = 2.25, T2 = (4-1+0-1) 2.25 = 4.5,
           total 9.
      S=2: stages (0,1),(1,2) on 1 GPU each, times (1,1): T1 = 2, k* = 0, T2 = (8-2+0-1) 1
           = 5, T3 = 2, total 9.
    Equal totals: the smaller S wins -> one stage.  (Larger-S-wins would return S=2.)"""
    fwd, bwd = _cd_profile([[1, 1.125], [1, 1.125]])
    assert closed_form([2.25])[0] == 9.0 and closed_form([1.0, 1.0])[0] == 9.0
    t = _both_oracles(fwd, bwd, 2, 1)
    assert (t["S"], t["total"]) == (1, 9.0)
    assert t["stages"] == [(0, 2, 2, 0, 0)]


def test_device_split_order_smaller_m_wins():
    """Reading R6 (smaller k, then m, then s): L=2, M=3, n=1; layer 0 costs
    F+B = 2 on 1 or 2 GPUs, layer 1 costs 1 on 1 or 2 GPUs, both cost 10 on 3 GPUs.
    W(1) with S'=2 splits only at k=1 into (I(m), I(3-m)):
      m=1: stage times (2, 1) on (1, 2) GPUs: T1 = 3, k* = 0, T2 = 5*2 = 10, T3 = 3 -> 16;
      m=2: stage times (2, 1) on (2, 1) GPUs -> 16 as well.
    S=1 (one stage on 3 GPUs) costs 4*20 = 80.  The tie goes to m=1: stage 0 gets 1 GPU
    (offset 0), stage 1 gets 2 GPUs (offset 1).  (Reversed m order returns (2 GPUs, 1 GPU).)"""
    fwd, bwd = _cd_profile([[2, 2, 10], [1, 1, 10]])
    assert closed_form([2.0, 1.0])[0] == 16.0
    t = _both_oracles(fwd, bwd, 3, 1)
    assert (t["S"], t["total"]) == (2, 16.0)
    assert t["stages"] == [(0, 1, 1, 0, 0), (1, 2, 2, 0, 1)]


def test_node_split_order_smaller_j_wins():
    """Reading R6 for whole-node splits W(q) -> (W(j), W(q-j)), smaller j first.  L=5, M=2,
    n=3, integer F+B (columns d=1, d=2): [[3,3],[1,1],[2,3],[3,2],[1,1]].  Two partitions
    tie at total 51 (closed form, Eq.1-3 / P:381-386):
      (0,1)x1, (1,3)x1 on node 0; (3,4)x2 on node 1; (4,5)x2 on node 2 — stage times
        3, 3, 2, 1: k* = 0, T1 = 9, T2 = (16-4+0-1)*3 = 33, T3 = 9, total 51;
      (0,1)x2 on node 0; (1,2)x1, (2,3)x1 on node 1; (3,5)x2 on node 2 — stage times
        3, 1, 2, 3: k* = 0, T1 = 9, T2 = 33, T3 = 9, total 51.
    The first is reached with the smaller j at the layer split k=3 (node split (W(1), W(2))),
    the second with (W(2), W(1)): the oracle keeps the smaller j."""
    cd = [[3, 3], [1, 1], [2, 3], [3, 2], [1, 1]]
    fwd, bwd = _cd_profile(cd)
    first = [(0, 1, 1, 0, 0), (1, 3, 1, 0, 1), (3, 4, 2, 1, 0), (4, 5, 2, 2, 0)]
    second = [(0, 1, 2, 0, 0), (1, 2, 1, 1, 0), (2, 3, 1, 1, 1), (3, 5, 2, 2, 0)]
    for st in (first, second):
        times = [stage_time(fwd, bwd, u, v, d) for (u, v, d, _, _) in st]
        assert closed_form(times)[0] == 51.0
    t = _both_oracles(fwd, bwd, 2, 3)
    assert t["total"] == 51.0
    assert t["stages"] == first


# ------------------------------------------------------------------ stage masks (reading R31)
from oracle.dp import stage_allowed  # noqa: E402


def test_pow2_mask_hand_example():
    """pow2_tp: with M = 3 a single stage on the whole node would use 3 GPUs (not a power of
    two), so the 1-node template must split into stages of (1, 2) or (2, 1) GPUs.  L = 2,
    F+B per layer: 1 GPU -> 4, 2 GPUs -> 2, 3 GPUs -> 1.
      unmasked: S=1 on 3 GPUs, t = 2: total 4*2 = 8 (vs S=2 splits >= 10);
      masked:   (I(1), I(2)): times (4, 2): T1 = 6, k* = 0, T2 = 5*4 = 20, T3 = 6 -> 32;
                (I(2), I(1)): times (2, 4): T1 = 6, k* = 1, T2 = 6*4 = 24, T3 = 4 -> 34."""
    fwd, bwd = _cd_profile([[4, 2, 1], [4, 2, 1]])
    free = TemplateDP(fwd, bwd, 3).template(1)
    assert (free["S"], free["total"]) == (1, 8.0)
    t = TemplateDP(fwd, bwd, 3, pow2_tp=True).template(1)
    assert (t["S"], t["total"]) == (2, 32.0)
    assert t["stages"] == [(0, 1, 1, 0, 0), (1, 2, 2, 0, 1)]
    c, _ = coracle.template_set(fwd, bwd, 3, 1, 1, pow2_tp=True)
    assert c[0] == t


def test_memory_mask_hand_example():
    """Stage memory (sum of the stage's layer bytes / d <= cap): L = 4 layers of 10 bytes,
    M = 1, n = 2, cap = 25: a 3-layer stage (30) does not fit, so only the 2+2 split is
    allowed although 1+3 / 3+1 exist; cap = 15 leaves no feasible 2-node template (None)."""
    fwd, bwd = _cd_profile([[1], [1], [1], [1]])
    sb = [10.0] * 4
    t = TemplateDP(fwd, bwd, 1, stage_bytes=sb, mem_cap=25.0).template(2)
    assert [s[:2] for s in t["stages"]] == [(0, 2), (2, 4)]
    assert TemplateDP(fwd, bwd, 1, stage_bytes=sb, mem_cap=15.0).template(2) is None
    assert stage_allowed(0, 3, 1, stage_bytes=sb, mem_cap=25.0) is False
    assert stage_allowed(0, 3, 2, stage_bytes=sb, mem_cap=25.0) is True


def test_masks_vs_brute_force_and_c_oracle():
    """With stage masks the recursion stays a heuristic over the allowed mappings: DP total
    >= brute force over allowed mappings, equal for S <= 2 templates, never a disallowed
    stage; the C oracle equals the Python oracle."""
    rng = random.Random(31)
    checked = 0
    for i in range(80):
        L, M = rng.randint(2, 6), rng.choice([2, 3, 4])
        n = rng.randint(1, min(3, L))
        p = random_profile(4400 + i, L, M, rng.choice(["integer", "uniform"]))
        sb = [float(rng.randint(1, 9)) for _ in range(L)]
        masks = rng.choice([{"pow2_tp": True}, {"stage_bytes": sb, "mem_cap": float(rng.randint(6, 30))},
                            {"pow2_tp": True, "stage_bytes": sb, "mem_cap": float(rng.randint(6, 30))}])
        ok = lambda u, v, d: stage_allowed(u, v, d, masks.get("pow2_tp", False), masks.get("stage_bytes"),
                                           masks.get("mem_cap"))
        t = TemplateDP(p.fwd_ms, p.bwd_ms, M, **masks).template(n)
        best, _ = brute_force(p.fwd_ms, p.bwd_ms, M, n, allowed=ok)
        c, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, M, n, n, **masks)
        assert c[0] == t
        if t is None:
            assert best == float("inf")
            continue
        assert all(ok(u, v, d) for (u, v, d, _, _) in t["stages"])
        assert t["total"] >= best - 1e-9 * best
        if t["S"] <= 2:
            b2, _ = brute_force(p.fwd_ms, p.bwd_ms, M, n, S_only=t["S"], allowed=ok)
            assert t["total"] <= b2 * (1 + 1e-12)
        checked += 1
    assert checked > 40
