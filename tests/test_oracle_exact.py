"""Pins for the exact-optimum oracle (oracle/exact.py, oracle/c/oob_exact.c) against brute
force over every mapping (oracle/brute.py) and the SURVEY §0.1 counterexamples: the exact
solver must reach the brute-force minimum, return a valid mapping whose closed form is
that minimum, and never be worse than the paper's recursion."""
import random

import pytest

from oracle.brute import brute_force
from oracle.dp import TemplateDP, closed_form, stage_time
from oracle.exact import exact_template
from workloads import costs_profile, random_profile


def _valid(st, L, M, n):
    assert st[0][0] == 0 and st[-1][1] == L
    for a, b in zip(st, st[1:]):
        assert a[1] == b[0] and a[0] < a[1]
    used = [0] * n
    for (_, _, d, node) in st:
        assert 1 <= d <= M
        used[node] += d
    assert used == [M] * n
    nodes = [s[3] for s in st]
    assert nodes == sorted(nodes)


@pytest.mark.parametrize("costs,n,bf", [
    ([1, 9, 1, 3, 9, 2], 3, 138.0),
    ([9, 4, 1, 7, 8, 6], 3, 182.0),
    ([6, 8, 3, 1, 4, 7, 4], 4, 192.0),
    ([8, 3, 2, 5, 5, 8, 3], 4, 189.0),
])
def test_exact_reaches_counterexample_optima(costs, n, bf):
    """SURVEY §0.1 vectors where the recursion is strictly above the optimum."""
    p = costs_profile(costs, 1)
    e = exact_template(p.fwd_ms, p.bwd_ms, 1, n)
    assert e["total"] == bf and e["dp_value"] == bf
    _valid(e["stages"], len(costs), 1, n)
    assert TemplateDP(p.fwd_ms, p.bwd_ms, 1).template(n)["total"] > bf


def test_exact_vs_brute_force_integers():
    """Integer costs: every sum is exact, so exact == brute force bit for bit, and the
    returned mapping is one of brute force's argmins."""
    rng = random.Random(5)
    for i in range(80):
        L = rng.randint(2, 7)
        M = rng.randint(1, 3)
        n = rng.randint(1, min(3, L))
        p = random_profile(9000 + i, L, M, rng.choice(["integer", "spiky"]))
        best, arg = brute_force(p.fwd_ms, p.bwd_ms, M, n)
        e = exact_template(p.fwd_ms, p.bwd_ms, M, n)
        _valid(e["stages"], L, M, n)
        assert e["total"] == best and e["dp_value"] == best
        assert tuple(e["stages"]) in [tuple(m) for m in arg]
        assert e["total"] <= TemplateDP(p.fwd_ms, p.bwd_ms, M).template(n)["total"]


def test_exact_vs_brute_force_real():
    """Real-valued costs: equal up to the summation order of the two objectives."""
    rng = random.Random(6)
    for i in range(60):
        L = rng.randint(2, 7)
        M = rng.randint(1, 3)
        n = rng.randint(1, min(3, L))
        p = random_profile(9500 + i, L, M, "uniform")
        best, _ = brute_force(p.fwd_ms, p.bwd_ms, M, n)
        e = exact_template(p.fwd_ms, p.bwd_ms, M, n)
        _valid(e["stages"], L, M, n)
        times = [stage_time(p.fwd_ms, p.bwd_ms, u, v, d) for (u, v, d, _) in e["stages"]]
        assert closed_form(times)[0] == e["total"]
        assert e["total"] == pytest.approx(best, rel=1e-12)
        assert e["dp_value"] == pytest.approx(best, rel=1e-12)
        dp = TemplateDP(p.fwd_ms, p.bwd_ms, M).template(n)["total"]
        assert e["total"] <= dp * (1 + 1e-12)


def test_exact_single_node_single_stage():
    """n = 1, M = 1: one stage of all layers (F+B = c per layer), total = 4 t (Eq.4)."""
    p = costs_profile([2, 3, 5], 1)
    e = exact_template(p.fwd_ms, p.bwd_ms, 1, 1)
    assert e["stages"] == [(0, 3, 1, 0)] and e["total"] == 4 * 10.0


def test_exact_too_few_layers():
    p = costs_profile([1, 2], 1)
    assert exact_template(p.fwd_ms, p.bwd_ms, 1, 3) is None


def test_exact_window_by_recursion_total():
    """ub = the recursion's total only narrows the bottleneck values searched: same optimum."""
    rng = random.Random(8)
    for i in range(40):
        L = rng.randint(3, 9)
        M = rng.randint(1, 4)
        n = rng.randint(1, min(4, L))
        p = random_profile(9800 + i, L, M, rng.choice(["integer", "uniform", "spiky"]))
        ub = TemplateDP(p.fwd_ms, p.bwd_ms, M).template(n)["total"]
        a = exact_template(p.fwd_ms, p.bwd_ms, M, n)
        b = exact_template(p.fwd_ms, p.bwd_ms, M, n, ub=ub)
        assert a["total"] == b["total"] and a["stages"] == b["stages"]


def test_exact_vs_brute_force_constant_ties():
    """Constant profiles (every layer alike: massive ties among mappings): exact == brute
    force bit for bit, and the returned mapping is one of brute force's argmins."""
    rng = random.Random(9)
    for i in range(30):
        L = rng.randint(2, 7)
        M = rng.randint(1, 3)
        n = rng.randint(1, min(3, L))
        p = random_profile(9900 + i, L, M, "constant")
        best, arg = brute_force(p.fwd_ms, p.bwd_ms, M, n)
        e = exact_template(p.fwd_ms, p.bwd_ms, M, n)
        _valid(e["stages"], L, M, n)
        assert e["total"] == best
        assert tuple(e["stages"]) in [tuple(m) for m in arg]
