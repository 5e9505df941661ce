"""Pins for oracle/instantiate.py (Eq.5, Eq.6, coverage) against paper/SPEC values,
brute force and invariants."""
import random

import pytest

from oracle.dp import node_sizes
from oracle.instantiate import (coverage_ok, distribute_batch_brute, enumerate_sets,
                                enumerate_sets_brute, recommend_batch, variance_objective)
from workloads import CONFIGS


def test_eq5_paper_13_nodes():
    """13 nodes with templates (2,3,4) include (1,1,2) and (0,3,1)."""
    xs = enumerate_sets([2, 3, 4], 13, 0)
    assert (1, 1, 2) in xs and (0, 3, 1) in xs


def test_eq5_fig6_seven_nodes():
    """`fig:instantiation_dyp` P:517-520 setup; N'=7, f=1 -> exactly
    {(2,1,0), (0,1,1)}."""
    assert sorted(enumerate_sets([2, 3, 4], 7, 1)) == [(0, 1, 1), (2, 1, 0)]
    assert enumerate_sets([2], 2, 0) == [(1,)]


def test_eq5_equals_brute_force():
    """exact set equality for N' <= 20, p <= 5; every set satisfies
    Requirements 1-2."""
    for n0 in range(1, 4):
        for p in range(1, 6):
            sizes = list(range(n0, n0 + p))
            for Np in range(0, 21):
                for f in range(0, 3):
                    a = enumerate_sets(sizes, Np, f)
                    b = enumerate_sets_brute(sizes, Np, f)
                    assert sorted(a) == sorted(b)
                    assert len(set(a)) == len(a)
                    for x in a:
                        assert sum(xi * ni for xi, ni in zip(x, sizes)) == Np
                        assert sum(x) >= f + 1


def test_coverage_theorem_configs():
    """App. A: every N' in [(f+1) n0, N] is reachable with >= f+1 pipelines,
    for every BASELINE config with sizes capped at L (reading R4)."""
    for cfg in CONFIGS.values():
        sizes = node_sizes(cfg.N, cfg.f, cfg.n0, L=cfg.L)
        assert coverage_ok(sizes, (cfg.f + 1) * cfg.n0, cfg.N, cfg.f)


def test_coverage_theorem_small():
    """p = n0 consecutive sizes n0..2n0-1 cover every N' in [n0, 100] (f=0);
    random (N, f, n0) with p > n0 - 1 cover [(f+1) n0, N]."""
    for n0 in range(1, 7):
        assert coverage_ok(list(range(n0, 2 * n0)), n0, 100, 0)
    rng = random.Random(3)
    done = 0
    while done < 300:
        N, f, n0 = rng.randint(1, 40), rng.randint(0, 3), rng.randint(1, 4)
        if N < (f + 1) * n0:
            continue
        sizes = node_sizes(N, f, n0)
        if len(sizes) <= n0 - 1:
            continue
        assert coverage_ok(sizes, (f + 1) * n0, N, f)
        done += 1


def test_eq6_spec_example():
    """times (10, 20), B=24, b=4 -> N_b = (4, 2), objective 0."""
    nb, obj = distribute_batch_brute([10.0, 20.0], 24, 4)
    assert nb == (4, 2) and obj == 0.0


def test_eq6_conservation_and_errors():
    rng = random.Random(5)
    for _ in range(200):
        x = rng.randint(1, 4)
        T = [rng.uniform(1, 30) for _ in range(x)]
        b = rng.choice([1, 2, 4])
        K = rng.randint(x, 14)
        nb, obj = distribute_batch_brute(T, K * b, b)
        assert sum(nb) * b == K * b and min(nb) >= 1
        assert obj == pytest.approx(variance_objective(nb, T))
    with pytest.raises(ValueError):
        distribute_batch_brute([1.0, 2.0], 4, 4)
    with pytest.raises(ValueError):
        distribute_batch_brute([1.0], 7, 2)


def test_recommend_batch_spec():
    """SPEC S:253-255."""
    assert recommend_batch(2, 4, 4) == 8
    assert recommend_batch(3, 2, 7) == 8
    assert recommend_batch(1, 4, 8) == 8
