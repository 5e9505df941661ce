"""CPU tests of the C-ABI library: loads, exports every declared symbol, host logic
(node spec, counts, JSON, Eq.5/Eq.6 solvers) against the oracle.  No GPU compute."""
import ctypes
import json
import os
import random
import re

import numpy as np
import pytest

from oracle.dp import node_sizes as oracle_node_sizes
from oracle.dp import template_set as oracle_template_set
from oracle.instantiate import (distribute_batch_brute, enumerate_sets_brute, recommend_batch,
                                select_plan_brute, variance_objective)
from tests.helpers import count_universe, pack_templates
from workloads import CONFIGS, random_profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def planner():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2309_08125_b200 import planner as p
    return p


def test_library_exports_every_declared_symbol(planner):
    from paper_2309_08125_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "oobleck_plan.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(oob_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 25
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in include/oobleck_plan.h but not exported"
    assert declared == set(_lib.EXPORTED)


@pytest.mark.parametrize("key,cells,splits", [
    ("cfg1", 145, 306), ("cfg2", 15405, 1136491), ("cfg3", 61886, 10390002),
    ("cfg4", 3501358, 14306501154), ("cfg5", 259210, 139149026)])
def test_work_counts_match_survey(planner, key, cells, splits):
    """SURVEY §8 table (derived there by a separate counting script)."""
    cfg = CONFIGS[key]
    info = planner.dp_info(cfg.L, cfg.M, cfg.n0, cfg.n_max)
    assert (info.cells_per_profile, info.splits_per_profile) == (cells, splits)


def test_work_counts_match_brute_enumeration(planner):
    rng = random.Random(1)
    for _ in range(12):
        L, M = rng.randint(1, 10), rng.randint(1, 5)
        n_hi = rng.randint(1, L)
        info = planner.dp_info(L, M, 1, n_hi)
        assert (info.cells_per_profile, info.splits_per_profile) == count_universe(L, M, n_hi)
    for key in ("cfg1", "cfg2"):
        cfg = CONFIGS[key]
        info = planner.dp_info(cfg.L, cfg.M, cfg.n0, cfg.n_max)
        assert (info.cells_per_profile, info.splits_per_profile) == count_universe(cfg.L, cfg.M, cfg.n_max)


def test_node_sizes(planner):
    from paper_2309_08125_b200._lib import OOB_E_INFEASIBLE, OobError
    for N, f, n0, L in [(13, 2, 2, 100), (7, 1, 2, 100), (4, 1, 2, 100), (512, 4, 3, 96), (64, 3, 1, 32)]:
        assert planner.node_sizes(N, f, n0, L) == oracle_node_sizes(N, f, n0, L)
    with pytest.raises(OobError) as e:
        planner.node_sizes(3, 1, 2, 10)
    assert e.value.status == OOB_E_INFEASIBLE and "f+1" in str(e.value)
    with pytest.raises(OobError):
        planner.node_sizes(40, 1, 12, 10)      # n0 > L: too few layers


def test_count_sets_vs_brute(planner):
    for n0 in range(1, 4):
        for p in range(1, 5):
            for Np in range(0, 19):
                for f in range(0, 3):
                    want = len(enumerate_sets_brute(list(range(n0, n0 + p)), Np, f))
                    assert planner.count_sets(n0, n0 + p - 1, Np, f) == want


def test_distribute_batch_spec_and_brute(planner):
    from paper_2309_08125_b200._lib import OOB_E_BATCH, OobError
    assert planner.distribute_batch([10.0, 20.0], 24, 4) == ((4, 2), 0.0)
    assert planner.distribute_batch([7.0], 64, 8)[0] == (8,)
    with pytest.raises(OobError) as e:
        planner.distribute_batch([1.0, 2.0], 4, 4)
    assert e.value.status == OOB_E_BATCH and e.value.payload["recommended_global_batch"] == 8
    rng = random.Random(7)
    for trial in range(500):
        x = rng.randint(1, 4)
        kind = trial % 3
        if kind == 0:
            T = [rng.uniform(0.5, 30.0) for _ in range(x)]
        elif kind == 1:
            T = [float(rng.randint(1, 6)) for _ in range(x)]        # integer, many ties
        else:
            base = [rng.uniform(1, 10) for _ in range(2)]
            T = [rng.choice(base) for _ in range(x)]                  # repeated templates
        b = rng.choice([1, 2, 4])
        K = rng.randint(x, 30 if x <= 3 else 20)
        nb, obj = planner.distribute_batch(T, K * b, b)
        assert sum(nb) == K and min(nb) >= 1
        _, best = distribute_batch_brute(T, K * b, b)
        assert obj == pytest.approx(variance_objective(nb, T), rel=1e-9, abs=1e-9)
        assert obj <= best * (1 + 1e-9) + 1e-9, (T, K, nb, obj, best)


def test_recommend_batch(planner):
    for x, b, B in [(2, 4, 4), (3, 2, 7), (1, 4, 8), (5, 3, 1), (1, 1, 1)]:
        assert planner.recommend_batch(x, b, B) == recommend_batch(x, b, B)


def _oracle_set(p, M, sizes):
    return oracle_template_set(p.fwd_ms, p.bwd_ms, M, sizes)


def test_instantiate_vs_brute(planner):
    """oob_instantiate on an oracle-made template set == brute-force plan choice."""
    from paper_2309_08125_b200 import planner as pl
    rng = random.Random(11)
    checked = 0
    for i in range(40):
        L, M = rng.randint(3, 7), rng.randint(1, 2)
        N, f, n0 = rng.randint(2, 9), rng.randint(0, 2), 1
        if N < (f + 1) * n0:
            continue
        sizes = oracle_node_sizes(N, f, n0, L)
        prof = random_profile(900 + i, L, M, rng.choice(["uniform", "lognormal"]))
        tpls = _oracle_set(prof, M, sizes)
        packed, info = pack_templates([tpls], L, M, sizes[0], sizes[-1])
        dinfo = pl.OobDpInfo(**info, wavefronts=0, cells_per_profile=0, splits_per_profile=0,
                             kernel_launches=0, workspace_bytes=0)
        h = ctypes.c_void_p()
        pl.check(pl.lib.oob_template_set_from_packed(packed.ctypes.data, ctypes.byref(dinfo), ctypes.byref(h)))
        ts = pl.TemplateSet(h)
        assert ts.templates(0) == tpls
        b = rng.choice([1, 2])
        B = b * rng.randint(N, 14)
        for Np in range((f + 1) * n0, N + 1):
            want = select_plan_brute(tpls, Np, f, B, b)
            if want is None:
                continue
            got = planner.instantiate(ts, 0, Np, f, B, b)
            assert got["throughput"] == pytest.approx(want[0], rel=1e-12)
            assert got["counts"] == want[1]
            assert sum(got["nb"]) * b == B                   # conservation
            assert sum(got["counts"]) >= f + 1
            checked += 1
    assert checked > 20


def _set_handle(pl, tpls, L, M, sizes):
    packed, info = pack_templates([tpls], L, M, sizes[0], sizes[-1])
    dinfo = pl.OobDpInfo(**info, wavefronts=0, cells_per_profile=0, splits_per_profile=0,
                         kernel_launches=0, workspace_bytes=0)
    h = ctypes.c_void_p()
    pl.check(pl.lib.oob_template_set_from_packed(packed.ctypes.data, ctypes.byref(dinfo), ctypes.byref(h)))
    return pl.TemplateSet(h)


def test_instantiate_capped_candidates(planner):
    """Above max_enumerated (cfg4: 2.2e19 sets) oob_instantiate scores knapsack candidates
    (reading R20): on enumerable random cases the plan is valid, never better than the
    exhaustive optimum, within 10% of it, and equal to it in >= 90% of the cases."""
    from oracle import coracle
    from paper_2309_08125_b200 import planner as pl
    rng = random.Random(123)
    cases = exact = 0
    for it in range(120):
        L, M = rng.randint(6, 24), rng.choice([1, 2, 4, 8])
        N, f, n0 = rng.randint(8, 40), rng.randint(0, 3), rng.randint(1, 2)
        if N < (f + 1) * n0 or n0 > L:
            continue
        sizes = oracle_node_sizes(N, f, n0, L)
        prof = random_profile(100 + it, L, M, rng.choice(["uniform", "lognormal", "spiky", "integer"]))
        tpls = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, sizes[0], sizes[-1])[0]
        ts = _set_handle(pl, tpls, L, M, sizes)
        b = rng.choice([1, 2, 4])
        B = b * rng.randint(max(1, N // 4), 3 * N)
        Np = rng.randint((f + 1) * n0, N)
        try:
            ex = planner.instantiate(ts, 0, Np, f, B, b, max_enumerated=10 ** 8)
        except pl.OobError:
            continue
        if not 1 < ex["num_feasible"] <= 3e5:
            continue
        ca = planner.instantiate(ts, 0, Np, f, B, b, max_enumerated=1)
        assert ca["capped"] and not ex["capped"]
        assert sum(c * (sizes[0] + i) for i, c in enumerate(ca["counts"])) == Np
        assert sum(ca["counts"]) >= f + 1 and sum(ca["nb"]) * b == B
        assert ca["throughput"] <= ex["throughput"] * (1 + 1e-12)
        assert ca["throughput"] >= 0.9 * ex["throughput"], (it, ca, ex)
        cases += 1
        exact += ca["throughput"] >= ex["throughput"] * (1 - 1e-12)
    assert cases >= 60 and exact >= 0.9 * cases, (cases, exact)


def test_instantiate_all_vs_brute(planner):
    """oob_instantiate_all: the plan for every N' in one call.  Exhaustive mode == brute force
    (select_plan_brute) for every N'; capped mode (max_enumerated = 1: knapsack candidates +
    the certified bound) never beats the optimum, its upper bound never falls below it, and
    it finds the optimum in >= 90% of the N'."""
    from oracle import coracle
    from paper_2309_08125_b200 import planner as pl
    rng = random.Random(321)
    n_ex = n_cap = hit = 0
    for it in range(40):
        L, M = rng.randint(6, 14), rng.choice([1, 2, 4])
        N, f, n0 = rng.randint(8, 16), rng.randint(0, 2), rng.randint(1, 2)
        if N < (f + 1) * n0 or n0 > L:
            continue
        sizes = oracle_node_sizes(N, f, n0, L)
        prof = random_profile(700 + it, L, M, rng.choice(["uniform", "lognormal", "spiky"]))
        tpls = coracle.template_set(prof.fwd_ms, prof.bwd_ms, M, sizes[0], sizes[-1])[0]
        ts = _set_handle(pl, tpls, L, M, sizes)
        b = rng.choice([1, 2])
        B = b * rng.randint(max(f + 1, 4), 12)          # brute-force Eq.6: K = B/b <= 12
        lo = (f + 1) * n0
        ex = planner.instantiate_all(ts, 0, lo, N, f, B, b, max_enumerated=10 ** 7)
        ca = planner.instantiate_all(ts, 0, lo, N, f, B, b, max_enumerated=1)
        for e, c in zip(ex, ca):
            want = select_plan_brute(tpls, e["nodes"], f, B, b)
            if want is None:
                assert e["status"] != 0 and c["status"] != 0
                continue
            assert e["exact"] and e["throughput"] == pytest.approx(want[0], rel=1e-12) and e["counts"] == want[1]
            assert e["upper_bound"] == e["throughput"]
            n_ex += 1
            if c["exact"]:
                continue
            assert c["throughput"] <= want[0] * (1 + 1e-12)
            assert c["upper_bound"] >= want[0] * (1 - 1e-12)
            assert sum(x * (sizes[0] + i) for i, x in enumerate(c["counts"])) == e["nodes"]
            n_cap += 1
            hit += c["throughput"] >= want[0] * (1 - 1e-12)
    assert n_ex > 100 and n_cap > 60 and hit >= 0.9 * n_cap, (n_ex, n_cap, hit)


def test_load_profile_json(planner, tmp_path):
    from paper_2309_08125_b200._lib import OOB_E_INVALID, OOB_E_PARSE, OobError
    prof = random_profile(5, 6, 2, "lognormal")
    doc = {"gpus_per_node": 2, "microbatch_reference": 4, "layers": [
        {"name": f"l{l}", "state_bytes": 1000 + l, "activation_bytes_per_sample": 10,
         "fwd_ms": {str(d): float(prof.fwd_ms[l, d - 1]) for d in (1, 2)},
         "bwd_ms": {str(d): float(prof.bwd_ms[l, d - 1]) for d in (1, 2)}} for l in range(6)]}
    text = json.dumps(doc)          # floats are written with repr: exact binary64 round trip
    path = tmp_path / "p.json"
    path.write_text(text)
    p = planner.load_profile(str(path))
    assert (p.L, p.M) == (6, 2)
    # the parsed costs are the written ones, bit for bit (repr round-trips binary64), so the
    # loaded profile plans exactly like the array profile
    f, b, st = p.costs()
    assert np.array_equal(f, prof.fwd_ms) and np.array_equal(b, prof.bwd_ms)
    assert list(st) == [1000 + l for l in range(6)]
    q = planner.Profile.from_arrays(prof.fwd_ms, prof.bwd_ms)
    qf, qb, _ = q.costs()
    assert np.array_equal(qf, f) and np.array_equal(qb, b)
    bad = dict(doc)
    bad["layers"] = [dict(doc["layers"][0])]
    bad["layers"][0]["fwd_ms"] = {"1": 1.0}
    (tmp_path / "bad.json").write_text(json.dumps(bad))
    with pytest.raises(OobError) as e:
        planner.load_profile(str(tmp_path / "bad.json"))
    assert e.value.status == OOB_E_INVALID and "device-count" in str(e.value)
    (tmp_path / "empty.json").write_text(json.dumps({"gpus_per_node": 1, "layers": []}))
    with pytest.raises(OobError) as e:
        planner.load_profile(str(tmp_path / "empty.json"))
    assert "empty model" in str(e.value)
    (tmp_path / "broken.json").write_text("{\"gpus_per_node\": 1, \"layers\": [")
    with pytest.raises(OobError) as e:
        planner.load_profile(str(tmp_path / "broken.json"))
    assert e.value.status == OOB_E_PARSE
    neg = {"gpus_per_node": 1, "layers": [{"fwd_ms": {"1": -1.0}, "bwd_ms": {"1": 1.0}}]}
    (tmp_path / "neg.json").write_text(json.dumps(neg))
    with pytest.raises(OobError) as e:
        planner.load_profile(str(tmp_path / "neg.json"))
    assert e.value.status == OOB_E_INVALID


def test_profile_validation(planner):
    from paper_2309_08125_b200._lib import OobError
    with pytest.raises(OobError):
        planner.Profile.from_arrays(np.zeros((0, 1)), np.zeros((0, 1)))
    with pytest.raises(OobError):
        planner.Profile.from_arrays(np.array([[1.0], [0.0]]), np.ones((2, 1)))
    with pytest.raises(OobError):
        planner.Profile.from_arrays(np.array([[np.nan]]), np.ones((1, 1)))


def test_min_nodes_spec(planner):
    """SPEC S:82-84 (reading R5)."""
    GB = 10 ** 9
    for total, N, want in [(100 * GB, 8, 1), (300 * GB, 8, 3)]:
        p = planner.Profile.from_arrays(np.ones((4, 4)), np.ones((4, 4)),
                                        np.full(4, total // 4, dtype=np.int64))
        assert p.min_nodes(N, 40 * GB, 0.8) == want
    p = planner.Profile.from_arrays(np.ones((4, 4)), np.ones((4, 4)), np.full(4, 2500 * GB, dtype=np.int64))
    from paper_2309_08125_b200._lib import OobError
    with pytest.raises(OobError):
        p.min_nodes(4, 40 * GB, 0.8)


def test_exact_entry_points_fail_cleanly_without_device(planner):
    """oob_exact_run / oob_exact_workspace_bytes: NULL buffers are OOB_E_INVALID before any
    CUDA call; without a device the size query reports OOB_E_CUDA (no crash, no fallback)."""
    from paper_2309_08125_b200._lib import OOB_E_CUDA, OOB_E_INVALID, OobError
    with pytest.raises(OobError) as e:
        planner.exact_run(12, 4, 1, 4, 1, 0, 0, 0, 0, 0, 0)
    assert e.value.status == OOB_E_INVALID
    import torch
    if torch.cuda.is_available():
        assert planner.exact_workspace_bytes(12, 4, 1, 4, 1) > 0
        return
    with pytest.raises(OobError) as e:
        planner.exact_workspace_bytes(12, 4, 1, 4, 1)
    assert e.value.status == OOB_E_CUDA
