"""Dynamic reconfiguration (PAPER §5; Appendix B).

Oracle pins (oracle/reconfig.py, readings R21-R27 in DESIGN.md §10): the three cases of
Fig. 7, Appendix B's merge guarantee as a property over random failure
sequences, and the invariants §3-§5 state.  Parity: the C++ engine behind the C ABI
(oob_exec_*) reproduces the oracle's actions, pipelines, batch split, copy plan and sync
groups on the same scenarios (host code: runs on CPU).
"""
import random

import pytest

from oracle import reconfig as R
from oracle.dp import template_set
from oracle.instantiate import enumerate_sets_brute
from workloads import random_profile


def _templates(L, M, n_lo, n_hi, seed=11, kind="uniform"):
    p = random_profile(seed, L, M, kind)
    return template_set(p.fwd_ms, p.bwd_ms, M, range(n_lo, n_hi + 1))


def _check_invariants(st, alive):
    nodes = [n for p in st.pipes for n in p]
    assert sorted(nodes) == sorted(alive), "every survivor in exactly one pipeline"
    assert len(st.pipes) >= st.f + 1, "f+1 replicas"
    for p in st.pipes:
        assert st.n_lo <= len(p) <= st.n_hi, "pipeline instantiated from a template"
    assert sum(st.nb) * st.b == st.B and all(x >= 1 for x in st.nb), "batch conserved"
    for layer, g in enumerate(st.sync_groups()):
        assert sorted(p for p, _ in g) == list(range(len(st.pipes))), "one sync entry per pipeline"


# ------------------------------------------------------------------ Fig. 7
def test_fig7a_simple_reinstantiation():
    """'A node failure in a 4-node pipeline.  We have a 3-node pipeline template, thus a new
    pipeline with 3 nodes is instantiated, which replaces the existing one.'"""
    tpls = _templates(8, 1, 2, 5)                      # sizes 2..5 (N = 7, f = 1, n0 = 2)
    st = R.State.from_counts(tpls, [0, 1, 1, 0], list(range(7)), f=1, B=12, b=1)
    assert [len(p) for p in st.pipes] == [3, 4]
    actions, _ = st.apply_failures({4})
    assert actions == [("reinstantiate", 1, 3)]
    assert [len(p) for p in st.pipes] == [3, 3] and st.pipes[1] == [3, 5, 6]
    _check_invariants(st, [0, 1, 2, 3, 5, 6])


def test_fig7b_borrow_a_node():
    """'A node failure in a 2-node pipeline.  Since there is no template for one node, it
    gets another node from another pipeline to keep the 2-node pipeline.  Two affected
    pipelines reinstantiate or reconfigure themselves.'  (n0 = 2; the 4-node pipeline
    yields its last node and becomes a 3-node pipeline.)"""
    tpls = _templates(8, 1, 2, 6)
    st = R.State.from_counts(tpls, [1, 0, 1, 0, 0], list(range(6)), f=1, B=12, b=1)
    actions, _ = st.apply_failures({1})
    assert actions == [("borrow", 1, 0), ("reinstantiate", 0, 2)]
    assert st.pipes == [[0, 5], [2, 3, 4]]
    _check_invariants(st, [0, 2, 3, 4, 5])


def test_fig7c_merge_pipelines():
    """'A node failure in a 2-node pipeline.  Because it cannot borrow a node from any other
    pipeline, it is merged with another pipeline.'  All pipelines at n0 = 2: the broken one
    (1 node) merges with the smallest other into 2 n0 - k = 3 nodes (Appendix B)."""
    tpls = _templates(8, 1, 2, 4)                      # N = 6, f = 1: sizes 2..4
    st = R.State.from_counts(tpls, [3, 0, 0], list(range(6)), f=1, B=12, b=1)
    actions, _ = st.apply_failures({3})
    assert actions == [("merge", 1, 0), ("reinstantiate", 1, 3)]
    assert st.pipes == [[2, 0, 1], [4, 5]]
    _check_invariants(st, [0, 1, 2, 4, 5])


def test_exit_below_f_plus_one_replicas():
    """P:298-300 / §5 'until we have fewer than (f+1) n0 nodes'."""
    tpls = _templates(8, 1, 2, 4)
    st = R.State.from_counts(tpls, [2, 0, 0], list(range(4)), f=1, B=8, b=1)
    with pytest.raises(R.Exit):
        st.apply_failures({0})


def test_copy_plan_and_unrecoverable():
    """Missing layers are copied from surviving owners; a layer whose every
    copy failed cannot be recovered."""
    tpls = _templates(8, 1, 2, 4)
    st = R.State.from_counts(tpls, [3, 0, 0], list(range(6)), f=1, B=12, b=1, layer_bytes=[10] * 8)
    before = st.owned()
    _, copies = st.apply_failures({3})
    after = st.owned()
    for (layer, donor, recv, nbytes) in copies:
        assert layer in before[donor] and donor != 3 and layer in after[recv] and nbytes == 10
    needed = {(n, l) for n, ls in after.items() for l in ls if l not in before.get(n, set())}
    assert needed == {(r, l) for (l, _, r, _) in copies}
    st2 = R.State.from_counts(tpls, [3, 0, 0], list(range(6)), f=1, B=12, b=1)
    owners0 = [n for n, ls in st2.owned().items() if 0 in ls]
    with pytest.raises((R.Unrecoverable, R.Exit)):
        st2.apply_failures(set(owners0))


def _random_scenario(rng, seed):
    M = rng.choice([1, 2])
    n0 = rng.choice([1, 2, 3])
    f = rng.randint(0, 2)
    L = rng.randint(max(2 * n0 - 1, n0 + 1), 9)
    N = (f + 1) * n0 + rng.randint(0, 3 * n0 + 2)
    n_hi = min(N - f * n0, L)
    tpls = _templates(L, M, n0, n_hi, seed=seed, kind=rng.choice(["uniform", "integer", "spiky"]))
    sets = enumerate_sets_brute([t["nodes"] for t in tpls], N, f)
    counts = rng.choice(sets)
    b = rng.choice([1, 2])
    B = b * (N + rng.randint(0, 3))
    return tpls, counts, N, f, B, b


def test_appendix_b_merge_guarantee_property():
    """Appendix B: whenever >= (f+1) n0 nodes survive, reinstantiation (with borrowing and
    merging) always finds a template and keeps >= f+1 pipelines — random failure sequences
    over random configurations (L >= 2 n0 - 1, so the L cap keeps sizes up to 2 n0 - 1)."""
    rng = random.Random(5)
    steps = 0
    for case in range(300):
        tpls, counts, N, f, B, b = _random_scenario(rng, 900 + case)
        st = R.State.from_counts(tpls, counts, list(range(N)), f=f, B=B, b=b)
        alive = list(range(N))
        while True:
            k = rng.choice([1, 1, 1, 2])
            failed = set(rng.sample(alive, min(k, len(alive))))
            owners = st.owned()
            lost_layer = any(all(n in failed for n, ls in owners.items() if layer in ls) for layer in range(st.L))
            try:
                st.apply_failures(failed)
            except R.Exit:
                assert len(alive) - len(failed) < (f + 1) * st.n_lo
                break
            except R.Unrecoverable:
                # only when every copy of some layer failed at once, which needs
                # more simultaneous failures than the f the replicas guarantee
                assert lost_layer and len(failed) > f
                break
            assert not lost_layer
            alive = [n for n in alive if n not in failed]
            _check_invariants(st, alive)
            steps += 1
    assert steps > 500


# ------------------------------------------------------------------ C++ engine (C ABI) vs oracle
def _cpp_set(tpls, L, M):
    import ctypes
    from paper_2309_08125_b200 import planner
    from tests.helpers import pack_templates
    n_lo, n_hi = tpls[0]["nodes"], tpls[-1]["nodes"]
    buf, info = pack_templates([tpls], L, M, n_lo, n_hi)
    dinfo = planner.OobDpInfo(**info)
    h = ctypes.c_void_p()
    planner.check(planner.lib.oob_template_set_from_packed(buf.ctypes.data, ctypes.byref(dinfo), ctypes.byref(h)))
    return planner.TemplateSet(h)


def _same_state(ex, st):
    got = ex.pipelines()
    assert [p for p, _ in got] == st.pipes
    from oracle.instantiate import variance_objective
    T = [st.tpl[len(p)]["tstar"] for p in st.pipes]
    nb = [n for _, n in got]
    assert sum(nb) == sum(st.nb) and min(nb) >= 1
    assert variance_objective(nb, T) == pytest.approx(variance_objective(st.nb, T), rel=1e-9, abs=1e-9)
    for layer, g in enumerate(st.sync_groups()):
        assert ex.sync_group(layer) == g


def test_engine_matches_oracle_random_failures():
    """oob_exec_* (C++) == oracle/reconfig.py: actions, pipelines (node order), Eq.6 objective,
    copy plans and sync groups after every failure, on random scenarios and sequences."""
    from paper_2309_08125_b200 import planner
    from paper_2309_08125_b200._lib import OOB_E_INFEASIBLE, OobError
    rng = random.Random(77)
    compared = 0
    for case in range(150):
        tpls, counts, N, f, B, b = _random_scenario(rng, 3000 + case)
        L, M = tpls[0]["stages"][-1][1], None
        M = sum(s[2] for s in tpls[0]["stages"]) // tpls[0]["nodes"]
        lb = [rng.randint(1, 100) for _ in range(L)]
        ids = rng.sample(range(10 * N), N)
        st = R.State.from_counts(tpls, counts, ids, f=f, B=B, b=b, layer_bytes=lb)
        ts = _cpp_set(tpls, L, M)
        ex = planner.ExecState(ts, 0, f, B, b, counts, ids, lb)
        _same_state(ex, st)
        alive = list(ids)
        while True:
            failed = set(rng.sample(alive, min(rng.choice([1, 1, 2]), len(alive))))
            try:
                want = st.apply_failures(failed)
            except (R.Exit, R.Unrecoverable):
                with pytest.raises(OobError) as e:
                    ex.fail(failed)
                assert e.value.status == OOB_E_INFEASIBLE
                break
            got = ex.fail(failed)
            assert got == (want[0], want[1])
            alive = [n for n in alive if n not in failed]
            _same_state(ex, st)
            compared += 1
    assert compared > 200


def test_masked_sets_instantiate_and_exec_rules():
    """A template set with an infeasible size (stage masks, reading R31): oob_instantiate
    never uses it (brute force over the feasible sizes agrees), and the reconfiguration
    state refuses the set (reinstantiation needs every size n_lo..n_hi)."""
    from paper_2309_08125_b200 import planner
    from paper_2309_08125_b200._lib import OOB_E_INVALID, OobError
    from oracle.instantiate import select_plan_brute
    tpls = _templates(8, 1, 2, 5)
    holed = [tpls[0], None, tpls[2], tpls[3]]            # size 3 infeasible
    ts = _cpp_set(holed, 8, 1)
    assert ts.templates(0)[1] is None
    from oracle.instantiate import distribute_for_plan, enumerate_sets_brute
    feas = [t for t in holed if t is not None]
    for Np in range(4, 12):
        best = None
        for X in enumerate_sets_brute([t["nodes"] for t in feas], Np, 1):
            pipes = [t for t, c in zip(feas, X) for _ in range(c)]
            try:
                _, it = distribute_for_plan(pipes, 12, 1)
            except ValueError:
                continue
            key = (-12 / it, sum(X), X)
            best = key if best is None or key < best else best
        if best is None:                                  # only size-3 pipelines would fit
            with pytest.raises(OobError):
                planner.instantiate(ts, 0, Np, 1, 12, 1)
            continue
        got = planner.instantiate(ts, 0, Np, 1, 12, 1)
        assert got["counts"][1] == 0
        assert got["throughput"] == pytest.approx(-best[0], rel=1e-12)
    with pytest.raises(OobError) as e:
        planner.ExecState(ts, 0, 1, 12, 1, [1, 0, 0, 1], list(range(7)))
    assert e.value.status == OOB_E_INVALID
