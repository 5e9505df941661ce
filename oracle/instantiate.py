"""ORACLE (test infrastructure only) — pipeline instantiation and batch distribution,
PAPER.md §4.2.  Plain definitions written out; exponential where the
definition is (small inputs only).

* `enumerate_sets`: Eq.5 (`eq:instantiation_dp`) literally —
  X(p', N') = X(p'-1, N') ++ theta(X(p', N' - n_{p'}), p'), then the Requirement-2 filter
  sum x >= f+1.
* `enumerate_sets_brute`: nested loops over every x_i <= N'/n_i (pin for Eq.5).
* `distribute_batch_brute`: Eq.6 (`eq:nonlinear_optimization`) by enumerating
  every integer assignment N_{b,i} >= 1 with sum N_{b,i} b = B (reading R18); T_i is the
  pipeline's per-microbatch steady cost t* (reading R19).
* `recommend_batch`: smallest distributable B' >= B.
* `iteration_ms`: T1 + max(0, N_b - S + k* - 1) t* + T3 (Eq.2 with the real N_b; SPEC S:131;
  reading R30 for N_b below the pipeline fill).
* `select_plan_brute`: max-throughput plan over all feasible sets.
* `distribute_for_plan`: Eq.6 for a plan's pipelines; Eq.6 can have several minimizers
  (pipelines with equal T_i), and the distributor exists to balance the pipelines'
  execution, so among the minimizers the one with the smallest plan iteration
  time max_i iteration_ms(N_b,i) is taken, remaining ties giving the larger count to the
  lower pipeline index (reading R29).
"""
from __future__ import annotations

from .brute import compositions


def enumerate_sets(sizes, Nprime: int, f: int):
    """Eq.5 with list concatenation; returns the feasible X (tuples), filtered by f."""
    p = len(sizes)
    memo = {}

    def X(pp: int, n: int):
        # pp = index of the last template allowed (-1: none)
        if n < 0:
            return []
        if pp < 0:
            return [tuple([0] * p)] if n == 0 else []
        key = (pp, n)
        if key in memo:
            return memo[key]
        keep = X(pp - 1, n)                          # X(p'-1, N')
        add = []
        for x in X(pp, n - sizes[pp]):               # theta(X(p', N' - n_p'), p')
            y = list(x)
            y[pp] += 1
            add.append(tuple(y))
        memo[key] = keep + add                       # concatenation
        return memo[key]

    return [x for x in X(p - 1, Nprime) if sum(x) >= f + 1]


def enumerate_sets_brute(sizes, Nprime: int, f: int):
    out = []

    def rec(i, rem, cur):
        if i == len(sizes):
            if rem == 0 and sum(cur) >= f + 1:
                out.append(tuple(cur))
            return
        for x in range(rem // sizes[i] + 1):
            rec(i + 1, rem - x * sizes[i], cur + [x])
    rec(0, Nprime, [])
    return out


def variance_objective(nb, T):
    """sum_i (N_{b,i} T_i - mean)^2 (Eq.6 objective)."""
    y = [n * t for n, t in zip(nb, T)]
    mean = sum(y) / len(y)
    return sum((v - mean) ** 2 for v in y)


def distribute_batch_brute(T, B: int, b: int):
    """Exact Eq.6 by enumeration; returns (nb tuple, objective) or raises ValueError."""
    x = len(T)
    if B % b != 0 or B // b < x:
        raise ValueError("infeasible distribution")
    K = B // b
    best = None
    for nb in compositions(K, x):
        obj = variance_objective(nb, T)
        if best is None or obj < best[1]:
            best = (nb, obj)
    return best


def distribute_for_plan(pipes, B: int, b: int):
    """Reading R29: (nb, iteration time) of the Eq.6 minimizer with the smallest plan
    iteration time (pipes: template dicts); raises ValueError if not distributable."""
    x = len(pipes)
    if B % b != 0 or B // b < x:
        raise ValueError("infeasible distribution")
    T = [t["tstar"] for t in pipes]
    cands = [(variance_objective(nb, T), nb) for nb in compositions(B // b, x)]
    best_obj = min(o for o, _ in cands)
    tol = 1e-12 * (B // b * max(T)) ** 2        # rounding of a sum of squares of size (K T)^2
    best = None
    for o, nb in cands:
        if o > best_obj + tol:
            continue
        it = max(iteration_ms(t, n) for t, n in zip(pipes, nb))
        key = (it, tuple(-n for n in nb))
        if best is None or key < best[0]:
            best = (key, nb, it)
    return best[1], best[2]


def recommend_batch(x: int, b: int, B: int) -> int:
    Bp = max(B, x * b)
    if Bp % b:
        Bp += b - Bp % b
    return Bp


def iteration_ms(tpl, Nb: int) -> float:
    """Eq.2 with the real N_b; with fewer microbatches than the pipeline's fill (N_b <
    S - k* + 1) the steady phase T2 is empty, not negative (reading R30)."""
    S = tpl["S"]
    return (tpl["T1"] + float(max(0, Nb - S + tpl["kstar"] - 1)) * tpl["tstar"]) + tpl["T3"]


def select_plan_brute(templates, Nprime: int, f: int, B: int, b: int):
    """Best plan over every Eq.5 set: (throughput, counts, nb) — highest throughput, then
    fewer pipelines, then lexicographically smallest counts."""
    sizes = [t["nodes"] for t in templates]
    best = None
    for X in enumerate_sets_brute(sizes, Nprime, f):
        pipes = []
        for i, cnt in enumerate(X):
            pipes += [templates[i]] * cnt
        try:
            nb, it = distribute_for_plan(pipes, B, b)
        except ValueError:
            continue
        thr = B / it
        key = (-thr, sum(X), X)
        if best is None or key < best[0]:
            best = (key, thr, X, nb)
    if best is None:
        return None
    return best[1], best[2], best[3]


def coverage_ok(sizes, lo: int, hi: int, f: int) -> bool:
    """Every N' in [lo, hi] is a combination of sizes with >= f+1 pipelines (App. A),
    by exhaustive reachability: most[n] = max number of pipelines summing to n."""
    NEG = -1
    most = [NEG] * (hi + 1)
    most[0] = 0
    for n in range(1, hi + 1):
        for s in sizes:
            if s <= n and most[n - s] != NEG:
                most[n] = max(most[n], most[n - s] + 1)
    return all(most[Np] >= f + 1 for Np in range(lo, hi + 1))
