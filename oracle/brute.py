"""ORACLE (test infrastructure only) — brute force over every GPU-stage mapping.

Used to pin `oracle/dp.py` to something other than itself.  It enumerates, for a template
of n nodes x M GPUs over L layers:
  * every stage count S in n..min(L, n*M),
  * every partition of the L layers into S contiguous non-empty stages,
  * every assignment of the S stages (in pipeline order) to the n nodes as contiguous
    non-empty runs, and every composition of each node's M GPUs over its stages
    (all GPUs used; no stage spans nodes),
and scores each mapping with the closed form of the 1F1B objective (`dp.closed_form`,
P:381-386, N_b = 4S).  Exponential: tiny inputs only.
"""
from __future__ import annotations

from itertools import combinations

from .dp import INF, closed_form, stage_time


def compositions(total: int, parts: int):
    """All ordered tuples of `parts` positive integers summing to `total`."""
    if parts <= 0 or parts > total:
        return
    for cuts in combinations(range(1, total), parts - 1):
        prev = 0
        out = []
        for c in cuts:
            out.append(c - prev)
            prev = c
        out.append(total - prev)
        yield tuple(out)


def _gpu_assignments(S: int, n: int, M: int):
    """Per-stage GPU counts for S stages on n nodes: (node_of_stage, gpus_of_stage)."""
    for runs in compositions(S, n):
        if any(r > M for r in runs):
            continue
        per_node = [list(compositions(M, r)) for r in runs]

        def rec(i):
            if i == len(runs):
                yield []
                return
            for comp in per_node[i]:
                for rest in rec(i + 1):
                    yield [(i, g) for g in comp] + rest
        yield from rec(0)


def brute_force(fwd, bwd, M: int, n: int, S_only: int | None = None, allowed=None):
    """Minimum closed-form total over all mappings; returns (best_total, [argmin mappings]).
    A mapping is a tuple of stages (u, v, d, node).  S_only restricts the stage count;
    allowed(u, v, d) (optional) excludes mappings with a disallowed stage (stage masks)."""
    L = len(fwd)
    best = INF
    arg = []
    for S in range(n, min(L, n * M) + 1):
        if S_only is not None and S != S_only:
            continue
        assigns = list(_gpu_assignments(S, n, M))
        for layers in compositions(L, S):
            bounds = []
            u = 0
            for c in layers:
                bounds.append((u, u + c))
                u += c
            for asg in assigns:
                if allowed is not None and not all(allowed(b[0], b[1], g) for b, (_, g) in zip(bounds, asg)):
                    continue
                times = [float(stage_time(fwd, bwd, b[0], b[1], g)) for b, (_, g) in zip(bounds, asg)]
                tot = closed_form(times)[0]
                mapping = tuple((b[0], b[1], g, node) for b, (node, g) in zip(bounds, asg))
                if tot < best:
                    best = tot
                    arg = [mapping]
                elif tot == best:
                    arg.append(mapping)
    return best, arg
