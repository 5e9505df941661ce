"""ORACLE (test infrastructure only) — pipeline-template generation, §4.1.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import this module.  It shares no code with `paper_2309_08125_b200/` (the CUDA
path) and never imports it.

This is the paper's divide-and-conquer GPU-stage mapping written out literally in plain
Python, in binary64, memoized on the key (S', u, v, alloc) as P:470-474 prescribes:

* Eq.4 (`eq:dc_init`) base case: one stage on d GPUs of one node,
  T1 = F+B = sum_{k=u}^{v-1}(F_{l_k,d}+B_{l_k,d}), T2 = 2(F+B), T3 = F+B; a stage whose
  GPUs span nodes is infinite.
* Eq.1-3 (`eq:T1dc` P:395-400, `eq:T2dc` P:402-407, `eq:T3dc` P:409-420) combine two
  sub-problems split at layer k (second half starts at k: DESIGN reading R1), device
  split m and stage split s; k* is the slowest stage, N_b = 4S'.
* "We iterate over s, k, and m globally, and find a (s,k,m) that minimizes
  T1+T2+T3" — first strictly-smaller total in (k, m, s) order (reading R6).
* Choice of S: S in n..min(L, n*M) (reading R3), smaller S wins ties (R8).

Arithmetic contract: every + and * below is one IEEE
binary64 operation in the order written; Python floats are binary64 with no FMA.

Parity: pinned (tests/test_oracle_dp.py): SPEC worked examples, Eq.4 = Eq.2
at S'=1, brute force over all mappings (equality for S<=2, lower bound otherwise, the
counterexample c=[1,9,1,3,9,2]), closed-form consistency of returned partitions,
unmemoized recursion, validity <=> finiteness.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass

INF = float("inf")


# ---------------------------------------------------------------- device allocations
# Two-level device allocation (DESIGN reading R2): ("I", r) = r GPUs
# inside one node (1 <= r <= M-1); ("W", q) = q whole nodes (W(1) = all M GPUs of a node).

def alloc_gpus(a, M):
    kind, n = a
    return n if kind == "I" else n * M


def device_splits(a, M):
    """D(a): the ways to divide a device allocation into two, in order."""
    kind, n = a
    if kind == "W" and n >= 2:
        return [(("W", j), ("W", n - j)) for j in range(1, n)]
    if kind == "W" and n == 1:
        return [(("I", m), ("I", M - m)) for m in range(1, M)]
    return [(("I", m), ("I", n - m)) for m in range(1, n)]


# ---------------------------------------------------------------- cell values
@dataclass(frozen=True)
class Cell:
    """Memo value of T(S', u, v, a): the T1/T3 terms, slowest-stage time t* and index k*
    (0-based), plus the argmin split (k, m-index, s) for the backtrack (None at S'=1)."""
    T1: float
    T3: float
    tstar: float
    kstar: int
    split: tuple | None

    def T2(self, Sp: int) -> float:
        Nb = 4 * Sp                                   # N_b = 4S'
        return float(Nb - Sp + self.kstar - 1) * self.tstar   # Eq.2

    def total(self, Sp: int) -> float:
        return (self.T1 + self.T2(Sp)) + self.T3


def stage_time(fwd, bwd, u, v, d):
    """F_{s,d} + B_{s,d} = sum_{k=u}^{v-1} (F_{l_k,d} + B_{l_k,d})  (Eq.4), summed
    left to right starting from 0.0 (reading R12)."""
    t = 0.0
    for k in range(u, v):
        t = t + (fwd[k][d - 1] + bwd[k][d - 1])
    return t


def combine(Lc: Cell, Rc: Cell, Sp: int, s: int):
    """Eq.1-3 for one split: left sub-problem has s stages, right S'-s."""
    T1 = Lc.T1 + Rc.T1                                # Eq.1
    if Lc.tstar >= Rc.tstar:                          # k* from the first half (R7: left on ties)
        kstar = Lc.kstar
        tstar = Lc.tstar
        T3 = Lc.T3 + Rc.T1                            # Eq.3, case k* == k1*
    else:
        kstar = s + Rc.kstar                          # global index of the second half's k2*
        tstar = Rc.tstar
        T3 = Rc.T3                                    # Eq.3, else-branch
    Nb = 4 * Sp
    T2 = float(Nb - Sp + kstar - 1) * tstar           # Eq.2
    total = (T1 + T2) + T3
    return total, T1, T3, tstar, kstar


def stage_allowed(u, v, d, pow2_tp=False, stage_bytes=None, mem_cap=None):
    """Variants the paper is silent on (DESIGN reading R31): a stage of
    layers [u, v) on d GPUs of one node is allowed only if d is a power of two (pow2_tp:
    tensor-parallel degrees 1, 2, 4, 8, ...) and its memory fits: the stage's per-layer
    bytes (model states + activations) split over its d GPUs (in-stage sharding),
    sum_{l=u}^{v-1} stage_bytes[l] / d <= mem_cap — summed left to right in binary64, the
    division last (the paper models memory only through n0: reading R14 is the
    default, no mask)."""
    if pow2_tp and (d & (d - 1)) != 0:
        return False
    if stage_bytes is not None and mem_cap is not None:
        tot = 0.0
        for k in range(u, v):
            tot = tot + float(stage_bytes[k])
        if tot / float(d) > mem_cap:
            return False
    return True


class TemplateDP:
    """Memoized T(S', u, v, a) over one profile (fwd/bwd: [L][M] nested sequences).
    Optional stage masks (reading R31): pow2_tp, stage_bytes + mem_cap — a masked-out stage
    is infinite like one spanning nodes, and a sub-problem without any allowed
    division is infinite (None)."""

    def __init__(self, fwd, bwd, M: int, memo: bool = True, pow2_tp: bool = False, stage_bytes=None,
                 mem_cap=None):
        self.fwd = [list(map(float, row)) for row in fwd]
        self.bwd = [list(map(float, row)) for row in bwd]
        self.L = len(self.fwd)
        self.M = M
        self.memo = {} if memo else None
        self.calls = 0
        self.pow2_tp = pow2_tp
        self.stage_bytes = None if stage_bytes is None else [float(x) for x in stage_bytes]
        self.mem_cap = mem_cap

    def T(self, Sp: int, u: int, v: int, a):
        key = (Sp, u, v, a)
        if self.memo is not None and key in self.memo:
            return self.memo[key]
        self.calls += 1
        M = self.M
        if Sp == 1:
            kind, n = a
            if kind == "W" and n >= 2:
                res = None                            # GPUs across nodes -> infinite
            else:
                d = M if kind == "W" else n
                if not stage_allowed(u, v, d, self.pow2_tp, self.stage_bytes, self.mem_cap):
                    res = None                        # masked stage (reading R31)
                else:
                    t = stage_time(self.fwd, self.bwd, u, v, d)
                    res = Cell(t, t, t, 0, None)      # Eq.4
        else:
            best = None
            best_total = INF
            splits = device_splits(a, M)
            for k in range(u + 1, v):                 # layer split point
                for mi, (a1, a2) in enumerate(splits):   # device split
                    for s in range(1, Sp):            # stages in the first half
                        Lc = self.T(s, u, k, a1)
                        if Lc is None:
                            continue
                        Rc = self.T(Sp - s, k, v, a2)
                        if Rc is None:
                            continue
                        total, T1, T3, tstar, kstar = combine(Lc, Rc, Sp, s)
                        if total < best_total:
                            best_total = total
                            best = Cell(T1, T3, tstar, kstar, (k, mi, s))
            res = best                                # None = no feasible division (infinite)
        if self.memo is not None:
            self.memo[key] = res
        return res

    # ------------------------------------------------------------ templates
    def template(self, n: int):
        """Pipeline template for n nodes: argmin over S in n..min(L, n*M);
        None when every S is infinite (only possible with stage masks)."""
        if n > self.L:
            raise ValueError("too few layers for node count")
        best = None
        for S in range(n, min(self.L, n * self.M) + 1):
            c = self.T(S, 0, self.L, ("W", n))
            if c is None:
                continue
            tot = c.total(S)
            if best is None or tot < best[0]:
                best = (tot, S, c)
        if best is None:
            if self.pow2_tp or self.mem_cap is not None:
                return None
            raise ValueError("no feasible template")
        tot, S, c = best
        stages = []
        self._backtrack(S, 0, self.L, ("W", n), 0, 0, stages)
        return {
            "nodes": n, "S": S, "stages": stages,
            "T1": c.T1, "T2": c.T2(S), "T3": c.T3, "kstar": c.kstar, "tstar": c.tstar,
            "total": tot,
        }

    def _backtrack(self, Sp, u, v, a, node, gpu_off, out):
        c = self.T(Sp, u, v, a)
        kind, n = a
        if Sp == 1:
            d = self.M if kind == "W" else n
            out.append((u, v, d, node, gpu_off))
            return
        k, mi, s = c.split
        a1, a2 = device_splits(a, self.M)[mi]
        if kind == "W" and n >= 2:
            # whole-node split: the left half gets the lower node indices
            self._backtrack(s, u, k, a1, node, 0, out)
            self._backtrack(Sp - s, k, v, a2, node + a1[1], 0, out)
        else:
            # GPUs inside one node: the left half gets the lower GPU offsets
            self._backtrack(s, u, k, a1, node, gpu_off, out)
            self._backtrack(Sp - s, k, v, a2, node, gpu_off + a1[1], out)


def node_sizes(N: int, f: int, n0: int, L: int | None = None):
    """Node specification: consecutive sizes n0 .. N - f*n0, capped at L
    (reading R4).  Raises when N < (f+1)*n0 ("cannot maintain f+1 replicas")."""
    if N < (f + 1) * n0:
        raise ValueError("cannot maintain f+1 replicas")
    hi = N - f * n0
    if L is not None:
        hi = min(hi, L)
    return list(range(n0, hi + 1))


def template_set(fwd, bwd, M, sizes, **masks):
    """All templates of a node specification from one shared memo; `masks`:
    TemplateDP's stage masks (reading R31), an infeasible size gives None."""
    sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
    dp = TemplateDP(fwd, bwd, M, **masks)
    # running the largest template first fills the caches for all others
    out = {}
    for n in sorted(sizes, reverse=True):
        out[n] = dp.template(n)
    return [out[n] for n in sorted(sizes)]


def closed_form(stage_times):
    """Closed form of the 1F1B objective for a fixed partition with per-stage times t_i
    (P:381-386): T1 = sum t_i; k* = first index of the max; T2 =
    (4S - S + k* - 1) t_{k*}; T3 = sum_{i >= k*} t_i.  Returns (total, T1, T2, T3, k*)."""
    S = len(stage_times)
    T1 = 0.0
    for t in stage_times:
        T1 = T1 + t
    kstar = 0
    for i in range(1, S):
        if stage_times[i] > stage_times[kstar]:
            kstar = i
    T2 = float(4 * S - S + kstar - 1) * stage_times[kstar]
    T3 = 0.0
    for i in range(kstar, S):
        T3 = T3 + stage_times[i]
    return (T1 + T2) + T3, T1, T2, T3, kstar
