"""The W kernel's split filter ("Exact filter") checked against the oracle.

k_wave_w skips a split unless a binary32 lower bound of its total, built from per-cell
shadows rounded toward -inf, can reach the output's current minimum.  Its exactness rests
on one claim: for EVERY split (X left, Y right, s / S_Y stages),

    lb = (rd32(X.t*) >= rd32(Y.t*)) ? A_X + 3 S_Y X.t* + 2 Y.T1 : A_Y + 4 s Y.t* + X.T1
    (A = T1 + T3 + C1 t*, C1 = 3S'-1+k*, every term rounded down)
    lb <= total * (1 + 2^-43)       (total = the oracle's binary64 Eq.1-3 value).

The kernel's filter threshold is float_ru(m (1 + 2^-40)), so a split with total <= m is
never dropped.  This test recomputes the bound here from the DESIGN formulas (no CUDA
code), with the directed roundings emulated exactly (fractions), for every split of every
cell of small random instances of all test kinds, and checks the claim and that the bound
is tight (it is the filter's whole point).  A dropped term or a swapped branch in the
derivation makes lb exceed the total by far more than 2^-43 on some split.
"""
import random
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import dp
from workloads import random_profile


def _rd32(x: F) -> float:
    """Largest binary32 value <= x (x exact, non-negative)."""
    d = float(x)                                  # nearest binary64
    if F(d) > x:
        d = float(np.nextafter(d, -np.inf))
    f = np.float32(d)
    if F(float(f)) > F(d):
        f = np.nextafter(f, np.float32(-np.inf))
    return float(f)


def _shadow(c: dp.Cell, Sp: int):
    C1 = 3 * Sp - 1 + c.kstar
    A = _rd32(F(c.T1) + F(c.T3) + F(C1) * F(c.tstar))
    t1 = _rd32(F(c.T1))
    return A, t1, _rd32(F(c.tstar)), _rd32(2 * F(t1))


def _lb(X, s, Y, SY):
    AX, X1, Xts, _ = _shadow(X, s)
    AY, _, Yts, Y2 = _shadow(Y, SY)
    # each kernel operation rounds toward -inf: fma(a, b, c) then + d
    tl = _rd32(F(_rd32(F(3 * SY) * F(Xts) + F(AX))) + F(Y2))
    tr = _rd32(F(4 * s) * F(Yts) + F(_rd32(F(AY) + F(X1))))
    return tl if Xts >= Yts else tr


def _allocs(L, M):
    return [("I", r) for r in range(1, M)] + [("W", q) for q in range(1, L + 1)]


KINDS = [("lognormal", "real"), ("lognormal", "dyadic"), ("uniform", "real"), ("integer", "real"),
         ("spiky", "real"), ("constant", "real")]


@pytest.mark.parametrize("case", range(len(KINDS)), ids=[f"{k}-{m}" for k, m in KINDS])
def test_filter_bound_every_split(case):
    kind, mode = KINDS[case]
    rng = random.Random(77 + case)
    worst = F(0)
    checked = 0
    for trial in range(6):
        L = rng.randint(5, 8)
        M = rng.choice([1, 2, 4])
        p = random_profile(900 + 10 * case + trial, L, M, kind=kind, mode=mode)
        T = dp.TemplateDP(p.fwd_ms, p.bwd_ms, M)
        for Sp in range(2, L + 1):
            for u in range(L):
                for v in range(u + 2, L + 1):
                    for a in _allocs(L, M):
                        for k in range(u + 1, v):
                            for a1, a2 in dp.device_splits(a, M):
                                for s in range(1, Sp):
                                    X, Y = T.T(s, u, k, a1), T.T(Sp - s, k, v, a2)
                                    if X is None or Y is None:
                                        continue
                                    total = dp.combine(X, Y, Sp, s)[0]
                                    r = F(_lb(X, s, Y, Sp - s)) / F(total)
                                    assert r <= 1 + F(1, 2 ** 43), (kind, mode, L, M, Sp, u, v, a, k, s, float(r))
                                    worst = max(worst, r)
                                    checked += 1
    assert checked > 1000
    assert worst > 1 - F(1, 2 ** 20)              # the bound is tight (within binary32 rounding)
