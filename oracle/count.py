"""ORACLE (test infrastructure only) — size of the template DP's cell universe and its
feasible split evaluations, counted from the definitions (DESIGN §2 R2-R4).

Only `tests/` and `bench.py`'s `--impl reference` / `cpu_baseline` legs use this: the
reference arm reports cells/s of the oracle without loading the product library.

Definitions (PAPER §4.1.2, with readings R2/R3):
* allocations I(r) = r GPUs inside one node (1 <= r <= M-1) and W(q) = q whole nodes; at
  wavefront length l only W(q) with q <= Q_l exist (Q_L = n_hi for the full range, n_hi - 1
  otherwise: a sub-range never holds all n_hi nodes' worth of a template);
* a cell (S', u, u+l, a) is valid iff lo(a) <= S' <= min(l, gpus(a)), lo(W(q)) = q,
  lo(I(r)) = 1 (no stage spans nodes P:450-452, pigeonhole P:459, >= 1 layer per stage P:390);
* a feasible split of a cell with S' >= 2 is (k, (a1, a2) in D(a), s) with both children
  valid; for children a1 on l1 layers and a2 on l2 layers the (s, S' - s) pairs range over
  the product of the two children's valid S'-intervals, each pair landing on exactly one
  parent S' (so the per-range split count is a sum of interval-length products, and the
  W x W part is a discrete convolution over the node counts).
Pinned by brute-force enumeration on small shapes (tests/helpers.count_universe) and by the
numbers SURVEY §8 records for cfg1-cfg5 (tests/test_oracle_count.py).
"""
from __future__ import annotations

import numpy as np


def _len(lo: int, g: int, l: int) -> int:
    hi = min(l, g)
    return hi - lo + 1 if hi >= lo else 0


def universe(L: int, M: int, n_hi: int) -> tuple[int, int]:
    """(cells, feasible splits) of one profile's template DP for sizes up to n_hi."""
    def Q(l):
        return n_hi if l == L else max(1, n_hi - 1)

    # lenW[l][q] = valid S' of W(q) on l layers (0 when q > Q_l); lenI[l][r] likewise for I(r)
    lenW = np.zeros((L + 1, n_hi + 1), dtype=np.int64)
    lenI = np.zeros((L + 1, M + 1), dtype=np.int64)
    for l in range(1, L + 1):
        for q in range(1, Q(l) + 1):
            lenW[l, q] = _len(q, q * M, l)
        for r in range(1, M):
            lenI[l, r] = _len(1, r, l)
    cells = 0
    splits = 0
    for l in range(1, L + 1):
        nr = L - l + 1
        cells += nr * (int(lenW[l].sum()) + int(lenI[l].sum()))
        if l < 2:
            continue
        per = 0
        for l1 in range(1, l):
            l2 = l - l1
            # W(q >= 2) -> (W(j), W(q - j)), parents q <= Q_l
            conv = np.convolve(lenW[l1], lenW[l2])          # conv[q] = sum_j lenW[l1][j] lenW[l2][q-j]
            per += int(conv[2:Q(l) + 1].sum())
            # W(1) -> (I(m), I(M - m)), m = 1..M-1
            for m in range(1, M):
                per += int(lenI[l1, m] * lenI[l2, M - m])
            # I(r) -> (I(m), I(r - m)), r = 2..M-1
            for r in range(2, M):
                for m in range(1, r):
                    per += int(lenI[l1, m] * lenI[l2, r - m])
        splits += nr * per
    return cells, splits
