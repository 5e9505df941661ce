// DP cell universe, HBM layout and work counts ("Work").
//
// The universe follows PAPER §4.1.2: a cell is a sub-problem T(S', u, v, a)
// with the two-level device allocation a (reading R2); it is finite iff
// lo(a) <= S' <= min(v-u, gpus(a)) (no stage across nodes P:450-452, pigeonhole P:459,
// at least one layer and one GPU per stage P:390), so only those cells are stored.
#include <algorithm>

#include "oob_internal.h"

namespace oob {

namespace {
// number of S' values of allocation with lower bound lo and GPU count g at length l
inline int64_t len_cells(int lo, int g, int l) {
    int hi = std::min(l, g);
    return hi >= lo ? (int64_t)(hi - lo + 1) : 0;
}
}  // namespace

bool build_geometry(int L, int M, int n_lo, int n_hi, Geometry &g) {
    if (L < 1 || L > 1023 || M < 1 || M > 64 || n_lo < 1 || n_hi < n_lo || n_hi > L) {
        set_error("build_geometry: need 1 <= L <= 1023, 1 <= M <= 64, 1 <= n_lo <= n_hi <= L");
        return false;
    }
    g.L = L; g.M = M; g.n_lo = n_lo; g.n_hi = n_hi;
    g.A = (M - 1) + n_hi;
    g.Q.assign(L + 1, 0);
    g.cells.assign(L + 1, 0);
    g.base.assign(L + 2, 0);
    g.off.assign((size_t)(L + 1) * g.A, -1);
    g.wave_splits.assign(L + 1, 0);
    g.wave_cells.assign(L + 1, 0);
    for (int l = 1; l <= L; ++l) {
        g.Q[l] = (l == L) ? n_hi : std::max(1, n_hi - 1);
        int32_t off = 0;
        for (int a = 0; a < g.A; ++a) {
            if (g.is_whole(a) && g.alloc_n(a) > g.Q[l]) continue;
            int64_t c = len_cells(g.lo(a), g.gpus(a), l);
            if (c == 0) continue;
            g.off[(size_t)l * g.A + a] = off;
            off += (int32_t)c;
        }
        g.cells[l] = off;
    }
    g.base[1] = 0;
    g.total_cells = 0;
    for (int l = 1; l <= L; ++l) {
        g.wave_cells[l] = (int64_t)(L - l + 1) * g.cells[l];
        g.base[l + 1] = g.base[l] + g.wave_cells[l] + WAVE_PAD;
        g.total_cells += g.wave_cells[l];
    }
    g.table_cells = g.base[L + 1];

    // Feasible splits.  For a split at l1 = k-u (l2 = l-l1) the valid (s, S-s) pairs of a
    // device split (a1, a2) are exactly len(a1, l1) x len(a2, l2): every such pair lands
    // on a valid parent cell (s + S_R <= l, <= gpus(a), >= lo(a)).  Summed per parent alloc.
    std::vector<int64_t> lenW((size_t)(L + 1) * (n_hi + 1), 0), lenI((size_t)(L + 1) * (M + 1), 0);
    for (int l = 1; l <= L; ++l) {
        for (int q = 1; q <= n_hi; ++q) lenW[(size_t)l * (n_hi + 1) + q] = len_cells(q, q * M, l);
        for (int r = 1; r <= M; ++r) lenI[(size_t)l * (M + 1) + r] = len_cells(1, r, l);
    }
    auto LW = [&](int l, int q) { return lenW[(size_t)l * (n_hi + 1) + q]; };
    auto LI = [&](int l, int r) { return lenI[(size_t)l * (M + 1) + r]; };
    g.total_splits = 0;
    std::vector<int64_t> pre((size_t)n_hi + 1, 0);
    for (int l = 2; l <= L; ++l) {
        int64_t per_range = 0;
        const int Q = g.Q[l];
        for (int l1 = 1; l1 < l; ++l1) {
            int l2 = l - l1;
            // W(q >= 2) -> (W(j), W(q-j)): sum over 2 <= q <= Q, 1 <= j < q of
            // LW(l1, j) LW(l2, q-j) = sum_j LW(l1, j) * (LW(l2, 1) + ... + LW(l2, Q-j))
            for (int m = 1; m <= Q; ++m) pre[m] = pre[m - 1] + LW(l2, m);
            for (int j = 1; j < Q; ++j) per_range += LW(l1, j) * pre[Q - j];
            // W(1) -> (I(m), I(M-m))
            for (int m = 1; m < M; ++m) per_range += LI(l1, m) * LI(l2, M - m);
            // I(r) -> (I(m), I(r-m))
            for (int r = 2; r < M; ++r)
                for (int m = 1; m < r; ++m) per_range += LI(l1, m) * LI(l2, r - m);
        }
        g.wave_splits[l] = per_range * (L - l + 1);
        g.total_splits += g.wave_splits[l];
    }
    return true;
}

}  // namespace oob
