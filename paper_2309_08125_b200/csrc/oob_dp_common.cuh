// Device-side DP table layout and index helpers shared by the DP kernels.
//
// Cell table (per profile, HBM): AoS records Cell4 {T1, T3, t*, C1} (32 B) + ARG (u32).
//   T1, T3, t*: the memo value of T(S', u, v, a) (PAPER Eq.1-4);
//   C1 = (3S'-1) + k*: the cell's own Eq.2 coefficient (N_b - S' + k* - 1 with N_b = 4S',
//        P:405) — an exact small integer in binary64, so T2 = C1 * t* and
//        k* = C1 - (3S'-1) exactly;
//   ARG: argmin split packed (l1-1) | m << 10 | s << 20 (0xFFFFFFFF for S' = 1).
// Shadow table SH (per cell, float4, written with every cell): binary32 LOWER BOUNDS of
//   {A = T1 + T3 + C1 t*, T1, t*, 2 T1} (fp64 ops rounded down, then rounded down to fp32),
//   used only by k_wave_w's filter (a split whose lower bound cannot reach the output's
//   current minimum is skipped; every candidate is re-evaluated exactly in binary64).
// Cell index: base[l] + u*cells[l] + off[l*A + a] + (S' - lo(a)).
#pragma once

#include <cstdint>

namespace oob {

struct __align__(32) Cell4 {
    double T1, T3, TS, C1;
};

struct DevGeom {
    int L, M, n_lo, n_hi, A, P;
    int64_t C;                // cells per profile
    const int32_t *cells;     // [L+1]
    const int64_t *base;      // [L+2]
    const int32_t *off;       // [(L+1)*A]
    const int32_t *wofs;      // [(L+1)*(L+2)]: offset of W row q (1..l+1) in a slab of length l (incl. I part)
    Cell4 *CELL;              // [P*C]
    float4 *SH;               // [P*C] shadow lower bounds (filter only)
    uint32_t *ARG;            // [P*C]
    // stage masks (DESIGN reading R31; masked = 0: none, every valid cell is finite)
    int masked;               // 1: some cells may be infinite (written by d_store_inf)
    int pow2;                 // a stage's GPU count must be a power of two
    const double *SB;         // [P][L] per-layer stage bytes (NULL: no memory mask)
    double mem_cap;           // sum_{l in stage} SB[l] / d <= mem_cap
};

__device__ __forceinline__ bool d_is_whole(const DevGeom &g, int a) { return a >= g.M - 1; }
// slab offset of W row q in a slab of length l (rows are contiguous: row q has
// d_wofs(l, q+1) - d_wofs(l, q) cells)
__device__ __forceinline__ int d_wofs(const DevGeom &g, int l, int q) { return __ldg(g.wofs + l * (g.L + 2) + q); }
__device__ __forceinline__ int d_alloc_n(const DevGeom &g, int a) {
    return d_is_whole(g, a) ? a - (g.M - 1) + 1 : a + 1;
}
__device__ __forceinline__ int d_lo(const DevGeom &g, int a) { return d_is_whole(g, a) ? d_alloc_n(g, a) : 1; }
__device__ __forceinline__ int d_gpus(const DevGeom &g, int a) {
    return d_is_whole(g, a) ? d_alloc_n(g, a) * g.M : d_alloc_n(g, a);
}
__device__ __forceinline__ int d_hi(const DevGeom &g, int a, int l) {
    int gg = d_gpus(g, a);
    return l < gg ? l : gg;
}
__device__ __forceinline__ int d_num_dsplits(const DevGeom &g, int a) {
    int n = d_alloc_n(g, a);
    return d_is_whole(g, a) ? (n >= 2 ? n - 1 : g.M - 1) : n - 1;
}
// j-th device split of a (same order as the oracle's device_splits)
__device__ __forceinline__ void d_dsplit(const DevGeom &g, int a, int j, int &a1, int &a2) {
    int n = d_alloc_n(g, a);
    int m = j + 1;
    if (d_is_whole(g, a) && n >= 2) { a1 = (g.M - 1) + m - 1; a2 = (g.M - 1) + (n - m) - 1; }
    else if (d_is_whole(g, a))      { a1 = m - 1; a2 = g.M - m - 1; }
    else                            { a1 = m - 1; a2 = n - m - 1; }
}
// k* <-> C1 = (3S'-1) + k* (both exact small integers in binary64)
__device__ __forceinline__ double d_kd(double c1, int S) { return __dadd_rn(c1, -(double)(3 * S - 1)); }
__device__ __forceinline__ double d_c1(double kd, int S) { return __dadd_rn((double)(3 * S - 1), kd); }
__device__ __forceinline__ int64_t d_cell(const DevGeom &g, int Sp, int u, int l, int a) {
    return g.base[l] + (int64_t)u * g.cells[l] + g.off[l * g.A + a] + (Sp - d_lo(g, a));
}
__device__ __forceinline__ Cell4 d_load(const Cell4 *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    Cell4 c;
    c.T1 = a.x; c.T3 = a.y; c.TS = b.x; c.C1 = b.y;
    return c;
}
// Shadow of a cell: every component rounds toward -inf, so each is <= the real value of
// the expression on the stored binary64 values (all positive).
__device__ __forceinline__ float4 d_shadow(double T1, double T3, double TS, double C1) {
    const double A = __dadd_rd(__dadd_rd(T1, T3), __dmul_rd(C1, TS));
    const float t1 = __double2float_rd(T1);
    return make_float4(__double2float_rd(A), t1, __double2float_rd(TS), __fmul_rd(2.0f, t1));
}
// Store cell c (table index incl. the profile offset) and its shadow.
__device__ __forceinline__ void d_store(const DevGeom &g, int64_t c, double T1, double T3, double TS, double C1) {
    reinterpret_cast<double2 *>(g.CELL + c)[0] = make_double2(T1, T3);
    reinterpret_cast<double2 *>(g.CELL + c)[1] = make_double2(TS, C1);
    g.SH[c] = d_shadow(T1, T3, TS, C1);
}
// Infinite cell (stage masks: no allowed stage / division): +inf values and shadow, so every
// split using it is +inf (never passes the filter, never enters an accumulator).
constexpr uint32_t ARG_INF = 0xFFFFFFFCu;
__device__ __forceinline__ void d_store_inf(const DevGeom &g, int64_t c, int Sp) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    reinterpret_cast<double2 *>(g.CELL + c)[0] = make_double2(inf, inf);
    reinterpret_cast<double2 *>(g.CELL + c)[1] = make_double2(inf, (double)(3 * Sp - 1));
    const float finf = __int_as_float(0x7f800000);
    g.SH[c] = make_float4(finf, finf, finf, finf);
    g.ARG[c] = ARG_INF;
}
// Reading R31: the stage [u, v) of profile p on d GPUs of one node is allowed iff d is a
// power of two (pow2) and sum_{l=u}^{v-1} SB[l] / d <= mem_cap (summed left to right).
__device__ __forceinline__ bool d_stage_allowed(const DevGeom &g, int p, int u, int v, int d) {
    if (g.pow2 && (d & (d - 1)) != 0) return false;
    if (g.SB) {
        const double *sb = g.SB + (size_t)p * g.L;
        double tot = 0.0;
        for (int k = u; k < v; ++k) tot = __dadd_rn(tot, sb[k]);
        if (__ddiv_rn(tot, (double)d) > g.mem_cap) return false;
    }
    return true;
}
// Poison cell c (no valid split found / corrupt key): NaN value, never passes the filter.
__device__ __forceinline__ void d_poison(const DevGeom &g, int64_t c, uint32_t code) {
    g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
    g.SH[c] = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                          __int_as_float(0x7fc00000));
    g.ARG[c] = code;
}

// Recompute the value of the cell (Sp, u, u+l, a) for its winning split (l1, j, s) from its
// two children (same arithmetic and order as the oracle's combine, oracle/dp.py) and store
// it with its ARG.  Used by every kernel that decides an argmin first and writes after.
__device__ __forceinline__ void d_write_winner(const DevGeom &g, int64_t pc, int Sp, int u, int l, int a,
                                               int l1, int j, int s) {
    const int k = u + l1, l2 = l - l1;
    int a1, a2;
    d_dsplit(g, a, j, a1, a2);
    const Cell4 Lc = d_load(g.CELL + pc + d_cell(g, s, u, l1, a1));
    const Cell4 Rc = d_load(g.CELL + pc + d_cell(g, Sp - s, k, l2, a2));
    const bool left = Lc.TS >= Rc.TS;
    const double kd = left ? d_kd(Lc.C1, s) : __dadd_rn((double)s, d_kd(Rc.C1, Sp - s));
    const int64_t c = pc + d_cell(g, Sp, u, l, a);
    d_store(g, c, __dadd_rn(Lc.T1, Rc.T1), left ? __dadd_rn(Lc.T3, Rc.T1) : Rc.T3,
            left ? Lc.TS : Rc.TS, d_c1(kd, Sp));
    g.ARG[c] = (uint32_t)(l1 - 1) | ((uint32_t)j << 10) | ((uint32_t)s << 20);
}

}  // namespace oob
