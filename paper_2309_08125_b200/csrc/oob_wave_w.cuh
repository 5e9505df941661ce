// Wavefront kernels for cells with S' >= 2 (the hot loop).
//
// k_wave_w — whole-node cells W(q >= 2).  For a range (u, v) of length l and a layer split
// k (l1 = k-u, l2 = v-k), W(q) cells combine left children W(j) of (u, k) with right
// children W(q-j) of (k, v) (PAPER Eq.1-3, two-level device split: reading R2).  In
// (nodes, stages) coordinates every pair (left cell, right cell) is a valid split of
// exactly one parent cell (q = j + j', S' = s + S_R): for each row pair (j, j') the work
// is a dense a_j x b_j' rectangle of splits.  Mapping (one CTA per (profile, range, item)):
//   * the child slab with more W cells ("big side") is register-tiled: a lane holds TE
//     consecutive cells of one row; 32 consecutive tiles (rows may straddle lanes) and one
//     chunk of small-side rows form a warp work unit; warps pull units from a counter;
//   * a unit walks its rows of the other slab ("small side") cell by cell; all lanes read
//     the same cell (L1 broadcast, 2 x 16-byte loads);
//   * each lane keeps the TE outputs its tile currently touches in a register ring (the
//     outputs slide by one cell per step); the output whose last contribution from this
//     lane has arrived is merged into the CTA's shared-memory accumulator, which holds per
//     parent cell the lexicographic minimum of (total, canonical split key), updated with
//     a 128-bit compare-and-swap — exact under any interleaving.
// Tie semantics: the oracle keeps the first strictly-smaller total in (k, m, s) order.
// Inside a ring slot the pairs of one (k, j) arrive in decreasing s, so "<=" keeps the
// smallest s; every merge compares (total, key) with key = l1<<20 | j<<10 | s, which is
// monotone in (k, m, s): the result is exactly the oracle's argmin.
//
// k_wave_small — cells inside one node (I(r), W(1)); k_wave_w_finalize — merge of the
// items' partial argmins and the winner's recomputation.
#pragma once

#include "oob_dp_common.cuh"

namespace oob {

constexpr int NT_MAX = 256;               // max threads per CTA of k_wave_w

struct WaveW {
    int l;                 // wavefront length
    int nranges;           // L - l + 1
    int nitems;            // work items per range
    const int4 *items;     // per item: (entry_lo, entry_hi, -, -)
    const int4 *ents;      // per (item, k): (l1, nblocks, nchunks, chunk_off)
    const int32_t *cb;     // chunk row boundaries: rows [cb[off+c], cb[off+c+1])
    int nout;              // W-part cells of a slab of length l (W(1)..W(Q_l))
    double *PB;            // partial best  [P][nranges][nitems][nout]
    uint32_t *PK;          // partial key
    const int32_t *tile_off;   // [L+1] offset of the flat tile list of a big side of length lb
    const int32_t *tile_cnt;   // [L+1] number of tiles
    const int32_t *tiles;      // packed (row << 16 | e0)
};

__device__ __forceinline__ int d_wcells(const DevGeom &g, int l) {
    return g.cells[l] - g.off[l * g.A + (g.M - 1)];
}
// offset of W(q) inside the W-part of a slab of length l (-1 if absent)
__device__ __forceinline__ int d_woff(const DevGeom &g, int l, int q) {
    const int o = g.off[l * g.A + (g.M - 1) + q - 1];
    return o < 0 ? -1 : o - g.off[l * g.A + (g.M - 1)];
}
__device__ __forceinline__ int d_wlen(const DevGeom &g, int l, int q) {
    const int hi = min(l, q * g.M);
    return hi >= q ? hi - q + 1 : 0;
}

// One split, operands in left / right roles.  The coefficient is cla + clb if the left
// half holds the slowest stage (3S'-1+k*_L) and cra + crb otherwise (3S'-1+s+k*_R), exact
// integers:
//   T1 = L.T1 + R.T1; left = L.t* >= R.t*; T3 = left ? L.T3 + R.T1 : R.T3;
//   T2 = coef * t*; total = (T1 + T2) + T3; keep if total <= best.
// skip_r / skip_l: the second operand of that coefficient is +0 (t == 0), use the first.
__device__ __forceinline__ void split_eval(double LT1, double LT3, double LTS, double cla, double clb,
                                           double RT1, double RT3, double RTS, double cra, double crb,
                                           double &best, int &widx, int code, bool skip_r = false) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double cL = __dadd_rn(cla, clb);
    const double cR = skip_r ? cra : __dadd_rn(cra, crb);
    const double TS = left ? LTS : RTS;
    const double T3 = left ? T3a : RT3;
    const double c = left ? cL : cR;
    const double T2 = __dmul_rn(c, TS);
    const double tot = __dadd_rn(__dadd_rn(T1, T2), T3);
    const bool upd = tot <= best;
    best = upd ? tot : best;
    widx = upd ? code : widx;
}

__device__ __forceinline__ void split_eval2(double LT1, double LT3, double LTS, double cla, double clb,
                                            double RT1, double RT3, double RTS, double cra, double crb,
                                            double &best, int &widx, int code, bool skip_l) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double cL = skip_l ? cla : __dadd_rn(cla, clb);
    const double cR = __dadd_rn(cra, crb);
    const double TS = left ? LTS : RTS;
    const double T3 = left ? T3a : RT3;
    const double c = left ? cL : cR;
    const double T2 = __dmul_rn(c, TS);
    const double tot = __dadd_rn(__dadd_rn(T1, T2), T3);
    const bool upd = tot <= best;
    best = upd ? tot : best;
    widx = upd ? code : widx;
}

// 128-bit shared-memory CAS (sm_90+ atom.shared.cas.b128)
__device__ __forceinline__ void cas128(unsigned addr, unsigned long long &olo, unsigned long long &ohi,
                                       unsigned long long clo, unsigned long long chi,
                                       unsigned long long nlo, unsigned long long nhi) {
    asm volatile("{\n\t.reg .b128 d, c, v;\n\t"
                 "mov.b128 c, {%2, %3};\n\t"
                 "mov.b128 v, {%4, %5};\n\t"
                 "atom.shared.cas.b128 d, [%6], c, v;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(olo), "=l"(ohi)
                 : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "r"(addr)
                 : "memory");
}

// acc entry = {double total bits, key}: lexicographic-min update (exact under races).
// The slow path (a CAS loop) is out of line: most flushes lose the comparison.
__device__ __noinline__ void acc_merge_slow(unsigned addr, unsigned long long cx, unsigned long long cy,
                                            double b, uint32_t key) {
    const unsigned long long nb = (unsigned long long)__double_as_longlong(b);
    for (;;) {
        unsigned long long olo, ohi;
        cas128(addr, olo, ohi, cx, cy, nb, (unsigned long long)key);
        if (olo == cx && ohi == cy) return;
        cx = olo;
        cy = ohi;
        const double A = __longlong_as_double((long long)cx);
        const uint32_t K = (uint32_t)cy;
        if (!(b < A || (b == A && key < K))) return;
    }
}

// flush one ring slot into the accumulator entry `idx` if `ok` (valid output, finite)
__device__ __forceinline__ void acc_flush(const ulonglong2 *acc, int idx, bool ok, double b, uint32_t key) {
    const unsigned addr = (unsigned)__cvta_generic_to_shared(acc + (ok ? idx : 0));
    unsigned long long cx, cy;   // one 16-byte shared load (single transaction)
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(cx), "=l"(cy) : "r"(addr) : "memory");
    const double A = __longlong_as_double((long long)cx);
    const uint32_t K = (uint32_t)cy;
    if (ok && (b < A || (b == A && key < K))) acc_merge_slow(addr, cx, cy, b, key);
}

constexpr double D_INF = __builtin_huge_val();

template <int TE>
__global__ void __launch_bounds__(NT_MAX, (TE <= 4 ? 2 : 1)) k_wave_w(DevGeom g, WaveW w) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int l = w.l;
    const int nout = w.nout;
    ulonglong2 *acc = reinterpret_cast<ulonglong2 *>(smem);
    int *outOff = reinterpret_cast<int *>(acc + nout);    // [L+2] W(q) offsets in slab l
    int *ucum = outOff + (g.L + 2);                        // [L+2] cumulative units per entry
    int *ctr = ucum + (g.L + 2);
    const int NT = blockDim.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    int bid = blockIdx.x;
    const int item = bid % w.nitems; bid /= w.nitems;
    const int u = bid % w.nranges;
    const int p = bid / w.nranges;
    const int64_t pc = (int64_t)p * g.C;
    const int4 it = w.items[item];
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);

    for (int i = tid; i < nout; i += NT)
        acc[i] = make_ulonglong2((unsigned long long)__double_as_longlong(D_INF), 0xFFFFFFFFull);
    for (int q = tid; q < g.L + 2; q += NT) outOff[q] = (q >= 1 && q <= Ql && q <= l) ? d_woff(g, l, q) : -1;
    if (tid == 0) {
        int c = 0;
        ucum[0] = 0;
        for (int e = it.x; e < it.y; ++e) {
            const int4 en = w.ents[e];
            c += en.y * en.z;
            ucum[e - it.x + 1] = c;
        }
        *ctr = 0;
    }
    __syncthreads();
    const int nunits = ucum[it.y - it.x];

    for (;;) {
        int un = 0;
        if (lane == 0) un = atomicAdd(ctr, 1);
        un = __shfl_sync(0xFFFFFFFFu, un, 0);
        if (un >= nunits) break;
        int ei = 0;
        while (ucum[ei + 1] <= un) ++ei;
        const int4 en = w.ents[it.x + ei];
        const int l1 = en.x;
        const int local = un - ucum[ei];
        const int chunk = local / en.y;
        const int blk = local % en.y;
        const int r_lo = w.cb[en.w + chunk], r_hi = w.cb[en.w + chunk + 1];
        const int k = u + l1;
        const int l2 = l - l1;
        const bool ltiled = d_wcells(g, l1) >= d_wcells(g, l2);   // big side = left
        const int ls = ltiled ? l2 : l1;                           // small side length
        const int lb = ltiled ? l1 : l2;
        const int us = ltiled ? k : u;                             // small slab start
        const int ub = ltiled ? u : k;
        const int ti = blk * 32 + lane;
        const bool has = ti < w.tile_cnt[lb];
        const int32_t code = has ? w.tiles[w.tile_off[lb] + ti] : 0;
        const int rowB = has ? (code >> 16) : 1;
        const int e0 = has ? (code & 0xFFFF) : 0;
        const int lenB = has ? d_wlen(g, lb, rowB) : 0;
        const Cell4 *bp = g.CELL + pc + g.base[lb] + (int64_t)ub * g.cells[lb] +
                          (has ? g.off[lb * g.A + (g.M - 1) + rowB - 1] : 0) + e0;
        // register tile: T1, T3, t*, C1 of TE big-side cells (sentinels beyond the row)
        double RT1[TE], RT3[TE], RTS[TE], RC1[TE];
#pragma unroll
        for (int t = 0; t < TE; ++t) {
            if (has && e0 + t < lenB) {
                const Cell4 c = d_load(bp + t);
                RT1[t] = c.T1; RT3[t] = c.T3; RTS[t] = c.TS; RC1[t] = c.C1;
            } else {
                RT1[t] = D_INF; RT3[t] = D_INF; RTS[t] = D_INF; RC1[t] = 1.0;
            }
        }
        // stage count of the tile's first cell (its c2 = 4s or 3S_R is folded per step)
        const double S0 = (double)(rowB + e0);
        const Cell4 *sp = g.CELL + pc + g.base[ls] + (int64_t)us * g.cells[ls] + g.off[ls * g.A + (g.M - 1)];
        for (int rs = r_lo; rs < r_hi; ++rs) {
            const int q = rowB + rs;
            const int ob = (has && q <= g.L + 1) ? outOff[q] : -1;
            const bool qok = ob >= 0;
            const int rl = d_wlen(g, ls, rs);
            const Cell4 *rp = sp + d_woff(g, ls, rs);
            double best[TE];
            int widx[TE];
#pragma unroll
            for (int t = 0; t < TE; ++t) { best[t] = D_INF; widx[t] = 0; }
            if (ltiled) {
                // big = left row j = rowB (s_t = S0 + t); iterate right row j' = rs, e'
                // ascending (S_R = rs + e').  coef_left = 3S_R + C1_L[t];
                // coef_right = 4 s_t + C1_R = (C1_R + 4 S0) + 4t.
                // Ring slot r <-> output E with (E - e0) % TE == r.
                const int j = rowB;
                const uint32_t kb = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) | (uint32_t)(j + e0);
                double c3 = (double)(3 * rs);          // 3 S_R
                const double s4 = 4.0 * S0;
                Cell4 x = d_load(rp);
                int ep = 0;
#define OOB_LT_STEP(I)                                                                          \
    {                                                                                           \
        const Cell4 nx = d_load(rp + min(ep + (I) + 1, rl - 1));                                \
        const double xr = __dadd_rn(x.C1, s4);                                                  \
        _Pragma("unroll") for (int t = 0; t < TE; ++t)                                          \
            split_eval(RT1[t], RT3[t], RTS[t], c3, RC1[t], x.T1, x.T3, x.TS, xr,                \
                       (double)(4 * t), best[((I) + t) % TE], widx[((I) + t) % TE], t, t == 0); \
        c3 = __dadd_rn(c3, 3.0);                                                                \
        acc_flush(acc, ob + e0 + ep + (I), qok && best[(I)] < D_INF, best[(I)],                \
                  kb + (uint32_t)widx[(I)]);                                                    \
        best[(I)] = D_INF;                                                                      \
        x = nx;                                                                                 \
    }
#pragma unroll 1
                for (; ep + TE <= rl; ep += TE) {
#pragma unroll
                    for (int i = 0; i < TE; ++i) OOB_LT_STEP(i)
                }
#pragma unroll
                for (int i = 0; i < TE - 1; ++i)
                    if (ep + i < rl) OOB_LT_STEP(i)
#undef OOB_LT_STEP
#pragma unroll
                for (int r = 0; r < TE; ++r) {
                    const int E = e0 + rl + (((r - rl) % TE) + TE) % TE;
                    acc_flush(acc, ob + E, qok && best[r] < D_INF, best[r], kb + (uint32_t)widx[r]);
                }
            } else {
                // big = right row j' = rowB (S_R,t = S0 + t); iterate left row j = rs, e
                // descending (s = rs + e).  coef_left = 3 S_R,t + C1_L = (C1_L + 3 S0) + 3t;
                // coef_right = 4s + C1_R[t].  Step i = rl-1-e; slot (t - i) % TE holds output
                // E = e + e0 + t; the t = TE-1 output completes at each step.
                const int jl = rs;
                const uint32_t kb = ((uint32_t)l1 << 20) | ((uint32_t)jl << 10);
                double c4 = (double)(4 * (rs + rl - 1));   // 4 s
                const double s3 = 3.0 * S0;
                Cell4 x = d_load(rp + rl - 1);
                int st = 0;
#define OOB_RT_STEP(I)                                                                          \
    {                                                                                           \
        const int e = rl - 1 - st - (I);                                                        \
        const Cell4 nx = d_load(rp + max(e - 1, 0));                                            \
        const double xl = __dadd_rn(x.C1, s3);                                                  \
        _Pragma("unroll") for (int t = 0; t < TE; ++t)                                          \
            split_eval2(x.T1, x.T3, x.TS, xl, (double)(3 * t), RT1[t], RT3[t], RTS[t], c4,      \
                       RC1[t], best[((t - (I)) % TE + TE) % TE], widx[((t - (I)) % TE + TE) % TE], t, t == 0); \
        c4 = __dadd_rn(c4, -4.0);                                                               \
        const int sf = ((TE - 1 - (I)) % TE + TE) % TE;                                         \
        const int E = e + e0 + TE - 1;                                                          \
        acc_flush(acc, ob + E, qok && best[sf] < D_INF, best[sf],                               \
                  kb + (uint32_t)(jl + E - e0 - widx[sf]));                                     \
        best[sf] = D_INF;                                                                       \
        x = nx;                                                                                 \
    }
#pragma unroll 1
                for (; st + TE <= rl; st += TE) {
#pragma unroll
                    for (int i = 0; i < TE; ++i) OOB_RT_STEP(i)
                }
#pragma unroll
                for (int i = 0; i < TE - 1; ++i)
                    if (st + i < rl) OOB_RT_STEP(i)
#undef OOB_RT_STEP
                // after the last step (i = rl-1, e = 0) slot sg holds t = (sg + rl - 1) % TE
#pragma unroll
                for (int sg = 0; sg < TE; ++sg) {
                    const int t = (sg + rl - 1) % TE;
                    const int E = e0 + t;
                    acc_flush(acc, ob + E, qok && best[sg] < D_INF, best[sg],
                              kb + (uint32_t)(jl + E - e0 - widx[sg]));
                }
            }
        }
    }
    __syncthreads();
    const size_t pb = (size_t)blockIdx.x * nout;
    for (int i = tid; i < nout; i += NT) {
        const ulonglong2 a = acc[i];
        w.PB[pb + i] = __longlong_as_double((long long)a.x);
        w.PK[pb + i] = (uint32_t)a.y;
    }
}

// Per W(q >= 2) cell: lexicographic min of the items' partials, then the winner's
// (T1, T3, t*, C1) recomputed from its two children (same arithmetic as the oracle).
__global__ void k_wave_w_finalize(DevGeom g, WaveW w) {
    const int l = w.l;
    const int nout = w.nout;
    const int64_t n = (int64_t)g.P * w.nranges * nout;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = (int)(t % nout);
    const int u = (int)((t / nout) % w.nranges);
    const int p = (int)(t / ((int64_t)nout * w.nranges));
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);
    int q = 0, Sp = 0;
    for (int qq = 2; qq <= min(Ql, l); ++qq) {
        const int o = d_woff(g, l, qq);
        const int len = d_wlen(g, l, qq);
        if (o >= 0 && i >= o && i < o + len) { q = qq; Sp = qq + (i - o); break; }
    }
    if (q == 0) return;       // W(1) cell (handled by k_wave_small)
    double best = D_INF;
    uint32_t key = 0xFFFFFFFFu;
    const size_t base = ((size_t)p * w.nranges + u) * w.nitems;
    for (int it = 0; it < w.nitems; ++it) {
        const size_t pi = (base + it) * nout + i;
        const double b = w.PB[pi];
        const uint32_t kk = w.PK[pi];
        if (b < best || (b == best && kk < key)) { best = b; key = kk; }
    }
    const int64_t pc = (int64_t)p * g.C;
    const int aW = (g.M - 1) + q - 1;
    if (!(best < D_INF)) {     // no split found: impossible for a valid cell; poison it
        const int64_t c = pc + d_cell(g, Sp, u, l, aW);
        g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
        g.ARG[c] = 0xFFFFFFFEu;
        return;
    }
    const int l1 = (int)(key >> 20), j = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
    d_write_winner(g, pc, Sp, u, l, aW, l1, j - 1, s);
}

// I(r) and W(1) cells with S' >= 2 (GPUs inside one node): one warp per cell, lanes take
// contiguous k ranges in the oracle's order (strict "<"), then a lexicographic
// (total, key) warp-shuffle argmin.
__global__ void k_wave_small(DevGeom g, int l) {
    const int nsmall = min(g.A, g.M);              // alloc indices 0..M-1: I(1..M-1), W(1)
    const int nr = g.L - l + 1;
    const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    int per_range = 0;
    for (int a = 0; a < nsmall; ++a) per_range += max(0, d_hi(g, a, l) - 1);
    if (per_range == 0) return;
    if (warp_id >= (int64_t)g.P * nr * per_range) return;
    int rem = (int)(warp_id % per_range);
    const int u = (int)((warp_id / per_range) % nr);
    const int p = (int)(warp_id / ((int64_t)per_range * nr));
    int a = 0, Sp = 0;
    for (int aa = 0; aa < nsmall; ++aa) {
        const int c = max(0, d_hi(g, aa, l) - 1);
        if (rem < c) { a = aa; Sp = 2 + rem; break; }
        rem -= c;
    }
    if (g.off[l * g.A + a] < 0) return;
    const int64_t pc = (int64_t)p * g.C;
    const double dSp3 = (double)(3 * Sp - 1);
    const int nd = d_num_dsplits(g, a);
    const int per_lane = (l - 1 + 31) / 32;
    const int l1_lo = 1 + lane * per_lane, l1_hi = min(l - 1, (lane + 1) * per_lane);
    double best = D_INF;
    uint32_t bkey = 0xFFFFFFFFu;
    for (int l1 = l1_lo; l1 <= l1_hi; ++l1) {
        const int k = u + l1, l2 = l - l1;
        for (int j = 0; j < nd; ++j) {
            int a1, a2;
            d_dsplit(g, a, j, a1, a2);
            if (g.off[l1 * g.A + a1] < 0 || g.off[l2 * g.A + a2] < 0) continue;
            const int s_lo = max(max(1, d_lo(g, a1)), Sp - d_hi(g, a2, l2));
            const int s_hi = min(min(Sp - 1, d_hi(g, a1, l1)), Sp - d_lo(g, a2));
            for (int s = s_lo; s <= s_hi; ++s) {
                const Cell4 Lc = d_load(g.CELL + pc + d_cell(g, s, u, l1, a1));
                const Cell4 Rc = d_load(g.CELL + pc + d_cell(g, Sp - s, k, l2, a2));
                const double T1 = __dadd_rn(Lc.T1, Rc.T1);
                const bool left = Lc.TS >= Rc.TS;
                const double T3 = left ? __dadd_rn(Lc.T3, Rc.T1) : Rc.T3;
                const double TS = left ? Lc.TS : Rc.TS;
                const double KD = left ? d_kd(Lc.C1, s) : __dadd_rn((double)s, d_kd(Rc.C1, Sp - s));
                const double T2 = __dmul_rn(__dadd_rn(KD, dSp3), TS);
                const double tot = __dadd_rn(__dadd_rn(T1, T2), T3);
                if (tot < best) {
                    best = tot;
                    bkey = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) | (uint32_t)s;
                }
            }
        }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const double ob = __shfl_down_sync(0xFFFFFFFFu, best, d);
        const uint32_t ok = __shfl_down_sync(0xFFFFFFFFu, bkey, d);
        if (ob < best || (ob == best && ok < bkey)) { best = ob; bkey = ok; }
    }
    if (lane != 0) return;
    d_write_winner(g, pc, Sp, u, l, a, (int)(bkey >> 20), (int)((bkey >> 10) & 1023u), (int)(bkey & 1023u));
}

}  // namespace oob
