// Wavefront kernels for cells with S' >= 2 (the hot loop).
//
// k_wave_w — whole-node cells W(q >= 2).  For a range (u, v) of length l and a layer split
// k (l1 = k-u, l2 = v-k), W(q) cells combine left children W(j) of (u, k) with right
// children W(q-j) of (k, v) (PAPER Eq.1-3, two-level device split: reading R2).  In
// (nodes, stages) coordinates every pair (left cell, right cell) is a valid split of
// exactly one parent cell (q = j + j', S' = s + S_R): for each row pair (j, j') the work is
// a dense a_j x b_j' rectangle of splits.  Mapping (one CTA per (item, profile, range);
// items are lists of layer splits k, ordered by decreasing cost so the block scheduler
// runs them longest-first):
//   * the child slab with more W cells ("big side") is register-tiled: a lane holds TE
//     consecutive cells of one row; 32 consecutive tiles (rows may straddle lanes) and one
//     chunk of small-side rows form a warp work unit; warps pull units from a counter;
//   * a unit walks its rows of the other slab ("small side") cell by cell; all lanes read
//     the same cell (L1 broadcast, 2 x 16-byte loads) and evaluate TE splits;
//   * the outputs a lane touches slide by one cell per step: a ring of TE slots keeps, per
//     in-flight output, only the minimum HIGH WORD of its totals (one 32-bit min per
//     split).  When an output's last contribution from this lane has arrived, the slot is
//     compared with the high word of the CTA's shared-memory accumulator entry; only if it
//     is <= (it can win or tie) does the lane recompute that output's TE splits exactly
//     (the same binary64 operations, hence the same bits) and merge the lexicographic
//     minimum of (total, split key) with a 128-bit compare-and-swap — exact under any
//     interleaving.  Since the high word of a positive binary64 is monotone in its value,
//     the filter never drops a winner.
//   * at the end of the task the CTA's accumulator is merged into the global accumulator
//     of the range (128-bit global CAS); k_fin recomputes each winner's cell.
// Tie semantics: the oracle keeps the first strictly smaller total in (k, m, s) order; the
// key l1<<20 | j<<10 | s is monotone in (k, m, s), so the lexicographic minimum of
// (total, key) is exactly the oracle's argmin.
//
// k_fin — per wavefront: the winners of the W(q >= 2) cells of wave l, and every cell
// inside one node (I(r), W(1)) of wave l+1 (those depend only on shorter cells inside a
// node), a group of threads per cell with a lexicographic argmin reduction.
#pragma once

#include "oob_dp_common.cuh"

namespace oob {

constexpr int NTW = 256;                                          // threads per k_wave_w CTA
constexpr unsigned long long ACC_EMPTY = 0x7FEFFFFFFFFFFFFFull;   // DBL_MAX: "no split yet"
constexpr double D_INF = __builtin_huge_val();

// Finalize / in-node work of one wavefront (k_fin, or k_wave_w's extra blocks and last CTAs).
struct FinArgs {
    int lw, nranges_w, nout_w;     // W finalize of wave lw (lw = 0: none)
    int nbw;                       // blocks of the W part
    ulonglong2 *GACC;              // accumulator of wave lw (this rank's)
    const ulonglong2 *GPART;       // world > 1: all ranks' partial accumulators [world][entries]
    int64_t part_stride;           // entries per rank in GPART
    int world;
    int lseed, nout_s, nbseed;     // seeds of wave lseed (0: none): W outputs per range, blocks
    ulonglong2 *GSEED;             // accumulator of wave lseed (the other parity buffer)
    int ls, nsmall;                // small cells of wave ls (ls = 0: none); cells per range
    int tpc;                       // threads per small cell
};

struct WaveW {
    int l;                 // wavefront length
    int nranges;           // L - l + 1
    int cpr;               // CTAs per (profile, range); they share the range's unit queue
    int nents;             // layer splits k with work (balanced splits first)
    const int4 *ents;      // per entry: (l1, nblocks, nchunks, chunk_off)
    const int32_t *upre;   // [nents + 1] unit prefix: entry e owns units [upre[e], upre[e+1])
    const int32_t *cb;     // chunk row boundaries: rows [cb[off+c], cb[off+c+1])
    int *ctr;              // [P][nranges] unit counters of this pass (zeroed before the launch)
    int unit_lo, unit_hi;  // this pass processes queue units [unit_lo, unit_hi)
    int seeded;            // 1: start from the global accumulator (an earlier pass's minima)
    long long perm_a;      // > 1: unit order permutation multiplier (coprime to the pass's unit count)
    int rev_lanes;         // 1: lane i holds the block's tile 31 - i (diagnostic)
    int rank, world;       // single-profile sharding: this rank takes units rank, rank+world, ...
    int nout;              // W-part cells of a slab of length l (W(1)..W(Q_l))
    ulonglong2 *GACC;      // global accumulator [P][nranges][nout]: {total bits, key}
    const int32_t *tile_off;   // [L+1] offset of the flat tile list of a big side of length lb
    const int32_t *tile_cnt;   // [L+1] number of tiles
    const int32_t *tiles;      // packed (row << 16 | e0)
    // fused finalize (unsharded waves): blocks >= nbmain run the in-node cells and seeds of
    // the next wave (fa: nbw = 0; independent of this wave, they fill its tail); the last CTA
    // of each range (rdone counter) finalizes the range's W outputs of this wave (fw: lw = l)
    int nbmain;
    int fin_inline;
    int *rdone;                // [P][nranges] CTAs of the range that have merged
    FinArgs fa, fw;
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

// One split with operands in left / right roles (DESIGN.md §2 arithmetic contract):
//   T1 = L.T1 + R.T1; left = L.t* >= R.t*; T3 = left ? L.T3 + R.T1 : R.T3;
//   T2 = c * t* with c = left ? cL : cR (exact small integers: 3S'-1+k*); total = (T1 + T2) + T3.
// cL / cR have zero low words (integers < 2^21), so the coefficient select is one 32-bit
// select of the high words.
__device__ __forceinline__ double split_total(double LT1, double LT3, double LTS, double cL,
                                              double RT1, double RT3, double RTS, double cR) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double ts = left ? LTS : RTS;
    const double T3 = left ? T3a : RT3;
    const double c = __hiloint2double(left ? __double2hiint(cL) : __double2hiint(cR), 0);
    return __dadd_rn(__dadd_rn(T1, __dmul_rn(c, ts)), T3);
}

// 128-bit compare-and-swap (sm_90+ atom.cas.b128), shared or global (generic address).
__device__ __forceinline__ void cas128_shared(unsigned addr, unsigned long long &olo, unsigned long long &ohi,
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
__device__ __forceinline__ void cas128_global(ulonglong2 *p, unsigned long long &olo, unsigned long long &ohi,
                                              unsigned long long clo, unsigned long long chi,
                                              unsigned long long nlo, unsigned long long nhi) {
    asm volatile("{\n\t.reg .b128 d, c, v;\n\t"
                 "mov.b128 c, {%2, %3};\n\t"
                 "mov.b128 v, {%4, %5};\n\t"
                 "atom.global.cas.b128 d, [%6], c, v;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(olo), "=l"(ohi)
                 : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "l"(p)
                 : "memory");
}

__device__ __forceinline__ bool lex_less(unsigned long long b, uint32_t key, unsigned long long A, uint32_t K) {
    return b < A || (b == A && key < K);
}

// Lexicographic-min merge of (total bits b, key) into the shared accumulator entry at addr.
__device__ __forceinline__ void acc_merge_shared(unsigned addr, unsigned long long b, uint32_t key) {
    unsigned long long cx, cy;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(cx), "=l"(cy) : "r"(addr) : "memory");
    while (lex_less(b, key, cx, (uint32_t)cy)) {
        unsigned long long ox, oy;
        cas128_shared(addr, ox, oy, cx, cy, b, (unsigned long long)key);
        if (ox == cx && oy == cy) return;
        cx = ox;
        cy = oy;
    }
}

// ---------------------------------------------------------------- closed-form slab geometry
// W rows of a slab of length l: row q (1 <= q <= min(Q_l, l)) holds S' = q..min(l, Mq).
__device__ __forceinline__ int c_wlen(int M, int l, int q) { return min(l, M * q) - q + 1; }
// offset of row q inside the W part of the slab
__device__ __forceinline__ int c_woff(int M, int l, int q) {
    const int a = min(q - 1, l / M);            // rows q' < q with M q' <= l
    const int r = q - 1 - a;
    return (M - 1) * (a * (a + 1) / 2) + a + r * (l + 1) - ((q - 1) * q / 2 - a * (a + 1) / 2);
}
// cells of I(1..M-1) at the start of a slab of length l
__device__ __forceinline__ int c_ipart(int M, int l) {
    return l >= M - 1 ? (M - 1) * M / 2 : l * (l + 1) / 2 + (M - 1 - l) * l;
}

// Flush one completed ring slot (exact minimum `b` of its TE contributions, split key
// `key`) into accumulator entry `idx`.  Fast path: compare the high word of `b` with the
// entry's filter word (u32, at most the high word of the entry's total; TE odd makes the
// lanes' filter words — TE entries apart — hit distinct banks).  Only if it can win or tie
// does the lane read the 16-byte entry and run the lexicographic CAS loop (entries only
// decrease, so a stale read is an upper bound and the loop stays exact), then lower the
// filter.  Dummy entries have filter 0 (nothing passes); +inf / NaN never pass ACC_EMPTY.
// diagnostic counters (flush tests passed, CAS successes): compiled in with -DOOB_FLUSH_STATS
// (scripts/flush_stats.py), enabled by oob_dbg_flush_stats
__device__ unsigned long long g_flush_stats[4];
__device__ int g_flush_stats_on;

__device__ __forceinline__ void acc_flush(unsigned acc_s, unsigned filt_s, int idx, double b, uint32_t key) {
    const unsigned bh = (unsigned)__double2hiint(b);
    unsigned fh;
    asm("ld.shared.u32 %0, [%1];" : "=r"(fh) : "r"(filt_s + 4u * (unsigned)idx));
    if (bh <= fh) {
#ifdef OOB_FLUSH_STATS
        if (g_flush_stats_on) {
            atomicAdd(&g_flush_stats[0], 1ull);
            if (bh < fh) atomicAdd(&g_flush_stats[2], 1ull);
        }
#endif
        const unsigned addr = acc_s + 16u * (unsigned)idx;
        const unsigned long long bb = (unsigned long long)__double_as_longlong(b);
        unsigned long long cx, cy;
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(cx), "=l"(cy) : "r"(addr) : "memory");
        while (lex_less(bb, key, cx, (uint32_t)cy)) {
            unsigned long long ox, oy;
            cas128_shared(addr, ox, oy, cx, cy, bb, (unsigned long long)key);
            if (ox == cx && oy == cy) {
#ifdef OOB_FLUSH_STATS
                if (g_flush_stats_on) atomicAdd(&g_flush_stats[1], 1ull);
#endif
                asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(filt_s + 4u * (unsigned)idx), "r"(bh) : "memory");
                break;
            }
            cx = ox;
            cy = oy;
        }
    }
}

// Streamed side staging: a per-warp ring of XR_CELLS cells in shared memory, filled with
// cp.async in batches of XR_BATCH cells (512 B: one 16-byte copy per lane) issued
// XR_AHEAD batches ahead of the step loop, so the steps read the streamed cell from shared
// memory (broadcast LDS) instead of waiting on L1/L2.  The first XR_MIRROR cells of the
// ring are mirrored after its end, so the TE+1 cells a block of steps reads are contiguous
// (one base address per block, immediate offsets).  Copies are unguarded: a chunk's last
// batches may read past the slab (the CELL allocation is padded by XR_CELLS cells).
constexpr int XR_CELLS = 64;
constexpr int XR_BATCH = 16;
constexpr int XR_AHEAD = 2;
constexpr int XR_MIRROR = 8;
constexpr int XR_BYTES = (XR_CELLS + XR_MIRROR) * 32;   // per warp

struct XRing {
    const double2 *ring;                  // this warp's ring (shared memory, 2 x double2 per cell)
    unsigned ring_s;                      // its shared-space address + lane * 16
    const char *src;                      // chunk start (global) + lane * 16
    int nb_iss, nb_ok;                    // batches issued / complete
    bool mirror;                          // this lane also writes the mirror cells
};

__device__ __forceinline__ void xr_issue(XRing &r) {
#ifdef OOB_XR_SYNC
    __syncwarp();
#endif
    const int b = r.nb_iss++;
    const unsigned pos = (unsigned)((b * XR_BATCH) & (XR_CELLS - 1)) * 32u;
    const char *g = r.src + (size_t)b * (XR_BATCH * 32);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(r.ring_s + pos), "l"(g) : "memory");
    if (pos == 0 && r.mirror)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(r.ring_s + XR_CELLS * 32u), "l"(g) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void xr_start(XRing &r, const double2 *ring, const Cell4 *src, int lane) {
    r.ring = ring;
    r.ring_s = (unsigned)__cvta_generic_to_shared(ring) + lane * 16;
    r.src = reinterpret_cast<const char *>(src) + lane * 16;
    r.mirror = lane < 2 * XR_MIRROR;
    r.nb_iss = 0;
    r.nb_ok = 0;
#pragma unroll
    for (int i = 0; i <= XR_AHEAD; ++i) xr_issue(r);
}
// make cells <= j available (warp-uniform; j grows by <= XR_BATCH between calls)
__device__ __forceinline__ void xr_ensure(XRing &r, int j) {
    if (j / XR_BATCH >= r.nb_ok) {
        xr_issue(r);
#ifdef OOB_XR_WAIT0
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#else
        asm volatile("cp.async.wait_group %0;" ::"n"(XR_AHEAD) : "memory");
#endif
        __syncwarp();                     // the other lanes' copies are visible
        r.nb_ok = r.nb_iss - XR_AHEAD;
    }
}
// cells c .. c + XR_MIRROR of the ring as one contiguous run
__device__ __forceinline__ const double2 *xr_at(const XRing &r, int c) { return r.ring + 2 * (c & (XR_CELLS - 1)); }
__device__ __forceinline__ Cell4 xr_cell(const double2 *q, int i) {
    const double2 a = q[2 * i], b = q[2 * i + 1];
    Cell4 x;
    x.T1 = a.x; x.T3 = a.y; x.TS = b.x; x.C1 = b.y;
    return x;
}

// The small-side rows r_lo..r_hi-1 of one unit against this lane's register tile.
//  LT = true : tile = LEFT child (row rowB = j, s_t = S0 + t), stream = RIGHT child (row
//              rs = j', S_R = rs + e).  cL = C1_L[t] + 3 S_R, cR = C1_R(e) + 4 s_t.
//              Ties: contributions to one output arrive with decreasing s -> "<=".
//              key = l1<<20 | rowB<<10 | (S0 + t).
//  LT = false: tile = RIGHT child (row rowB = j', S_R,t = S0 + t), stream = LEFT child (row
//              rs = j, s = rs + e).  cL = C1_L(e) + 3 S_R,t, cR = C1_R[t] + 4 s.
//              Ties: arrivals with increasing s -> "<".  key = l1<<20 | rs<<10 | (rs + e).
// Output E' = e + t (index relative to the tile's first output) lives in ring slot
// E' mod TE; its first contribution (t = TE-1) assigns the slot, t = 0 completes it (flush).
// Each row runs in blocks of TE steps (static slots) plus a guarded tail.  The streamed
// cells (rows r_lo..r_hi-1 are contiguous in the slab) come through the warp's XRing.
template <int TE, bool LT>
__device__ __forceinline__ void run_rows(XRing &xr, int M, int ls, int r_lo, int r_hi,
                                         const double (&RT1)[TE], const double (&RT3)[TE], const double (&RTS)[TE],
                                         const double (&RC1)[TE], int rowB, int e0, int l1, int L,
                                         const int *outOff, int nout, unsigned acc_s, unsigned filt_s) {
    const int S0 = rowB + e0;
    const double xadd = (double)((LT ? 4 : 3) * S0);
    int rb = 0;                                           // chunk cell of the row's first cell
    for (int rs = r_lo; rs < r_hi; ++rs) {
        const int rl = c_wlen(M, ls, rs);
        const int q = rowB + rs;
        const int ob = outOff[min(q, L + 1)];
        const int idx0 = (ob == nout) ? nout : ob + e0;  // accumulator entry of E' = 0
        double cst = (double)((LT ? 3 : 4) * rs);
        const uint32_t kb = LT ? (((uint32_t)l1 << 20) | ((uint32_t)rowB << 10) | (uint32_t)S0)
                               : (((uint32_t)l1 << 20) | ((uint32_t)rs << 10) | (uint32_t)rs);
        double best[TE];
        int widx[TE];
#pragma unroll
        for (int t = 0; t < TE; ++t) { best[t] = D_INF; widx[t] = 0; }
        xr_ensure(xr, rb + TE);
        int blk = 0;
        const double2 *xq = xr_at(xr, rb);
#define OOB_STEP(I)                                                                             \
    {                                                                                           \
        const Cell4 x = xr_cell(xq, (I));                                                       \
        const double xc = __dadd_rn(x.C1, xadd);                                                \
        _Pragma("unroll") for (int t = 0; t < TE; ++t) {                                        \
            const int sl = ((I) + t) % TE;                                                      \
            const double cs = t == 0 ? xc : __dadd_rn(xc, (double)((LT ? 4 : 3) * t));          \
            const double ct = __dadd_rn(RC1[t], cst);                                           \
            const double tot = LT ? split_total(RT1[t], RT3[t], RTS[t], ct, x.T1, x.T3, x.TS, cs) \
                                  : split_total(x.T1, x.T3, x.TS, cs, RT1[t], RT3[t], RTS[t], ct); \
            if (t == TE - 1) {                                                                  \
                best[sl] = tot;                                                                 \
                widx[sl] = t;                                                                   \
            } else {                                                                            \
                const bool upd = LT ? (tot <= best[sl]) : (tot < best[sl]);                     \
                best[sl] = upd ? tot : best[sl];                                                \
                widx[sl] = upd ? t : widx[sl];                                                  \
            }                                                                                   \
        }                                                                                       \
        cst = __dadd_rn(cst, LT ? 3.0 : 4.0);                                                   \
        acc_flush(acc_s, filt_s, idx0 + blk + (I), best[(I)],                                   \
                  LT ? kb + (uint32_t)widx[(I)] : kb + (uint32_t)(blk + (I) - widx[(I)]));      \
    }
        // blocks of TE steps; the last one stops at the row end (one copy of the step code
        // keeps the kernel inside the instruction cache)
#pragma unroll 1
        for (; blk < rl; blk += TE) {
            xr_ensure(xr, rb + blk + TE);
            xq = xr_at(xr, rb + blk);
#pragma unroll
            for (int I = 0; I < TE; ++I)
                if (I == 0 || blk + I < rl) OOB_STEP(I)
        }
#undef OOB_STEP
        // pending: slot sl holds E' = rl + ((sl - rl) mod TE); E' = rl + TE - 1 is the slot of
        // E' = rl - 1, already flushed
#pragma unroll
        for (int sl = 0; sl < TE; ++sl) {
            const int Ep = rl + (((sl - rl) % TE) + TE) % TE;
            if (Ep <= rl + TE - 2)
                acc_flush(acc_s, filt_s, idx0 + Ep, best[sl],
                          LT ? kb + (uint32_t)widx[sl] : kb + (uint32_t)(Ep - widx[sl]));
        }
        rb += rl;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");   // no copy of this chunk outlives the unit
    __syncwarp();
}

// Per-wave finalize + small cells.  Blocks [0, nbw): one thread per (profile, range, W-part
// cell) of wave lw (lw >= 2): read + reset the global accumulator, recompute the winner.
// Blocks [nbw, ...): cells inside one node (I(r), W(1), S' >= 2) of wave ls (2 <= ls <= L):
// `tpc` threads per cell (1..32, power of two) split the layer splits of the cell, scan
// (m, s), keep the first strictly smaller total, then a lexicographic (total, key) reduction.

__device__ __forceinline__ void fin_w_one(const DevGeom &g, const FinArgs &f, int64_t t) {
    const int l = f.lw;
    const int nout = f.nout_w;
    const int i = (int)(t % nout);
    const int u = (int)((t / nout) % f.nranges_w);
    const int p = (int)(t / ((int64_t)nout * f.nranges_w));
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);
    // row q of the W-part cell i: largest q with c_woff(q) <= i (binary search, closed form)
    int lo = 1, hi = min(Ql, l);
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (c_woff(g.M, l, mid) <= i) lo = mid; else hi = mid - 1;
    }
    const int q = lo, Sp = q + (i - c_woff(g.M, l, q));
    if (q < 2) return;        // W(1) cell (computed with the small cells)
    ulonglong2 *ga = f.GACC + t;
    ulonglong2 a = __ldcg(ga);
    __stcg(ga, make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull));
    for (int r = 0; r < f.world && f.world > 1; ++r) {   // lexicographic min over the ranks
        const ulonglong2 b = __ldcg(f.GPART + (int64_t)r * f.part_stride + t);
        if (lex_less(b.x, (uint32_t)b.y, a.x, (uint32_t)a.y)) a = b;
    }
    const int64_t pc = (int64_t)p * g.C;
    const int aW = (g.M - 1) + q - 1;
    if (a.x >= ACC_EMPTY) {   // no split found: impossible for a valid cell; poison it
        const int64_t c = pc + d_cell(g, Sp, u, l, aW);
        g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
        g.ARG[c] = 0xFFFFFFFEu;
        return;
    }
    const uint32_t key = (uint32_t)a.y;
    const int l1 = (int)(key >> 20), j = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
    // bounds check of the decoded split (a corrupt key must not read outside the table)
    const int l2 = l - l1, jr = q - j, sr = Sp - s;
    if (l1 < 1 || l2 < 1 || j < 1 || jr < 1 || s < j || sr < jr || s > min(l1, g.M * j) ||
        sr > min(l2, g.M * jr)) {
        const int64_t c = pc + d_cell(g, Sp, u, l, aW);
        g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
        g.ARG[c] = 0xFFFFFFFDu;
        return;
    }
    d_write_winner(g, pc, Sp, u, l, aW, l1, j - 1, s);
    return;
}

// The W finalize of one range (profile-range index pr) of wave f.lw by one CTA (k_wave_w's
// last CTA of the range): fin_w_one's steps in three phases over FB outputs per thread
// (accumulator loads; child loads; recompute + store) so their memory latencies overlap.
template <int NT>
__device__ __forceinline__ void fin_w_range(const DevGeom &g, const FinArgs &f, int pr, int tid) {
    constexpr int FB = 4;
    const int l = f.lw, nout = f.nout_w, M = g.M;
    const int u = pr % f.nranges_w, p = pr / f.nranges_w;
    const int64_t pc = (int64_t)p * g.C;
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);
    for (int i0 = tid; i0 < nout; i0 += FB * NT) {
        int q[FB], Sp[FB];
        ulonglong2 a[FB];
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            const int i = i0 + j * NT;
            q[j] = 0;
            Sp[j] = 0;
            a[j] = make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull);
            if (i >= nout) continue;
            int lo = 1, hi = min(Ql, l);
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (c_woff(M, l, mid) <= i) lo = mid; else hi = mid - 1;
            }
            q[j] = lo;
            Sp[j] = lo + (i - c_woff(M, l, lo));
            if (lo < 2) continue;
            ulonglong2 *ga = f.GACC + (int64_t)pr * nout + i;
            a[j] = __ldcg(ga);
            __stcg(ga, make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull));
        }
        Cell4 Lc[FB], Rc[FB];
        int l1v[FB], sv[FB], ok[FB];
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            ok[j] = 0;
            l1v[j] = 0;
            sv[j] = 0;
            if (q[j] < 2) continue;
            const int aW = (M - 1) + q[j] - 1;
            if (a[j].x >= ACC_EMPTY) {       // no split found: impossible for a valid cell; poison it
                const int64_t c = pc + d_cell(g, Sp[j], u, l, aW);
                g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
                g.ARG[c] = 0xFFFFFFFEu;
                continue;
            }
            const uint32_t key = (uint32_t)a[j].y;
            const int l1 = (int)(key >> 20), jj = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
            const int l2 = l - l1, jr = q[j] - jj, sr = Sp[j] - s;
            if (l1 < 1 || l2 < 1 || jj < 1 || jr < 1 || s < jj || sr < jr || s > min(l1, M * jj) ||
                sr > min(l2, M * jr)) {      // corrupt key: flag, never read outside the table
                const int64_t c = pc + d_cell(g, Sp[j], u, l, aW);
                g.CELL[c].T1 = __longlong_as_double(0x7ff8000000000000LL);
                g.ARG[c] = 0xFFFFFFFDu;
                continue;
            }
            // children W(jj) of (u, u+l1) and W(jr) of (u+l1, u+l)
            Lc[j] = d_load(g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + c_ipart(M, l1) + c_woff(M, l1, jj) +
                           (s - jj));
            Rc[j] = d_load(g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] + c_ipart(M, l2) +
                           c_woff(M, l2, jr) + (sr - jr));
            l1v[j] = l1;
            sv[j] = s | (jj << 16);
            ok[j] = 1;
        }
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            if (!ok[j]) continue;
            const int s = sv[j] & 0xFFFF, jj = sv[j] >> 16;
            const bool left = Lc[j].TS >= Rc[j].TS;
            const double kd = left ? d_kd(Lc[j].C1, s) : __dadd_rn((double)s, d_kd(Rc[j].C1, Sp[j] - s));
            const int64_t c = pc + d_cell(g, Sp[j], u, l, (M - 1) + q[j] - 1);
            d_store(g.CELL + c, __dadd_rn(Lc[j].T1, Rc[j].T1), left ? __dadd_rn(Lc[j].T3, Rc[j].T1) : Rc[j].T3,
                    left ? Lc[j].TS : Rc[j].TS, d_c1(kd, Sp[j]));
            g.ARG[c] = (uint32_t)(l1v[j] - 1) | ((uint32_t)(jj - 1) << 10) | ((uint32_t)s << 20);
        }
    }
}

__device__ __forceinline__ void fin_seed_one(const DevGeom &g, const FinArgs &f, int64_t t) {
    // ---------------- seeds of wave lseed: per W(q >= 2) output (S', u, u+l, W(q)), the
    // lexicographic minimum over a few proportional splits (j ~ q/2, s ~ S' j/q,
    // l1 ~ l s/S'), evaluated exactly as k_wave_w evaluates them (split_total), so the
    // accumulator starts near the optimum and the flush filter rarely passes.  Children
    // come from waves <= l-2 (2 <= l1 <= l-2), all final when this kernel runs.
    const int l = f.lseed;
    const int nr = g.L - l + 1;
    const int nout = f.nout_s;
    if (t >= (int64_t)g.P * nr * nout) return;
    const int i = (int)(t % nout);
    const int u = (int)((t / nout) % nr);
    const int p = (int)(t / ((int64_t)nout * nr));
    const int M = g.M;
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);
    int lo = 1, hi = min(Ql, l);
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (c_woff(M, l, mid) <= i) lo = mid; else hi = mid - 1;
    }
    const int q = lo, Sp = q + (i - c_woff(M, l, q));
    unsigned long long bb = ACC_EMPTY;
    uint32_t bk = 0xFFFFFFFFu;
    if (q >= 2) {
        const int64_t pc = (int64_t)p * g.C;
        const int Qc = max(1, g.n_hi - 1);                 // children are shorter than L
        for (int jj = 0; jj < 2; ++jj) {
            const int j = jj == 0 ? q / 2 : (q + 1) / 2;
            if (jj == 1 && j == q / 2) continue;
            const int jr = q - j;
            if (j < 1 || jr < 1 || j > Qc || jr > Qc) continue;
            for (int ss = 0; ss < 2; ++ss) {
                const int s = ss == 0 ? (Sp * j) / q : (Sp * j + q - 1) / q;
                if (ss == 1 && s == (Sp * j) / q) continue;
                const int sr = Sp - s;
                if (s < j || sr < jr || s > M * j || sr > M * jr) continue;
                for (int kk = 0; kk < 3; ++kk) {
                    const int l1 = (l * s) / Sp + kk - 1;
                    const int l2 = l - l1;
                    if (l1 < 2 || l2 < 2 || s > l1 || sr > l2 || j > l1 || jr > l2) continue;
                    const Cell4 *lc = g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + c_ipart(M, l1) +
                                      c_woff(M, l1, j) + (s - j);
                    const Cell4 *rc = g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] +
                                      c_ipart(M, l2) + c_woff(M, l2, jr) + (sr - jr);
                    const Cell4 L = d_load(lc), R = d_load(rc);
                    const double cL = __dadd_rn(L.C1, (double)(3 * sr));
                    const double cR = __dadd_rn(R.C1, (double)(4 * s));
                    const double tot = split_total(L.T1, L.T3, L.TS, cL, R.T1, R.T3, R.TS, cR);
                    const unsigned long long tb = (unsigned long long)__double_as_longlong(tot);
                    const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) | (uint32_t)s;
                    if (lex_less(tb, key, bb, bk)) { bb = tb; bk = key; }
                }
            }
        }
    }
    // warm start: the argmin splits (l1', j', s') of the same output (q, S') on the two
    // length-(l-2) sub-ranges [u, u+l-2) and [u+2, u+l), shifted to [u, u+l)
    if (q >= 2 && l >= 8) {
        const int64_t pc = (int64_t)p * g.C;
        const int lp = l - 2;
        const int Qp = max(1, g.n_hi - 1);
        if (q <= Qp && q <= lp && Sp <= min(lp, M * q)) {
#pragma unroll 1
            for (int side = 0; side < 2; ++side) {
                const int up = u + 2 * side;
                const uint32_t arg = g.ARG[pc + g.base[lp] + (int64_t)up * g.cells[lp] + c_ipart(M, lp) +
                                           c_woff(M, lp, q) + (Sp - q)];
                if (arg >= 0xFFFFFFFEu) continue;
                const int l1p = (int)(arg & 1023u) + 1 + 2 * side, j = (int)((arg >> 10) & 1023u) + 1;
                const int s = (int)(arg >> 20);
                const int jr = q - j, sr = Sp - s;
#pragma unroll 1
                for (int d = 0; d < 3; ++d) {
                    const int l1 = l1p + d - side;   // shifts 0..2 (left range) / 1..3 - 1 (right)
                    const int l2 = l - l1;
                    if (l1 < 2 || l2 < 2 || s > l1 || sr > l2 || j > l1 || jr > l2 || jr < 1) continue;
                    const Cell4 *lc = g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + c_ipart(M, l1) +
                                      c_woff(M, l1, j) + (s - j);
                    const Cell4 *rc = g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] +
                                      c_ipart(M, l2) + c_woff(M, l2, jr) + (sr - jr);
                    if (s < j || sr < jr || s > M * j || sr > M * jr) continue;
                    const Cell4 Lc = d_load(lc), Rc = d_load(rc);
                    const double cL = __dadd_rn(Lc.C1, (double)(3 * sr));
                    const double cR = __dadd_rn(Rc.C1, (double)(4 * s));
                    const double tot = split_total(Lc.T1, Lc.T3, Lc.TS, cL, Rc.T1, Rc.T3, Rc.TS, cR);
                    const unsigned long long tb = (unsigned long long)__double_as_longlong(tot);
                    const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) | (uint32_t)s;
                    if (lex_less(tb, key, bb, bk)) { bb = tb; bk = key; }
                }
            }
        }
    }
    __stcg(f.GSEED + t, make_ulonglong2(bb, (unsigned long long)bk));
    return;
}

// Small cells of wave f.ls: block `bid` of the small part (256 threads, f.tpc <= 32 threads per cell).
__device__ __forceinline__ void fin_small_block(const DevGeom &g, const FinArgs &f, int64_t bid) {
    const int l = f.ls;
    const int nr = g.L - l + 1;
    const int cpb = blockDim.x / f.tpc;                      // cells per block
    const int sub = threadIdx.x / f.tpc, tl = threadIdx.x % f.tpc;
    const int64_t cell = bid * cpb + sub;
    const bool active = cell < (int64_t)g.P * nr * f.nsmall;
    double best = D_INF;
    uint32_t bkey = 0xFFFFFFFFu;
    int u = 0, p = 0, a = 0, Sp = 0;
    if (active) {
        int rem = (int)(cell % f.nsmall);
        u = (int)((cell / f.nsmall) % nr);
        p = (int)(cell / ((int64_t)f.nsmall * nr));
        const int nsm = min(g.A, g.M);                       // alloc indices 0..M-1: I(1..M-1), W(1)
        for (int aa = 0; aa < nsm; ++aa) {
            const int c = max(0, d_hi(g, aa, l) - 1);
            if (rem < c) { a = aa; Sp = 2 + rem; break; }
            rem -= c;
        }
        const int64_t pc = (int64_t)p * g.C;
        const double dSp3 = (double)(3 * Sp - 1);
        const int r = d_is_whole(g, a) ? g.M : d_alloc_n(g, a);  // GPUs of the cell's node part
        const int nd = r - 1;                                    // device splits (I(m), I(r-m))
        // a thread takes layer splits l1 = 1 + tl, 1 + tl + tpc, ... and, for each, every
        // device split m and stage split s (ascending, strict "<": the first minimum in
        // (k, m, s) order).  I(m) of a slab of length l' starts at c_ipart(m, l') (I(1..m-1)
        // before it; W(1) plays "I(M)" right after I(M-1)).
        const Cell4 *CP = g.CELL + pc;
        for (int l1 = 1 + tl; l1 < l; l1 += f.tpc) {
            const int k = u + l1, l2 = l - l1;
            const Cell4 *lrow = CP + g.base[l1] + (int64_t)u * g.cells[l1] - 1;
            const Cell4 *rrow = CP + g.base[l2] + (int64_t)k * g.cells[l2] - 1;
            for (int m = 1; m <= nd; ++m) {
                const int s_lo = max(1, Sp - min(l2, r - m));
                const int s_hi = min(Sp - 1, min(l1, m));
                const Cell4 *lb = lrow + c_ipart(m, l1);
                const Cell4 *rb = rrow + c_ipart(r - m, l2) + Sp;
                for (int s = s_lo; s <= s_hi; ++s) {
                    const Cell4 Lc = d_load(lb + s);
                    const Cell4 Rc = d_load(rb - s);
                    const double T1 = __dadd_rn(Lc.T1, Rc.T1);
                    const bool left = Lc.TS >= Rc.TS;
                    const double T3 = left ? __dadd_rn(Lc.T3, Rc.T1) : Rc.T3;
                    const double TS = left ? Lc.TS : Rc.TS;
                    const double KD = left ? d_kd(Lc.C1, s) : __dadd_rn((double)s, d_kd(Rc.C1, Sp - s));
                    const double T2 = __dmul_rn(__dadd_rn(KD, dSp3), TS);
                    const double tot = __dadd_rn(__dadd_rn(T1, T2), T3);
                    if (tot < best) {
                        best = tot;
                        bkey = ((uint32_t)l1 << 20) | ((uint32_t)(m - 1) << 10) | (uint32_t)s;
                    }
                }
            }
        }
    }
    // lexicographic (total, key) reduction over the tpc threads of the cell (segments of
    // width tpc <= 32 inside a warp)
    const int wd = min(f.tpc, 32);
    for (int d = wd >> 1; d >= 1; d >>= 1) {
        const double ob = __shfl_down_sync(0xFFFFFFFFu, best, d, wd);
        const uint32_t ok = __shfl_down_sync(0xFFFFFFFFu, bkey, d, wd);
        if (ob < best || (ob == best && ok < bkey)) { best = ob; bkey = ok; }
    }
    if (tl != 0) return;
    if (!active) return;
    d_write_winner(g, (int64_t)p * g.C, Sp, u, l, a, (int)(bkey >> 20), (int)((bkey >> 10) & 1023u),
                   (int)(bkey & 1023u));
}

__global__ void __launch_bounds__(256) k_fin(DevGeom g, FinArgs f) {
    if ((int)blockIdx.x < f.nbw) {
        const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (t < (int64_t)g.P * f.nranges_w * f.nout_w) fin_w_one(g, f, t);
        return;
    }
    if ((int)blockIdx.x < f.nbw + f.nbseed) {
        fin_seed_one(g, f, (int64_t)(blockIdx.x - f.nbw) * blockDim.x + threadIdx.x);
        return;
    }
    fin_small_block(g, f, (int64_t)blockIdx.x - f.nbw - f.nbseed);
}

template <int TE>
__global__ void __launch_bounds__(NTW, 2) k_wave_w(DevGeom g, WaveW w) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_last;
    if ((int)blockIdx.x >= w.nbmain) {        // next wave's seeds and in-node cells
        const int ab = (int)blockIdx.x - w.nbmain;
        if (ab < w.fa.nbseed)
            fin_seed_one(g, w.fa, (int64_t)ab * NTW + threadIdx.x);
        else
            fin_small_block(g, w.fa, (int64_t)ab - w.fa.nbseed);
        return;
    }
    const int l = w.l;
    const int nout = w.nout;
    const int L = g.L, M = g.M;
    const int ndum = L + 2 * TE + 2;                              // dummy entries
    ulonglong2 *acc = reinterpret_cast<ulonglong2 *>(smem);     // [nout] + dummy[ndum]
    unsigned *filt = reinterpret_cast<unsigned *>(acc + nout + ndum);  // [nout + ndum] high words
    int4 *sents = reinterpret_cast<int4 *>(filt + ((nout + ndum + 3) & ~3));   // [nents] (16 B aligned)
    int64_t *sbase = reinterpret_cast<int64_t *>(sents + w.nents);               // [L+2]
    int *scells = reinterpret_cast<int *>(sbase + L + 2);        // [L+1]
    int *outOff = scells + (L + 1);                              // [L+2] W(q) offsets (nout: none)
    int *upre = outOff + (L + 2);                                // [nents + 1]
    // per-warp streamed-side rings (16 B aligned) after upre
    const size_t ring_off = ((size_t)(reinterpret_cast<unsigned char *>(upre + w.nents + 1) - smem) + 15) & ~(size_t)15;
    double2 *rings = reinterpret_cast<double2 *>(smem + ring_off);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int pr = blockIdx.x / w.cpr;
    const int u = pr % w.nranges;
    const int p = pr / w.nranges;
    const int64_t pc = (int64_t)p * g.C;
    const int Ql = (l == L) ? g.n_hi : max(1, g.n_hi - 1);

    const ulonglong2 *gseed = w.GACC + ((size_t)(blockIdx.x / w.cpr)) * nout;   // this range's entries
    for (int i = tid; i < nout + ndum; i += NTW) {
        const bool real = i < nout;
        ulonglong2 a = real ? make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull) : make_ulonglong2(0ull, 0ull);
        if (real && w.seeded) a = __ldcg(gseed + i);
        acc[i] = a;
        filt[i] = real ? (unsigned)(a.x >> 32) : 0u;
    }
    for (int i = tid; i < L + 2; i += NTW) {
        sbase[i] = g.base[i];
        if (i <= L) scells[i] = g.cells[i];
        outOff[i] = (i >= 2 && i <= Ql && i <= l) ? c_woff(M, l, i) : nout;
    }
    for (int i = tid; i <= w.nents; i += NTW) {
        upre[i] = w.upre[i];
        if (i < w.nents) sents[i] = w.ents[i];
    }
    __syncthreads();
    const int nunits = w.unit_hi;
    const unsigned acc_s = (unsigned)__cvta_generic_to_shared(acc);
    const unsigned filt_s = (unsigned)__cvta_generic_to_shared(filt);
    int *gctr = w.ctr + pr;

    for (;;) {
        int un = 0;
        if (lane == 0) un = w.unit_lo + w.rank + w.world * atomicAdd(gctr, 1);
        un = __shfl_sync(0xFFFFFFFFu, un, 0);
        if (un >= nunits) break;
        if (w.perm_a > 1)    // visit the queue in a pseudo-random order (a permutation of the pass's units)
            un = w.unit_lo + (int)(((long long)(un - w.unit_lo) * w.perm_a) % (nunits - w.unit_lo));
        int lo = 0, hi = w.nents - 1;                // entry: upre[ei] <= un < upre[ei+1]
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (upre[mid] <= un) lo = mid; else hi = mid - 1;
        }
        const int ei = lo;
        const int4 en = sents[ei];
        const int l1 = en.x & 0xFFFF;
        const int local = un - upre[ei];
        const int chunk = local / en.y;
        const int blk = local % en.y;
        const int r_lo = w.cb[en.w + chunk], r_hi = w.cb[en.w + chunk + 1];
        const int k = u + l1;
        const int l2 = l - l1;
        const bool ltiled = (en.x >> 16) & 1;                     // tiled side = left child
        const int ls = ltiled ? l2 : l1;                           // small side length
        const int lb = ltiled ? l1 : l2;
        const int us = ltiled ? k : u;                             // small slab start
        const int ub = ltiled ? u : k;
        const int ti = blk * 32 + (w.rev_lanes ? 31 - lane : lane);
        const bool has = ti < w.tile_cnt[lb];
        const int32_t code = has ? w.tiles[w.tile_off[lb] + ti] : 0;
        const int rowB = has ? (code >> 16) : 1;
        const int e0 = has ? (code & 0xFFFF) : 0;
        const int lenB = has ? c_wlen(M, lb, rowB) : 0;
        const int ncell = max(0, min(TE, lenB - e0));             // valid cells of the tile
        const Cell4 *bp = g.CELL + pc + sbase[lb] + (int64_t)ub * scells[lb] + c_ipart(M, lb) +
                          (has ? c_woff(M, lb, rowB) : 0) + e0;
        // register tile: T1, T3, t*, C1 of TE big-side cells (sentinels beyond the row)
        double RT1[TE], RT3[TE], RTS[TE], RC1[TE];
#pragma unroll
        for (int t = 0; t < TE; ++t) {
            if (t < ncell) {
                const Cell4 c = d_load(bp + t);
                RT1[t] = c.T1; RT3[t] = c.T3; RTS[t] = c.TS; RC1[t] = c.C1;
            } else {
                RT1[t] = D_INF; RT3[t] = D_INF; RTS[t] = D_INF; RC1[t] = 1.0;
            }
        }
        const Cell4 *sp = g.CELL + pc + sbase[ls] + (int64_t)us * scells[ls] + c_ipart(M, ls);
        XRing xr;                                            // rows r_lo.. are contiguous
        xr_start(xr, rings + (size_t)(tid >> 5) * (XR_BYTES / 16), sp + c_woff(M, ls, r_lo), lane);
        if (ltiled)
            run_rows<TE, true>(xr, M, ls, r_lo, r_hi, RT1, RT3, RTS, RC1, rowB, e0, l1, L, outOff, nout, acc_s,
                               filt_s);
        else
            run_rows<TE, false>(xr, M, ls, r_lo, r_hi, RT1, RT3, RTS, RC1, rowB, e0, l1, L, outOff, nout, acc_s,
                                filt_s);
    }
    __syncthreads();
    // merge into the range's global accumulator (L2-coherent loads; a stale value is an
    // upper bound of the current one, so the CAS loop stays exact).  Loads are batched so
    // their latencies overlap.
    ulonglong2 *ga = w.GACC + ((size_t)p * w.nranges + u) * nout;
    constexpr int MB = 4;
    for (int i0 = tid; i0 < nout; i0 += MB * NTW) {
        ulonglong2 a[MB], cur[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int i = i0 + j * NTW;
            a[j] = i < nout ? acc[i] : make_ulonglong2(ACC_EMPTY, 0ull);
            cur[j] = a[j].x < ACC_EMPTY ? __ldcg(ga + i) : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int i = i0 + j * NTW;
            while (lex_less(a[j].x, (uint32_t)a[j].y, cur[j].x, (uint32_t)cur[j].y)) {
                unsigned long long ox, oy;
                cas128_global(ga + i, ox, oy, cur[j].x, cur[j].y, a[j].x, a[j].y);
                if (ox == cur[j].x && oy == cur[j].y) break;
                cur[j].x = ox;
                cur[j].y = oy;
            }
        }
    }
    if (w.fin_inline) {                        // the range's last CTA finalizes its W outputs
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(w.rdone + pr, 1) == w.cpr - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            fin_w_range<NTW>(g, w.fw, pr, tid);
        }
    }
}

__global__ void k_gacc_init(ulonglong2 *gacc, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) gacc[i] = make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull);
}

}  // namespace oob
