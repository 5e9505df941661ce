// Wavefront kernels for cells with S' >= 2 (the hot loop).
//
// k_wave_w — whole-node cells W(q >= 2) of wavefront l.  For a range (u, v) and a layer
// split k (l1 = k-u, l2 = v-k), W(q) cells combine left children W(j) of (u, k) with right
// children W(q-j) of (k, v) (PAPER Eq.1-3, two-level device split: reading R2).  In
// (nodes, stages) coordinates every pair (left cell, right cell) is a valid split of
// exactly one parent (q = j + j', S' = s + S_R): each row pair (j, j') is a dense rectangle.
//   * Work: per wave one unit queue (layer split k, chunk of streamed rows, block of 32
//     register tiles of TE cells), balanced splits first; `cpr` CTAs per (profile, range)
//     pull units; a lane streams its unit's rows cell by cell (all lanes the same cell,
//     from a per-warp shared-memory ring filled by cp.async) against its TE tile cells.
//   * Screen: per split a binary32 lower bound of the binary64 total from the children's
//     round-down shadows (6 FMA/ALU instructions, no FP64); per output (slot ring: outputs
//     slide by one cell per step) the minimum bound is compared with the output's filter
//     F(min) = float_ru(min (1 + 2^-40)); the bound never exceeds the total by more than
//     2^-43, so winners and ties always pass (derivation: DESIGN.md §6; checked against the
//     oracle by tests/test_filter_bound.py).
//   * Exact path: passing outputs are queued per warp and re-evaluated in binary64 in the
//     oracle's operation order, one output per lane, merged as the lexicographic minimum of
//     (total, key) with a 128-bit CAS into the CTA's accumulator (exact under any
//     interleaving: the key l1<<20 | j<<10 | s is monotone in the oracle's (k, m, s) order,
//     so the lexicographic minimum is the oracle's first strict minimum).
//   * End: the CTA merges its improved entries into the range's global accumulator; the
//     range's co-resident CTAs then finalize the winners' cells in shares; extra blocks of
//     the launch compute the next wave's in-node cells and seeds.  Single-profile sets
//     pipeline the waves (programmatic dependent launches + per-wave counters).
//
// k_fin — per wavefront (unfused / sharded modes and wave 2): the winners of the W(q >= 2)
// cells of wave l, the in-node cells (I(r), W(1)) of wave l+1 and the seeds of wave l+1.
#pragma once

#include "oob_dp_common.cuh"

namespace oob {

constexpr int NTW = 256;                                          // threads per k_wave_w CTA
#ifndef OOB_WAVE_MINB
#define OOB_WAVE_MINB 2
#endif
constexpr int WAVE_CTAS_PER_SM = OOB_WAVE_MINB;                   // register budget: 65536 / (256 x this)
constexpr unsigned long long ACC_EMPTY = 0x7FEFFFFFFFFFFFFFull;   // DBL_MAX: "no split yet"
constexpr double D_INF = __builtin_huge_val();
constexpr unsigned long long ACC_DIRTY = 1ull << 32;   // accumulator key word: improved by this CTA

// Wavefront pipeline state (see pipe_wait below)
struct Pipe {
    int *cnt;              // [3][L+2]: seeds, in-node cells, finalize shares done per wave
    const int *expc;       // [3][L+2]: the counts that make each part ready
    int *err;              // timeout flag (k_extract turns it into a template status: OOB_E_CUDA)
    int on;
    long long spin_max;    // polls before a wait gives up (~200 ns each)
};

#ifndef OOB_MAX_WORLD
#define OOB_MAX_WORLD 8
#endif

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
    unsigned *GFW, *GFS;           // global filters (binary32 bits of F(min)) of waves lw / lseed
    int ls, nsmall;                // small cells of wave ls (ls = 0: none); cells per range
    int tpc;                       // threads per small cell
    int small_range;               // 1: one warp per (profile, range) stages the child I-parts in smem
};

struct WaveW {
    int l;                 // wavefront length
    int nranges;           // L - l + 1
    int cpr;               // CTAs per (profile, range); they share the range's unit queue
    int nents;             // layer splits k with work (balanced splits first)
    const int4 *ents;      // per entry: (l1, nblocks, nchunks, chunk_off)
    const int32_t *upre;   // [nents + 1] unit prefix: entry e owns units [upre[e], upre[e+1])
    const int32_t *cb;     // chunk row boundaries: rows [cb[off+c], cb[off+c+1])
    int ncb;               // entries of cb (staged in shared memory)
    int *ctr;              // [P][nranges] unit counters (zeroed before the launch)
    int nunits;            // units of the range's queue
    int seeded;            // 1: start from the global accumulator (the seeds' minima)
    int rank, world;       // single-profile sharding: this rank takes units rank, rank+world, ...
    int nout;              // W-part cells of a slab of length l (W(1)..W(Q_l))
    ulonglong2 *GACC;      // global accumulator [P][nranges][nout]: {total bits, key}
    unsigned *GFILT;       // global filter [P][nranges][nout]: F(min) over every CTA's improvements
    const int32_t *tile_off;   // [L+1] offset of the flat tile list of a big side of length lb
    const int32_t *tile_cnt;   // [L+1] number of tiles
    const int32_t *tiles;      // packed (row << 16 | e0)
    // fused finalize (unsharded waves): blocks >= nbmain run the in-node cells and seeds of
    // the next wave (fa: nbw = 0; independent of this wave, they fill its tail); the last CTA
    // of each range (rdone counter) finalizes the range's W outputs of this wave (fw: lw = l)
    int nbmain;
    int fin_inline;
    int *rdone;                // [P][nranges] CTAs of the range that have merged
    int *rclaim;               // [P][nranges] finalize shares claimed
    Pipe pp;                   // wavefront pipeline (pp.on = 0: plain kernel boundaries)
    int refresh;               // 1: each unit refreshes its filter entries from the range's global filter
    int fin_spin;              // polls a merged CTA waits for its range's others (0: exit; the last finalizes alone)
    int fin_helpers;           // the range's last fin_helpers merged CTAs wait (for the others / the ranks) and share the finalize
    int warp_mode;             // 1: one WARP per (profile, range) (batched sweeps' short waves: the
                               // per-range work is a few units, a CTA per range idles on its prologue,
                               // barrier and finalize); no pipeline, cpr = 1, no merge
    int prefetch;              // 1: each unit prefetches its tile and chunk cells into L1 (one CTA per range)
    // fused exchange over NVLink peer memory (single-profile sharding, oob_dp_set_comm):
    // the range's last local CTA stores the range's partial argmins into every rank's
    // gather slot of this rank (plain remote stores), fences, and counts itself in every
    // rank's per-range counter; the finalize waits for all ranks' partials (epoch-based
    // counters, never reset) and takes the lexicographic minimum over them
    int peer;                  // 1: this wave exchanges through peer memory
    unsigned epoch;            // run number (counter targets epoch x world)
    ulonglong2 *xpart[OOB_MAX_WORLD];   // rank r's gather buffer of this wave (slot of this rank: + rank * part_stride)
    int *xdone[OOB_MAX_WORLD];          // rank r's per-range "ranks published" counters of this wave
    FinArgs fa, fw;
};

__device__ __forceinline__ int L_of(const DevGeom &g) { return g.L; }

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

// ---------------------------------------------------------------- closed-form slab geometry
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

// diagnostic counters (outputs whose bound passed the filter, CAS successes): compiled in
// with -DOOB_FLUSH_STATS (scripts/flush_stats.py), enabled by oob_dbg_flush_stats
__device__ unsigned long long g_flush_stats[4];
__device__ int g_flush_stats_on;

// diagnostic timeline (compiled in with -DOOB_TIMELINE, scripts/timeline.py): per wave the
// global-timer ns of [0] first main-CTA start, [1] first CTA past its prologue waits, [2] last
// CTA done with its units, [3] last CTA done (finalize included), [4] first aux block start,
// [5] last aux block end, [6] last seed block end, [7] last in-node block end
#ifdef OOB_TIMELINE
__device__ unsigned long long g_tl[1024][8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define OOB_TL_MIN(l, i) atomicMin(&g_tl[l][i], gtime())
#define OOB_TL_MAX(l, i) atomicMax(&g_tl[l][i], gtime())
#else
#define OOB_TL_MIN(l, i) ((void)0)
#define OOB_TL_MAX(l, i) ((void)0)
#endif

// ---------------------------------------------------------------- exact filter (fast path)
// A split's binary64 total is bounded from below by a binary32 expression of the children's
// shadows (oob_dp_common.cuh d_shadow; every operation rounds toward -inf):
//   left child X, right child Y, s = stages of X, S_Y = stages of Y,
//   totL = A_X + 3 S_Y X.t* + 2 Y.T1   (= the total when X holds the slowest stage)
//   totR = A_Y + 4 s Y.t* + X.T1       (= the total when Y holds it)
//   lb   = (X.t*_f >= Y.t*_f) ? totL : totR
// (expand Eqs.1-3 with C1 = 3S'-1+k*: T1 + (C1_X + 3 S_Y) X.t* + X.T3 + Y.T1, resp.
// T1 + (C1_Y + 4 s) Y.t* + Y.T3).  Rounding t* down is monotone, so the binary32 compare
// can only misjudge an exact tie of the rounded t*'s, where X.t* < Y.t* and lb takes totL:
// then totL <= totR + 2^-44 totR, because X.T3 sums s - k*_X stages <= X.t* and
// Y.T1 - Y.T3 sums k*_Y stages <= Y.t* (up to the binary64 rounding of those sums, <= 192 ulp).
// The binary64 total is >= (1 - 3u) times the real expression, so a split can reach a
// current minimum m (its total <= m) only if lb <= m (1 + 2^-43).  The filter therefore
// compares lb with F(m) = float_ru(m (1 + 2^-40)) and never drops a winner or a tie.
constexpr unsigned FILT_EMPTY = 0x7F7FFFFFu;   // FLT_MAX: nothing known yet
__device__ __forceinline__ float filt_of(unsigned long long bits) {
    if (bits >= 0x7FEFFFFFFFFFFFFFull) return 3.402823466e38f;   // empty entry: FLT_MAX
    return __double2float_ru(__dmul_ru(__longlong_as_double((long long)bits), 1.0 + 0x1p-40));
}

// Streamed side staging: a per-warp ring of XR_CELLS shadow cells (float4) in shared memory,
// filled with cp.async in batches of XR_BATCH cells (512 B: one 16-byte copy per lane)
// issued XR_AHEAD batches ahead of the step loop, so the steps read the streamed shadow
// from shared memory (broadcast LDS.128).  The first XR_MIRROR cells of the ring are
// mirrored after its end, so the TE cells a block of steps reads are contiguous (one base
// address per block, immediate offsets).  Copies are unguarded: a chunk's last batches may
// read past the slab (the SH allocation is padded by XR_CELLS cells).
#ifndef OOB_XR_BATCH
#define OOB_XR_BATCH 32
#endif
#ifndef OOB_XR_AHEAD
#define OOB_XR_AHEAD 2
#endif
constexpr int XR_BATCH = OOB_XR_BATCH;                  // cells per copy batch (<= 32: one 16-B copy per lane)
constexpr int XR_AHEAD = OOB_XR_AHEAD;                  // batches in flight ahead of the steps
constexpr int xr_pow2(int x) { return x <= 1 ? 1 : 2 * xr_pow2((x + 1) / 2); }
constexpr int XR_CELLS = xr_pow2(XR_BATCH * (XR_AHEAD + 2));   // ring: >= the batch in use, the previous one
                                                                // and XR_AHEAD in flight (power of two)
static_assert(XR_BATCH <= 32 && (XR_BATCH & (XR_BATCH - 1)) == 0, "one 16-B copy per lane per batch");
constexpr int XR_MIRROR = 8;
constexpr int XR_BYTES = (XR_CELLS + XR_MIRROR) * 16;   // per warp

struct XRing {
    const float4 *ring;                   // this warp's ring (shared memory)
    unsigned ring_s;                      // its shared-space address + lane * 16
    const char *src;                      // chunk start (global shadow) + lane * 16
    int nb_iss, nb_ok;                    // batches issued / complete
    bool mirror;                          // this lane also writes a mirror cell
};

__device__ __forceinline__ void xr_issue(XRing &r) {
    const int b = r.nb_iss++;
    const unsigned pos = (unsigned)((b * XR_BATCH) & (XR_CELLS - 1)) * 16u;
    const char *g = r.src + (size_t)b * (XR_BATCH * 16);
    if (XR_BATCH == 32 || (threadIdx.x & 31) < XR_BATCH)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(r.ring_s + pos), "l"(g) : "memory");
    if (pos == 0 && r.mirror)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(r.ring_s + XR_CELLS * 16u), "l"(g) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void xr_start(XRing &r, const float4 *ring, const float4 *src, int lane) {
    r.ring = ring;
    r.ring_s = (unsigned)__cvta_generic_to_shared(ring) + lane * 16;
    r.src = reinterpret_cast<const char *>(src) + lane * 16;
    r.mirror = lane < XR_MIRROR;
    r.nb_iss = 0;
    r.nb_ok = 0;
#pragma unroll
    for (int i = 0; i <= XR_AHEAD; ++i) xr_issue(r);
}
// make cells <= j available (warp-uniform; j grows by <= XR_BATCH between calls)
__device__ __forceinline__ void xr_ensure(XRing &r, int j) {
    if (j / XR_BATCH >= r.nb_ok) {
        // lanes diverge on the exact path: none may still read the region this copy
        // overwrites (write-after-read across lanes)
        __syncwarp();
        xr_issue(r);
        asm volatile("cp.async.wait_group %0;" ::"n"(XR_AHEAD) : "memory");
        __syncwarp();                     // the other lanes' copies are visible
        r.nb_ok = r.nb_iss - XR_AHEAD;
    }
}
// cells c .. c + XR_MIRROR of the ring as one contiguous run
__device__ __forceinline__ const float4 *xr_at(const XRing &r, int c) { return r.ring + (c & (XR_CELLS - 1)); }

// Lower bound of one split from the tile shadow (TA/TB/TS/TC, lane constants) and the
// streamed shadow x (see the filter derivation above); fst = LT ? 3 S_R : 4 s.
template <bool LT>
__device__ __forceinline__ float split_lb(float TA, float TB, float TS, float TC, const float4 x, float fst) {
    if (LT) {   // tile X: TA = A_X, TB = X.T1, TS = X.t*, TC = 4 s; x = Y
        const float tl = __fadd_rd(__fmaf_rd(fst, TS, TA), x.w);
        const float tr = __fmaf_rd(TC, x.z, __fadd_rd(x.x, TB));
        return TS >= x.z ? tl : tr;
    } else {    // tile Y: TA = A_Y, TB = 2 Y.T1, TS = Y.t*, TC = 3 S_Y; x = X
        const float tl = __fadd_rd(__fmaf_rd(TC, x.z, x.x), TB);
        const float tr = __fmaf_rd(fst, TS, __fadd_rd(TA, x.y));
        return x.z >= TS ? tl : tr;
    }
}

// Candidate queue: the outputs whose slot bound passes the filter are not re-evaluated in
// place (divergent, global-latency bound) but appended to a per-warp queue in shared memory
// and re-evaluated by the whole warp, one output per lane, when the queue is full and at the
// end of each unit.  An entry (20 B) names one output E' of one (tile, streamed row) pair:
//   x = tile cell index, y = streamed row's first cell index, z = key base kb,
//   w = accumulator entry (16 bits) | ncell << 16 | LT << 19,
//   v = (the stage count the key does not carry: LT: rs, else S0; 10 bits) | E' << 10 | rl << 21
// (11 bits each: rows hold <= L <= 1023 cells, E' <= rl + TE - 2; the accumulator entries of
// a wave, nout + dummies, are < 2^16 — oob_dp_plan_create falls back to k_wave_v1 otherwise).
constexpr int XQ_CAP = 32;
constexpr int XQ_BYTES = XQ_CAP * 20;     // per warp

// Exact evaluation of the queued outputs (warp-collective; lane i takes entry i): every
// valid contribution t (tile cell t, streamed cell e = E' - t) in binary64 in the oracle's
// operation order, the lexicographic minimum of (total, key), merged with the 128-bit CAS
// into the CTA's accumulator entry (entries only decrease: a stale read is an upper bound,
// the loop stays exact); then the CTA's and the range's global filters are lowered.
//  LT = true : tile = LEFT child (s = S0 + t), stream = RIGHT child (S_R = rs + e);
//              key = kb + t, kb = l1<<20 | rowB<<10 | S0.
//  LT = false: tile = RIGHT child (S_R = S0 + t), stream = LEFT child (s = rs + e);
//              key = kb + e, kb = l1<<20 | rs<<10 | rs.
template <int TE>
__device__ __noinline__ void xq_flush(const uint4 *q4, const unsigned *q1, int count, const Cell4 *CELL,
                                      unsigned acc_s, unsigned filt_s, unsigned *gfr) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    if (lane < count) {
        const uint4 en = q4[lane];
        const unsigned v = q1[lane];
        const int idx = (int)(en.w & 0xFFFFu), ncell = (int)((en.w >> 16) & 7u);
        const bool lt = (en.w >> 19) & 1u;
        const int v0 = (int)(v & 1023u), Ep = (int)((v >> 10) & 2047u), rl = (int)(v >> 21);
        const int rs = lt ? v0 : (int)(en.z & 1023u), S0 = lt ? (int)(en.z & 1023u) : v0;
        unsigned long long bb = ACC_EMPTY;
        uint32_t bk = 0xFFFFFFFFu;
#pragma unroll
        for (int t = 0; t < TE; ++t) {
            const int e = Ep - t;
            if (t < ncell && e >= 0 && e < rl) {
                const Cell4 tc = d_load(CELL + en.x + t), sc = d_load(CELL + en.y + e);
                const Cell4 &Lc = lt ? tc : sc, &Rc = lt ? sc : tc;
                const int sL = lt ? S0 + t : rs + e, sR = lt ? rs + e : S0 + t;   // stages of left / right
                const double cL = __dadd_rn(Lc.C1, (double)(3 * sR));
                const double cR = __dadd_rn(Rc.C1, (double)(4 * sL));
                const double tot = split_total(Lc.T1, Lc.T3, Lc.TS, cL, Rc.T1, Rc.T3, Rc.TS, cR);
                const unsigned long long tb = (unsigned long long)__double_as_longlong(tot);
                const uint32_t key = en.z + (uint32_t)(lt ? t : e);
                if (lex_less(tb, key, bb, bk)) { bb = tb; bk = key; }
            }
        }
        if (bb < ACC_EMPTY) {
            const unsigned addr = acc_s + 16u * (unsigned)idx;
            unsigned long long cx, cy;
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(cx), "=l"(cy) : "r"(addr) : "memory");
#ifdef OOB_FLUSH_STATS
            if (g_flush_stats_on) {
                atomicAdd(&g_flush_stats[0], 1ull);
                if (bb == cx) atomicAdd(&g_flush_stats[2], 1ull);
                else if (bb > cx) atomicAdd(&g_flush_stats[3], 1ull);
                if (bb == cx && bk == (uint32_t)cy) atomicAdd(&g_flush_stats[1], 1ull << 32);   // same split
            }
#endif
            while (lex_less(bb, bk, cx, (uint32_t)cy)) {
                unsigned long long ox, oy;
                cas128_shared(addr, ox, oy, cx, cy, bb, (unsigned long long)bk | ACC_DIRTY);
                if (ox == cx && oy == cy) {
#ifdef OOB_FLUSH_STATS
                    if (g_flush_stats_on) atomicAdd(&g_flush_stats[1], 1ull);
#endif
                    const unsigned fb = __float_as_uint(filt_of(bb));
                    asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(filt_s + 4u * (unsigned)idx), "r"(fb) : "memory");
                    atomicMin(gfr + idx, fb);     // share with the range's other CTAs (refreshed per unit)
                    break;
                }
                cx = ox;
                cy = oy;
            }
        }
    }
    __syncwarp();
}

// Queue the outputs flagged in `mask` (bit b: output E' = base + b of this lane's tile and
// the current streamed row; warp-collective, a no-op when no lane has a bit).
template <int TE, bool LT>
__device__ __noinline__ int xq_push(unsigned mask, int base, unsigned bidx, int ncell, unsigned srow, int rl, int S0,
                                    int rs, uint32_t kb, int idx0, uint4 *q4, unsigned *q1, int count,
                                    const Cell4 *CELL, unsigned acc_s, unsigned filt_s, unsigned *gfr) {
    const unsigned lane_lt = (1u << (threadIdx.x & 31)) - 1u;
    for (;;) {
        const bool h = mask != 0;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, h);
        if (!bal) break;
        const int n = __popc(bal);
        if (h) {
            const int slot = count + __popc(bal & lane_lt);
            if (slot < XQ_CAP) {           // lanes past a full queue keep their bit for the next round
                const int Ep = base + __ffs(mask) - 1;
                mask &= mask - 1;
                q4[slot] = make_uint4(bidx, srow, kb,
                                      (unsigned)(idx0 + Ep) | ((unsigned)ncell << 16) | (LT ? 1u << 19 : 0u));
                q1[slot] = (LT ? (unsigned)rs : (unsigned)S0) | ((unsigned)Ep << 10) | ((unsigned)rl << 21);
            }
        }
        count = min(count + n, XQ_CAP);
        if (count == XQ_CAP) {              // flush full queues only
            xq_flush<TE>(q4, q1, count, CELL, acc_s, filt_s, gfr);
            count = 0;
        }
    }
    return count;
}


// One step (streamed cell x, uniform factor fst: LT 3 S_R, else 4 s) of a lane's TE splits:
// lower bounds into the ring slots (output E' = e + t lives in slot E' mod TE; its first
// contribution t = TE-1 assigns the slot).
template <int TE, bool LT>
__device__ __forceinline__ void fast_step(const float4 x, float fst, int I, const float (&TA)[TE],
                                          const float (&TB)[TE], const float (&TS)[TE], const float (&TC)[TE],
                                          float (&mn)[TE]) {
#pragma unroll
    for (int t = 0; t < TE; ++t) {
        const int sl = (I + t) % TE;
        const float lb = split_lb<LT>(TA[t], TB[t], TS[t], TC[t], x, fst);
        mn[sl] = (t == TE - 1) ? lb : fminf(mn[sl], lb);
    }
}

// Pass bits (bit r + d) of the pending outputs E' = rl + d, d = 0..TE-2, when rl mod TE = R
// (slot (R + d) mod TE), against their filter entries fp[d].
template <int TE, int R>
__device__ __forceinline__ unsigned pending_mask(const float (&mn)[TE], const float *fp) {
    unsigned pm = 0;
    if (R < TE) {
#pragma unroll
        for (int d = 0; d <= TE - 2; ++d)
            pm |= (mn[(R + d) % TE] <= fp[d]) ? (1u << (R + d)) : 0u;
    }
    return pm;
}

// The small-side rows r_lo..r_hi-1 of one unit against this lane's register tile (shadow
// lower bounds TA/TB/TS/TC; binary64 tile at bp for the exact path).  Each row runs full
// blocks of TE steps (no guards) and a guarded tail; the outputs whose bounds pass the
// filter are collected per block (bit mask) and re-evaluated exactly.
template <int TE, bool LT>
__device__ __forceinline__ int run_rows(XRing &xr, int64_t sidx, const int32_t *wls, int r_lo, int r_hi,
                                        const float (&TA)[TE], const float (&TB)[TE], const float (&TS)[TE],
                                        const float (&TC)[TE], int64_t bidx, int ncell, int rowB, int e0,
                                        int l1, int L, const int *outOff, int nout, unsigned acc_s,
                                        unsigned filt_s, unsigned *gfr, uint4 *q4, unsigned *q1,
                                        const Cell4 *CELL, int qn) {
    static_assert(TE == 4, "the pending-output switch below covers TE = 4");
    // qn: outputs queued so far by this warp (warp-uniform); the queue carries over to the
    // warp's next unit of the same range and is flushed when full or after the last unit
    const int S0 = rowB + e0;
    const float *filt = reinterpret_cast<const float *>(__cvta_shared_to_generic(filt_s));
    int rb = 0;                                           // chunk cell of the row's first cell
    for (int rs = r_lo; rs < r_hi; ++rs) {
        const int rl = __ldg(wls + rs + 1) - __ldg(wls + rs);
        const int q = rowB + rs;
        const int ob = outOff[min(q, L + 1)];
        const int idx0 = (ob == nout) ? nout : ob + e0;  // accumulator entry of E' = 0
        const uint32_t kb = LT ? (((uint32_t)l1 << 20) | ((uint32_t)rowB << 10) | (uint32_t)S0)
                               : (((uint32_t)l1 << 20) | ((uint32_t)rs << 10) | (uint32_t)rs);
        const int64_t srow = sidx + rb;
        const float *fr = filt + idx0;
        float fst = (float)((LT ? 3 : 4) * rs);
        float mn[TE];
#pragma unroll
        for (int t = 0; t < TE; ++t) mn[t] = __int_as_float(0x7f800000);
        int blk = 0;
        const int full = rl - rl % TE;
        unsigned pmask = 0;                               // passed outputs E' = mbase + bit
        int mbase = 0;
#pragma unroll 1
        for (; blk < full; blk += TE) {
            xr_ensure(xr, rb + blk + TE);
            const float4 *xq = xr_at(xr, rb + blk);
            if (blk - mbase > 32 - TE) {                  // the mask window is full: queue it
                if (__any_sync(0xFFFFFFFFu, pmask != 0))
                    qn = xq_push<TE, LT>(pmask, mbase, (unsigned)bidx, ncell, (unsigned)srow, rl, S0, rs, kb, idx0, q4,
                                         q1, qn, CELL, acc_s, filt_s, gfr);
                pmask = 0;
                mbase = blk;
            }
            unsigned pm4 = 0;                             // this block's passes (static bits)
            const float *fb = fr + blk;
#pragma unroll
            for (int I = 0; I < TE; ++I) {
                fast_step<TE, LT>(xq[I], fst, I, TA, TB, TS, TC, mn);
                fst += LT ? 3.0f : 4.0f;
                pm4 |= (mn[I] <= fb[I]) ? (1u << I) : 0u;
            }
            pmask |= pm4 << (blk - mbase);
        }
        // tail block (rl % TE steps) and the pending outputs E' = rl .. rl + TE - 2
        {
            xr_ensure(xr, rb + blk + TE);
            const float4 *xq = xr_at(xr, rb + blk);
            unsigned pm = 0;
#pragma unroll
            for (int I = 0; I < TE - 1; ++I) {
                if (blk + I < rl) {
                    fast_step<TE, LT>(xq[I], fst, I, TA, TB, TS, TC, mn);
                    fst += LT ? 3.0f : 4.0f;
                    pm |= (mn[I] <= fr[blk + I]) ? (1u << I) : 0u;
                }
            }
            // pending outputs E' = rl + d (d = 0..TE-2) live in slot (rl + d) mod TE; rl mod TE
            // is warp-uniform, so a switch branches to one case with static slot indices
            switch (rl - blk) {                           // = rl mod TE
                case 0: pm |= pending_mask<TE, 0>(mn, fr + rl); break;
                case 1: pm |= pending_mask<TE, 1>(mn, fr + rl); break;
                case 2: pm |= pending_mask<TE, 2>(mn, fr + rl); break;
                case 3: pm |= pending_mask<TE, 3>(mn, fr + rl); break;
                default: pm |= pending_mask<TE, 4>(mn, fr + rl); break;
            }
            // the row's last window and its tail / pending outputs in one push when they fit
            if (blk - mbase + 2 * TE - 3 <= 31) {
                pmask |= pm << (blk - mbase);
                pm = 0;
            }
            if (__any_sync(0xFFFFFFFFu, pmask != 0))
                qn = xq_push<TE, LT>(pmask, mbase, (unsigned)bidx, ncell, (unsigned)srow, rl, S0, rs, kb, idx0, q4, q1,
                                     qn, CELL, acc_s, filt_s, gfr);
            if (__any_sync(0xFFFFFFFFu, pm != 0))
                qn = xq_push<TE, LT>(pm, blk, (unsigned)bidx, ncell, (unsigned)srow, rl, S0, rs, kb, idx0, q4, q1, qn,
                                     CELL, acc_s, filt_s, gfr);
        }
        rb += rl;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");   // no copy of this chunk outlives the unit
    __syncwarp();
    return qn;
}

// One warp unit (inlined: an out-of-line unit measured 9% slower on cfg4, and capping the
// kernel at 80 registers for 3 CTAs/SM spills in the step loop, +70%): start the streamed
// chunk's ring, load the register tile (shadow lower bounds
// of TE big-side cells; +inf beyond the row, so a sentinel's bound never passes), refresh
// the filter entries of the outputs [olo, ohi) the unit can touch from the range's global
// filter (minima the range's other CTAs found), then run the rows.
template <int TE, bool LT>
__device__ __forceinline__ int run_unit(const float4 *__restrict__ SH, const Cell4 *CELL, int64_t sidx, const int32_t *wls,
                                     int r_lo, int r_hi, int64_t bidx, int ncell, int rowB, int e0, int l1, int L,
                                     const int *outOff, int nout, unsigned acc_s, unsigned filt_s, unsigned *gfr,
                                     unsigned char *wsm, int olo, int ohi, int qn) {
    const int lane = threadIdx.x & 31;
    uint4 *q4 = reinterpret_cast<uint4 *>(wsm + XR_BYTES);         // this warp's candidate queue
    unsigned *q1 = reinterpret_cast<unsigned *>(q4 + XQ_CAP);
    XRing xr;                                            // rows r_lo.. are contiguous
    xr_start(xr, reinterpret_cast<float4 *>(wsm), SH + sidx, lane);
    float TA[TE], TB[TE], TS[TE], TC[TE];
#pragma unroll
    for (int t = 0; t < TE; ++t) {
        const float inf = __int_as_float(0x7f800000);
        float4 c = make_float4(inf, inf, inf, inf);
        if (t < ncell) c = __ldg(SH + bidx + t);
        TA[t] = c.x;
        TB[t] = LT ? c.y : c.w;
        TS[t] = c.z;
        TC[t] = (float)((LT ? 4 : 3) * (rowB + e0 + t));
    }
    unsigned *filt = reinterpret_cast<unsigned *>(__cvta_shared_to_generic(filt_s));
    for (int i0 = olo + lane; i0 < ohi; i0 += 128) {   // 4 loads in flight per lane
        unsigned gv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) gv[j] = i0 + 32 * j < ohi ? __ldcg(gfr + i0 + 32 * j) : 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (gv[j] < filt[i0 + 32 * j]) atomicMin(filt + i0 + 32 * j, gv[j]);
    }
    return run_rows<TE, LT>(xr, sidx, wls, r_lo, r_hi, TA, TB, TS, TC, bidx, ncell, rowB, e0, l1, L, outOff, nout, acc_s,
                            filt_s, gfr, q4, q1, CELL, qn);
}

// The warp's queued candidates after its last unit of a range.
template <int TE>
__device__ __forceinline__ void flush_rest(unsigned char *wsm, int qn, const Cell4 *CELL, unsigned acc_s, unsigned filt_s,
                                           unsigned *gfr) {
    if (qn) {
        const uint4 *q4 = reinterpret_cast<const uint4 *>(wsm + XR_BYTES);
        xq_flush<TE>(q4, reinterpret_cast<const unsigned *>(q4 + XQ_CAP), qn, CELL, acc_s, filt_s, gfr);
    }
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
        if (d_wofs(g, l, mid) - d_wofs(g, l, 1) <= i) lo = mid; else hi = mid - 1;
    }
    const int q = lo, Sp = q + (i - (d_wofs(g, l, q) - d_wofs(g, l, 1)));
    if (q < 2) return;        // W(1) cell (computed with the small cells)
    ulonglong2 *ga = f.GACC + t;
    ulonglong2 a = __ldcg(ga);
    __stcg(ga, make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull));
    __stcg(f.GFW + t, FILT_EMPTY);
    for (int r = 0; r < f.world && f.world > 1; ++r) {   // lexicographic min over the ranks
        const ulonglong2 b = __ldcg(f.GPART + (int64_t)r * f.part_stride + t);
        if (lex_less(b.x, (uint32_t)b.y, a.x, (uint32_t)a.y)) a = b;
    }
    const int64_t pc = (int64_t)p * g.C;
    const int aW = (g.M - 1) + q - 1;
    if (a.x >= ACC_EMPTY) {   // no finite split: infinite under stage masks, else impossible (poison)
        if (g.masked) d_store_inf(g, pc + d_cell(g, Sp, u, l, aW), Sp);
        else d_poison(g, pc + d_cell(g, Sp, u, l, aW), 0xFFFFFFFEu);
        return;
    }
    const uint32_t key = (uint32_t)a.y;
    const int l1 = (int)(key >> 20), j = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
    // bounds check of the decoded split (a corrupt key must not read outside the table)
    const int l2 = l - l1, jr = q - j, sr = Sp - s;
    if (l1 < 1 || l2 < 1 || j < 1 || jr < 1 || s < j || sr < jr || s > min(l1, g.M * j) ||
        sr > min(l2, g.M * jr)) {
        d_poison(g, pc + d_cell(g, Sp, u, l, aW), 0xFFFFFFFDu);
        return;
    }
    d_write_winner(g, pc, Sp, u, l, aW, l1, j - 1, s);
    return;
}

// The W finalize of one range (profile-range index pr) of wave f.lw by one CTA (k_wave_w's
// last CTA of the range): fin_w_one's steps in three phases over FB outputs per thread
// (accumulator loads; child loads; recompute + store) so their memory latencies overlap.
template <int NT>
__device__ __forceinline__ void fin_w_range(const DevGeom &g, const FinArgs &f, int pr, int tid, int part = 0,
                                            int nparts = 1, const ulonglong2 *sacc = nullptr) {
    // sacc: the range's accumulator in this CTA's shared memory (the range's only CTA); the
    // global entries are then only reset
    constexpr int FB = 4;
    const int l = f.lw, nout = f.nout_w, M = g.M;
    const int u = pr % f.nranges_w, p = pr / f.nranges_w;
    const int64_t pc = (int64_t)p * g.C;
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);
    const int stride = NT * nparts;               // share `part`: outputs part NT + tid + k stride
    for (int i0 = part * NT + tid; i0 < nout; i0 += FB * stride) {
        int q[FB], Sp[FB];
        ulonglong2 a[FB];
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            const int i = i0 + j * stride;
            q[j] = 0;
            Sp[j] = 0;
            a[j] = make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull);
            if (i >= nout) continue;
            int lo = 1, hi = min(Ql, l);
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (d_wofs(g, l, mid) - d_wofs(g, l, 1) <= i) lo = mid; else hi = mid - 1;
            }
            q[j] = lo;
            Sp[j] = lo + (i - (d_wofs(g, l, lo) - d_wofs(g, l, 1)));
            if (lo < 2) continue;
            ulonglong2 *ga = f.GACC + (int64_t)pr * nout + i;
            a[j] = sacc ? sacc[i] : __ldcg(ga);
            for (int r = 0; r < f.world && f.world > 1; ++r) {   // lexicographic min over the ranks' partials
                const ulonglong2 b = __ldcg(f.GPART + (int64_t)r * f.part_stride + (int64_t)pr * nout + i);
                if (lex_less(b.x, (uint32_t)b.y, a[j].x, (uint32_t)a[j].y)) a[j] = b;
            }
            __stcg(ga, make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull));
            __stcg(f.GFW + (int64_t)pr * nout + i, FILT_EMPTY);
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
            if (a[j].x >= ACC_EMPTY) {       // no finite split: infinite under masks, else poison
                if (g.masked) d_store_inf(g, pc + d_cell(g, Sp[j], u, l, aW), Sp[j]);
                else d_poison(g, pc + d_cell(g, Sp[j], u, l, aW), 0xFFFFFFFEu);
                continue;
            }
            const uint32_t key = (uint32_t)a[j].y;
            const int l1 = (int)(key >> 20), jj = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
            const int l2 = l - l1, jr = q[j] - jj, sr = Sp[j] - s;
            if (l1 < 1 || l2 < 1 || jj < 1 || jr < 1 || s < jj || sr < jr || s > min(l1, M * jj) ||
                sr > min(l2, M * jr)) {      // corrupt key: flag, never read outside the table
                d_poison(g, pc + d_cell(g, Sp[j], u, l, aW), 0xFFFFFFFDu);
                continue;
            }
            // children W(jj) of (u, u+l1) and W(jr) of (u+l1, u+l)
            Lc[j] = d_load(g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + d_wofs(g, l1, jj) +
                           (s - jj));
            Rc[j] = d_load(g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] + d_wofs(g, l2, jr) + (sr - jr));
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
            d_store(g, c, __dadd_rn(Lc[j].T1, Rc[j].T1), left ? __dadd_rn(Lc[j].T3, Rc[j].T1) : Rc[j].T3,
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
        if (d_wofs(g, l, mid) - d_wofs(g, l, 1) <= i) lo = mid; else hi = mid - 1;
    }
    const int q = lo, Sp = q + (i - (d_wofs(g, l, q) - d_wofs(g, l, 1)));
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
                Cell4 Lk[3], Rk[3];                         // the 3 l1 candidates' loads in flight together
                bool okk[3];
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    const int l1 = (l * s) / Sp + kk - 1;
                    const int l2 = l - l1;
                    okk[kk] = !(l1 < 2 || l2 < 2 || s > l1 || sr > l2 || j > l1 || jr > l2);
                    if (!okk[kk]) continue;
                    Lk[kk] = d_load(g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + d_wofs(g, l1, j) + (s - j));
                    Rk[kk] = d_load(g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] + d_wofs(g, l2, jr) +
                                    (sr - jr));
                }
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    if (!okk[kk]) continue;
                    const int l1 = (l * s) / Sp + kk - 1;
                    const double cL = __dadd_rn(Lk[kk].C1, (double)(3 * sr));
                    const double cR = __dadd_rn(Rk[kk].C1, (double)(4 * s));
                    const double tot = split_total(Lk[kk].T1, Lk[kk].T3, Lk[kk].TS, cL, Rk[kk].T1, Rk[kk].T3, Rk[kk].TS, cR);
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
            uint32_t args[2];                               // both sides' argmins in flight together
#pragma unroll
            for (int side = 0; side < 2; ++side)
                args[side] = g.ARG[pc + g.base[lp] + (int64_t)(u + 2 * side) * g.cells[lp] + d_wofs(g, lp, q) + (Sp - q)];
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const uint32_t arg = args[side];
                if (arg >= ARG_INF) continue;
                const int l1p = (int)(arg & 1023u) + 1 + 2 * side, j = (int)((arg >> 10) & 1023u) + 1;
                const int s = (int)(arg >> 20);
                const int jr = q - j, sr = Sp - s;
                Cell4 Lk[3], Rk[3];
                bool okk[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const int l1 = l1p + d - side;   // shifts 0..2 (left range) / 1..3 - 1 (right)
                    const int l2 = l - l1;
                    okk[d] = !(l1 < 2 || l2 < 2 || s > l1 || sr > l2 || j > l1 || jr > l2 || jr < 1 || s < j || sr < jr ||
                               s > M * j || sr > M * jr);
                    if (!okk[d]) continue;
                    Lk[d] = d_load(g.CELL + pc + g.base[l1] + (int64_t)u * g.cells[l1] + d_wofs(g, l1, j) + (s - j));
                    Rk[d] = d_load(g.CELL + pc + g.base[l2] + (int64_t)(u + l1) * g.cells[l2] + d_wofs(g, l2, jr) +
                                   (sr - jr));
                }
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (!okk[d]) continue;
                    const int l1 = l1p + d - side;
                    const double cL = __dadd_rn(Lk[d].C1, (double)(3 * sr));
                    const double cR = __dadd_rn(Rk[d].C1, (double)(4 * s));
                    const double tot = split_total(Lk[d].T1, Lk[d].T3, Lk[d].TS, cL, Rk[d].T1, Rk[d].T3, Rk[d].TS, cR);
                    const unsigned long long tb = (unsigned long long)__double_as_longlong(tot);
                    const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) | (uint32_t)s;
                    if (lex_less(tb, key, bb, bk)) { bb = tb; bk = key; }
                }
            }
        }
    }
    __stcg(f.GSEED + t, make_ulonglong2(bb, (unsigned long long)bk));
    __stcg(f.GFS + t, __float_as_uint(filt_of(bb)));
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
    if (tl == 0 && active) {
        if (bkey == 0xFFFFFFFFu) d_store_inf(g, (int64_t)p * g.C + d_cell(g, Sp, u, l, a), Sp);   // masks
        else d_write_winner(g, (int64_t)p * g.C, Sp, u, l, a, (int)(bkey >> 20), (int)((bkey >> 10) & 1023u),
                            (int)(bkey & 1023u));
    }
}

// Small cells of wave f.ls, one WARP per (profile, range) (f.small_range; M <= 8): lane i
// owns the range's in-node cell i (I(r) or W(1), S' >= 2; chunks of 32 when there are
// more) and scans the layer splits l1 ascending — for each, the warp stages the I-parts of
// the two child slabs ([u, u+l1) and [u+l1, v), <= (M-1)M/2 cells each) in shared memory,
// the next l1's cells in flight in registers — then every device split m and stage split s
// ascending with a strict "<": the oracle's first minimum in (k, m, s) order, read from
// shared memory instead of one global load per child (the cells of a range share them).
constexpr int SR_IPMAX = 28;       // (M-1)M/2 for M <= 8
constexpr int SR_SMEM = (NTW / 32) * 2 * SR_IPMAX * 32;   // bytes per 256-thread block
__device__ __forceinline__ void fin_small_range(const DevGeom &g, const FinArgs &f, int64_t bid,
                                                unsigned char *smem) {
    const int l = f.ls, M = g.M;
    const int nr = g.L - l + 1;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t pr = bid * (blockDim.x >> 5) + wi;
    if (pr >= (int64_t)g.P * nr) return;
    const int u = (int)(pr % nr), p = (int)(pr / nr);
    const int64_t pc = (int64_t)p * g.C;
    const Cell4 *CP = g.CELL + pc;
    Cell4 *buf = reinterpret_cast<Cell4 *>(smem) + (size_t)wi * 2 * SR_IPMAX;   // [left I-part][right I-part]
    const int nsm = min(g.A, M);                                   // alloc indices 0..M-1: I(1..M-1), W(1)
    for (int c0 = 0; c0 < f.nsmall; c0 += 32) {
        const int ci = c0 + lane;
        const bool active = ci < f.nsmall;
        int a = 0, Sp = 2;
        if (active) {
            int rem = ci;
            for (int aa = 0; aa < nsm; ++aa) {
                const int c = max(0, d_hi(g, aa, l) - 1);
                if (rem < c) { a = aa; Sp = 2 + rem; break; }
                rem -= c;
            }
        }
        const int r = d_is_whole(g, a) ? M : d_alloc_n(g, a);   // GPUs of the cell's node part
        const double dSp3 = (double)(3 * Sp - 1);
        double best = D_INF;
        uint32_t bkey = 0xFFFFFFFFu;
        // staged cells of layer split l1: lane j holds cells j and j + 32 of [left | right]
        Cell4 nx[2 * ((2 * SR_IPMAX + 31) / 32)];
        auto fetch = [&](int l1) {
            const int l2 = l - l1;
            const int nl = c_ipart(M, l1), nrt = c_ipart(M, l2);
            const Cell4 *lrow = CP + g.base[l1] + (int64_t)u * g.cells[l1];
            const Cell4 *rrow = CP + g.base[l2] + (int64_t)(u + l1) * g.cells[l2];
#pragma unroll
            for (int t = 0; t < (int)(sizeof(nx) / sizeof(nx[0])); ++t) {
                const int i = lane + 32 * t;
                if (i < nl) nx[t] = d_load(lrow + i);
                else if (i >= SR_IPMAX && i - SR_IPMAX < nrt) nx[t] = d_load(rrow + (i - SR_IPMAX));
            }
        };
        fetch(1);
        for (int l1 = 1; l1 < l; ++l1) {
            __syncwarp();
#pragma unroll
            for (int t = 0; t < (int)(sizeof(nx) / sizeof(nx[0])); ++t) {
                const int i = lane + 32 * t;
                if (i < 2 * SR_IPMAX) buf[i] = nx[t];
            }
            __syncwarp();
            if (l1 + 1 < l) fetch(l1 + 1);                        // next split's cells in flight
            if (!active) continue;
            const int l2 = l - l1;
            const Cell4 *lrow = buf - 1;                           // I(m) cell s at lrow[c_ipart(m, l1) + s]
            const Cell4 *rrow = buf + SR_IPMAX - 1;
            for (int m = 1; m <= r - 1; ++m) {
                const int s_lo = max(1, Sp - min(l2, r - m));
                const int s_hi = min(Sp - 1, min(l1, m));
                const Cell4 *lb = lrow + c_ipart(m, l1);
                const Cell4 *rb = rrow + c_ipart(r - m, l2) + Sp;
                for (int s = s_lo; s <= s_hi; ++s) {
                    const Cell4 Lc = lb[s];
                    const Cell4 Rc = rb[-s];
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
        if (active && bkey == 0xFFFFFFFFu) d_store_inf(g, pc + d_cell(g, Sp, u, l, a), Sp);   // masks
        else if (active)
            d_write_winner(g, pc, Sp, u, l, a, (int)(bkey >> 20), (int)((bkey >> 10) & 1023u), (int)(bkey & 1023u));
    }
}

// ---------------------------------------------------------------- wavefront pipeline
// With OOB_DP_PIPE, wavefront l+1's kernel is launched as a programmatic dependent of wave
// l's (it starts once every CTA of wave l has started) and synchronises through per-wave
// counters instead of kernel boundaries.  Per wave c: seeds (aux blocks of launch c-1),
// in-node cells (aux blocks of launch c-1, or k_fin for c = 2) and the W-part finalize
// shares (main CTAs of launch c); each producer block fences and increments its counter
// after writing.  Readiness is monotone in c (a wave's finalize follows units that waited
// for the previous wave), so "wave c ready" covers every shorter wave.  Every cell of a
// wave is read only after its wave is ready (and the tables pad each wave to whole 32-byte
// sectors plus the streams' read-ahead), so L1-cached loads never see a stale line.  Waits
// are bounded; a timeout sets the error word and releases every later wait: the results
// are then wrong, so k_extract marks every template (status 2) and oob_generate_templates /
// oob_template_set_from_packed return OOB_E_CUDA; the GPU never hangs.
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// one thread waits until the parts in `mask` (bit kind: 0 seeds, 1 in-node cells,
// 2 finalize shares) of wave c are ready
__device__ __noinline__ void pipe_wait_raw(int *cnt, const int *expc, int *err, int L, int c, int mask,
                                           long long spin_max) {
    for (long long it = 0;; ++it) {
        bool ok = true;
        for (int kind = 0; kind < 3; ++kind)
            if ((mask >> kind) & 1) ok = ok && ld_acquire(cnt + kind * (L + 2) + c) >= expc[kind * (L + 2) + c];
        if (ok || *(volatile int *)err) break;
        if (it >= spin_max) { atomicExch(err, 1); break; }
        __nanosleep(200);
    }
    __threadfence();
}
__device__ __forceinline__ void pipe_wait(const Pipe &pp, int L, int c, int mask) {
    if (pp.on && c >= 2) pipe_wait_raw(pp.cnt, pp.expc, pp.err, L, c, mask, pp.spin_max);
}
// the calling block has finished writing its part of wave c (all threads reach this)
__device__ __forceinline__ void pipe_signal(const Pipe &pp, int L, int kind, int c) {
    if (!pp.on) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(pp.cnt + kind * (L + 2) + c, 1);
    }
}

// Warp mode of k_wave_w (w.warp_mode): every warp of the CTA owns one (profile, range) of
// the wave — its accumulator and filter in its own shared-memory region, initialised from
// the seeds — runs all of the range's units itself (in queue order, no unit counter) and
// finalizes the range's W outputs from shared memory; the wave-constant tables are staged
// once per CTA.  Same units, same exact path, same (total, key) minimum as the CTA mode.
template <int TE>
__device__ __forceinline__ void warp_ranges(const DevGeom &g, const WaveW &w, unsigned char *smem, ulonglong2 *acc0,
                                            unsigned *filt0, int4 *sents, int64_t *sbase, int *scells, int *outOff,
                                            int *upre, int *stoff, int *stcnt, int *scb, float4 *rings) {
    const int l = w.l, nout = w.nout, L = g.L, M = g.M;
    const int ndum = L + 2 * TE + 2;
    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const int Ql = (l == L) ? g.n_hi : max(1, g.n_hi - 1);
    if (tid == 0) OOB_TL_MIN(l, 0);
    for (int i = tid; i <= L; i += NTW) {
        stoff[i] = w.tile_off[i];
        stcnt[i] = w.tile_cnt[i];
    }
    for (int i = tid; i < w.ncb; i += NTW) scb[i] = w.cb[i];
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
    const int pr = (int)blockIdx.x * (NTW / 32) + wi;
    if (pr >= g.P * w.nranges) return;
    const int u = pr % w.nranges, p = pr / w.nranges;
    const int64_t pc = (int64_t)p * g.C;
    ulonglong2 *acc = acc0 + (size_t)wi * (nout + ndum);
    unsigned *filt = filt0 + (size_t)wi * (nout + ndum);
    const ulonglong2 *gseed = w.GACC + (size_t)pr * nout;
    unsigned *gfilt = w.GFILT + (size_t)pr * nout;
    for (int i0 = lane; i0 < nout + ndum; i0 += 4 * 32) {
        ulonglong2 a[4];
        unsigned fv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + j * 32;
            const bool real = i < nout;
            a[j] = real ? make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull) : make_ulonglong2(0ull, 0ull);
            if (real && w.seeded) a[j] = __ldcg(gseed + i);
            fv[j] = real ? __ldcg(gfilt + i) : 0xBF800000u;   // dummies: -1 (nothing passes)
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + j * 32;
            if (i < nout + ndum) {
                acc[i] = a[j];
                filt[i] = fv[j];
            }
        }
    }
    __syncwarp();
    const unsigned acc_s = (unsigned)__cvta_generic_to_shared(acc);
    const unsigned filt_s = (unsigned)__cvta_generic_to_shared(filt);
    unsigned char *wsm = reinterpret_cast<unsigned char *>(rings) + (size_t)wi * (XR_BYTES + XQ_BYTES);
    int ei = 0, qn = 0;
    for (int un = 0; un < w.nunits; ++un) {
        while (upre[ei + 1] <= un) ++ei;
        const int4 en = sents[ei];
        const int l1 = en.x & 0xFFFF;
        const int local = un - upre[ei];
        const int chunk = local / en.y;
        const int blk = local % en.y;
        const int r_lo = scb[en.w + chunk], r_hi = scb[en.w + chunk + 1];
        const int k = u + l1;
        const int l2 = l - l1;
        const bool ltiled = (en.x >> 16) & 1;
        const int ls = ltiled ? l2 : l1, lb = ltiled ? l1 : l2;
        const int us = ltiled ? k : u, ub = ltiled ? u : k;
        const int ti = blk * 32 + lane;
        const bool has = ti < stcnt[lb];
        const int32_t code = has ? w.tiles[stoff[lb] + ti] : 0;
        const int rowB = has ? (code >> 16) : 1;
        const int e0 = has ? (code & 0xFFFF) : 0;
        const int wb0 = has ? d_wofs(g, lb, rowB) : 0;
        const int lenB = has ? d_wofs(g, lb, rowB + 1) - wb0 : 0;
        const int ncell = max(0, min(TE, lenB - e0));
        const int64_t sidx = pc + sbase[ls] + (int64_t)us * scells[ls] + d_wofs(g, ls, r_lo);
        const int64_t bidx = pc + sbase[lb] + (int64_t)ub * scells[lb] + (has ? wb0 : d_wofs(g, lb, 1)) + e0;
        if (ltiled)
            qn = run_unit<TE, true>(g.SH, g.CELL, sidx, g.wofs + ls * (L + 2), r_lo, r_hi, bidx, ncell, rowB, e0, l1, L,
                                    outOff, nout, acc_s, filt_s, gfilt, wsm, 0, 0, qn);
        else
            qn = run_unit<TE, false>(g.SH, g.CELL, sidx, g.wofs + ls * (L + 2), r_lo, r_hi, bidx, ncell, rowB, e0, l1, L,
                                     outOff, nout, acc_s, filt_s, gfilt, wsm, 0, 0, qn);
    }
    flush_rest<TE>(wsm, qn, g.CELL, acc_s, filt_s, gfilt);
    __syncwarp();
    if (tid % 32 == 0) OOB_TL_MAX(l, 2);
    fin_w_range<32>(g, w.fw, pr, lane, 0, 1, acc);
    if (lane == 0) OOB_TL_MAX(l, 3);
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
    extern __shared__ __align__(16) unsigned char fsm[];
    if (f.small_range) fin_small_range(g, f, (int64_t)blockIdx.x - f.nbw - f.nbseed, fsm);
    else fin_small_block(g, f, (int64_t)blockIdx.x - f.nbw - f.nbseed);
}

template <int TE>
__global__ void __launch_bounds__(NTW, WAVE_CTAS_PER_SM) k_wave_w(DevGeom g, WaveW w) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_last;
    // block order: [main CTAs][extra blocks]
    const int bid = (int)blockIdx.x;          // main CTA index
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the next wave may start (pipeline)
    if (bid >= w.nbmain) {                    // next wave's seeds and in-node cells
        const int ab = (int)blockIdx.x - w.nbmain;
        if (threadIdx.x == 0) OOB_TL_MIN(w.l, 4);
        if (ab < w.fa.nbseed) {
            // seeds of wave l+1 read cells of waves <= l-1 and reuse wave l-1's accumulator buffer
            if (threadIdx.x == 0) pipe_wait(w.pp, L_of(g), w.fa.lseed - 2, 7);
            __syncthreads();
            fin_seed_one(g, w.fa, (int64_t)ab * NTW + threadIdx.x);
            pipe_signal(w.pp, L_of(g), 0, w.fa.lseed);
            if (threadIdx.x == 0) OOB_TL_MAX(w.l, 6);
        } else {
            // in-node cells of wave l+1 read in-node cells of waves <= l
            if (threadIdx.x == 0) pipe_wait(w.pp, L_of(g), w.fa.ls - 1, 2);
            __syncthreads();
            if (w.fa.small_range) fin_small_range(g, w.fa, (int64_t)ab - w.fa.nbseed, smem);
            else fin_small_block(g, w.fa, (int64_t)ab - w.fa.nbseed);
            pipe_signal(w.pp, L_of(g), 1, w.fa.ls);
            if (threadIdx.x == 0) OOB_TL_MAX(w.l, 7);
        }
        if (threadIdx.x == 0) OOB_TL_MAX(w.l, 5);
        return;
    }
    const int l = w.l;
    const int nout = w.nout;
    const int L = g.L, M = g.M;
    const int ndum = L + 2 * TE + 2;                              // dummy entries (absent parent rows)
    const bool wm = w.warp_mode;
    const int nacc = wm ? (NTW / 32) * (nout + ndum) : nout + ndum;   // warp mode: one region per warp
    ulonglong2 *acc = reinterpret_cast<ulonglong2 *>(smem);     // [nout] + dummy[ndum]  (x warps)
    unsigned *filt = reinterpret_cast<unsigned *>(acc + nacc);  // [nout + ndum] binary32 filters F(min)  (x warps)
    int4 *sents = reinterpret_cast<int4 *>(filt + ((nacc + 3) & ~3));   // [nents] (16 B aligned)
    int64_t *sbase = reinterpret_cast<int64_t *>(sents + w.nents);               // [L+2]
    int *scells = reinterpret_cast<int *>(sbase + L + 2);        // [L+1]
    int *outOff = scells + (L + 1);                              // [L+2] W(q) offsets (nout: none)
    int *upre = outOff + (L + 2);                                // [nents + 1]
    int *stoff = upre + w.nents + 1;                             // [L+1] tile list offsets
    int *stcnt = stoff + (L + 1);                                // [L+1] tile counts
    int *scb = stcnt + (L + 1);                                  // [ncb] chunk row boundaries
    // per-warp streamed-side rings (16 B aligned) after the tables
    const size_t ring_off = ((size_t)(reinterpret_cast<unsigned char *>(scb + w.ncb) - smem) + 15) & ~(size_t)15;
    float4 *rings = reinterpret_cast<float4 *>(smem + ring_off);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    if (wm) {
        warp_ranges<TE>(g, w, smem, acc, filt, sents, sbase, scells, outOff, upre, stoff, stcnt, scb, rings);
        return;
    }
    const int pr = bid / w.cpr;
    const int u = pr % w.nranges;
    const int p = pr / w.nranges;
    const int64_t pc = (int64_t)p * g.C;
    const int Ql = (l == L) ? g.n_hi : max(1, g.n_hi - 1);

    const ulonglong2 *gseed = w.GACC + (size_t)pr * nout;   // this range's entries
    unsigned *gfilt = w.GFILT + (size_t)pr * nout;
    __shared__ int s_rdy;                      // every wave <= s_rdy is ready (pipeline)
    if (tid == 0) {
        OOB_TL_MIN(l, 0);
        if (w.seeded) pipe_wait(w.pp, L, l, 1);   // this wave's seeds (launch l-1's extra blocks)
        // the accumulator buffer's previous user (wave l-3) has finalized: wave l-2 ready
        pipe_wait(w.pp, L, l - 2, 6);
        s_rdy = w.pp.on ? max(1, l - 2) : L;
        OOB_TL_MIN(l, 1);
    }
    __syncthreads();
    // accumulator from the seeds, filter from the range's global filter (F of the seeds and
    // of every improvement so far: <= F(seed)); 4 entries per thread in flight together
    for (int i0 = tid; i0 < nout + ndum; i0 += 4 * NTW) {
        ulonglong2 a[4];
        unsigned fv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + j * NTW;
            const bool real = i < nout;
            a[j] = real ? make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull) : make_ulonglong2(0ull, 0ull);
            if (real && w.seeded) a[j] = __ldcg(gseed + i);
            fv[j] = real ? __ldcg(gfilt + i) : 0xBF800000u;   // dummies: -1 (nothing passes)
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + j * NTW;
            if (i < nout + ndum) {
                acc[i] = a[j];
                filt[i] = fv[j];
            }
        }
    }
    for (int i = tid; i <= L; i += NTW) {
        stoff[i] = w.tile_off[i];
        stcnt[i] = w.tile_cnt[i];
    }
    for (int i = tid; i < w.ncb; i += NTW) scb[i] = w.cb[i];
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
    const int nunits = w.nunits;
    const unsigned acc_s = (unsigned)__cvta_generic_to_shared(acc);
    const unsigned filt_s = (unsigned)__cvta_generic_to_shared(filt);
    int *gctr = w.ctr + pr;
    unsigned char *wsm = reinterpret_cast<unsigned char *>(rings) + (size_t)(tid >> 5) * (XR_BYTES + XQ_BYTES);
    int qn = 0;                                                   // this warp's queued candidates

    for (;;) {
        int un = 0;
        if (lane == 0) un = w.rank + w.world * atomicAdd(gctr, 1);
        un = __shfl_sync(0xFFFFFFFFu, un, 0);
        if (un >= nunits) break;
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
        const int r_lo = scb[en.w + chunk], r_hi = scb[en.w + chunk + 1];
        const int k = u + l1;
        const int l2 = l - l1;
        if (w.pp.on) {                                           // both children's waves ready?
            const int cmax = max(l1, l2);
            if (cmax > *(volatile int *)&s_rdy) {
                if (lane == 0) {
                    pipe_wait(w.pp, L, cmax, 6);                 // in-node cells + W finalize
                    atomicMax(&s_rdy, cmax);
                }
                __syncwarp();
            }
        }
        const bool ltiled = (en.x >> 16) & 1;                     // tiled side = left child
        const int ls = ltiled ? l2 : l1;                           // small side length
        const int lb = ltiled ? l1 : l2;
        const int us = ltiled ? k : u;                             // small slab start
        const int ub = ltiled ? u : k;
        const int ti = blk * 32 + lane;
        const bool has = ti < stcnt[lb];
        const int32_t code = has ? w.tiles[stoff[lb] + ti] : 0;
        const int rowB = has ? (code >> 16) : 1;
        const int e0 = has ? (code & 0xFFFF) : 0;
        const int wb0 = has ? d_wofs(g, lb, rowB) : 0;
        const int lenB = has ? d_wofs(g, lb, rowB + 1) - wb0 : 0;
        const int ncell = max(0, min(TE, lenB - e0));             // valid cells of the tile
        // the streamed chunk's first batches are in flight while the tile and the filter load
        const int64_t sidx = pc + sbase[ls] + (int64_t)us * scells[ls] + d_wofs(g, ls, r_lo);
        if (w.prefetch) {   // warm L1 with the binary64 cells the exact path may load
            const Cell4 *tp = g.CELL + pc + sbase[lb] + (int64_t)ub * scells[lb] + (has ? d_wofs(g, lb, rowB) : 0) + e0;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + TE - 1));
            const Cell4 *sp0 = g.CELL + sidx + lane * 8;       // 32 lanes x 256 B covers a 256-cell chunk
            asm volatile("prefetch.global.L1 [%0];" ::"l"(sp0));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(sp0 + 4));
        }
        const int64_t bidx = pc + sbase[lb] + (int64_t)ub * scells[lb] + (has ? wb0 : d_wofs(g, lb, 1)) + e0;
        int olo = 0, ohi = 0;   // outputs of the parent rows q = rowB + rs this unit can touch
        if (w.refresh) {
            const int tb0 = blk * 32, tb1 = min(blk * 32 + 31, stcnt[lb] - 1);
            const int rmin = w.tiles[stoff[lb] + tb0] >> 16, rmax = w.tiles[stoff[lb] + tb1] >> 16;
            olo = outOff[min(rmin + r_lo, L + 1)];
            ohi = outOff[min(rmax + r_hi, L + 1)];
        }
        if (ltiled)
            qn = run_unit<TE, true>(g.SH, g.CELL, sidx, g.wofs + ls * (L + 2), r_lo, r_hi, bidx, ncell, rowB, e0, l1, L,
                                    outOff, nout, acc_s, filt_s, gfilt, wsm, olo, ohi, qn);
        else
            qn = run_unit<TE, false>(g.SH, g.CELL, sidx, g.wofs + ls * (L + 2), r_lo, r_hi, bidx, ncell, rowB, e0, l1, L,
                                     outOff, nout, acc_s, filt_s, gfilt, wsm, olo, ohi, qn);
    }
    flush_rest<TE>(wsm, qn, g.CELL, acc_s, filt_s, gfilt);
    __syncthreads();
    if (tid == 0) OOB_TL_MAX(l, 2);
    // merge into the range's global accumulator (L2-coherent loads; a stale value is an
    // upper bound of the current one, so the CAS loop stays exact).  Loads are batched so
    // their latencies overlap.
    if (w.cpr == 1 && w.fin_inline && w.world == 1) {   // the range's only CTA: finalize from shared memory
        fin_w_range<NTW>(g, w.fw, pr, tid, 0, 1, acc);
        pipe_signal(w.pp, L, 2, l);
        if (tid == 0) OOB_TL_MAX(l, 3);
        return;
    }
    ulonglong2 *ga = w.GACC + ((size_t)p * w.nranges + u) * nout;
    constexpr int MB = 4;
    for (int i0 = tid; i0 < nout; i0 += MB * NTW) {
        ulonglong2 a[MB], cur[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int i = i0 + j * NTW;
            a[j] = i < nout ? acc[i] : make_ulonglong2(ACC_EMPTY, 0ull);
            if (!(a[j].y & ACC_DIRTY)) a[j] = make_ulonglong2(ACC_EMPTY, 0ull);   // only this CTA's improvements
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
    if (w.fin_inline && w.peer) {
        // Peer exchange: the range's last local CTA publishes the local minima to every rank;
        // every local CTA of the range then waits for all ranks' partials and claims
        // finalize shares (fin_w_range takes the minimum over the gathered partials).
        __threadfence();
        __syncthreads();
        __shared__ int s_help;
        if (tid == 0) {
            const int ticket = atomicAdd(w.rdone + pr, 1) + 1;   // merge order, 1..cpr
            s_last = ticket == w.cpr;
            s_help = ticket > w.cpr - w.fin_helpers;            // the last fin_helpers CTAs finalize
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (int r = 0; r < w.world; ++r) {
                ulonglong2 *dst = w.xpart[r] + (int64_t)w.rank * w.fw.part_stride + ((int64_t)p * w.nranges + u) * nout;
                for (int i = tid; i < nout; i += NTW) dst[i] = __ldcg(ga + i);   // NVLink store into rank r
            }
            __threadfence_system();
            __syncthreads();
            if (tid < w.world) atomicAdd(w.xdone[tid] + pr, 1);
        } else if (!s_help) {
            // merged CTAs other than the range's last fin_helpers leave (their slots go to
            // the next wave); the helpers wait for the other ranks and share the finalize
            if (tid == 0) OOB_TL_MAX(l, 3);
            return;
        }
        if (tid == 0) {
            const int target = (int)w.epoch * w.world;
            int ok = 0;
            for (long long it = 0; it < w.pp.spin_max; ++it) {
                int v;
                asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(w.xdone[w.rank] + pr) : "memory");
                if (v >= target) { ok = 1; break; }
                if (*(volatile int *)w.pp.err) break;
                __nanosleep(200);
            }
            if (!ok) atomicExch(w.pp.err, 1);   // surfaces as OOB_E_CUDA (k_extract)
            s_last = ok;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (;;) {
                __syncthreads();
                if (tid == 0) s_last = atomicAdd(w.rclaim + pr, 1);
                __syncthreads();
                const int c = s_last;
                if (c >= w.cpr) break;
                fin_w_range<NTW>(g, w.fw, pr, tid, c, w.cpr);
                pipe_signal(w.pp, L, 2, l);
            }
        }
    } else if (w.fin_inline) {
        // The range's W outputs are final once all its cpr CTAs have merged.  The host sizes
        // the main grid to the resident CTA slots whenever cpr > 1 (the extra blocks come
        // after it), so the range's CTAs are co-resident: each waits for the others, then
        // they claim the cpr shares of the finalize from a counter.  The wait is bounded: on
        // timeout (a GPU shared with other work) a CTA just exits; the last CTA to merge never
        // waits and claims every share left, so each share is finalized exactly once.
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int ticket = atomicAdd(w.rdone + pr, 1) + 1;   // merge order, 1..cpr
            int ok = ticket == w.cpr;
            // only the range's last fin_helpers CTAs wait and share; the others leave
            const int spin = ticket > w.cpr - w.fin_helpers ? w.fin_spin : 0;
            for (int it = 0; !ok && it < spin; ++it) {
                __nanosleep(128);
                ok = *(volatile int *)(w.rdone + pr) >= w.cpr;
            }
            s_last = ok;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (;;) {
                __syncthreads();
                if (tid == 0) s_last = atomicAdd(w.rclaim + pr, 1);
                __syncthreads();
                const int c = s_last;
                if (c >= w.cpr) break;
                fin_w_range<NTW>(g, w.fw, pr, tid, c, w.cpr);
                pipe_signal(w.pp, L, 2, l);
            }
        }
    }
    if (tid == 0) OOB_TL_MAX(l, 3);
}

// Start of every run: empty accumulators and filters (the finalize resets what it reads,
// but a run that failed part-way, or another plan's run in the same workspace, leaves
// entries behind) and zero counters (unit counters, pipeline counters, error word).
__global__ void k_init(ulonglong2 *gacc, unsigned *gfilt, int64_t nacc, int *ctr, int64_t nctr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nacc) {
        gacc[i] = make_ulonglong2(ACC_EMPTY, 0xFFFFFFFFull);
        gfilt[i] = FILT_EMPTY;
    }
    if (i < nctr) ctr[i] = 0;
}

}  // namespace oob
