// CUDA DP engine for pipeline-template generation (PAPER §4.1.2, Eqs.1-4) on sm_100a.
//
// The memoized recursion T(S', u, v, a) is evaluated bottom-up as a wavefront over the
// layer-range length l = v - u (every sub-problem of a length-l range has a shorter
// range), all cells of one wavefront in parallel:
//   K_base      : every S' = 1 cell (Eq.4), all lengths at once;
//   K_wave(l)   : every S' >= 2 cell of length l, min over splits (k, m, s) of
//                 T1 + T2 + T3 combined per Eqs.1-3 with N_b = 4S';
//   K_extract   : per template size n, argmin over S and the backtrack.
// Arithmetic contract: binary64 with explicit __dadd_rn/__dmul_rn (no FMA
// contraction; the file is also built with --fmad=false), in the oracle's order:
//   T1 = L.T1 + R.T1; left = L.t* >= R.t*; T3 = left ? L.T3 + R.T1 : R.T3;
//   k* = left ? L.k* : s + R.k*; T2 = (double)(3S' + k* - 1) * t*; total = (T1 + T2) + T3;
//   the first split (in (k, m, s) order) with a strictly smaller total wins.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cstring>
#include <mutex>
#include <numeric>
#include <vector>

#include "oob_internal.h"
#include "oob_dp_common.cuh"
#include "oob_wave_w.cuh"

namespace oob {

// ------------------------------------------------------------------ K_base: Eq.4
// One thread per (profile, u, base alloc) of wavefront l = blockIdx.y + 1.  Base allocs:
// I(r), r = 1..M-1 (d = r) and W(1) (d = M).  t = sum_{k=u}^{v-1}(F + B) left to right.
__global__ void k_base(DevGeom g, const double *__restrict__ fwd, const double *__restrict__ bwd) {
    const int l = blockIdx.y + 1;
    const int nu = g.L - l + 1;
    const int per_prof = nu * g.M;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)per_prof * g.P) return;
    const int p = (int)(t / per_prof);
    const int r = (int)(t % per_prof);
    const int u = r / g.M;
    const int a = r % g.M;                 // 0..M-2 -> I(a+1); M-1 -> W(1)
    const int d = a + 1;                   // I(r): r GPUs; W(1): M GPUs
    if (g.off[l * g.A + a] < 0) return;
    const double *F = fwd + (size_t)p * g.L * g.M;
    const double *B = bwd + (size_t)p * g.L * g.M;
    const int64_t c = (int64_t)p * g.C + d_cell(g, 1, u, l, a);
    if (g.masked && !d_stage_allowed(g, p, u, u + l, d)) {   // masked stage (reading R31)
        d_store_inf(g, c, 1);
        return;
    }
    double s = 0.0;
    for (int k = u; k < u + l; ++k) s = __dadd_rn(s, __dadd_rn(F[k * g.M + d - 1], B[k * g.M + d - 1]));
    d_store(g, c, s, s, s, 2.0);    // T1 = T3 = t* = t; C1 = 3*1 - 1 + k*(=0)
    g.ARG[c] = 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ K_wave (v1)
// Reference kernel: one thread per (profile, u, cell of the slab) for wavefront l; loops the
// splits in the oracle's (k, m, s) order with a strict "<".  S' = 1 cells are skipped.
__global__ void k_wave_v1(DevGeom g, int l) {
    const int nu = g.L - l + 1;
    const int cl = g.cells[l];
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nu * cl * g.P) return;
    const int p = (int)(t / ((int64_t)nu * cl));
    const int rem = (int)(t % ((int64_t)nu * cl));
    const int u = rem / cl;
    const int i = rem % cl;
    int a = 0, Sp = 0;
    for (int aa = 0; aa < g.A; ++aa) {
        int o = g.off[l * g.A + aa];
        if (o < 0 || o > i) continue;
        int cnt = d_hi(g, aa, l) - d_lo(g, aa) + 1;
        if (i < o + cnt) { a = aa; Sp = d_lo(g, aa) + (i - o); break; }
    }
    if (Sp < 2) return;
    const int v = u + l;
    const int64_t pc = (int64_t)p * g.C;
    const double dSp3 = (double)(3 * Sp - 1);
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int bl1 = 0, bj = 0, bs = 0;
    const int nd = d_num_dsplits(g, a);
    for (int k = u + 1; k < v; ++k) {
        const int l1 = k - u, l2 = v - k;
        for (int j = 0; j < nd; ++j) {
            int a1, a2;
            d_dsplit(g, a, j, a1, a2);
            if (g.off[l1 * g.A + a1] < 0 || g.off[l2 * g.A + a2] < 0) continue;
            int s_lo = max(max(1, d_lo(g, a1)), Sp - d_hi(g, a2, l2));
            int s_hi = min(min(Sp - 1, d_hi(g, a1, l1)), Sp - d_lo(g, a2));
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
                if (tot < best) { best = tot; bl1 = l1; bj = j; bs = s; }
            }
        }
    }
    if (bl1 == 0) { d_store_inf(g, pc + d_cell(g, Sp, u, l, a), Sp); return; }   // no finite split (masks)
    d_write_winner(g, pc, Sp, u, l, a, bl1, bj, bs);
}

// ------------------------------------------------------------------ K_extract
// One warp per (profile, template size n).  Choice of S: the lanes evaluate
// S = n + lane, n + lane + 32, ... and the warp takes the lexicographic minimum of
// (total, S) — the oracle's "first strictly smaller total" scan in ascending S (smaller S
// wins ties, reading R8).  Backtrack: the split tree level by level, the warp expanding a
// level's nodes in parallel; a node carries the index of its first stage (its left child
// keeps it, its right child starts s stages later), so every leaf (S' = 1) writes its stage
// record straight into pipeline order.  Frontier: two buffers of <= L + 1 nodes in shared
// memory (dynamic, 2 x (L+1) x 16 bytes per warp).
struct XNode {
    uint64_t key;      // Sp | u << 10 | v << 20 | a << 30 | node << 41 | goff << 51 (goff < 64)
    int32_t first;     // stage index of the node's first stage
    int32_t pad;
};

__global__ void k_extract(DevGeom g, unsigned char *packed, size_t tpl_bytes, Pipe pp) {
    extern __shared__ __align__(16) unsigned char xsm[];
    __shared__ int s_err;
    if (threadIdx.x == 0) {
        s_err = 0;
        if (pp.on) {                  // the pipelined waves' last cells (and, by monotonicity, all)
            pipe_wait(pp, g.L, g.L, 6);
            s_err = *(volatile int *)pp.err;   // a timed-out wait: the table may be wrong
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int p_cnt = g.n_hi - g.n_lo + 1;
    const int t = blockIdx.x * (blockDim.x >> 5) + wib;
    if (t >= p_cnt * g.P) return;
    const int p = t / p_cnt;
    const int n = g.n_lo + t % p_cnt;
    const int64_t pc = (int64_t)p * g.C;
    const int L = g.L;
    const int aW = (g.M - 1) + n - 1;
    PackedHeader *h = reinterpret_cast<PackedHeader *>(packed + (size_t)t * tpl_bytes);
    int32_t *st = reinterpret_cast<int32_t *>(h + 1);
    // argmin over S: lexicographic (total, S)
    const int Smax = min(L, n * g.M);
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bestS = 0x7FFFFFFF;
    for (int S = n + lane; S <= Smax; S += 32) {
        const Cell4 c = d_load(g.CELL + pc + d_cell(g, S, 0, L, aW));
        const double T2 = __dmul_rn(c.C1, c.TS);      // (4S - S + k* - 1) t*, Eq.2
        const double tot = __dadd_rn(__dadd_rn(c.T1, T2), c.T3);
        if (tot < best || (tot == best && S < bestS)) { best = tot; bestS = S; }
    }
    for (int d = 16; d >= 1; d >>= 1) {
        const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, d);
        const int os = __shfl_xor_sync(0xFFFFFFFFu, bestS, d);
        if (ob < best || (ob == best && os < bestS)) { best = ob; bestS = os; }
    }
    int status = s_err ? 2 : 0;       // 2: pipeline wait timed out (OOB_E_CUDA on the host)
    if (!(best < __longlong_as_double(0x7ff0000000000000LL))) {
        // every S infinite: no allowed mapping under the stage masks (reading R31) —
        // an infeasible template (status 3, S = 0)
        if (lane == 0) {
            const double inf = __longlong_as_double(0x7ff0000000000000LL);
            h->nodes = n; h->S = 0; h->kstar = 0; h->status = status ? status : 3;
            h->T1 = h->T2 = h->T3 = h->tstar = h->iter = inf;
            h->pad = 0.0;
        }
        for (int i = lane; i < L; i += 32) {
            int32_t *r = st + 5 * i;
            r[0] = r[1] = r[2] = r[3] = r[4] = -1;
        }
        return;
    }
    if (lane == 0) {
        const Cell4 c = d_load(g.CELL + pc + d_cell(g, bestS, 0, L, aW));
        h->nodes = n; h->S = bestS; h->kstar = (int)d_kd(c.C1, bestS);
        h->T1 = c.T1; h->T3 = c.T3; h->tstar = c.TS;
        h->T2 = __dmul_rn(c.C1, c.TS);
        h->iter = best;
        h->pad = 0.0;
    }
    auto pack = [](int Sp, int u, int v, int a, int node, int goff) -> uint64_t {
        return (uint64_t)Sp | ((uint64_t)u << 10) | ((uint64_t)v << 20) | ((uint64_t)a << 30) |
               ((uint64_t)node << 41) | ((uint64_t)goff << 51);
    };
    XNode *fr[2];
    fr[0] = reinterpret_cast<XNode *>(xsm) + (size_t)wib * 2 * (L + 1);
    fr[1] = fr[0] + (L + 1);
    int cnt = 1, cur = 0;
    if (lane == 0) fr[0][0] = XNode{pack(bestS, 0, L, aW, 0, 0), 0, 0};
    __syncwarp();
    bool bad = false;
    while (cnt > 0) {
        int next = 0;
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            XNode c0{0, 0, 0}, c1{0, 0, 0};
            int nout = 0;
            if (i < cnt) {
                const XNode nd = fr[cur][i];
                const uint64_t e = nd.key;
                const int Sp = (int)(e & 1023u), u = (int)((e >> 10) & 1023u), v = (int)((e >> 20) & 1023u);
                const int a = (int)((e >> 30) & 2047u), node = (int)((e >> 41) & 1023u), goff = (int)((e >> 51) & 63u);
                if (Sp == 1) {
                    if (nd.first < L) {
                        int32_t *r = st + 5 * nd.first;
                        r[0] = u; r[1] = v; r[2] = d_is_whole(g, a) ? g.M : d_alloc_n(g, a); r[3] = node; r[4] = goff;
                    } else {
                        bad = true;
                    }
                } else {
                    const uint32_t arg = g.ARG[pc + d_cell(g, Sp, u, v - u, a)];
                    const int k = u + (int)(arg & 1023u) + 1;
                    const int j = (int)((arg >> 10) & 1023u);
                    const int s = (int)(arg >> 20);
                    if (arg >= 0xFFFFFFFDu || k <= u || k >= v || s < 1 || s >= Sp || j >= d_num_dsplits(g, a)) {
                        bad = true;           // corrupt split (never for a valid table)
                    } else {
                        int a1, a2;
                        d_dsplit(g, a, j, a1, a2);
                        const bool wsplit = d_is_whole(g, a) && d_alloc_n(g, a) >= 2;
                        c0 = XNode{pack(s, u, k, a1, node, wsplit ? 0 : goff), nd.first, 0};
                        c1 = XNode{wsplit ? pack(Sp - s, k, v, a2, node + d_alloc_n(g, a1), 0)
                                          : pack(Sp - s, k, v, a2, node, goff + d_alloc_n(g, a1)),
                                   nd.first + s, 0};
                        nout = 2;
                    }
                }
            }
            // compact the children into the next frontier
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, nout > 0);
            const int pos = next + 2 * __popc(bal & ((1u << lane) - 1u));
            if (nout > 0 && pos + 1 <= L) {
                fr[cur ^ 1][pos] = c0;
                fr[cur ^ 1][pos + 1] = c1;
            } else if (nout > 0) {
                bad = true;
            }
            next += 2 * __popc(bal);
        }
        __syncwarp();
        cnt = min(next, L + 1);
        cur ^= 1;
    }
    if (__any_sync(0xFFFFFFFFu, bad) && !status) status = 1;
    for (int i = bestS + lane; i < L; i += 32) {
        int32_t *r = st + 5 * i;
        r[0] = r[1] = r[2] = r[3] = r[4] = -1;
    }
    if (lane == 0) h->status = status;
}

}  // namespace oob

// ==================================================================== plan + C ABI
using namespace oob;

namespace {

constexpr int TE_W = 4;                    // k_wave_w register tile: TE cells per lane
constexpr double SHARD_MIN_SPLITS = 2e7;   // wavefronts sharded across ranks (per-wave ncclAllGather)
constexpr double SHARD_MIN_SPLITS_PEER = 5e6;   // ... with the fused peer exchange (cfg4 4 GPUs: 9.57 -> 9.15 ms)
constexpr int SEED_MIN_L = 6;              // waves seeded with proportional splits (k_fin)
constexpr int CTAS_PER_SM = WAVE_CTAS_PER_SM;   // k_wave_w: resident CTAs per SM (register bound; smem may allow fewer)

// Plan-time switches (read once at oob_dp_plan_create; every OOB_DP_* variable is part of
// the plan-cache key of oob_generate_templates).  All select variants with identical
// results; the effective values are reported by oob_dp_plan_info (oob_dp_info.switches).
struct Knobs {
    int kernel = 2;            // OOB_DP_KERNEL=v1: thread-per-cell reference kernel (1)
    int fuse_fin = 1;          // OOB_DP_FUSE=0: separate k_fin launch per wave
    int pipe = 1;              // OOB_DP_PIPE=0: plain kernel boundaries between wavefronts
    int seed_init = 1;         // OOB_DP_SEEDINIT=0: no proportional-split seeds
    double seed_spo = 0.0;     // OOB_DP_SEEDSPO: seed waves with >= this many splits per W output
    int seed_min_l = SEED_MIN_L;   // OOB_DP_SEEDMINL: first seeded wavefront
    int small_pairs = 1;       // OOB_DP_SMALLPAIRS: layer splits per thread of an in-node cell
    int chunk_max = 0;         // OOB_DP_CHMAX: streamed cells per unit (upper bound; 0: 320, 192 / 96 sharded over 2-3 / >= 4)
    int units_per_cta = 0;     // OOB_DP_UPC: minimum queue units per CTA (chunk size)
    int units_per_warp = 4;    // OOB_DP_UPW: chunks shrink until every warp slot has this many units
    int refresh = 1;           // OOB_DP_REFRESH=0: no per-unit filter refresh
    int refresh_lmin = 64;     // OOB_DP_REFRESHL: refresh only from this wavefront on (shorter waves:
                               // small units, the refresh costs more than it filters; cfg4 13.84 -> 13.76 ms)
    double shard_min = -1.0;   // OOB_DP_SHARDMIN: waves with fewer splits run redundantly (default:
                               // 5e6 with the peer exchange, 2e7 with per-wave ncclAllGather)
    long long spin_max = 1ll << 24;        // OOB_DP_PIPE_SPIN: polls before a pipeline wait times out
    int fin_wait = -1;         // OOB_DP_FINWAIT=0/1: merged CTAs exit (the range's last one finalizes
                               // alone) / all wait and share; default: the last ceil(nout / fin_help)
    int fin_help = 0;          // OOB_DP_FINHELP: outputs of a range per finalize helper CTA (0: 512, 768 with a peer exchange)
    int shard_x = 1;           // OOB_DP_SHARDX=nccl: per-wave ncclAllGather + k_fin instead of peer stores
    int small_range = 1;       // OOB_DP_SMALLRANGE=0: in-node cells thread(s) per cell instead of warp per range
    double slot_frac = 1.0;    // OOB_DP_SLOTFRAC: share of the resident CTA slots one wave's grid fills
    int slot_frac_lmax = 1 << 30;   // OOB_DP_SLOTFRAC_LMAX: ... for waves l <= this only
    int warp_units = 64;       // OOB_DP_WARPMAX: batched waves with <= this many units per range run one
                               // warp per (profile, range) (0: never)
    int debug = 0;             // OOB_DP_DEBUG: per-wave plan on stderr
};

Knobs read_knobs() {
    Knobs k;
    auto env = [](const char *n) { return std::getenv(n); };
    if (const char *v = env("OOB_DP_KERNEL")) k.kernel = std::string(v) == "v1" ? 1 : 2;
    if (const char *v = env("OOB_DP_FUSE")) k.fuse_fin = std::atoi(v) != 0;
    if (const char *v = env("OOB_DP_PIPE")) k.pipe = std::atoi(v) != 0;
    if (const char *v = env("OOB_DP_SEEDINIT")) k.seed_init = std::atoi(v) != 0;
    if (const char *v = env("OOB_DP_SEEDSPO")) k.seed_spo = std::atof(v);
    if (const char *v = env("OOB_DP_SEEDMINL")) k.seed_min_l = std::max(3, std::atoi(v));
    if (const char *v = env("OOB_DP_SMALLPAIRS")) k.small_pairs = std::max(1, std::atoi(v));
    if (const char *v = env("OOB_DP_CHMAX")) k.chunk_max = std::max(12, std::atoi(v));
    if (const char *v = env("OOB_DP_UPC")) k.units_per_cta = std::max(0, std::atoi(v));
    if (const char *v = env("OOB_DP_UPW")) k.units_per_warp = std::max(1, std::atoi(v));
    if (const char *v = env("OOB_DP_REFRESH")) k.refresh = std::atoi(v) != 0;
    if (const char *v = env("OOB_DP_REFRESHL")) k.refresh_lmin = std::max(0, std::atoi(v));
    if (const char *v = env("OOB_DP_SHARDMIN")) k.shard_min = std::atof(v);
    if (const char *v = env("OOB_DP_PIPE_SPIN")) k.spin_max = std::max(0ll, std::atoll(v));
    if (const char *v = env("OOB_DP_FINWAIT")) k.fin_wait = std::atoi(v) != 0 ? 1 : 0;
    if (const char *v = env("OOB_DP_FINHELP")) k.fin_help = std::max(1, std::atoi(v));
    if (const char *v = env("OOB_DP_SHARDX")) k.shard_x = std::string(v) == "nccl" ? 0 : 1;
    if (const char *v = env("OOB_DP_WARPMAX")) k.warp_units = std::max(0, std::atoi(v));
    if (const char *v = env("OOB_DP_SMALLRANGE")) k.small_range = std::max(0, std::min(2, std::atoi(v)));
    if (const char *v = env("OOB_DP_SLOTFRAC")) k.slot_frac = std::max(0.05, std::min(1.0, std::atof(v)));
    if (const char *v = env("OOB_DP_SLOTFRAC_LMAX")) k.slot_frac_lmax = std::atoi(v);
    if (env("OOB_DP_DEBUG")) k.debug = 1;
    if (k.shard_min < 0) k.shard_min = k.shard_x ? SHARD_MIN_SPLITS_PEER : SHARD_MIN_SPLITS;
    return k;
}

struct WaveHost {
    int nents = 0, nunits = 0, nout = 0, cpr = 1;
    size_t ents_off = 0, upre_off = 0, cb_off = 0;   // byte offsets in the geometry's items region
    std::vector<int32_t> ents;     // 4 ints per entry: (l1, nblocks, nchunks, chunk_off)
    std::vector<int32_t> upre;     // unit prefix per entry [nents + 1]
    std::vector<int32_t> cb;       // chunk row boundaries
    size_t smem = 0;
    size_t ctr_off = 0;            // first unit counter of this wave (ints)
    size_t done_off = 0;           // per-range finished-CTA counters (fused finalize)
    int max_row = 0;               // longest streamed W row (queue entry fields)
    int nsmall = 0;                // cells inside one node with S' >= 2 per range
    bool seed = false;             // accumulator seeded by k_fin (proportional + warm-start splits)
    bool warp = false;             // one warp per (profile, range) (k_wave_w warp mode)
    double cost = 0.0;             // modelled issue cycles of the wave (all ranges, profiles)
};

int Q_of(const Geometry &g, int l) { return (l == g.L) ? g.n_hi : std::max(1, g.n_hi - 1); }
int wlen_h(const Geometry &g, int l, int q) {
    int hi = std::min(l, q * g.M);
    return hi >= q ? hi - q + 1 : 0;
}
int wcells_h(const Geometry &g, int l) { return g.cells[l] - g.off[(size_t)l * g.A + (g.M - 1)]; }

// SMs of the current device (148 on B200; the CPU build box has no device)
int device_sms() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
        return n;
    cudaGetLastError();   // clear the sticky "no device" error of the query
    return 148;
}

}  // namespace

struct oob_dp_plan {
    Geometry g;
    int32_t P = 1;
    Knobs kn;
    int kernel = 2;                      // 1 = v1 (thread per cell), 2 = tiled W kernel
    int num_sms = 148;                   // SMs the wave grids were sized for
    bool pipe_on = false;                // pipelined wavefronts (single-profile, unsharded)
    size_t pipe_cnt_off = 0;             // ints into the counter region: [3][L+2] + error word
    size_t geom_bytes = 0, ws_bytes = 0, tpl_bytes = 0;
    std::vector<unsigned char> geom_blob;   // host image of the device geometry (read-only)
    std::vector<std::pair<int, void *>> dev_geom;   // plan-owned device copies, per device
    size_t off_cells = 0, off_base = 0, off_off = 0, off_wofs = 0, off_pexp = 0, off_tiles = 0, off_tile_off = 0,
           off_tile_cnt = 0, off_items = 0;
    size_t off_CELL = 0, off_SH = 0, off_ARG = 0, off_GACC = 0, off_GFILT = 0, off_CTR = 0;
    int64_t gacc_n = 0;
    void *comm = nullptr;                // ncclComm_t (single-profile sharding), world > 1
    int rank = 0, world = 1;
    // fused exchange over peer memory (sharded waves; default with a communicator):
    // plan-owned exchange buffer XB = [3 parities][world][gacc_n] partial argmins + [ctr_n]
    // epoch-based "ranks published" counters, IPC-mapped into every rank
    bool xpeer = false;
    void *xb = nullptr;                  // this rank's exchange buffer (cudaMalloc)
    int xb_dev = -1;
    std::vector<void *> xb_peer;         // [world] every rank's buffer in this process (own = xb)
    size_t xb_off_done = 0, xb_bytes = 0;
    unsigned epoch = 0;                  // runs so far (peer counters are never reset)
    size_t off_GPART = 0;                // [world][wave partial] gathered partial accumulators
    size_t ws_bytes_base = 0;
    size_t ctr_n = 0;
    std::vector<int32_t> tiles;          // flat tile lists of TE_W cells
    std::vector<int32_t> tile_off, tile_cnt;   // [L+1]
    std::vector<double> stream_steps;    // [L+1] cost-model steps of streaming a slab of length ls
    std::vector<WaveHost> waves;         // [L+1]
    size_t max_smem = 0;
    int chunk_eff = 320;                 // effective OOB_DP_CHMAX of the sizing (size_plan)
    int sized_world = 1;                 // the world size_plan last sized the waves for
    int timing = 0;
    int mask_pow2 = 0;                   // stage masks (oob_dp_set_stage_masks, reading R31)
    const double *mask_sb = nullptr;     // device [P][L] stage bytes (borrowed)
    double mask_cap = 0.0;
    std::vector<cudaEvent_t> ev;
    int ev_used = 0;
    double acc_ms = 0.0;
    int64_t acc_launches = 0;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static oob_status cuda_fail(cudaError_t e, const char *what) {
    return fail(OOB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Flat tile lists: for a big side of length lb, its W rows j = 1..min(Q, lb) cut into
// ceil(len/TE) tiles of TE consecutive cells, in row order; 32 consecutive tiles form one
// warp work unit of k_wave_w.
static void build_tiles(oob_dp_plan *pl) {
    const Geometry &g = pl->g;
    pl->tile_off.assign(g.L + 1, 0);
    pl->tile_cnt.assign(g.L + 1, 0);
    for (int lb = 1; lb <= g.L; ++lb) {
        const int J = std::min(Q_of(g, lb), lb);
        pl->tile_off[lb] = (int32_t)pl->tiles.size();
        for (int j = 1; j <= J; ++j) {
            const int len = wlen_h(g, lb, j);
            for (int e0 = 0; e0 < len; e0 += TE_W) pl->tiles.push_back((j << 16) | e0);
        }
        pl->tile_cnt[lb] = (int32_t)pl->tiles.size() - pl->tile_off[lb];
    }
}

// Issue-cycle model of one k: every unit (32 lanes) walks its rows; a step costs TE splits
// (~20 instructions each) plus the load and the merge (~24).
static double k_cost(const oob_dp_plan *pl, int l, int l1, bool lt) {
    const int l2 = l - l1;
    const int ls = lt ? l2 : l1, lb = lt ? l1 : l2;       // streamed side, tiled side
    const double steps = pl->stream_steps[ls];             // rows + per-row tail/flush/setup
    const double units = (pl->tile_cnt[lb] + 31) / 32;
    return units * (steps * (TE_W * 20.0 + 24.0) + 400.0);
}

// Unit queue of wavefront l (identical for every range and profile): one entry per layer
// split k with work, balanced splits (l1 near l/2) first so the accumulator sees good
// totals early; an entry's small-side rows are cut into chunks of ~CH steps; a warp unit is
// (entry, chunk, block of 32 big-side tiles).  `slots` = resident CTAs of the GPU: ranges
// get several CTAs (sharing the range's queue) when there are fewer ranges than slots.
static void build_wave(oob_dp_plan *pl, int l, int slots, WaveHost &wh, int CH) {
    const Geometry &g = pl->g;
    const int nr = g.L - l + 1;
    std::vector<int> order;
    for (int l1 = 1; l1 < l; ++l1) order.push_back(l1);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return std::abs(2 * a - l) < std::abs(2 * b - l); });
    wh.ents.clear();
    wh.upre.assign(1, 0);
    wh.cb.clear();
    wh.max_row = 0;
    double total = 0.0;
    for (int l1 : order) {
        const int l2 = l - l1;
        // tile the left child (stream the right) or the reverse, whichever the model finds
        // cheaper: tiling the bigger side fills the 32 lanes, streaming the longer rows cuts
        // the per-row overhead
        const double cl = k_cost(pl, l, l1, true), cr = k_cost(pl, l, l1, false);
        const bool lt = cl <= cr;
        const int ls = lt ? l2 : l1, lb = lt ? l1 : l2;
        const int JS = std::min(Q_of(g, ls), ls);
        const int nblocks = (pl->tile_cnt[lb] + 31) / 32;
        const int coff = (int)wh.cb.size();
        int nchunks = 0, acc = 0, last = -1;
        for (int r = 1; r <= JS; ++r) {
            const int c = acc / CH;
            if (c != last) { wh.cb.push_back(r); ++nchunks; last = c; }
            acc += wlen_h(g, ls, r);
            wh.max_row = std::max(wh.max_row, wlen_h(g, ls, r));
        }
        wh.cb.push_back(JS + 1);
        if (nchunks == 0 || nblocks == 0) { wh.cb.resize(coff); continue; }
        wh.ents.insert(wh.ents.end(), {l1 | (lt ? 1 << 16 : 0), nblocks, nchunks, coff});
        wh.upre.push_back(wh.upre.back() + nblocks * nchunks);
        total += std::min(cl, cr);
    }
    wh.nents = (int)wh.ents.size() / 4;
    wh.nunits = wh.upre.back();
    wh.nout = wcells_h(g, l);
    const int ranges = pl->P * nr;
    wh.cpr = std::max(1, std::min(wh.nunits / 8, slots / std::max(1, ranges)));
    // acc[nout + dummy] (16 B) + filter (4 B) + base[L+2] (8 B) + cells[L+1] + outOff[L+2]
    // + upre[L+4] + ents[nents] (16 B)
    const size_t nent = (size_t)(wh.nout + g.L + 2 * TE_W + 2) * (wh.warp ? NTW / 32 : 1);
    const size_t before_ring = nent * 16 + (nent + 3) / 4 * 16 + (size_t)wh.nents * 16 + (size_t)(g.L + 2) * 8 +
                               (size_t)(g.L + 1) * 4 + (size_t)(g.L + 2) * 4 + (size_t)(g.L + 4) * 4 +
                               2 * (size_t)(g.L + 1) * 4 + wh.cb.size() * 4;   // + tile tables, chunk bounds
    wh.smem = before_ring + 32 + (size_t)(NTW / 32) * (XR_BYTES + XQ_BYTES);   // + per-warp rings and queues
    wh.cost = total * ranges;
}

// cells inside one node with S' >= 2 per range of length l (I(r), r < M, and W(1))
static int small_cells(const Geometry &g, int l) {
    int per = 0;
    for (int a = 0; a < std::min(g.A, g.M); ++a) per += std::max(0, std::min(l, g.gpus(a)) - 1);
    return per;
}

// threads per small cell: about `per` layer splits l1 per thread, 1..32 (one warp segment)
static int small_tpc(const Geometry &g, int l, int per) {
    int t = 1;
    while (t < 32 && t * per < l - 1) t *= 2;
    return t;
}

// in-node cells one warp per (profile, range) (fin_small_range): batched sweeps with M <= 8,
// unless OOB_DP_SMALLRANGE=0 (a single profile has too few ranges: one warp walking all
// layer splits of a range sits on the pipelined critical path, cfg4 +16%; =2 forces it)
static bool small_range_on(const oob_dp_plan *pl, int l) {
    // enough (profile, range) pairs for every resident warp slot to get >= 2 of them
    const int64_t pairs = (int64_t)pl->P * (pl->g.L - l + 1);
    const int64_t warp_slots = (int64_t)CTAS_PER_SM * pl->num_sms * (NTW / 32);
    return pl->g.M <= 8 && (pl->kn.small_range == 2 || (pl->kn.small_range == 1 && pairs >= 2 * warp_slots));
}

// blocks of 256 threads computing the in-node cells of wave l (all profiles)
static int64_t small_blocks(const oob_dp_plan *pl, int l) {
    const Geometry &g = pl->g;
    if (small_range_on(pl, l)) return ((int64_t)pl->P * (g.L - l + 1) + NTW / 32 - 1) / (NTW / 32);
    const int tpc = small_tpc(g, l, pl->kn.small_pairs);
    const int64_t ns = (int64_t)pl->P * (g.L - l + 1) * small_cells(g, l);
    return (ns + (256 / tpc) - 1) / (256 / tpc);
}

// Pipelined wavefronts (k_wave_w as programmatic dependent launches synchronised by
// counters): only the fused single-pass, unsharded W kernel, and only when every wave's main
// grid fits the resident CTA slots (a single profile); batched sweeps have far more CTAs
// than slots and gain nothing from the overlap.
static bool plan_pipe_on(const oob_dp_plan *pl) {
    const Geometry &G = pl->g;
    bool on = pl->kn.pipe && pl->kernel == 2 && (pl->world == 1 || pl->xpeer) && pl->kn.fuse_fin;
    for (int l = 2; l <= G.L && on; ++l)
        on = pl->waves[l].nents > 0 && !pl->waves[l].warp &&
             (int64_t)pl->P * (G.L - l + 1) * pl->waves[l].cpr <= (int64_t)CTAS_PER_SM * pl->num_sms;
    return on;
}

// Wave sizing (chunks, CTAs per range, seeds), workspace layout and the geometry blob, for
// `world` ranks sharing every wave's units: 320-cell chunks on one GPU (cfg4 13.96 -> 13.84 ms
// with the carried-over candidate queue), 192 on 2-3 ranks, 96 from 4 (each rank's share of a
// range still has enough units; 4 GPUs 7.35 -> 7.20 ms).  Host only; run by
// oob_dp_plan_create and again by oob_dp_set_comm / oob_dp_set_virtual_shards.
static void size_plan(oob_dp_plan *pl, int world) {
    const Geometry &g = pl->g;
    const int L = g.L, M = g.M, num_profiles = pl->P, SMS = pl->num_sms;
    pl->kernel = pl->kn.kernel;
    pl->max_smem = 0;
    const int chmax = pl->kn.chunk_max > 0 ? pl->kn.chunk_max : (world >= 4 ? 96 : world >= 2 ? 192 : 320);
    pl->chunk_eff = chmax;
    pl->waves.assign(L + 1, WaveHost());
    size_t items_total = 0, gacc_max = 0, ctr_total = 0;
    bool fits = true;                    // queue-entry fields and shared memory of k_wave_w
    for (int l = 2; l <= L; ++l) {
        WaveHost &wh = pl->waves[l];
        // smaller chunks (more, shorter units) until every warp slot has ~4 units and every
        // CTA has >= units_per_cta units of its range's queue (short tails per CTA);
        // resident CTAs per SM: launch bounds (registers), then shared memory
        int per_sm = CTAS_PER_SM;
        for (int pass = 0; pass < 2; ++pass) {
            for (int CH = chmax;; CH /= 2) {
                const double frac = l <= pl->kn.slot_frac_lmax ? pl->kn.slot_frac : 1.0;
                build_wave(pl, l, std::max(1, (int)(per_sm * SMS * frac)), wh, CH);
                if (CH <= 12 || ((int64_t)wh.nunits * num_profiles * (L - l + 1) >=
                                     (int64_t)pl->kn.units_per_warp * per_sm * SMS * (NTW / 32) &&
                                 wh.nunits >= pl->kn.units_per_cta * wh.cpr))
                    break;
            }
            const int by_smem = std::max<int>(1, (int)((228 * 1024) / (std::max<size_t>(wh.smem, 1) + 1024)));
            const int ps = std::max(1, std::min(CTAS_PER_SM, by_smem));
            if (ps == per_sm) break;
            per_sm = ps;
        }
        // batched sweeps: short waves (few units per range) one warp per (profile, range)
        // ... when there are enough (profile, range) pairs for >= 2 per resident warp slot
        if (num_profiles > 1 && pl->kn.fuse_fin && wh.nunits <= pl->kn.warp_units &&
            (int64_t)num_profiles * (L - l + 1) >= 2LL * CTAS_PER_SM * SMS * (NTW / 32)) {
            WaveHost ww = wh;
            ww.warp = true;
            build_wave(pl, l, per_sm * SMS, ww, chmax);
            ww.warp = true;
            ww.cpr = 1;
            if (ww.smem <= 113 * 1024) wh = ww;
        }
        // queue entries carry the accumulator entry in 16 bits and E', rl in 11 bits each
        if (wh.nout + L + 2 * TE_W + 2 > 0xFFFF || wh.max_row + TE_W > 2047) fits = false;
        wh.ents_off = items_total;
        items_total += align_up(wh.ents.size() * sizeof(int32_t), 16);
        wh.upre_off = items_total;
        items_total += align_up(wh.upre.size() * sizeof(int32_t), 16);
        wh.cb_off = items_total;
        items_total += align_up(wh.cb.size() * sizeof(int32_t), 16);
        gacc_max = std::max(gacc_max, (size_t)num_profiles * (L - l + 1) * wh.nout);
        // seeds cost ~18 scattered split evaluations per W output; they pay off where an output
        // has many splits (long rows: many flushes the seeded filter rejects)
        {
            int64_t wout = 0;
            for (int q = 2; q <= std::min(Q_of(g, l), l); ++q) wout += wlen_h(g, l, q);
            const double spo = wout ? (double)g.wave_splits[l] / ((double)(L - l + 1) * wout) : 0.0;
            wh.seed = pl->kn.seed_init && l >= pl->kn.seed_min_l && spo >= pl->kn.seed_spo;
        }
        wh.ctr_off = ctr_total;
        ctr_total += (size_t)num_profiles * (L - l + 1);
        wh.done_off = ctr_total;
        ctr_total += 2 * (size_t)num_profiles * (L - l + 1);   // merged CTAs, claimed finalize shares
        pl->max_smem = std::max(pl->max_smem, wh.smem);
    }
    pl->pipe_cnt_off = ctr_total;
    ctr_total += 3 * (size_t)(L + 2) + 1;
    pl->ctr_n = ctr_total;
    if (pl->max_smem > 227 * 1024 || !fits) pl->kernel = 1;
    pl->pipe_on = plan_pipe_on(pl);
    if (pl->kn.debug) {
        for (int l = 2; l <= L; ++l) {
            const WaveHost &wh = pl->waves[l];
            std::fprintf(stderr, "l=%d ents=%d units=%d cpr=%d ctas=%lld smem=%zu cost=%.3g seed=%d\n", l, wh.nents,
                         wh.nunits, wh.cpr, (long long)wh.cpr * (L - l + 1) * num_profiles, wh.smem, wh.cost,
                         (int)wh.seed);
        }
    }

    // plan-owned device geometry (read-only): uploaded once per device by oob_dp_run
    size_t o = 0;
    pl->off_cells = o; o = align_up(o + sizeof(int32_t) * (L + 1), 256);
    pl->off_base = o;  o = align_up(o + sizeof(int64_t) * (L + 2), 256);
    pl->off_off = o;   o = align_up(o + sizeof(int32_t) * (size_t)(L + 1) * g.A, 256);
    pl->off_wofs = o;  o = align_up(o + sizeof(int32_t) * (size_t)(L + 1) * (L + 2), 256);
    pl->off_pexp = o;  o = align_up(o + sizeof(int32_t) * 3 * (size_t)(L + 2), 256);
    pl->off_tiles = o; o = align_up(o + sizeof(int32_t) * std::max<size_t>(1, pl->tiles.size()), 256);
    pl->off_tile_off = o; o = align_up(o + sizeof(int32_t) * (L + 1), 256);
    pl->off_tile_cnt = o; o = align_up(o + sizeof(int32_t) * (L + 1), 256);
    pl->off_items = o;    o = align_up(o + items_total, 256);
    pl->geom_bytes = o;
    // caller-owned workspace: tables, accumulators, counters (re-initialised every run)
    o = 0;
    const size_t n = (size_t)g.table_cells * num_profiles;
    pl->off_CELL = o; o = align_up(o + 32 * (n + 16 + XR_CELLS), 256);   // + padding: row streams read ahead
    pl->off_SH = o; o = align_up(o + 16 * (n + 16 + XR_CELLS), 256);     // shadow lower bounds (+ padding)
    pl->off_ARG = o; o = align_up(o + 4 * n, 256);
    pl->gacc_n = (int64_t)gacc_max;
    pl->off_GACC = o; o = align_up(o + 3 * 16 * gacc_max, 256);   // three buffers (wave mod 3)
    pl->off_GFILT = o; o = align_up(o + 3 * 4 * gacc_max, 256);   // their filters
    pl->off_CTR = o; o = align_up(o + 4 * pl->ctr_n + 4, 256);
    pl->ws_bytes_base = o;
    pl->ws_bytes = o;
    pl->tpl_bytes = packed_template_bytes(L);
    pl->geom_blob.assign(pl->geom_bytes, 0);
    unsigned char *b = pl->geom_blob.data();
    std::memcpy(b + pl->off_cells, g.cells.data(), sizeof(int32_t) * (L + 1));
    std::memcpy(b + pl->off_base, g.base.data(), sizeof(int64_t) * (L + 2));
    std::memcpy(b + pl->off_off, g.off.data(), sizeof(int32_t) * (size_t)(L + 1) * g.A);
    {   // pipeline: blocks / shares that make each wave's seeds, in-node cells and W part ready
        int32_t *ex = reinterpret_cast<int32_t *>(b + pl->off_pexp);
        for (int l = 2; l <= L; ++l) {
            const WaveHost &wh = pl->waves[l];
            const int64_t nr = L - l + 1;
            if (l >= 3) {                       // produced by launch l-1's extra blocks
                const int64_t nsd = wh.seed ? (int64_t)num_profiles * nr * wh.nout : 0;
                ex[l] = (int32_t)((nsd + 255) / 256);
                ex[(L + 2) + l] = small_cells(g, l) > 0 ? (int32_t)small_blocks(pl, l) : 0;
            }
            ex[2 * (L + 2) + l] = wh.nents > 0 ? (int32_t)((int64_t)num_profiles * nr * wh.cpr) : 0;
        }
    }
    {   // W row offsets per slab length (I part + rows 1..q-1), DevGeom::wofs
        int32_t *wo = reinterpret_cast<int32_t *>(b + pl->off_wofs);
        for (int l = 0; l <= L; ++l) {
            const int ip = l >= M - 1 ? (M - 1) * M / 2 : l * (l + 1) / 2 + (M - 1 - l) * l;   // I(1..M-1) cells
            int acc = ip;
            wo[(size_t)l * (L + 2)] = ip;
            for (int q = 1; q <= L + 1; ++q) {
                wo[(size_t)l * (L + 2) + q] = acc;
                const int hi = std::min(l, M * q);
                acc += hi >= q ? hi - q + 1 : 0;
            }
        }
    }
    if (!pl->tiles.empty()) std::memcpy(b + pl->off_tiles, pl->tiles.data(), sizeof(int32_t) * pl->tiles.size());
    std::memcpy(b + pl->off_tile_off, pl->tile_off.data(), sizeof(int32_t) * (L + 1));
    std::memcpy(b + pl->off_tile_cnt, pl->tile_cnt.data(), sizeof(int32_t) * (L + 1));
    for (int l = 2; l <= L; ++l) {
        const WaveHost &wh = pl->waves[l];
        if (!wh.ents.empty())
            std::memcpy(b + pl->off_items + wh.ents_off, wh.ents.data(), wh.ents.size() * sizeof(int32_t));
        if (!wh.upre.empty())
            std::memcpy(b + pl->off_items + wh.upre_off, wh.upre.data(), wh.upre.size() * sizeof(int32_t));
        if (!wh.cb.empty())
            std::memcpy(b + pl->off_items + wh.cb_off, wh.cb.data(), wh.cb.size() * sizeof(int32_t));
    }
}

extern "C" oob_status oob_dp_plan_create(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi,
                                         int32_t num_profiles, oob_dp_plan **out) {
    if (!out) return fail(OOB_E_INVALID, "oob_dp_plan_create: out is NULL");
    if (num_profiles < 1) return fail(OOB_E_INVALID, "oob_dp_plan_create: num_profiles < 1");
    oob_dp_plan *pl = new (std::nothrow) oob_dp_plan();
    if (!pl) return fail(OOB_E_NOMEM, "oob_dp_plan_create: out of memory");
    if (!build_geometry(L, M, n_lo, n_hi, pl->g)) { delete pl; return OOB_E_INVALID; }
    pl->P = num_profiles;
    pl->kn = read_knobs();
    pl->kernel = pl->kn.kernel;
    pl->num_sms = device_sms();
    build_tiles(pl);
    pl->stream_steps.assign(L + 1, 0.0);
    for (int ls = 1; ls <= L; ++ls) {
        const int JS = std::min(Q_of(pl->g, ls), ls);
        for (int r = 1; r <= JS; ++r) pl->stream_steps[ls] += wlen_h(pl->g, ls, r) + 6.0;
    }
    size_plan(pl, 1);
    *out = pl;
    return OOB_OK;
}

// Device copies of the geometry blob (stale after size_plan; re-uploaded on the next run).
static void drop_device_geometry(oob_dp_plan *pl) {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &dg : pl->dev_geom)
        if (cudaSetDevice(dg.first) == cudaSuccess) cudaFree(dg.second);
    cudaSetDevice(cur);
    pl->dev_geom.clear();
}

// Peer exchange buffers of a sharded plan (see oob_dp_set_comm).
static void release_exchange(oob_dp_plan *pl) {
    if (!pl->xb) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->xb_dev);
    for (int r = 0; r < (int)pl->xb_peer.size(); ++r)
        if (r != pl->rank && pl->xb_peer[r]) cudaIpcCloseMemHandle(pl->xb_peer[r]);
    cudaFree(pl->xb);
    cudaSetDevice(cur);
    pl->xb = nullptr;
    pl->xb_peer.clear();
    pl->xpeer = false;
}

extern "C" void oob_dp_plan_free(oob_dp_plan *pl) {
    if (!pl) return;
    for (auto e : pl->ev) cudaEventDestroy(e);
    for (auto &dg : pl->dev_geom) {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cudaSetDevice(dg.first) == cudaSuccess) {
            cudaFree(dg.second);
            cudaSetDevice(cur);
        }
    }
    release_exchange(pl);
    delete pl;
}

// The plan's read-only device geometry on the current device (uploaded on first use).
static oob_status plan_geometry(oob_dp_plan *pl, unsigned char **geo) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    for (auto &dg : pl->dev_geom)
        if (dg.first == dev) { *geo = (unsigned char *)dg.second; return OOB_OK; }
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (sms != pl->num_sms)
        return fail(OOB_E_INVALID, "oob_dp_run: the plan was built for a device with " + std::to_string(pl->num_sms) +
                                       " SMs, the current device has " + std::to_string(sms) +
                                       " (create the plan with that device current)");
    void *p = nullptr;
    e = cudaMalloc(&p, pl->geom_bytes);
    if (e != cudaSuccess) return fail(OOB_E_NOMEM, std::string("cudaMalloc plan geometry: ") + cudaGetErrorString(e));
    e = cudaMemcpy(p, pl->geom_blob.data(), pl->geom_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(p); return cuda_fail(e, "plan geometry upload"); }
    {
        const size_t xs = 2 * 2 * (size_t)(pl->g.L + 1) * sizeof(XNode);
        if (xs > 48 * 1024 && (e = cudaFuncSetAttribute(k_extract, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs)) !=
                                  cudaSuccess) {
            cudaFree(p);
            return cuda_fail(e, "cudaFuncSetAttribute(k_extract)");
        }
    }
    if (pl->kernel == 2) {
        const int sm = (int)std::max<size_t>(pl->max_smem, 48 * 1024);
        e = cudaFuncSetAttribute(k_wave_w<TE_W>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        if (e != cudaSuccess) { cudaFree(p); return cuda_fail(e, "cudaFuncSetAttribute(k_wave_w)"); }
    }
    pl->dev_geom.emplace_back(dev, p);
    *geo = (unsigned char *)p;
    return OOB_OK;
}

// Kernels one oob_dp_run enqueues: k_init (accumulators + counters), k_base, k_fin
// (in-node cells of wave 2), per wave k_wave_w and, unless fused, k_fin; k_extract.
// v1: k_init, k_base, one kernel per wave, k_extract.
static int64_t count_launches(const oob_dp_plan *pl) {
    const Geometry &G = pl->g;
    if (pl->kernel == 1) return 3 + (G.L - 1);
    int64_t n = 4;
    for (int l = 2; l <= G.L; ++l) {
        const WaveHost &wh = pl->waves[l];
        const bool shard = pl->world > 1 && !wh.warp && (double)G.wave_splits[l] * pl->P >= pl->kn.shard_min;
        const bool has = wh.nents > 0;
        n += has ? 1 : 0;
        n += (pl->kn.fuse_fin && has && (!shard || pl->xpeer)) ? 0 : 1;
    }
    return n;
}

extern "C" oob_status oob_dp_plan_info(const oob_dp_plan *pl, oob_dp_info *out) {
    if (!pl || !out) return fail(OOB_E_INVALID, "oob_dp_plan_info: NULL argument");
    const Geometry &g = pl->g;
    out->L = g.L; out->M = g.M; out->n_lo = g.n_lo; out->n_hi = g.n_hi;
    out->num_profiles = pl->P;
    out->wavefronts = g.L - 1;
    out->cells_per_profile = g.total_cells;
    out->splits_per_profile = g.total_splits;
    out->kernel_launches = count_launches(pl);
    out->workspace_bytes = pl->ws_bytes;
    out->packed_template_bytes = pl->tpl_bytes;
    out->packed_profile_bytes = pl->tpl_bytes * (size_t)(g.n_hi - g.n_lo + 1);
    out->packed_bytes = out->packed_profile_bytes * pl->P;
    out->kernel = pl->kernel;
    out->pipelined = pl->pipe_on ? 1 : 0;
    out->fused = (pl->kernel == 2 && pl->kn.fuse_fin) ? 1 : 0;
    out->seeded = 0;
    for (int l = 2; l <= g.L; ++l) out->seeded += pl->waves[l].seed ? 1 : 0;
    out->chunk_max = pl->chunk_eff;
    out->refresh = pl->kn.refresh;
    out->small_pairs = pl->kn.small_pairs;
    out->num_sms = pl->num_sms;
    out->world = pl->world;
    out->warp_waves = 0;
    for (int l = 2; l <= g.L; ++l) out->warp_waves += pl->waves[l].warp ? 1 : 0;
    out->small_range = 0;
    for (int l = 2; l <= g.L; ++l) out->small_range += small_range_on(pl, l) ? 1 : 0;   // waves
    out->exchange = pl->world > 1 ? (pl->xpeer ? 1 : (pl->comm ? 2 : 3)) : 0;
    return OOB_OK;
}

extern "C" oob_status oob_dp_set_comm(oob_dp_plan *pl, void *comm, int32_t world, int32_t rank) {
    if (!pl || world < 1 || rank < 0 || rank >= world || (world > 1 && !comm))
        return fail(OOB_E_INVALID, "oob_dp_set_comm: bad argument");
    if (world > 1 && pl->kernel != 2)
        return fail(OOB_E_INVALID, "oob_dp_set_comm: sharding needs the W-kernel path");
    if (world > OOB_MAX_WORLD) return fail(OOB_E_INVALID, "oob_dp_set_comm: world above OOB_MAX_WORLD");
    release_exchange(pl);
    if (world != pl->sized_world) {          // per-rank unit shares: re-size the waves
        drop_device_geometry(pl);
        size_plan(pl, world);
        pl->sized_world = world;
    }
    pl->comm = world > 1 ? comm : nullptr;
    pl->world = world;
    pl->rank = world > 1 ? rank : 0;
    pl->off_GPART = pl->ws_bytes_base;
    pl->ws_bytes = pl->ws_bytes_base + (world > 1 ? align_up(16 * (size_t)world * pl->gacc_n, 256) : 0);
    if (world > 1 && pl->kn.shard_x && pl->kn.fuse_fin) {
        // peer exchange buffer, IPC handles all-gathered over the communicator (collective:
        // every rank calls oob_dp_set_comm)
        cudaError_t e;
        const size_t part = 3 * 16 * (size_t)world * pl->gacc_n;
        pl->xb_off_done = align_up(part, 256);
        pl->xb_bytes = pl->xb_off_done + align_up(4 * pl->ctr_n + 4, 256);
        if ((e = cudaGetDevice(&pl->xb_dev)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        if ((e = cudaMalloc(&pl->xb, pl->xb_bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc exchange buffer");
        if ((e = cudaMemset(pl->xb, 0, pl->xb_bytes)) != cudaSuccess) return cuda_fail(e, "cudaMemset exchange buffer");
        cudaIpcMemHandle_t h;
        if ((e = cudaIpcGetMemHandle(&h, pl->xb)) != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
        void *dh = nullptr;
        if ((e = cudaMalloc(&dh, sizeof(h) * (world + 1))) != cudaSuccess) return cuda_fail(e, "cudaMalloc handles");
        std::vector<cudaIpcMemHandle_t> all((size_t)world);
        e = cudaMemcpy(dh, &h, sizeof(h), cudaMemcpyHostToDevice);
        oob_status st = e == cudaSuccess ? nccl_allgather_bytes(comm, dh, (char *)dh + sizeof(h), sizeof(h),
                                                                 sizeof(h) * world, world, nullptr)
                                         : cuda_fail(e, "H2D handle");
        if (st == OOB_OK) {
            e = cudaMemcpy(all.data(), (char *)dh + sizeof(h), sizeof(h) * world, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) st = cuda_fail(e, "D2H handles");
        }
        cudaFree(dh);
        if (st != OOB_OK) { release_exchange(pl); return st; }
        pl->xb_peer.assign((size_t)world, nullptr);
        for (int r = 0; r < world; ++r) {
            if (r == rank) { pl->xb_peer[r] = pl->xb; continue; }
            e = cudaIpcOpenMemHandle(&pl->xb_peer[r], all[r], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) { release_exchange(pl); return cuda_fail(e, "cudaIpcOpenMemHandle (peer exchange)"); }
        }
        pl->xpeer = true;
    }
    pl->pipe_on = plan_pipe_on(pl);
    return OOB_OK;
}

extern "C" oob_status oob_dp_set_stage_masks(oob_dp_plan *pl, int32_t pow2_tp, const double *d_stage_bytes,
                                             double mem_cap_bytes) {
    if (!pl) return fail(OOB_E_INVALID, "oob_dp_set_stage_masks: NULL plan");
    if (d_stage_bytes && !(mem_cap_bytes > 0.0)) return fail(OOB_E_INVALID, "oob_dp_set_stage_masks: cap must be > 0");
    pl->mask_pow2 = pow2_tp ? 1 : 0;
    pl->mask_sb = d_stage_bytes;
    pl->mask_cap = mem_cap_bytes;
    return OOB_OK;
}

extern "C" oob_status oob_dp_set_timing(oob_dp_plan *pl, int32_t enable) {
    if (!pl) return fail(OOB_E_INVALID, "oob_dp_set_timing: NULL plan");
    pl->timing = enable ? 1 : 0;
    return OOB_OK;
}

static oob_status harvest_events(oob_dp_plan *pl) {
    for (int i = 0; i + 1 < pl->ev_used; i += 2) {
        cudaError_t e = cudaEventSynchronize(pl->ev[i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, pl->ev[i], pl->ev[i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        pl->acc_ms += ms;
        pl->acc_launches += 1;
    }
    pl->ev_used = 0;
    return OOB_OK;
}

extern "C" oob_status oob_dp_kernel_time(oob_dp_plan *pl, double *ms_out, int64_t *launches_out,
                                         int32_t reset) {
    if (!pl) return fail(OOB_E_INVALID, "oob_dp_kernel_time: NULL plan");
    oob_status s = harvest_events(pl);
    if (s != OOB_OK) return s;
    if (ms_out) *ms_out = pl->acc_ms;
    if (launches_out) *launches_out = pl->acc_launches;
    if (reset) { pl->acc_ms = 0.0; pl->acc_launches = 0; }
    return OOB_OK;
}

// accumulator of wave l: three buffers (wave mod 3): k_fin / the fused finalize reads wave
// l-1's while the seeds of wave l+1 fill another
static ulonglong2 *gacc_of(const oob_dp_plan *pl, ulonglong2 *gacc, int l) {
    return gacc + (size_t)(l % 3) * (size_t)pl->gacc_n;
}
// global filter of wave l's accumulator (same buffer and index)
static unsigned *gfilt_of(const oob_dp_plan *pl, ulonglong2 *gacc, int l) {
    return (unsigned *)((unsigned char *)gacc - pl->off_GACC + pl->off_GFILT) + (size_t)(l % 3) * (size_t)pl->gacc_n;
}

// Finalize arguments for wave lw (0: none) and in-node cells + seeds of wave ls (0: none);
// *nbsmall receives the blocks of the small-cell part.
static FinArgs make_fin(const oob_dp_plan *pl, const DevGeom &dg, ulonglong2 *gacc, int lw, int ls, bool sharded,
                        int64_t *nbsmall, const ulonglong2 *gpart = nullptr) {
    const int lsd = ls;                 // seeds of the same wave as the in-node cells
    const Geometry &G = pl->g;
    FinArgs f;
    f.lw = lw;
    f.nranges_w = lw ? G.L - lw + 1 : 0;
    f.nout_w = lw ? pl->waves[lw].nout : 0;
    const int64_t nw = (int64_t)pl->P * f.nranges_w * f.nout_w;
    f.nbw = (int)((nw + 255) / 256);
    f.GACC = gacc_of(pl, gacc, lw);
    f.GFW = gfilt_of(pl, gacc, lw);
    f.world = sharded ? pl->world : 1;
    f.part_stride = (int64_t)pl->P * f.nranges_w * f.nout_w;   // all-gather: rank r at r x (wave partial)
    f.GPART = gpart ? gpart : (const ulonglong2 *)((const unsigned char *)dg.CELL - pl->off_CELL + pl->off_GPART);
    // seeds for wave ls (children of length <= ls-2: final before this launch)
    f.lseed = (lsd >= 2 && lsd <= G.L && pl->waves[lsd].seed) ? lsd : 0;
    f.nout_s = f.lseed ? pl->waves[lsd].nout : 0;
    const int64_t nsd = f.lseed ? (int64_t)pl->P * (G.L - lsd + 1) * f.nout_s : 0;
    f.nbseed = (int)((nsd + 255) / 256);
    f.GSEED = gacc_of(pl, gacc, lsd);
    f.GFS = gfilt_of(pl, gacc, lsd);
    f.ls = ls;
    f.nsmall = ls ? small_cells(G, ls) : 0;
    f.tpc = ls ? small_tpc(G, ls, pl->kn.small_pairs) : 32;
    f.small_range = (ls && small_range_on(pl, ls)) ? 1 : 0;
    *nbsmall = (ls && f.nsmall > 0) ? small_blocks(pl, ls) : 0;
    return f;
}

static cudaError_t launch_fin(const oob_dp_plan *pl, const DevGeom &dg, ulonglong2 *gacc, int lw, int ls,
                              cudaStream_t stream, bool sharded = false) {
    int64_t nbs = 0;
    const FinArgs f = make_fin(pl, dg, gacc, lw, ls, sharded, &nbs);
    const int64_t blocks = f.nbw + f.nbseed + nbs;
    if (blocks == 0) return cudaSuccess;
    k_fin<<<(unsigned)blocks, 256, f.small_range ? SR_SMEM : 0, stream>>>(dg, f);
    return cudaGetLastError();
}

// One rank's state of a run: its workspace (tables, accumulators, counters) and output.
struct RankRun {
    unsigned char *ws;
    unsigned char *packed;
    int rank;
    DevGeom dg;
    ulonglong2 *gacc;
    int *ctr;
    Pipe pp;
};

// The template set for `nr` local rank contexts on the current device and stream.
// nr = 1: one GPU (world = 1) or this process's rank of an NCCL-sharded plan; nr = world > 1
// with comm = NULL: virtual shards — every rank's kernels run on this device, one after the
// other per wavefront, and the all-gather of the partial argmins is a set of device copies
// (the sharded algorithm, checkable on one GPU).
static oob_status run_ranks(oob_dp_plan *pl, const double *d_fwd, const double *d_bwd, RankRun *rr, int nr,
                            cudaStream_t stream) {
    const Geometry &G = pl->g;
    unsigned char *geo = nullptr;
    oob_status gs = plan_geometry(pl, &geo);
    if (gs != OOB_OK) return gs;
    cudaError_t e;
    const bool pipe_on = pl->pipe_on;
    if (pl->xpeer) ++pl->epoch;           // peer counters: targets epoch x world (never reset)
    for (int i = 0; i < nr; ++i) {
        RankRun &R = rr[i];
        DevGeom &dg = R.dg;
        dg.L = G.L; dg.M = G.M; dg.n_lo = G.n_lo; dg.n_hi = G.n_hi; dg.A = G.A; dg.P = pl->P;
        dg.C = G.table_cells;
        dg.cells = (const int32_t *)(geo + pl->off_cells);
        dg.base = (const int64_t *)(geo + pl->off_base);
        dg.off = (const int32_t *)(geo + pl->off_off);
        dg.wofs = (const int32_t *)(geo + pl->off_wofs);
        dg.CELL = (Cell4 *)(R.ws + pl->off_CELL);
        dg.SH = (float4 *)(R.ws + pl->off_SH);
        dg.ARG = (uint32_t *)(R.ws + pl->off_ARG);
        dg.pow2 = pl->mask_pow2;
        dg.SB = pl->mask_sb;
        dg.mem_cap = pl->mask_cap;
        dg.masked = (pl->mask_pow2 || pl->mask_sb) ? 1 : 0;
        R.gacc = (ulonglong2 *)(R.ws + pl->off_GACC);
        R.ctr = (int *)(R.ws + pl->off_CTR);
        R.pp.cnt = R.ctr + pl->pipe_cnt_off;
        R.pp.expc = (const int *)(geo + pl->off_pexp);
        R.pp.err = R.pp.cnt + 3 * (G.L + 2);
        R.pp.on = pipe_on ? 1 : 0;
        R.pp.spin_max = pl->kn.spin_max;
        {   // every run starts from a clean workspace state: accumulators, filters, counters
            const int64_t nacc = pl->kernel == 2 ? 3 * pl->gacc_n : 0;
            const int64_t nmax = std::max<int64_t>(nacc, (int64_t)pl->ctr_n + 1);
            k_init<<<(unsigned)((nmax + 255) / 256), 256, 0, stream>>>(R.gacc, gfilt_of(pl, R.gacc, 0), nacc, R.ctr,
                                                                      (int64_t)pl->ctr_n + 1);
            if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_init launch");
        }
        {   // K_base: grid.y = l
            int64_t maxn = (int64_t)G.L * G.M * pl->P;
            dim3 grid((unsigned)((maxn + 255) / 256), (unsigned)G.L);
            k_base<<<grid, 256, 0, stream>>>(dg, d_fwd, d_bwd);
            if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_base launch");
        }
        if (pl->kernel == 2 && G.L >= 2 && (e = launch_fin(pl, dg, R.gacc, 0, 2, stream)) != cudaSuccess)
            return cuda_fail(e, "k_fin launch");
    }
    if (pl->timing) {
        size_t need = 2 * (size_t)(G.L - 1) + pl->ev_used;
        while (pl->ev.size() < need) {
            cudaEvent_t ev;
            e = cudaEventCreate(&ev);
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
            pl->ev.push_back(ev);
        }
    }
    for (int l = 2; l <= G.L; ++l) {
        if (pl->kernel == 1) {
            int64_t n = (int64_t)(G.L - l + 1) * G.cells[l] * pl->P;
            if (n == 0) continue;
            if (pl->timing) cudaEventRecord(pl->ev[pl->ev_used], stream);
            for (int i = 0; i < nr; ++i) k_wave_v1<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(rr[i].dg, l);
            if (pl->timing) { cudaEventRecord(pl->ev[pl->ev_used + 1], stream); pl->ev_used += 2; }
            if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_wave_v1 launch");
            continue;
        }
        const WaveHost &wh = pl->waves[l];
        // shard only wavefronts whose work outweighs the all-gather (~10-20 us on NVLink);
        // short wavefronts run redundantly on every rank (identical results, no exchange)
        const bool shard = pl->world > 1 && !wh.warp && (double)G.wave_splits[l] * pl->P >= pl->kn.shard_min;
        const bool peer = shard && pl->xpeer;   // fused exchange through peer memory
        const int64_t ctas = wh.nents == 0 ? 0
                             : wh.warp ? ((int64_t)pl->P * (G.L - l + 1) + NTW / 32 - 1) / (NTW / 32)
                                       : (int64_t)pl->P * (G.L - l + 1) * wh.cpr;
        // fused finalize (OOB_DP_FUSE=1): unsharded waves finalize in k_wave_w's last CTAs
        // and run the next wave's in-node cells and seeds in extra blocks
        const bool fused = pl->kn.fuse_fin && ctas > 0 && (!shard || peer);
        if (pl->timing && (!pipe_on || l == 2)) cudaEventRecord(pl->ev[pl->ev_used], stream);
        for (int i = 0; i < nr && ctas > 0; ++i) {
            RankRun &R = rr[i];
            WaveW w{};
            w.l = l;
            w.nranges = G.L - l + 1;
            w.cpr = wh.cpr;
            w.nents = wh.nents;
            w.ents = (const int4 *)(geo + pl->off_items + wh.ents_off);
            w.upre = (const int32_t *)(geo + pl->off_items + wh.upre_off);
            w.cb = (const int32_t *)(geo + pl->off_items + wh.cb_off);
            w.ncb = (int)wh.cb.size();
            w.ctr = R.ctr + wh.ctr_off;
            w.nunits = wh.nunits;
            w.seeded = wh.seed;
            w.nout = wh.nout;
            w.GACC = gacc_of(pl, R.gacc, l);
            w.GFILT = gfilt_of(pl, R.gacc, l);
            w.tile_off = (const int32_t *)(geo + pl->off_tile_off);
            w.tile_cnt = (const int32_t *)(geo + pl->off_tile_cnt);
            w.tiles = (const int32_t *)(geo + pl->off_tiles);
            w.rank = shard ? R.rank : 0;
            w.world = shard ? pl->world : 1;
            int64_t aux = 0;
            w.nbmain = (int)ctas;
            w.refresh = pl->kn.refresh && wh.cpr > 1 && l >= pl->kn.refresh_lmin;   // one CTA per range: its own filter is current
            w.fin_spin = pl->kn.fin_wait != 0 ? (1 << 22) : 0;
            // only the range's last merged CTAs (~512 outputs each) wait — for the range's other
            // CTAs, and with a peer exchange for the other ranks' partials — and share the
            // finalize; the others leave at once and their slots go to the next wave
            // (OOB_DP_FINWAIT=1: every CTA helps, 0: the last alone; cfg4 14.54 -> 14.24 ms,
            // sharded over 4 GPUs 9.04 -> 7.43 ms)
            // (peer exchange: 768 outputs per helper, 4 GPUs 7.43 -> 7.35 ms)
            const int fin_help = pl->kn.fin_help > 0 ? pl->kn.fin_help : (peer ? 768 : 512);
            w.fin_helpers = pl->kn.fin_wait > 0 ? wh.cpr
                            : pl->kn.fin_wait == 0 ? 1
                                                   : std::max(1, std::min(wh.cpr, (wh.nout + fin_help - 1) / fin_help));
            w.warp_mode = wh.warp ? 1 : 0;
            // batched sweeps (one CTA per range, small shared memory, a larger L1): the exact
            // path's children are worth warming in L1 (cfg5 -2%; neutral to negative for cfg4)
            w.prefetch = wh.cpr == 1 && pl->P > 1;
            w.fin_inline = fused ? 1 : 0;
            w.rdone = R.ctr + wh.done_off;
            w.rclaim = w.rdone + (size_t)pl->P * w.nranges;
            w.peer = peer ? 1 : 0;
            w.epoch = pl->epoch;
            const size_t xpar = (size_t)(l % 3) * 16 * (size_t)pl->world * pl->gacc_n;   // this wave's gather buffer
            for (int r = 0; r < OOB_MAX_WORLD; ++r) {
                w.xpart[r] = (peer && r < pl->world) ? (ulonglong2 *)((unsigned char *)pl->xb_peer[r] + xpar) : nullptr;
                w.xdone[r] = (peer && r < pl->world)
                                 ? (int *)((unsigned char *)pl->xb_peer[r] + pl->xb_off_done) + wh.done_off
                                 : nullptr;
            }
            if (fused) {
                int64_t nbs = 0, nbw = 0;
                w.fa = make_fin(pl, R.dg, R.gacc, 0, l < G.L ? l + 1 : 0, false, &nbs);
                w.fw = make_fin(pl, R.dg, R.gacc, l, 0, peer, &nbw,
                                peer ? (const ulonglong2 *)((unsigned char *)pl->xb + xpar) : nullptr);
                aux = w.fa.nbseed + nbs;
            }
            w.pp = R.pp;
            const unsigned grid = (unsigned)(ctas + aux);
            if (pipe_on && l >= 3) {   // programmatic dependent of wave l-1 (counters, not the boundary)
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(grid);
                lc.blockDim = dim3(NTW);
                lc.dynamicSmemBytes = wh.smem;
                lc.stream = stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                e = cudaLaunchKernelEx(&lc, k_wave_w<TE_W>, R.dg, w);
                if (e != cudaSuccess) return cuda_fail(e, "k_wave_w launch (pipelined)");
            } else {
                k_wave_w<TE_W><<<grid, NTW, wh.smem, stream>>>(R.dg, w);
            }
            if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_wave_w launch");
        }
        if (pl->timing && (!pipe_on || l == G.L)) {
            cudaEventRecord(pl->ev[pl->ev_used + 1], stream);
            pl->ev_used += 2;
        }
        if (shard && !peer) {   // all-gather of the wave's partial argmins (every rank finalizes all)
            const size_t bytes = 16 * (size_t)pl->P * (G.L - l + 1) * wh.nout;
            if (pl->comm) {
                oob_status st = nccl_allgather_bytes(pl->comm, gacc_of(pl, rr[0].gacc, l), rr[0].ws + pl->off_GPART,
                                                     bytes, 16 * (size_t)pl->gacc_n, pl->world, stream);
                if (st != OOB_OK) return st;
            } else {   // virtual shards: rank r's partial into slot r of every rank's gather buffer
                for (int d = 0; d < nr; ++d)
                    for (int r = 0; r < nr; ++r) {
                        e = cudaMemcpyAsync(rr[d].ws + pl->off_GPART + (size_t)rr[r].rank * bytes,
                                            gacc_of(pl, rr[r].gacc, l), bytes, cudaMemcpyDeviceToDevice, stream);
                        if (e != cudaSuccess) return cuda_fail(e, "virtual-shard gather copy");
                    }
            }
        }
        for (int i = 0; i < nr && !fused; ++i)   // (peer-exchanged waves finalize inside k_wave_w)
            if ((e = launch_fin(pl, rr[i].dg, rr[i].gacc, l, l < G.L ? l + 1 : 0, stream, shard)) != cudaSuccess)
                return cuda_fail(e, "k_fin launch");
    }
    for (int i = 0; i < nr; ++i) {
        // one warp per template; 2 warps per block (frontier: 2 x (L+1) nodes of 16 B per warp)
        const int n = (G.n_hi - G.n_lo + 1) * pl->P;
        const size_t xs = 2 * 2 * (size_t)(G.L + 1) * sizeof(XNode);
        k_extract<<<(n + 1) / 2, 64, xs, stream>>>(rr[i].dg, rr[i].packed, pl->tpl_bytes, rr[i].pp);
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_extract launch");
    }
    return OOB_OK;
}

extern "C" oob_status oob_dp_run(oob_dp_plan *pl, const double *d_fwd, const double *d_bwd,
                                 void *d_ws, size_t ws_bytes, void *d_packed, void *stream_) {
    if (!pl || !d_fwd || !d_bwd || !d_ws || !d_packed)
        return fail(OOB_E_INVALID, "oob_dp_run: NULL argument");
    if (ws_bytes < pl->ws_bytes) return fail(OOB_E_NOMEM, "oob_dp_run: workspace too small");
    if (pl->world > 1 && !pl->comm)
        return fail(OOB_E_INVALID, "oob_dp_run: plan has virtual shards; use oob_dp_run_virtual");
    RankRun r{(unsigned char *)d_ws, (unsigned char *)d_packed, pl->rank, {}, nullptr, nullptr, {}};
    return run_ranks(pl, d_fwd, d_bwd, &r, 1, (cudaStream_t)stream_);
}

extern "C" oob_status oob_dp_set_virtual_shards(oob_dp_plan *pl, int32_t world) {
    if (!pl || world < 1 || world > 64) return fail(OOB_E_INVALID, "oob_dp_set_virtual_shards: bad argument");
    if (world > 1 && pl->kernel != 2)
        return fail(OOB_E_INVALID, "oob_dp_set_virtual_shards: sharding needs the W-kernel path");
    release_exchange(pl);
    if (world != pl->sized_world) {
        drop_device_geometry(pl);
        size_plan(pl, world);
        pl->sized_world = world;
    }
    pl->comm = nullptr;
    pl->world = world;
    pl->rank = 0;
    pl->off_GPART = pl->ws_bytes_base;
    pl->ws_bytes = pl->ws_bytes_base + (world > 1 ? align_up(16 * (size_t)world * pl->gacc_n, 256) : 0);
    pl->pipe_on = plan_pipe_on(pl);
    return OOB_OK;
}

extern "C" oob_status oob_dp_run_virtual(oob_dp_plan *pl, const double *d_fwd, const double *d_bwd,
                                         void *const *d_ws, size_t ws_bytes, void *const *d_packed, void *stream_) {
    if (!pl || !d_fwd || !d_bwd || !d_ws || !d_packed)
        return fail(OOB_E_INVALID, "oob_dp_run_virtual: NULL argument");
    if (pl->comm) return fail(OOB_E_INVALID, "oob_dp_run_virtual: plan has an NCCL communicator");
    if (ws_bytes < pl->ws_bytes) return fail(OOB_E_NOMEM, "oob_dp_run_virtual: workspace too small");
    std::vector<RankRun> rr((size_t)pl->world);
    for (int r = 0; r < pl->world; ++r) {
        if (!d_ws[r] || !d_packed[r]) return fail(OOB_E_INVALID, "oob_dp_run_virtual: NULL workspace or output");
        rr[r] = RankRun{(unsigned char *)d_ws[r], (unsigned char *)d_packed[r], r, {}, nullptr, nullptr, {}};
    }
    return run_ranks(pl, d_fwd, d_bwd, rr.data(), pl->world, (cudaStream_t)stream_);
}

// Diagnostic (not part of the C ABI header): enable/read the flush counters of k_wave_w.
extern "C" int oob_dbg_flush_stats(int enable, unsigned long long *out4) {
    if (out4) {
        if (cudaMemcpyFromSymbol(out4, oob::g_flush_stats, sizeof(unsigned long long) * 4) != cudaSuccess) return 1;
    }
    unsigned long long z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(oob::g_flush_stats, z, sizeof(z)) != cudaSuccess) return 1;
    return cudaMemcpyToSymbol(oob::g_flush_stats_on, &enable, sizeof(int)) == cudaSuccess ? 0 : 1;
}

// Diagnostic (not part of the C ABI header; -DOOB_TIMELINE builds only): read and reset the
// per-wave timeline of k_wave_w (8 x u64 per wave, see g_tl).
extern "C" int oob_dbg_timeline(unsigned long long *out, int nwaves) {
#ifdef OOB_TIMELINE
    if (nwaves > 1024) return 1;
    if (out && cudaMemcpyFromSymbol(out, oob::g_tl, sizeof(unsigned long long) * 8 * nwaves) != cudaSuccess) return 1;
    static unsigned long long init[1024][8];
    for (int i = 0; i < 1024; ++i)
        for (int j = 0; j < 8; ++j) init[i][j] = (j == 0 || j == 1 || j == 4) ? ~0ull : 0ull;
    return cudaMemcpyToSymbol(oob::g_tl, init, sizeof(init)) == cudaSuccess ? 0 : 1;
#else
    (void)out; (void)nwaves;
    return 2;
#endif
}
