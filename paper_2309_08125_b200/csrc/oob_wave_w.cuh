// Wavefront kernel for whole-node cells W(q >= 2) — the hot loop.
//
// For a range (u, v) of length l and a layer split k (l1 = k-u, l2 = v-k), the W(q) cells
// of the range combine left children W(j) of (u, k) with right children W(q-j) of (k, v)
// (PAPER Eq.1-3 with the two-level device split, reading R2).  In (nodes, stages)
// coordinates every pair (left cell, right cell) is a valid split of exactly one parent
// cell (q = j + j', S' = s + S_R), so for each row pair (j, j') the work is a dense
// a_j x b_j' rectangle of splits.  Mapping:
//   * the child slab with more W cells ("big side") is register-tiled: each lane holds TE
//     consecutive cells of one row (one (j, e-block) tile); tiles of one row stay in one
//     warp; several passes when tiles > threads;
//   * the other slab ("small side") is staged in shared memory and iterated row by row,
//     cell by cell, in lock-step by the whole CTA (shared-memory broadcast);
//   * each lane keeps the TE outputs its tile currently touches in a register ring (the
//     outputs slide by one cell per step); the output whose last contribution from this
//     lane has arrived is flushed into a shared-memory accumulator holding, per parent
//     cell, the lexicographic minimum of (total, canonical split key).
// Tie semantics: the oracle keeps the first strictly-smaller total in (k, m, s) order.
// Inside a ring slot the pairs of one (k, j) arrive in decreasing s, so "<=" keeps the
// smallest s; every flush and every cross-CTA merge compares (total, key) with
// key = l1<<20 | j<<10 | s, which is monotone in (k, m, s) — so the result is exactly the
// oracle's argmin, whatever the CTA / pass / row processing order.
// Races (no CTA barrier per row): warp w holds tiles of a contiguous block of big-side
// rows [a_w, b_w) with b_w <= a_{w+1} (rows never straddle warps), and every warp walks
// the staged rows j' in increasing order.  Warp w starts row j' only after warp w+1 has
// started row j' (neighbour chain through shared-memory progress counters, published
// after a block fence).  Then at any time j'_w <= j'_{w+1}, and the output rows touched,
// q in [a_w + j'_w, b_w - 1 + j'_w], are disjoint between warps.  Inside a warp the
// lanes of one row flush distinct outputs per step and __syncwarp orders the steps.
#pragma once

namespace oob {

constexpr int NT_MAX = 256;               // max threads per CTA of k_wave_w

struct WaveW {
    int l;                 // wavefront length
    int nranges;           // L - l + 1
    int nitems;            // work items per range
    const int4 *items;     // per item: (l1_lo, l1_hi excl, it_lo, it_hi excl)  (it rows 1-based)
    int nout;              // W-part cells of a slab of length l (W(1)..W(Q_l))
    int ns_max;            // max W-part cells of the staged (small) side over the items
    double *PB;            // partial best  [P][nranges][nitems][nout]
    uint32_t *PK;          // partial key
    const int32_t *tile_off;   // [L+1] offset of the tile table of a big side of length l_big
    const int32_t *tile_np;    // [L+1] number of passes
    const int32_t *tiles;      // packed (row << 16 | e0) or -1, [pass][blockDim]
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

struct Reg5 { double T1, T3, TS, c1, c2; };

// One split, operands already in "left / right" roles.  c1 = (3S-1)+k* of its own cell;
// c2 = 4s for the left cell, 3S_R for the right cell, so that
//   left wins : coef = 3S'-1+k*_L      = R.c2 + L.c1
//   right wins: coef = 3S'-1+s+k*_R    = L.c2 + R.c1     (exact small integers)
__device__ __forceinline__ void split_eval(double LT1, double LT3, double LTS, double Lc1, double Lc2,
                                           double RT1, double RT3, double RTS, double Rc1, double Rc2,
                                           double &best, int &widx, int code) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double cL = __dadd_rn(Rc2, Lc1);
    const double cR = __dadd_rn(Lc2, Rc1);
    const double TS = left ? LTS : RTS;
    const double T3 = left ? T3a : RT3;
    const double c = left ? cL : cR;
    const double T2 = __dmul_rn(c, TS);
    const double tot = __dadd_rn(__dadd_rn(T1, T2), T3);
    const bool upd = tot <= best;
    best = upd ? tot : best;
    widx = upd ? code : widx;
}

__device__ __forceinline__ void acc_merge(double *accB, uint32_t *accK, int idx, double b, uint32_t key) {
    const double A = accB[idx];
    const uint32_t K = accK[idx];
    if (b < A || (b == A && key < K)) {
        accB[idx] = b;
        accK[idx] = key;
    }
}

constexpr double D_INF = __builtin_huge_val();

template <int TE>
__global__ void __launch_bounds__(NT_MAX, (TE <= 4 ? 2 : 1)) k_wave_w(DevGeom g, WaveW w) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int l = w.l;
    const int nout = w.nout;
    double *accB = reinterpret_cast<double *>(smem);
    uint32_t *accK = reinterpret_cast<uint32_t *>(accB + nout);
    size_t o = ((size_t)nout * 12 + 15) / 16 * 16;
    double2 *sA = reinterpret_cast<double2 *>(smem + o);            // (T1, T3)
    double2 *sB = sA + w.ns_max;                                      // (TS, c1)
    double *sC = reinterpret_cast<double *>(sB + w.ns_max);           // c2
    int *outOff = reinterpret_cast<int *>(sC + w.ns_max);             // [L+2] W(q) offsets in slab l
    int *itOff = outOff + (g.L + 2);                                  // [L+2] staged rows
    int *itLen = itOff + (g.L + 2);
    volatile int *prog = reinterpret_cast<volatile int *>(itLen + (g.L + 2));   // [NT/32]
    const int NT = blockDim.x;
    const int nwarps = NT >> 5;
    const int warp = threadIdx.x >> 5;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    int bid = blockIdx.x;
    const int item = bid % w.nitems; bid /= w.nitems;
    const int u = bid % w.nranges;
    const int p = bid / w.nranges;
    const int64_t pc = (int64_t)p * g.C;
    const int4 it = w.items[item];
    const int Ql = (l == g.L) ? g.n_hi : max(1, g.n_hi - 1);

    for (int i = tid; i < nout; i += NT) { accB[i] = D_INF; accK[i] = 0xFFFFFFFFu; }
    for (int q = tid; q < g.L + 2; q += NT) outOff[q] = (q >= 1 && q <= Ql && q <= l) ? d_woff(g, l, q) : -1;

    for (int l1 = it.x; l1 < it.y; ++l1) {
        const int k = u + l1;
        const int l2 = l - l1;
        const bool ltiled = d_wcells(g, l1) >= d_wcells(g, l2);   // big side = left
        const int ls = ltiled ? l2 : l1;                           // staged (small) side length
        const int lb = ltiled ? l1 : l2;
        const int us = ltiled ? k : u;                             // staged slab start
        const int ub = ltiled ? u : k;
        const int Qs = (ls == g.L) ? g.n_hi : max(1, g.n_hi - 1);
            const int JS = min(Qs, ls);                                 // rows of the staged side
        const int it_lo = max(1, it.z), it_hi = min(JS + 1, it.w);
        __syncthreads();   // previous k done with the staging buffers
        // ---- stage the small side's W rows it_lo..it_hi-1 (with derived c1, c2)
        const int64_t sbase = pc + g.base[ls] + (int64_t)us * g.cells[ls] + g.off[ls * g.A + (g.M - 1)];
        for (int r = tid; r < g.L + 2; r += NT) {
            itOff[r] = (r >= 1 && r <= JS) ? d_woff(g, ls, r) : 0;
            itLen[r] = (r >= 1 && r <= JS) ? d_wlen(g, ls, r) : 0;
        }
        {
            for (int r = it_lo + warp; r < it_hi; r += nwarps) {
                const int ro = d_woff(g, ls, r), rl = d_wlen(g, ls, r);
                for (int e = lane; e < rl; e += 32) {
                    const int64_t c = sbase + ro + e;
                    const int S = r + e;
                    const double kd = g.KD[c];
                    sA[ro + e] = make_double2(g.T1[c], g.T3[c]);
                    sB[ro + e] = make_double2(g.TS[c], __dadd_rn((double)(3 * S - 1), kd));
                    sC[ro + e] = ltiled ? (double)(3 * S) : (double)(4 * S);
                }
            }
        }
        __syncthreads();
        // ---- passes over the big side's tiles
        const int np = w.tile_np[lb];
        const int32_t *tt = w.tiles + w.tile_off[lb];
        const int64_t bbase = pc + g.base[lb] + (int64_t)ub * g.cells[lb];
        for (int pass = 0; pass < np; ++pass) {
            const int32_t code = tt[pass * NT + tid];
            const bool has = code >= 0;
            const int rowB = has ? (code >> 16) : 1;
            const int e0 = has ? (code & 0xFFFF) : 0;
            const int lenB = has ? d_wlen(g, lb, rowB) : 0;
            const int offB = has ? g.off[lb * g.A + (g.M - 1) + rowB - 1] : 0;
            Reg5 R[TE];
#pragma unroll
            for (int t = 0; t < TE; ++t) {
                if (has && e0 + t < lenB) {
                    const int64_t c = bbase + offB + e0 + t;
                    const int S = rowB + e0 + t;
                    R[t].T1 = g.T1[c]; R[t].T3 = g.T3[c]; R[t].TS = g.TS[c];
                    R[t].c1 = __dadd_rn((double)(3 * S - 1), g.KD[c]);
                    R[t].c2 = ltiled ? (double)(4 * S) : (double)(3 * S);
                } else {
                    R[t].T1 = D_INF; R[t].T3 = D_INF; R[t].TS = D_INF; R[t].c1 = 1.0; R[t].c2 = 1.0;
                }
            }
            // warps without any tile in this pass step aside (progress = +inf)
            const bool wactive = __any_sync(0xFFFFFFFFu, has);
            if (lane == 0) prog[warp] = wactive ? it_lo - 1 : 0x3FFFFFFF;
            __syncthreads();
            for (int rs = it_lo; wactive && rs < it_hi; ++rs) {
                // publish "started rs" (our flushes of rs-1 are done), then wait for w+1
                __threadfence_block();
                if (lane == 0) {
                    prog[warp] = rs;
                    if (warp + 1 < nwarps)
                        while (prog[warp + 1] < rs) { }
                }
                __syncwarp();
                __threadfence_block();
                const int q = rowB + rs;
                const int ob = (has && q <= g.L + 1) ? outOff[q] : -1;
                const bool qok = ob >= 0;
                const int rl = itLen[rs];
                const int ro = itOff[rs];
                double best[TE];
                int widx[TE];
#pragma unroll
                for (int t = 0; t < TE; ++t) { best[t] = D_INF; widx[t] = 0; }
                if (ltiled) {
                    // big = left row j = rowB (tile e0..e0+TE-1); iterate right row j' = rs,
                    // e' ascending.  Ring slot r <-> output E with (E - e0) % TE == r.
                    const int j = rowB;
#pragma unroll 1
                    for (int base = 0; base < rl; base += TE) {
#pragma unroll
                        for (int i = 0; i < TE; ++i) {
                            const int ep = base + i;
                            if (ep < rl) {
                                const double2 a = sA[ro + ep];
                                const double2 bb = sB[ro + ep];
                                const double cc = sC[ro + ep];
#pragma unroll
                                for (int t = 0; t < TE; ++t)
                                    split_eval(R[t].T1, R[t].T3, R[t].TS, R[t].c1, R[t].c2,
                                               a.x, a.y, bb.x, bb.y, cc, best[(i + t) % TE], widx[(i + t) % TE], t);
                                if (qok && best[i] < D_INF) {
                                    const int E = e0 + ep;
                                    const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) |
                                                         (uint32_t)(j + e0 + widx[i]);
                                    acc_merge(accB, accK, ob + E, best[i], key);
                                }
                                best[i] = D_INF;
                                __syncwarp();
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < TE; ++r) {
                        if (qok && best[r] < D_INF) {
                            const int E = e0 + rl + (((r - rl) % TE) + TE) % TE;
                            const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)j << 10) |
                                                 (uint32_t)(j + e0 + widx[r]);
                            acc_merge(accB, accK, ob + E, best[r], key);
                        }
                    }
                } else {
                    // big = right row j' = rowB (tile e0'..); iterate left row j = rs,
                    // e descending.  Step i = rl-1-e; slot (t - i) % TE holds output
                    // E = e + e0 + t; the t = TE-1 output completes at each step.
                    const int jl = rs;
#pragma unroll 1
                    for (int base = 0; base < rl; base += TE) {
#pragma unroll
                        for (int i = 0; i < TE; ++i) {
                            const int st = base + i;
                            if (st < rl) {
                                const int e = rl - 1 - st;
                                const double2 a = sA[ro + e];
                                const double2 bb = sB[ro + e];
                                const double cc = sC[ro + e];
#pragma unroll
                                for (int t = 0; t < TE; ++t)
                                    split_eval(a.x, a.y, bb.x, bb.y, cc,
                                               R[t].T1, R[t].T3, R[t].TS, R[t].c1, R[t].c2,
                                               best[((t - i) % TE + TE) % TE], widx[((t - i) % TE + TE) % TE], t);
                                const int sf = ((TE - 1 - i) % TE + TE) % TE;
                                if (qok && best[sf] < D_INF) {
                                    const int E = e + e0 + TE - 1;
                                    const int s = jl + E - e0 - widx[sf];
                                    const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)jl << 10) | (uint32_t)s;
                                    acc_merge(accB, accK, ob + E, best[sf], key);
                                }
                                best[sf] = D_INF;
                                __syncwarp();
                            }
                        }
                    }
                    // pending: after the last step (i = rl-1, e = 0) slot sigma holds
                    // t = (sigma + rl - 1) % TE, output E = e0 + t.
#pragma unroll
                    for (int sg = 0; sg < TE; ++sg) {
                        if (qok && best[sg] < D_INF) {
                            const int t = (sg + rl - 1) % TE;
                            const int E = e0 + t;
                            const int s = jl + E - e0 - widx[sg];
                            const uint32_t key = ((uint32_t)l1 << 20) | ((uint32_t)jl << 10) | (uint32_t)s;
                            acc_merge(accB, accK, ob + E, best[sg], key);
                        }
                    }
                }
            }
            __syncthreads();   // pass done (all flushes visible before the next pass/k)
        }
    }
    __syncthreads();
    const size_t pb = (size_t)blockIdx.x * nout;
    for (int i = tid; i < nout; i += NT) {
        w.PB[pb + i] = accB[i];
        w.PK[pb + i] = accK[i];
    }
}

// Per W(q >= 2) cell: lexicographic min of the items' partials, then the winner's
// (T1, T3, t*, k*) recomputed from its two children (same arithmetic as the oracle).
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
    // which W(q) row holds W-part offset i
    int q = 0, Sp = 0;
    for (int qq = 2; qq <= min(Ql, l); ++qq) {
        const int o = d_woff(g, l, qq);
        const int len = d_wlen(g, l, qq);
        if (o >= 0 && i >= o && i < o + len) { q = qq; Sp = qq + (i - o); break; }
    }
    if (q == 0) return;       // W(1) cell (handled by k_wave_small) or padding
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
    const int64_t c = pc + g.base[l] + (int64_t)u * g.cells[l] + g.off[l * g.A + (g.M - 1)] + i;
    if (!(best < D_INF)) {     // no split found: impossible for a valid cell; poison it
        g.T1[c] = __longlong_as_double(0x7ff8000000000000LL);
        g.ARG[c] = 0xFFFFFFFEu;
        return;
    }
    const int l1 = (int)(key >> 20), j = (int)((key >> 10) & 1023u), s = (int)(key & 1023u);
    const int k = u + l1, l2 = l - l1;
    const int aL = (g.M - 1) + j - 1, aR = (g.M - 1) + (q - j) - 1;
    const int64_t cL = pc + d_cell(g, s, u, l1, aL);
    const int64_t cR = pc + d_cell(g, Sp - s, k, l2, aR);
    const double LT1 = g.T1[cL], LT3 = g.T3[cL], LTS = g.TS[cL], LKD = g.KD[cL];
    const double RT1 = g.T1[cR], RT3 = g.T3[cR], RTS = g.TS[cR], RKD = g.KD[cR];
    const double T1 = __dadd_rn(LT1, RT1);
    const bool left = LTS >= RTS;
    g.T1[c] = T1;
    g.T3[c] = left ? __dadd_rn(LT3, RT1) : RT3;
    g.TS[c] = left ? LTS : RTS;
    g.KD[c] = left ? LKD : __dadd_rn((double)s, RKD);
    g.ARG[c] = (uint32_t)(l1 - 1) | ((uint32_t)(j - 1) << 10) | ((uint32_t)s << 20);
}

// I(r) and W(1) cells with S' >= 2 (GPUs inside one node): one warp per cell, lanes take
// contiguous k ranges, then a lexicographic (total, key) warp-shuffle argmin.
__global__ void k_wave_small(DevGeom g, int l) {
    const int nsmall = min(g.A, g.M);              // alloc indices 0..M-1: I(1..M-1), W(1)
    const int nr = g.L - l + 1;
    const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    // cells per range: for a in 0..M-1 and S' in 2..hi(a, l)
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
                const int64_t cL = pc + d_cell(g, s, u, l1, a1);
                const int64_t cR = pc + d_cell(g, Sp - s, k, l2, a2);
                const double LT1 = g.T1[cL], LT3 = g.T3[cL], LTS = g.TS[cL], LKD = g.KD[cL];
                const double RT1 = g.T1[cR], RT3 = g.T3[cR], RTS = g.TS[cR], RKD = g.KD[cR];
                const double T1 = __dadd_rn(LT1, RT1);
                const bool left = LTS >= RTS;
                const double T3 = left ? __dadd_rn(LT3, RT1) : RT3;
                const double TS = left ? LTS : RTS;
                const double KD = left ? LKD : __dadd_rn((double)s, RKD);
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
    const int l1 = (int)(bkey >> 20), j = (int)((bkey >> 10) & 1023u), s = (int)(bkey & 1023u);
    const int k = u + l1, l2 = l - l1;
    int a1, a2;
    d_dsplit(g, a, j, a1, a2);
    const int64_t cL = pc + d_cell(g, s, u, l1, a1);
    const int64_t cR = pc + d_cell(g, Sp - s, k, l2, a2);
    const double LT1 = g.T1[cL], LT3 = g.T3[cL], LTS = g.TS[cL], LKD = g.KD[cL];
    const double RT1 = g.T1[cR], RT3 = g.T3[cR], RTS = g.TS[cR], RKD = g.KD[cR];
    const bool left = LTS >= RTS;
    const int64_t c = pc + d_cell(g, Sp, u, l, a);
    g.T1[c] = __dadd_rn(LT1, RT1);
    g.T3[c] = left ? __dadd_rn(LT3, RT1) : RT3;
    g.TS[c] = left ? LTS : RTS;
    g.KD[c] = left ? LKD : __dadd_rn((double)s, RKD);
    g.ARG[c] = (uint32_t)(l1 - 1) | ((uint32_t)j << 10) | ((uint32_t)s << 20);
}

}  // namespace oob
