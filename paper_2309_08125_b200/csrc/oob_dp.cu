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
#include <cstring>
#include <mutex>
#include <vector>

#include "oob_internal.h"

namespace oob {

// ------------------------------------------------------------------ device geometry
struct DevGeom {
    int L, M, n_lo, n_hi, A, P;
    int64_t C;                // cells per profile
    const int32_t *cells;     // [L+1]
    const int64_t *base;      // [L+2]
    const int32_t *off;       // [(L+1)*A]
    double *T1, *T3, *TS, *KD;  // [P*C]
    uint32_t *ARG;              // [P*C]
    uint64_t *STK;              // [P*p*(L+1)] backtrack stacks
};

__device__ __forceinline__ bool d_is_whole(const DevGeom &g, int a) { return a >= g.M - 1; }
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
__device__ __forceinline__ int64_t d_cell(const DevGeom &g, int Sp, int u, int l, int a) {
    return g.base[l] + (int64_t)u * g.cells[l] + g.off[l * g.A + a] + (Sp - d_lo(g, a));
}

// ------------------------------------------------------------------ K_base: Eq.4
// One thread per (profile, u, base alloc) of wavefront l = blockIdx.y + 1.  Base allocs:
// I(r), r = 1..M-1 (d = r) and W(1) (d = M).
__global__ void k_base(DevGeom g, const double *__restrict__ fwd, const double *__restrict__ bwd) {
    const int l = blockIdx.y + 1;
    const int nu = g.L - l + 1;
    const int per_prof = nu * g.M;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)per_prof * g.P) return;
    const int p = (int)(t / per_prof);
    const int r = (int)(t % per_prof);
    const int u = r / g.M;
    const int ai = r % g.M;                 // 0..M-2 -> I(ai+1); M-1 -> W(1)
    const int a = ai;                        // alloc index coincides (W(1) = M-1)
    const int d = ai + 1;                    // I(r): r GPUs; W(1): M GPUs
    if (g.off[l * g.A + a] < 0) return;
    const double *F = fwd + (size_t)p * g.L * g.M;
    const double *B = bwd + (size_t)p * g.L * g.M;
    double s = 0.0;
    for (int k = u; k < u + l; ++k) s = __dadd_rn(s, __dadd_rn(F[k * g.M + d - 1], B[k * g.M + d - 1]));
    const int64_t c = (int64_t)p * g.C + d_cell(g, 1, u, l, a);
    g.T1[c] = s; g.T3[c] = s; g.TS[c] = s; g.KD[c] = 0.0;
    g.ARG[c] = 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ K_wave (v1)
// One thread per (profile, u, cell of the slab) for wavefront l; S' = 1 cells are skipped.
__global__ void k_wave_v1(DevGeom g, int l) {
    const int nu = g.L - l + 1;
    const int cl = g.cells[l];
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nu * cl * g.P) return;
    const int p = (int)(t / ((int64_t)nu * cl));
    const int rem = (int)(t % ((int64_t)nu * cl));
    const int u = rem / cl;
    const int i = rem % cl;
    // find the allocation holding slab offset i
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
    double bT1 = 0, bT3 = 0, bTS = 0, bKD = 0;
    uint32_t barg = 0xFFFFFFFFu;
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
                    best = tot; bT1 = T1; bT3 = T3; bTS = TS; bKD = KD;
                    barg = (uint32_t)(l1 - 1) | ((uint32_t)j << 10) | ((uint32_t)s << 20);
                }
            }
        }
    }
    const int64_t c = pc + d_cell(g, Sp, u, l, a);
    g.T1[c] = bT1; g.T3[c] = bT3; g.TS[c] = bTS; g.KD[c] = bKD; g.ARG[c] = barg;
}

// ------------------------------------------------------------------ K_extract
// One thread per (profile, template size n): argmin over S (strict <, smaller S wins),
// then the split-tree backtrack (left child first => stages in pipeline order).
__global__ void k_extract(DevGeom g, unsigned char *packed, size_t tpl_bytes) {
    const int p_cnt = g.n_hi - g.n_lo + 1;
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= p_cnt * g.P) return;
    const int p = t / p_cnt;
    const int n = g.n_lo + t % p_cnt;
    const int64_t pc = (int64_t)p * g.C;
    const int L = g.L;
    const int aW = (g.M - 1) + n - 1;
    PackedHeader *h = reinterpret_cast<PackedHeader *>(packed + (size_t)t * tpl_bytes);
    int32_t *st = reinterpret_cast<int32_t *>(h + 1);
    int bestS = -1;
    double best = 0.0;
    const int Smax = min(L, n * g.M);
    for (int S = n; S <= Smax; ++S) {
        const int64_t c = pc + d_cell(g, S, 0, L, aW);
        const double T2 = __dmul_rn(__dadd_rn(g.KD[c], (double)(3 * S - 1)), g.TS[c]);
        const double tot = __dadd_rn(__dadd_rn(g.T1[c], T2), g.T3[c]);
        if (bestS < 0 || tot < best) { best = tot; bestS = S; }
    }
    const int64_t c = pc + d_cell(g, bestS, 0, L, aW);
    h->nodes = n; h->S = bestS; h->kstar = (int)g.KD[c]; h->status = 0;
    h->T1 = g.T1[c]; h->T3 = g.T3[c]; h->tstar = g.TS[c];
    h->T2 = __dmul_rn(__dadd_rn(g.KD[c], (double)(3 * bestS - 1)), g.TS[c]);
    h->iter = best;
    h->pad = 0.0;
    // explicit DFS stack in the workspace (<= L pending entries): packed
    // Sp | u<<10 | v<<20 | a<<30 | node<<41 | goff<<51
    uint64_t *stk = g.STK + (size_t)t * (size_t)(L + 1);
    auto pack = [](int Sp, int u, int v, int a, int node, int goff) -> uint64_t {
        return (uint64_t)Sp | ((uint64_t)u << 10) | ((uint64_t)v << 20) | ((uint64_t)a << 30) |
               ((uint64_t)node << 41) | ((uint64_t)goff << 51);
    };
    int top = 0, ns = 0;
    stk[top++] = pack(bestS, 0, L, aW, 0, 0);
    while (top > 0) {
        const uint64_t e = stk[--top];
        const int Sp = (int)(e & 1023u), u = (int)((e >> 10) & 1023u), v = (int)((e >> 20) & 1023u);
        const int a = (int)((e >> 30) & 2047u), node = (int)((e >> 41) & 1023u), goff = (int)((e >> 51) & 63u);
        if (Sp == 1) {
            int32_t *r = st + 5 * ns;
            r[0] = u; r[1] = v; r[2] = d_is_whole(g, a) ? g.M : d_alloc_n(g, a); r[3] = node; r[4] = goff;
            ++ns;
            continue;
        }
        const uint32_t arg = g.ARG[pc + d_cell(g, Sp, u, v - u, a)];
        const int k = u + (int)(arg & 1023u) + 1;
        const int j = (int)((arg >> 10) & 1023u);
        const int s = (int)(arg >> 20);
        int a1, a2;
        d_dsplit(g, a, j, a1, a2);
        const bool wsplit = d_is_whole(g, a) && d_alloc_n(g, a) >= 2;
        // push right, then left (popped first => stages come out in pipeline order)
        stk[top++] = wsplit ? pack(Sp - s, k, v, a2, node + d_alloc_n(g, a1), 0)
                            : pack(Sp - s, k, v, a2, node, goff + d_alloc_n(g, a1));
        stk[top++] = pack(s, u, k, a1, node, wsplit ? 0 : goff);
    }
    for (int i = ns; i < L; ++i) {
        int32_t *r = st + 5 * i;
        r[0] = r[1] = r[2] = r[3] = r[4] = -1;
    }
}

}  // namespace oob

// ==================================================================== plan + C ABI
using namespace oob;

struct oob_dp_plan {
    Geometry g;
    int32_t P = 1;
    size_t geom_bytes = 0, ws_bytes = 0, tpl_bytes = 0;
    std::vector<unsigned char> geom_blob;   // host image of the geometry region
    size_t off_cells = 0, off_base = 0, off_off = 0, off_T1 = 0, off_T3 = 0, off_TS = 0, off_KD = 0, off_ARG = 0, off_STK = 0;
    void *uploaded_to = nullptr;
    int timing = 0;
    std::vector<cudaEvent_t> ev;            // pairs per wavefront launch
    int ev_used = 0;
    double acc_ms = 0.0;
    int64_t acc_launches = 0;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static oob_status cuda_fail(cudaError_t e, const char *what) {
    return fail(OOB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

extern "C" oob_status oob_dp_plan_create(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi,
                                         int32_t num_profiles, oob_dp_plan **out) {
    if (!out) return fail(OOB_E_INVALID, "oob_dp_plan_create: out is NULL");
    if (num_profiles < 1) return fail(OOB_E_INVALID, "oob_dp_plan_create: num_profiles < 1");
    oob_dp_plan *pl = new (std::nothrow) oob_dp_plan();
    if (!pl) return fail(OOB_E_NOMEM, "oob_dp_plan_create: out of memory");
    if (!build_geometry(L, M, n_lo, n_hi, pl->g)) { delete pl; return OOB_E_INVALID; }
    pl->P = num_profiles;
    const Geometry &g = pl->g;
    size_t o = 0;
    pl->off_cells = o; o = align_up(o + sizeof(int32_t) * (L + 1), 256);
    pl->off_base = o;  o = align_up(o + sizeof(int64_t) * (L + 2), 256);
    pl->off_off = o;   o = align_up(o + sizeof(int32_t) * (size_t)(L + 1) * g.A, 256);
    pl->geom_bytes = o;
    const size_t n = (size_t)g.total_cells * num_profiles;
    pl->off_T1 = o;  o = align_up(o + 8 * n, 256);
    pl->off_T3 = o;  o = align_up(o + 8 * n, 256);
    pl->off_TS = o;  o = align_up(o + 8 * n, 256);
    pl->off_KD = o;  o = align_up(o + 8 * n, 256);
    pl->off_ARG = o; o = align_up(o + 4 * n, 256);
    pl->off_STK = o; o = align_up(o + 8 * (size_t)num_profiles * (n_hi - n_lo + 1) * (L + 1), 256);
    pl->ws_bytes = o;
    pl->tpl_bytes = packed_template_bytes(L);
    pl->geom_blob.assign(pl->geom_bytes, 0);
    std::memcpy(pl->geom_blob.data() + pl->off_cells, g.cells.data(), sizeof(int32_t) * (L + 1));
    std::memcpy(pl->geom_blob.data() + pl->off_base, g.base.data(), sizeof(int64_t) * (L + 2));
    std::memcpy(pl->geom_blob.data() + pl->off_off, g.off.data(), sizeof(int32_t) * (size_t)(L + 1) * g.A);
    *out = pl;
    return OOB_OK;
}

extern "C" void oob_dp_plan_free(oob_dp_plan *pl) {
    if (!pl) return;
    for (auto e : pl->ev) cudaEventDestroy(e);
    delete pl;
}

extern "C" oob_status oob_dp_plan_info(const oob_dp_plan *pl, oob_dp_info *out) {
    if (!pl || !out) return fail(OOB_E_INVALID, "oob_dp_plan_info: NULL argument");
    const Geometry &g = pl->g;
    out->L = g.L; out->M = g.M; out->n_lo = g.n_lo; out->n_hi = g.n_hi;
    out->num_profiles = pl->P;
    out->wavefronts = g.L - 1;
    out->cells_per_profile = g.total_cells;
    out->splits_per_profile = g.total_splits;
    out->kernel_launches = 1 + (g.L - 1) + 1;
    out->workspace_bytes = pl->ws_bytes;
    out->packed_template_bytes = pl->tpl_bytes;
    out->packed_profile_bytes = pl->tpl_bytes * (size_t)(g.n_hi - g.n_lo + 1);
    out->packed_bytes = out->packed_profile_bytes * pl->P;
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

extern "C" oob_status oob_dp_run(oob_dp_plan *pl, const double *d_fwd, const double *d_bwd,
                                 void *d_ws, size_t ws_bytes, void *d_packed, void *stream_) {
    if (!pl || !d_fwd || !d_bwd || !d_ws || !d_packed)
        return fail(OOB_E_INVALID, "oob_dp_run: NULL argument");
    if (ws_bytes < pl->ws_bytes) return fail(OOB_E_NOMEM, "oob_dp_run: workspace too small");
    cudaStream_t stream = (cudaStream_t)stream_;
    const Geometry &G = pl->g;
    unsigned char *ws = (unsigned char *)d_ws;
    cudaError_t e;
    if (pl->uploaded_to != d_ws) {
        e = cudaMemcpyAsync(ws, pl->geom_blob.data(), pl->geom_bytes, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return cuda_fail(e, "geometry upload");
        e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_fail(e, "geometry upload sync");
        pl->uploaded_to = d_ws;
    }
    DevGeom dg;
    dg.L = G.L; dg.M = G.M; dg.n_lo = G.n_lo; dg.n_hi = G.n_hi; dg.A = G.A; dg.P = pl->P;
    dg.C = G.total_cells;
    dg.cells = (const int32_t *)(ws + pl->off_cells);
    dg.base = (const int64_t *)(ws + pl->off_base);
    dg.off = (const int32_t *)(ws + pl->off_off);
    dg.T1 = (double *)(ws + pl->off_T1);
    dg.T3 = (double *)(ws + pl->off_T3);
    dg.TS = (double *)(ws + pl->off_TS);
    dg.KD = (double *)(ws + pl->off_KD);
    dg.ARG = (uint32_t *)(ws + pl->off_ARG);
    dg.STK = (uint64_t *)(ws + pl->off_STK);

    {   // K_base: grid.y = l
        int64_t maxn = (int64_t)G.L * G.M * pl->P;
        dim3 grid((unsigned)((maxn + 255) / 256), (unsigned)G.L);
        k_base<<<grid, 256, 0, stream>>>(dg, d_fwd, d_bwd);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "k_base launch");
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
        int64_t n = (int64_t)(G.L - l + 1) * G.cells[l] * pl->P;
        if (n == 0) continue;
        if (pl->timing) cudaEventRecord(pl->ev[pl->ev_used], stream);
        k_wave_v1<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(dg, l);
        if (pl->timing) { cudaEventRecord(pl->ev[pl->ev_used + 1], stream); pl->ev_used += 2; }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "k_wave launch");
    }
    {
        int n = (G.n_hi - G.n_lo + 1) * pl->P;
        k_extract<<<(n + 63) / 64, 64, 0, stream>>>(dg, (unsigned char *)d_packed, pl->tpl_bytes);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "k_extract launch");
    }
    return OOB_OK;
}
