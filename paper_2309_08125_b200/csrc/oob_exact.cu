// Exact optimum of the paper's 1F1B objective per template, on the GPU (SURVEY §0.1's
// "exact variant", §8(f) row 4).  The paper's recursion (Eqs.1-4, oob_dp.cu) keeps one
// argmin per memo cell and is a heuristic: on random profiles it misses the optimum of its
// own objective by up to 15%.  This solver returns, for every template size n,
// the minimum of the closed form over EVERY mapping of the L layers onto n nodes x M GPUs
// (contiguous stages, no stage across nodes, every GPU used).
//
// With stage times t_i, bottleneck tau = t_{k*} (k* = first maximum) and N_b = 4S
// (P:381-386):
//     total = sum_{i<k*} (t_i + 4 tau) + sum_{i>k*} (2 t_i + 3 tau) + 4 tau,
// so for a fixed tau the stages before the bottleneck (t < tau) and after it (t <= tau) are
// two independent shortest paths over (layer boundary, GPUs used):
//     Pre[l][m]  = min over tilings of layers [0, l) x GPUs [0, m)        of sum (t + 4 tau)
//     Suf[l][r]  = min over tilings of layers [l, L) x the LAST r GPUs    of sum (2t + 3 tau)
// (Suf is indexed by the GPUs remaining, so one table serves every n: node boundaries are
// multiples of M from either end), and the optimum for n is the minimum over every stage
// time tau and every placement (a, b, d, m) of a bottleneck stage with t(a, b, d) = tau of
//     (Pre[a][m] + Suf[b][nM - m - d]) + 4 tau.
// Only tau <= ub_n / (3n + 1) can beat a known total ub_n (every stage adds >= 3 tau, the
// bottleneck 4 tau, S >= n): the heuristic's own templates bound the search.
//
// Results are bit-identical to the CPU oracle (oracle/c/oob_exact.c, a separate per-n
// push-form implementation): every path cost is accumulated in the same order with the
// same binary64 operations (--fmad=false), ties between equal values go to the smallest
// tau, then the first (a, m, d, b), then the oracle's parent priorities (prefix: smallest
// previous boundary, then most GPUs; suffix: largest next boundary, then most GPUs), and
// the returned costs are the closed form of the chosen stages summed left to right.
//
// Kernels (all enqueued on the caller's stream, no host synchronisation):
//   k_ex_times  stage times T[p][d][v][u] (left-to-right sums, reading R12)
//   k_ex_hash   one representative entry per distinct stage time (open-addressing hash)
//   k_ex_window per-n windows tau <= ub_n / (3n + 1) (1 + 1e-12); accumulators reset
//   k_ex_tasks  task list: (profile, representative entry) with tau inside some window
//   k_ex_solve  persistent CTAs: per task Pre, Suf, then per n a block min of the
//               bottleneck placements -> 128-bit lexicographic atomic min of (total, tau)
//   k_ex_recon  persistent CTAs: per (profile, n) re-run the winning tau with parents,
//               walk them, write the packed template (oob_dp_run's layout)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "oob_internal.h"

namespace {

constexpr int EXT = 256;                            // threads per CTA
constexpr int EXS = 256;                            // k_ex_solve threads per CTA
constexpr int EX_CTAS_PER_SM = 6;                  // k_ex_solve (latency bound: many resident tasks)
constexpr int EX_RECON_PER_SM = 2;
constexpr double EX_INF = __builtin_huge_val();
// a stage-time loop whose sums are not built from one start point may see an out-of-order
// rounding: stop only clearly past tau (rounding of <= 1023 positive terms is ~1e-13 relative)
constexpr double EX_BRK = 1.0 + 0x1p-30;

struct ExGeom {
    int L, M, n_lo, n_hi, nsz, P;
    int Gmax, W;        // W = Gmax + 1: row stride of the DP tables
    int E;              // T entries per profile: M (L+1)^2
    int H;              // hash slots per profile
    int slots;          // k_ex_solve persistent CTAs (value scratch owners)
    int rslots;         // k_ex_recon persistent CTAs (value + parent scratch owners)
    int list_cap;       // bottleneck stage list (shared memory)
    size_t tpl_bytes, prof_bytes;
};

struct ExWs {
    unsigned long long *ctr;   // [0] tasks, [1] next task, [2] next (profile, n), [3] list overflow
    double *T;                 // [P][E]
    unsigned long long *hkey;  // [P][H]
    int *hidx;                 // [P][H]
    double *tw;                // [P][nsz]
    double *twmax;             // [P]
    int2 *tasks;               // [P * M * L (L+1) / 2]
    ulonglong2 *acc;           // [P][nsz]: x = total bits, y = tau bits
    double *dp;                // [slots][2][(L+1) W]
    int *par;                  // [slots][2][(L+1) W]
};

__host__ __device__ inline size_t t_index(int L, int d, int v, int u) {
    return ((size_t)(d - 1) * (L + 1) + v) * (L + 1) + u;
}

__device__ __forceinline__ unsigned hash_bits(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (unsigned)x;
}

__device__ __forceinline__ void cas128(ulonglong2 *p, unsigned long long &olo, unsigned long long &ohi,
                                       unsigned long long clo, unsigned long long chi, unsigned long long nlo,
                                       unsigned long long nhi) {
    asm volatile("{\n\t.reg .b128 d, c, v;\n\t"
                 "mov.b128 c, {%2, %3};\n\t"
                 "mov.b128 v, {%4, %5};\n\t"
                 "atom.global.cas.b128 d, [%6], c, v;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(olo), "=l"(ohi)
                 : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "l"(p)
                 : "memory");
}

// lexicographic min of (total, tau) — both positive binary64, so their bit patterns order
// like the values
__device__ void acc_min(ulonglong2 *a, unsigned long long v, unsigned long long tau) {
    unsigned long long cx = a->x, cy = a->y;
    while (v < cx || (v == cx && tau < cy)) {
        unsigned long long ox, oy;
        cas128(a, ox, oy, cx, cy, v, tau);
        if (ox == cx && oy == cy) break;
        cx = ox;
        cy = oy;
    }
}

// ------------------------------------------------------------------ stage times, dedupe
__global__ void k_ex_times(ExGeom g, const double *__restrict__ fwd, const double *__restrict__ bwd, double *T) {
    const int p = blockIdx.x / g.M, d = blockIdx.x % g.M + 1;
    const double *F = fwd + (size_t)p * g.L * g.M, *B = bwd + (size_t)p * g.L * g.M;
    double *Tp = T + (size_t)p * g.E;
    for (int u = threadIdx.x; u < g.L; u += blockDim.x) {
        double s = 0.0;
        for (int v = u + 1; v <= g.L; ++v) {
            s = __dadd_rn(s, __dadd_rn(F[(size_t)(v - 1) * g.M + d - 1], B[(size_t)(v - 1) * g.M + d - 1]));
            Tp[t_index(g.L, d, v, u)] = s;
        }
    }
}

__device__ __forceinline__ bool entry_valid(const ExGeom &g, int e, int &d, int &v, int &u) {
    u = e % (g.L + 1);
    const int r = e / (g.L + 1);
    v = r % (g.L + 1);
    d = r / (g.L + 1) + 1;
    return u < v;
}

__global__ void k_ex_hash(ExGeom g, const double *__restrict__ T, unsigned long long *hkey, int *hidx) {
    const int64_t n = (int64_t)g.P * g.E;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(i / g.E), e = (int)(i % g.E);
        int d, v, u;
        if (!entry_valid(g, e, d, v, u)) continue;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(T[i]);
        unsigned long long *K = hkey + (size_t)p * g.H;
        int *I = hidx + (size_t)p * g.H;
        unsigned h = hash_bits(bits) & (unsigned)(g.H - 1);
        for (;;) {
            const unsigned long long prev = atomicCAS(K + h, 0ull, bits);
            if (prev == 0ull || prev == bits) {
                atomicMin(I + h, e);
                break;
            }
            h = (h + 1) & (unsigned)(g.H - 1);
        }
    }
}

__global__ void k_ex_window(ExGeom g, const double *__restrict__ fwd, const double *__restrict__ bwd,
                            const unsigned char *__restrict__ packed_ub, double *tw, double *twmax, ulonglong2 *acc) {
    const int p = blockIdx.x;
    __shared__ double s_max, s_clb;
    if (threadIdx.x == 0) {
        // C_lb <= sum of all stage times of any mapping (every layer runs on some d <= M
        // GPUs), shrunk by 2^-30 for rounding: total >= (C_lb - tau) + (3n + 1) tau
        const double *F = fwd + (size_t)p * g.L * g.M, *B = bwd + (size_t)p * g.L * g.M;
        double c = 0.0;
        for (int l = 0; l < g.L; ++l) {
            double m = EX_INF;
            for (int d = 0; d < g.M; ++d) m = fmin(m, __dadd_rn(F[(size_t)l * g.M + d], B[(size_t)l * g.M + d]));
            c = __dadd_rn(c, m);
        }
        s_clb = __dmul_rn(c, 1.0 - 0x1p-30);
        s_max = 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < g.nsz; i += blockDim.x) {
        const int n = g.n_lo + i;
        double w = EX_INF;
        if (packed_ub) {
            const oob::PackedHeader *h =
                (const oob::PackedHeader *)(packed_ub + (size_t)p * g.prof_bytes + (size_t)i * g.tpl_bytes);
            if (h->status == 0 && h->S > 0) {
                // every stage adds >= 3 tau, the bottleneck 4 tau, S >= n: total >= (3n + 1) tau;
                // and total >= C_lb + 3n tau (above) — only tau under both bounds can win
                const double w1 = __ddiv_rn(h->iter, __dadd_rn(__dmul_rn(3.0, (double)n), 1.0));
                const double w2 = __ddiv_rn(__dadd_rn(h->iter, -s_clb), __dmul_rn(3.0, (double)n));
                w = __dmul_rn(fmin(w1, w2), __dadd_rn(1.0, 1e-12));
            }
        }
        tw[(size_t)p * g.nsz + i] = w;
        acc[(size_t)p * g.nsz + i] = make_ulonglong2(~0ull, ~0ull);
        atomicMax((unsigned long long *)&s_max, (unsigned long long)__double_as_longlong(w));
    }
    __syncthreads();
    if (threadIdx.x == 0) twmax[p] = s_max;
}

__global__ void k_ex_tasks(ExGeom g, const double *__restrict__ T, const unsigned long long *__restrict__ hkey,
                           const int *__restrict__ hidx, const double *__restrict__ twmax, int2 *tasks,
                           unsigned long long *ctr) {
    const int64_t n = (int64_t)g.P * g.E;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(i / g.E), e = (int)(i % g.E);
        int d, v, u;
        if (!entry_valid(g, e, d, v, u)) continue;
        const double tau = T[i];
        if (!(tau <= twmax[p])) continue;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(tau);
        const unsigned long long *K = hkey + (size_t)p * g.H;
        unsigned h = hash_bits(bits) & (unsigned)(g.H - 1);
        while (K[h] != bits) h = (h + 1) & (unsigned)(g.H - 1);
        if (hidx[(size_t)p * g.H + h] != e) continue;       // not the representative of its value
        const unsigned long long k = atomicAdd(ctr + 0, 1ull);
        tasks[k] = make_int2(p, e);
    }
}

// ------------------------------------------------------------------ the two shortest paths
// Pre over rows l = 0..L and m = 0..G; Suf over rows l = L..0 and r = 0..G (GPUs remaining),
// one thread per target, recording the parent (previous boundary << 8 | GPUs) with the
// oracle's priorities on equal values (k_ex_recon).
__device__ void ex_paths(const ExGeom &g, const double *__restrict__ Tp, int G, double tau, double *pre, double *suf,
                         int *ppar, int *spar) {
    const int L = g.L, M = g.M, W = g.W;
    const double t4 = __dmul_rn(4.0, tau), t3 = __dmul_rn(3.0, tau), brk = __dmul_rn(tau, EX_BRK);
    for (int m = threadIdx.x; m <= G; m += blockDim.x) {
        pre[m] = m == 0 ? 0.0 : EX_INF;
        suf[(size_t)L * W + m] = m == 0 ? 0.0 : EX_INF;
    }
    __syncthreads();
    for (int l2 = 1; l2 <= L; ++l2) {
        for (int m = threadIdx.x; m <= G; m += blockDim.x) {
            double best = EX_INF;
            int bl = 0, bd = 0;
            if (m > 0) {
                const int dm = (m - 1) % M + 1;                 // the stage stays inside its node
                for (int d = 1; d <= dm; ++d) {
                    const double *tc = Tp + t_index(L, d, l2, 0);
                    for (int l = l2 - 1; l >= 0; --l) {
                        const double t = tc[l];
                        if (t >= brk) break;
                        if (!(t < tau)) continue;
                        const double pv = pre[(size_t)l * W + m - d];
                        if (pv == EX_INF) continue;
                        const double v = __dadd_rn(pv, __dadd_rn(t, t4));
                        if (v < best || (v == best && (l < bl || (l == bl && d > bd)))) {
                            best = v;
                            bl = l;
                            bd = d;
                        }
                    }
                }
            }
            pre[(size_t)l2 * W + m] = best;
            ppar[(size_t)l2 * W + m] = (bl << 8) | bd;
        }
        __syncthreads();
    }
    for (int l0 = L - 1; l0 >= 0; --l0) {
        for (int r = threadIdx.x; r <= G; r += blockDim.x) {
            double best = EX_INF;
            int bl = 0, bd = 0;
            if (r > 0) {
                const int dm = (r - 1) % M + 1;
                for (int d = 1; d <= dm; ++d) {
                    for (int l = l0 + 1; l <= L; ++l) {
                        const double t = Tp[t_index(L, d, l, l0)];
                        if (t > brk) break;
                        if (!(t <= tau)) continue;
                        const double sv = suf[(size_t)l * W + r - d];
                        if (sv == EX_INF) continue;
                        const double v = __dadd_rn(sv, __dadd_rn(__dmul_rn(2.0, t), t3));
                        if (v < best || (v == best && (l > bl || (l == bl && d > bd)))) {
                            best = v;
                            bl = l;
                            bd = d;
                        }
                    }
                }
            }
            suf[(size_t)l0 * W + r] = best;
            spar[(size_t)l0 * W + r] = (bl << 8) | bd;
        }
        __syncthreads();
    }
}

// Value-only paths (k_ex_solve): the same recurrences as ex_paths, with the (GPU count,
// stage GPUs) pairs of a row spread over the threads (few GPUs but long stage ranges for
// large tau) and a shared-memory min per target; equal values need no tie rule here.
__device__ void ex_paths_fast(const ExGeom &g, const double *__restrict__ Tp, int G, double tau, double *pre,
                              double *suf, unsigned long long *s_row) {
    const int L = g.L, M = g.M, W = g.W;
    const double t4 = __dmul_rn(4.0, tau), t3 = __dmul_rn(3.0, tau), brk = __dmul_rn(tau, EX_BRK);
    const unsigned long long INFB = 0x7FF0000000000000ull;
    for (int m = threadIdx.x; m <= G; m += blockDim.x) {
        pre[m] = m == 0 ? 0.0 : EX_INF;
        suf[(size_t)L * W + m] = m == 0 ? 0.0 : EX_INF;
        s_row[m] = INFB;
    }
    __syncthreads();
    const int nt = blockDim.x, sq = nt / M, sr = nt % M;    // pair index i = (m - 1) M + (d - 1)
    for (int l2 = 1; l2 <= L; ++l2) {
        // targets m <= M l2 only (every stage has >= 1 layer and <= M GPUs)
        const int pairs = min(G, M * l2) * M;
        int m = threadIdx.x / M + 1, d = threadIdx.x % M + 1;
        for (int i = threadIdx.x; i < pairs; i += nt) {
            const int mc = m, dc = d;
            m += sq;
            d += sr;
            if (d > M) { d -= M; ++m; }
            if (dc > (mc - 1) % M + 1) continue;
            double best = EX_INF;
            const double *tc = Tp + t_index(L, dc, l2, 0);
            for (int l = l2 - 1; l >= 0; --l) {
                const double t = tc[l];
                if (t >= brk) break;
                if (!(t < tau)) continue;
                const double pv = pre[(size_t)l * W + mc - dc];
                if (pv == EX_INF) continue;
                best = fmin(best, __dadd_rn(pv, __dadd_rn(t, t4)));
            }
            if (best < EX_INF) atomicMin(s_row + mc, (unsigned long long)__double_as_longlong(best));
        }
        __syncthreads();
        for (int m = threadIdx.x; m <= G; m += blockDim.x) {
            pre[(size_t)l2 * W + m] = __longlong_as_double((long long)s_row[m]);
            s_row[m] = INFB;
        }
        __syncthreads();
    }
    for (int l0 = L - 1; l0 >= 0; --l0) {
        const int pairs = min(G, M * (L - l0)) * M;             // r <= M (L - l0)
        int r = threadIdx.x / M + 1, d = threadIdx.x % M + 1;
        for (int i = threadIdx.x; i < pairs; i += nt) {
            const int rc = r, dc = d;
            r += sq;
            d += sr;
            if (d > M) { d -= M; ++r; }
            if (dc > (rc - 1) % M + 1) continue;
            double best = EX_INF;
            const double *tc = Tp + t_index(L, dc, 0, l0);
            for (int l = l0 + 1; l <= L; ++l) {
                const double t = tc[(size_t)l * (L + 1)];
                if (t > brk) break;
                if (!(t <= tau)) continue;
                const double sv = suf[(size_t)l * W + rc - dc];
                if (sv == EX_INF) continue;
                best = fmin(best, __dadd_rn(sv, __dadd_rn(__dmul_rn(2.0, t), t3)));
            }
            if (best < EX_INF) atomicMin(s_row + rc, (unsigned long long)__double_as_longlong(best));
        }
        __syncthreads();
        for (int r = threadIdx.x; r <= G; r += blockDim.x) {
            suf[(size_t)l0 * W + r] = __longlong_as_double((long long)s_row[r]);
            s_row[r] = INFB;
        }
        __syncthreads();
    }
}

// bottleneck stages (a, b, d) with t(a, b, d) == tau, packed a | b << 10 | d << 20
__device__ int ex_bottlenecks(const ExGeom &g, const double *__restrict__ Tp, double tau, int *list, int *s_n,
                              unsigned long long *ctr) {
    if (threadIdx.x == 0) *s_n = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < g.L * g.M; i += blockDim.x) {
        const int a = i / g.M, d = i % g.M + 1;
        for (int b = a + 1; b <= g.L; ++b) {
            const double t = Tp[t_index(g.L, d, b, a)];
            if (t > tau) break;
            if (t == tau) {
                const int k = atomicAdd(s_n, 1);
                if (k < g.list_cap) list[k] = a | (b << 10) | (d << 20);
                else atomicExch(ctr + 3, 1ull);
            }
        }
    }
    __syncthreads();
    return min(*s_n, g.list_cap);
}

__device__ unsigned long long block_min_u64(unsigned long long v, unsigned long long *red) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = w < v ? w : v;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : ~0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
            v = w < v ? w : v;
        }
    }
    __syncthreads();
    return v;    // valid in warp 0
}

__global__ void __launch_bounds__(EXS, EX_CTAS_PER_SM) k_ex_solve(ExGeom g, ExWs w) {
    extern __shared__ unsigned long long s_dyn[];
    unsigned long long *s_row = s_dyn;                       // [Gmax + 1]
    int *s_list = (int *)(s_dyn + g.W);                      // [list_cap]
    __shared__ unsigned long long s_red[EXS / 32];
    __shared__ int s_task, s_n;
    double *pre = w.dp + (size_t)blockIdx.x * 2 * (g.L + 1) * g.W;
    double *suf = pre + (size_t)(g.L + 1) * g.W;
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned long long k = atomicAdd(w.ctr + 1, 1ull);
            s_task = k < w.ctr[0] ? (int)k : -1;
        }
        __syncthreads();
        const int k = s_task;
        __syncthreads();
        if (k < 0) break;
        const int2 tk = w.tasks[k];
        const int p = tk.x;
        const double *Tp = w.T + (size_t)p * g.E;
        const double tau = Tp[tk.y];
        const double *tw = w.tw + (size_t)p * g.nsz;
        int nmax = 0;
        for (int i = g.nsz - 1; i >= 0; --i)
            if (tau <= tw[i]) { nmax = g.n_lo + i; break; }
        const int Gt = nmax * g.M;
        ex_paths_fast(g, Tp, Gt, tau, pre, suf, s_row);
        const int nent = ex_bottlenecks(g, Tp, tau, s_list, &s_n, w.ctr);
        const double t4 = __dmul_rn(4.0, tau);
        const unsigned long long tbits = (unsigned long long)__double_as_longlong(tau);
        for (int i = 0; i < g.nsz; ++i) {
            if (!(tau <= tw[i])) continue;
            const int G = (g.n_lo + i) * g.M;
            unsigned long long best = ~0ull;
            for (int j = threadIdx.x; j < nent * G; j += blockDim.x) {
                const int c = s_list[j / G], m = j % G;
                const int a = c & 1023, b = (c >> 10) & 1023, d = c >> 20;
                if ((m % g.M) + d > g.M) continue;
                const double pv = pre[(size_t)a * g.W + m];
                const double sv = suf[(size_t)b * g.W + G - m - d];
                if (pv == EX_INF || sv == EX_INF) continue;
                const unsigned long long v = (unsigned long long)__double_as_longlong(__dadd_rn(__dadd_rn(pv, sv), t4));
                best = v < best ? v : best;
            }
            best = block_min_u64(best, s_red);
            if (threadIdx.x == 0 && best != ~0ull) acc_min(w.acc + (size_t)p * g.nsz + i, best, tbits);
        }
    }
}

__global__ void __launch_bounds__(EXT) k_ex_recon(ExGeom g, ExWs w, unsigned char *packed_out) {
    __shared__ int s_item;
    __shared__ unsigned long long s_key;
    double *pre = w.dp + (size_t)blockIdx.x * 2 * (g.L + 1) * g.W;
    double *suf = pre + (size_t)(g.L + 1) * g.W;
    int *ppar = w.par + (size_t)blockIdx.x * 2 * (g.L + 1) * g.W;
    int *spar = ppar + (size_t)(g.L + 1) * g.W;
    const int items = g.P * g.nsz;
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned long long k = atomicAdd(w.ctr + 2, 1ull);
            s_item = k < (unsigned long long)items ? (int)k : -1;
            s_key = ~0ull;
        }
        __syncthreads();
        const int it = s_item;
        if (it < 0) break;
        const int p = it / g.nsz, i = it % g.nsz, n = g.n_lo + i, G = n * g.M;
        const double *Tp = w.T + (size_t)p * g.E;
        oob::PackedHeader *hd = (oob::PackedHeader *)(packed_out + (size_t)p * g.prof_bytes + (size_t)i * g.tpl_bytes);
        int32_t *st = (int32_t *)(hd + 1);
        const ulonglong2 a = w.acc[(size_t)p * g.nsz + i];
        if (a.x == ~0ull || w.ctr[3] != 0) {    // no mapping (n > L) or a list overflow
            __syncthreads();
            if (threadIdx.x == 0) {
                hd->nodes = n; hd->S = 0; hd->kstar = 0; hd->status = w.ctr[3] != 0 ? 4 : 3;
                hd->T1 = hd->T2 = hd->T3 = hd->tstar = hd->iter = EX_INF;
            }
            continue;
        }
        const double tau = __longlong_as_double((long long)a.y);
        const double t4 = __dmul_rn(4.0, tau);
        ex_paths(g, Tp, G, tau, pre, suf, ppar, spar);
        // the first placement (a, m, d, b) in the oracle's scan order reaching the optimum
        for (int j = threadIdx.x; j < g.L * g.M; j += blockDim.x) {
            const int A = j / g.M, d = j % g.M + 1;
            for (int b = A + 1; b <= g.L; ++b) {
                const double t = Tp[t_index(g.L, d, b, A)];
                if (t > tau) break;
                if (t != tau) continue;
                for (int m = 0; m + d <= G; ++m) {
                    if ((m % g.M) + d > g.M) continue;
                    const double pv = pre[(size_t)A * g.W + m], sv = suf[(size_t)b * g.W + G - m - d];
                    if (pv == EX_INF || sv == EX_INF) continue;
                    if ((unsigned long long)__double_as_longlong(__dadd_rn(__dadd_rn(pv, sv), t4)) != a.x) continue;
                    const unsigned long long key =
                        (((unsigned long long)A * (G + 1) + m) * (g.M + 1) + d) * (g.L + 1) + b;
                    atomicMin(&s_key, key);
                    break;                    // larger m of this (A, b, d) come later in the scan
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long key = s_key;
            const int b = (int)(key % (g.L + 1));
            key /= (g.L + 1);
            const int d = (int)(key % (g.M + 1));
            key /= (g.M + 1);
            const int m = (int)(key % (G + 1));
            const int A = (int)(key / (G + 1));
            // prefix stages, walked backwards into the tail of the record, then moved
            int S = 0, l = A, mm = m;
            while (l > 0) {
                const int c = ppar[(size_t)l * g.W + mm], l0 = c >> 8, dd = c & 255;
                ++S;
                int32_t *r = st + 5 * (g.L - S);
                r[0] = l0; r[1] = l; r[2] = dd; r[3] = (mm - dd) / g.M; r[4] = (mm - dd) % g.M;
                l = l0;
                mm -= dd;
            }
            for (int j = 0; j < S; ++j)
                for (int q = 0; q < 5; ++q) st[5 * j + q] = st[5 * (g.L - S + j) + q];
            int32_t *r = st + 5 * S;
            r[0] = A; r[1] = b; r[2] = d; r[3] = m / g.M; r[4] = m % g.M;
            ++S;
            l = b;
            int rem = G - m - d;
            while (l < g.L) {
                const int c = spar[(size_t)l * g.W + rem], l2 = c >> 8, dd = c & 255;
                r = st + 5 * S;
                r[0] = l; r[1] = l2; r[2] = dd; r[3] = (G - rem) / g.M; r[4] = (G - rem) % g.M;
                ++S;
                rem -= dd;
                l = l2;
            }
            // closed form of the chosen stages (N_b = 4S), summed left to right
            double T1 = 0.0, ts = 0.0;
            int ks = 0;
            for (int j = 0; j < S; ++j) {
                const double t = Tp[t_index(g.L, st[5 * j + 2], st[5 * j + 1], st[5 * j + 0])];
                T1 = __dadd_rn(T1, t);
                if (j == 0 || t > ts) { ts = t; ks = j; }
            }
            double T3 = 0.0;
            for (int j = ks; j < S; ++j) T3 = __dadd_rn(T3, Tp[t_index(g.L, st[5 * j + 2], st[5 * j + 1], st[5 * j + 0])]);
            const double T2 = __dmul_rn((double)(4 * S - S + ks - 1), ts);
            hd->nodes = n; hd->S = S; hd->kstar = ks; hd->status = 0;
            hd->T1 = T1; hd->T2 = T2; hd->T3 = T3; hd->tstar = ts;
            hd->iter = __dadd_rn(__dadd_rn(T1, T2), T3);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host
bool ex_geom(int L, int M, int n_lo, int n_hi, int P, int sms, ExGeom &g) {
    if (L < 1 || L > 1023 || M < 1 || M > 64 || n_lo < 1 || n_hi < n_lo || n_hi > L || P < 1 || sms < 1) return false;
    g.L = L; g.M = M; g.n_lo = n_lo; g.n_hi = n_hi; g.nsz = n_hi - n_lo + 1; g.P = P;
    g.Gmax = n_hi * M;
    g.W = g.Gmax + 1;
    g.E = M * (L + 1) * (L + 1);
    const int valid = M * L * (L + 1) / 2;
    g.H = 1;
    while (g.H < 2 * valid) g.H <<= 1;
    g.slots = sms * EX_CTAS_PER_SM;
    g.rslots = sms * EX_RECON_PER_SM;
    g.list_cap = std::min(2 * L * M, 8192);
    // k_ex_solve's shared memory: one row of targets + the bottleneck list
    if (sizeof(unsigned long long) * (size_t)g.W + sizeof(int) * (size_t)g.list_cap > 200 * 1024) return false;
    g.tpl_bytes = oob::packed_template_bytes(L);
    g.prof_bytes = g.tpl_bytes * (size_t)g.nsz;
    return true;
}

size_t ex_layout(const ExGeom &g, unsigned char *base, ExWs *w) {
    using oob::align_up_host;
    const size_t rows = (size_t)(g.L + 1) * g.W;
    const size_t valid = (size_t)g.M * g.L * (g.L + 1) / 2;
    const size_t sz[] = {align_up_host(8 * sizeof(unsigned long long)),
                         align_up_host(sizeof(double) * (size_t)g.P * g.E),
                         align_up_host(sizeof(unsigned long long) * (size_t)g.P * g.H),
                         align_up_host(sizeof(int) * (size_t)g.P * g.H),
                         align_up_host(sizeof(double) * (size_t)g.P * g.nsz),
                         align_up_host(sizeof(double) * (size_t)g.P),
                         align_up_host(sizeof(int2) * (size_t)g.P * valid),
                         align_up_host(sizeof(ulonglong2) * (size_t)g.P * g.nsz),
                         align_up_host(sizeof(double) * (size_t)g.slots * 2 * rows),
                         align_up_host(sizeof(int) * (size_t)g.rslots * 2 * rows)};
    size_t off[10], tot = 0;
    for (int i = 0; i < 10; ++i) { off[i] = tot; tot += sz[i]; }
    if (w) {
        w->ctr = (unsigned long long *)(base + off[0]);
        w->T = (double *)(base + off[1]);
        w->hkey = (unsigned long long *)(base + off[2]);
        w->hidx = (int *)(base + off[3]);
        w->tw = (double *)(base + off[4]);
        w->twmax = (double *)(base + off[5]);
        w->tasks = (int2 *)(base + off[6]);
        w->acc = (ulonglong2 *)(base + off[7]);
        w->dp = (double *)(base + off[8]);
        w->par = (int *)(base + off[9]);
    }
    return tot;
}

int current_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return sms;
}

}  // namespace

extern "C" oob_status oob_exact_workspace_bytes(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi, int32_t num_profiles,
                                                size_t *bytes) {
    if (!bytes) return oob::fail(OOB_E_INVALID, "oob_exact_workspace_bytes: NULL argument");
    ExGeom g;
    const int sms = current_sms();
    if (sms < 1) return oob::fail(OOB_E_CUDA, "oob_exact_workspace_bytes: no CUDA device");
    if (!ex_geom(L, M, n_lo, n_hi, num_profiles, sms, g))
        return oob::fail(OOB_E_INVALID, "oob_exact_workspace_bytes: bad shape");
    *bytes = ex_layout(g, nullptr, nullptr);
    return OOB_OK;
}

extern "C" oob_status oob_exact_run(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi, int32_t num_profiles,
                                    const double *d_fwd, const double *d_bwd, const void *d_packed_ub, void *d_workspace,
                                    size_t workspace_bytes, void *d_packed_out, void *stream) {
    if (!d_fwd || !d_bwd || !d_workspace || !d_packed_out) return oob::fail(OOB_E_INVALID, "oob_exact_run: NULL argument");
    ExGeom g;
    const int sms = current_sms();
    if (sms < 1) return oob::fail(OOB_E_CUDA, "oob_exact_run: no CUDA device");
    if (!ex_geom(L, M, n_lo, n_hi, num_profiles, sms, g)) return oob::fail(OOB_E_INVALID, "oob_exact_run: bad shape");
    ExWs w;
    const size_t need = ex_layout(g, (unsigned char *)d_workspace, &w);
    if (workspace_bytes < need)
        return oob::fail(OOB_E_NOMEM, "oob_exact_run: workspace too small: need " + std::to_string(need) + " bytes");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(w.ctr, 0, 8 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(w.hkey, 0, sizeof(unsigned long long) * (size_t)g.P * g.H, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(w.hidx, 0x7f, sizeof(int) * (size_t)g.P * g.H, s);
    if (e != cudaSuccess) return oob::fail(OOB_E_CUDA, std::string("oob_exact_run memset: ") + cudaGetErrorString(e));
    const int64_t flat = (int64_t)g.P * g.E;
    const int grid = (int)std::min<int64_t>((flat + EXT - 1) / EXT, (int64_t)sms * 16);
    k_ex_times<<<g.P * g.M, 128, 0, s>>>(g, d_fwd, d_bwd, w.T);
    k_ex_hash<<<grid, EXT, 0, s>>>(g, w.T, w.hkey, w.hidx);
    k_ex_window<<<g.P, 128, 0, s>>>(g, d_fwd, d_bwd, (const unsigned char *)d_packed_ub, w.tw, w.twmax, w.acc);
    k_ex_tasks<<<grid, EXT, 0, s>>>(g, w.T, w.hkey, w.hidx, w.twmax, w.tasks, w.ctr);
    const size_t smem = sizeof(unsigned long long) * (size_t)g.W + sizeof(int) * (size_t)g.list_cap;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_ex_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return oob::fail(OOB_E_CUDA, std::string("oob_exact_run smem: ") + cudaGetErrorString(e));
    }
    k_ex_solve<<<g.slots, EXS, smem, s>>>(g, w);
    k_ex_recon<<<g.rslots, EXT, 0, s>>>(g, w, (unsigned char *)d_packed_out);
    e = cudaGetLastError();
    if (e != cudaSuccess) return oob::fail(OOB_E_CUDA, std::string("oob_exact_run launch: ") + cudaGetErrorString(e));
    return OOB_OK;
}
