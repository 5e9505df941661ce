/*
 * ORACLE (test infrastructure only) — plain C version of oracle/dp.py, for the configs
 * the Python oracle cannot finish in seconds.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant with the CUDA path (paper_2309_08125_b200/).
 *
 * PAPER.md §4.1.2 "GPU--Stage Mapping", literally:
 *   - memoized T(S', u, v, a) over the key (S', u, v, alloc);
 *   - base case Eq.4: T1 = T3 = t* = sum_{k=u}^{v-1}(F+B), k* = 0;
 *     GPUs spanning nodes -> infinite;
 *   - recursive case Eq.1-3 over k (layer split, second half starts at k),
 *     m (device split, two-level scheme) and s (stages of the first half), keeping the
 *     first strictly smaller T1+T2+T3 with N_b = 4S';
 *   - infinite when the division is impossible: more stages than layers or GPUs (P:390,
 *     P:457) or fewer stages than nodes (pigeonhole).  The Python oracle
 *     reaches the same infinities by plain recursion; tests check the two agree.
 *   - template: argmin over S in n..min(L, n*M) of T(S, 0, L, W(n)).
 * Arithmetic: binary64, operations exactly in the order written, built with
 * -ffp-contract=off (no FMA) and without -ffast-math.
 *
 * Single-threaded; not tuned.  Memory: one lazily-allocated array per (u, v, alloc).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double T1, T3, tstar;
    int32_t kstar;
    int16_t k, m, s;      /* argmin split (layer split k, device split m, stages s) */
    int8_t state;         /* 0 = not computed, 1 = finite, 2 = infinite */
} ocell;

typedef struct {
    int L, M, Qmax, A;    /* A = number of allocation kinds: I(1..M-1), W(1..Qmax) */
    const double *fwd, *bwd;
    int pow2;             /* stage masks (reading R31): d must be a power of two */
    const double *stage_bytes;   /* [L] or NULL: sum/d <= mem_cap */
    double mem_cap;
    ocell **memo;         /* [(u*(L+1)+v)*A + a] -> array indexed by S' (1..cap) */
    long long cells, splits;
} oracle_t;

/* allocation index: a < M-1 -> I(a+1);  a >= M-1 -> W(a-(M-1)+1) */
static int is_whole(const oracle_t *o, int a) { return a >= o->M - 1; }
static int alloc_n(const oracle_t *o, int a) { return is_whole(o, a) ? a - (o->M - 1) + 1 : a + 1; }
static int alloc_gpus(const oracle_t *o, int a) { return is_whole(o, a) ? alloc_n(o, a) * o->M : alloc_n(o, a); }
static int alloc_nodes(const oracle_t *o, int a) { return is_whole(o, a) ? alloc_n(o, a) : 1; }
static int idx_I(const oracle_t *o, int r) { (void)o; return r - 1; }
static int idx_W(const oracle_t *o, int q) { return (o->M - 1) + q - 1; }

static int num_device_splits(const oracle_t *o, int a) {
    int n = alloc_n(o, a);
    if (is_whole(o, a)) return n >= 2 ? n - 1 : o->M - 1;
    return n - 1;
}

/* m-th device split of a (in the order of oracle/dp.py device_splits) */
static void device_split(const oracle_t *o, int a, int m, int *a1, int *a2) {
    int n = alloc_n(o, a);
    int j = m + 1;
    if (is_whole(o, a) && n >= 2) { *a1 = idx_W(o, j); *a2 = idx_W(o, n - j); }
    else if (is_whole(o, a))      { *a1 = idx_I(o, j); *a2 = idx_I(o, o->M - j); }
    else                          { *a1 = idx_I(o, j); *a2 = idx_I(o, n - j); }
}

static double stage_time(const oracle_t *o, int u, int v, int d) {
    double t = 0.0;
    for (int k = u; k < v; ++k)
        t = t + (o->fwd[(size_t)k * o->M + (d - 1)] + o->bwd[(size_t)k * o->M + (d - 1)]);
    return t;
}

/* reading R31 (variants): the stage [u, v) on d GPUs is allowed iff d is a
 * power of two (pow2) and sum_{l=u}^{v-1} stage_bytes[l] / d <= mem_cap (left to right) */
static int stage_allowed(const oracle_t *o, int u, int v, int d) {
    if (o->pow2 && (d & (d - 1)) != 0) return 0;
    if (o->stage_bytes) {
        double tot = 0.0;
        for (int k = u; k < v; ++k) tot = tot + o->stage_bytes[k];
        if (tot / (double)d > o->mem_cap) return 0;
    }
    return 1;
}

static int stage_cap(const oracle_t *o, int u, int v, int a) {
    int c = v - u, g = alloc_gpus(o, a);
    return c < g ? c : g;
}

static const ocell INF_CELL = {0, 0, 0, 0, 0, 0, 0, 2};

static const ocell *T(oracle_t *o, int Sp, int u, int v, int a) {
    /* division impossible -> infinite */
    if (Sp > stage_cap(o, u, v, a) || Sp < alloc_nodes(o, a)) return &INF_CELL;
    size_t key = ((size_t)u * (o->L + 1) + v) * o->A + a;
    ocell *arr = o->memo[key];
    if (!arr) {
        arr = (ocell *)calloc((size_t)stage_cap(o, u, v, a) + 1, sizeof(ocell));
        o->memo[key] = arr;
    }
    ocell *c = &arr[Sp];
    if (c->state) return c;
    if (Sp == 1) {
        if (is_whole(o, a) && alloc_n(o, a) >= 2) { c->state = 2; return c; }
        int d = is_whole(o, a) ? o->M : alloc_n(o, a);
        if (!stage_allowed(o, u, v, d)) { c->state = 2; return c; }           /* masked (R31) */
        double t = stage_time(o, u, v, d);                                      /* Eq.4 */
        c->T1 = t; c->T3 = t; c->tstar = t; c->kstar = 0;
        c->k = c->m = c->s = -1;
        c->state = 1;
        o->cells++;
        return c;
    }
    double best_total = 1.0 / 0.0;
    int found = 0;
    int nd = num_device_splits(o, a);
    for (int k = u + 1; k < v; ++k) {
        for (int m = 0; m < nd; ++m) {
            int a1, a2;
            device_split(o, a, m, &a1, &a2);
            /* s outside [s_lo, s_hi] makes a child infinite by T()'s first test (more
             * stages than layers/GPUs, or fewer than nodes), so those s are skipped
             * exactly as the `continue`s below would skip them. */
            int s_lo = alloc_nodes(o, a1), s_hi = stage_cap(o, u, k, a1);
            if (s_lo < Sp - stage_cap(o, k, v, a2)) s_lo = Sp - stage_cap(o, k, v, a2);
            if (s_hi > Sp - alloc_nodes(o, a2)) s_hi = Sp - alloc_nodes(o, a2);
            if (s_lo < 1) s_lo = 1;
            if (s_hi > Sp - 1) s_hi = Sp - 1;
            for (int s = s_lo; s <= s_hi; ++s) {
                const ocell *Lc = T(o, s, u, k, a1);
                if (Lc->state != 1) continue;
                const ocell *Rc = T(o, Sp - s, k, v, a2);
                if (Rc->state != 1) continue;
                o->splits++;
                double T1 = Lc->T1 + Rc->T1;                     /* Eq.1 */
                double T3, tstar;
                int kstar;
                if (Lc->tstar >= Rc->tstar) {                    /* k* in the first half */
                    kstar = Lc->kstar; tstar = Lc->tstar;
                    T3 = Lc->T3 + Rc->T1;                         /* Eq.3 first case */
                } else {
                    kstar = s + Rc->kstar; tstar = Rc->tstar;
                    T3 = Rc->T3;                                  /* Eq.3 else-branch */
                }
                int Nb = 4 * Sp;
                double T2 = (double)(Nb - Sp + kstar - 1) * tstar;  /* Eq.2 */
                double total = (T1 + T2) + T3;
                if (total < best_total) {
                    best_total = total;
                    found = 1;
                    c->T1 = T1; c->T3 = T3; c->tstar = tstar; c->kstar = kstar;
                    c->k = (int16_t)k; c->m = (int16_t)m; c->s = (int16_t)s;
                }
            }
        }
    }
    c->state = found ? 1 : 2;
    if (found) o->cells++;
    return c;
}

static void backtrack(oracle_t *o, int Sp, int u, int v, int a, int node, int goff,
                      int32_t *stages, int *ns) {
    const ocell *c = T(o, Sp, u, v, a);
    if (Sp == 1) {
        int32_t *st = stages + 5 * (*ns);
        st[0] = u; st[1] = v; st[2] = is_whole(o, a) ? o->M : alloc_n(o, a);
        st[3] = node; st[4] = goff;
        (*ns)++;
        return;
    }
    int a1, a2;
    device_split(o, a, c->m, &a1, &a2);
    if (is_whole(o, a) && alloc_n(o, a) >= 2) {
        backtrack(o, c->s, u, c->k, a1, node, 0, stages, ns);
        backtrack(o, Sp - c->s, c->k, v, a2, node + alloc_n(o, a1), 0, stages, ns);
    } else {
        backtrack(o, c->s, u, c->k, a1, node, goff, stages, ns);
        backtrack(o, Sp - c->s, c->k, v, a2, node, goff + alloc_n(o, a1), stages, ns);
    }
}

/*
 * Template set for sizes n_lo..n_hi (largest first, one shared memo).
 * Outputs per template i = n - n_lo: S[i], kstar[i], costs[i*6 + {T1,T2,T3,tstar,total,0}],
 * stages[i*L*5 + j*5 + {u, v, d, node, gpu_offset}] for j < S[i].
 * Returns 0 on success, 1 when some template is infeasible, 2 on bad arguments.
 */
int oob_oracle_template_set_masked(int L, int M, const double *fwd, const double *bwd,
                                   int n_lo, int n_hi, int pow2, const double *stage_bytes, double mem_cap,
                                   int32_t *S_out, int32_t *kstar_out, double *costs_out, int32_t *stages_out,
                                   long long *cells_out, long long *splits_out) {
    if (L < 1 || M < 1 || n_lo < 1 || n_hi < n_lo || n_hi > L) return 2;
    oracle_t o;
    memset(&o, 0, sizeof o);
    o.L = L; o.M = M; o.Qmax = n_hi; o.A = (M - 1) + n_hi;
    o.fwd = fwd; o.bwd = bwd;
    o.pow2 = pow2; o.stage_bytes = stage_bytes; o.mem_cap = mem_cap;
    size_t nkeys = (size_t)(L + 1) * (L + 1) * o.A;
    o.memo = (ocell **)calloc(nkeys, sizeof(ocell *));
    if (!o.memo) return 2;
    int rc = 0;
    for (int n = n_hi; n >= n_lo; --n) {
        int i = n - n_lo;
        int a = idx_W(&o, n);
        double best = 0; int bestS = -1;
        int Smax = L < n * M ? L : n * M;
        for (int S = n; S <= Smax; ++S) {
            const ocell *c = T(&o, S, 0, L, a);
            if (c->state != 1) continue;
            double T2 = (double)(4 * S - S + c->kstar - 1) * c->tstar;
            double tot = (c->T1 + T2) + c->T3;
            if (bestS < 0 || tot < best) { best = tot; bestS = S; }
        }
        if (bestS < 0) { rc = 1; S_out[i] = 0; continue; }
        const ocell *c = T(&o, bestS, 0, L, a);
        S_out[i] = bestS;
        kstar_out[i] = c->kstar;
        double T2 = (double)(4 * bestS - bestS + c->kstar - 1) * c->tstar;
        costs_out[i * 6 + 0] = c->T1;
        costs_out[i * 6 + 1] = T2;
        costs_out[i * 6 + 2] = c->T3;
        costs_out[i * 6 + 3] = c->tstar;
        costs_out[i * 6 + 4] = best;
        costs_out[i * 6 + 5] = 0.0;
        int ns = 0;
        backtrack(&o, bestS, 0, L, a, 0, 0, stages_out + (size_t)i * L * 5, &ns);
    }
    if (cells_out) *cells_out = o.cells;
    if (splits_out) *splits_out = o.splits;
    for (size_t i = 0; i < nkeys; ++i) free(o.memo[i]);
    free(o.memo);
    return rc;
}

int oob_oracle_template_set(int L, int M, const double *fwd, const double *bwd,
                            int n_lo, int n_hi, int32_t *S_out, int32_t *kstar_out,
                            double *costs_out, int32_t *stages_out,
                            long long *cells_out, long long *splits_out) {
    return oob_oracle_template_set_masked(L, M, fwd, bwd, n_lo, n_hi, 0, NULL, 0.0, S_out, kstar_out, costs_out,
                                          stages_out, cells_out, splits_out);
}
