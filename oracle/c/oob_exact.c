/*
 * ORACLE (test infrastructure only) — the EXACT minimum of the paper's 1F1B objective for one
 * template, over every GPU-stage mapping, to measure how far the paper's per-cell argmin
 * recursion (a heuristic) is from the optimum at config scale.  Only tests/
 * and scripts/heuristic_gap.py use it; it shares nothing with paper_2309_08125_b200/.
 *
 * Mappings (reading R2): S contiguous stages tiling the layers
 * [0, L) in pipeline order and, in the same order, the n*M GPUs of n nodes, stage i on d_i
 * GPUs that do not cross a node boundary (every node's GPUs used, no stage spanning nodes).
 * Objective (closed form, N_b = 4S): with stage times t_i, k* the
 * first index of the maximum tau = t_{k*}:
 *     total = T1 + (3S - 1 + k*) tau + T3,   T1 = sum t_i,   T3 = sum_{i >= k*} t_i
 *           = sum_{i < k*} t_i + 2 sum_{i > k*} t_i + (3S + 1 + k*) tau
 *           = sum_{i < k*} (t_i + 4 tau) + sum_{i > k*} (2 t_i + 3 tau) + 4 tau.
 * So for a fixed bottleneck value tau the stages before the bottleneck stage (all t_i < tau,
 * k* is the FIRST maximum) and after it (t_i <= tau) decouple into two shortest-path DPs over
 * (layer boundary, GPUs used) with per-stage costs t + 4 tau and 2t + 3 tau; the optimum is
 * the minimum over every stage time tau and every placement of a bottleneck stage with
 * t = tau.  Stage times are summed left to right from 0.0 (reading R12), as the recursion's.
 * Pinned against brute force over all mappings (tests/test_oracle_exact.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int L, M, n, G;          /* G = n*M GPUs */
    double *t;               /* [u][v][d]: (L+1)*(L+1)*(M+1) */
} ctx_t;

static double T(const ctx_t *c, int u, int v, int d) {
    return c->t[((size_t)u * (c->L + 1) + v) * (c->M + 1) + d];
}

static int cmp_d(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : x > y;
}

/* prefix/suffix DPs for one tau; pre/suf: (L+1)*(G+1); parents optional */
static void dps(const ctx_t *c, double tau, double *pre, double *suf, int *ppar, int *spar) {
    const int L = c->L, M = c->M, G = c->G;
    const size_t W = (size_t)G + 1;
    for (size_t i = 0; i < (size_t)(L + 1) * W; ++i) { pre[i] = INFINITY; suf[i] = INFINITY; }
    pre[0] = 0.0;
    for (int l = 0; l < L; ++l)
        for (int m = 0; m < G; ++m) {
            const double p = pre[l * W + m];
            if (p == INFINITY) continue;
            for (int d = 1; d <= M && (m % M) + d <= M; ++d)
                for (int l2 = l + 1; l2 <= L; ++l2) {
                    const double t = T(c, l, l2, d);
                    if (!(t < tau)) break;                   /* times grow with the range */
                    const double v = p + (t + 4.0 * tau);
                    if (v < pre[l2 * W + m + d]) {
                        pre[l2 * W + m + d] = v;
                        if (ppar) ppar[l2 * W + m + d] = l * 64 + d;
                    }
                }
        }
    suf[(size_t)L * W + G] = 0.0;
    for (int l = L; l >= 1; --l)
        for (int m = G; m >= 1; --m) {
            const double s = suf[l * W + m];
            if (s == INFINITY) continue;
            /* a stage [l0, l) on GPUs [m-d, m) ending here */
            for (int d = 1; d <= M && d <= m && ((m - d) % M) + d <= M; ++d)
                for (int l0 = l - 1; l0 >= 0; --l0) {
                    /* sums from different start layers: stop only clearly past tau (an
                       out-of-order rounding is ~1e-13 relative), skip the rest exactly */
                    const double t = T(c, l0, l, d);
                    if (t > tau * (1.0 + 0x1p-30)) break;
                    if (!(t <= tau)) continue;
                    const double v = s + (2.0 * t + 3.0 * tau);
                    if (v < suf[l0 * W + m - d]) {
                        suf[l0 * W + m - d] = v;
                        if (spar) spar[l0 * W + m - d] = l * 64 + d;
                    }
                }
        }
}

/* Returns 0 and fills the optimum's stages (u, v, d, node) and S; 1 if no mapping (or none
 * with total <= ub).  ub (> 0, else ignored) is a known total (e.g. the recursion's): since
 * every stage contributes >= 3 tau and the bottleneck 4 tau, total >= (3S + 1) tau >=
 * (3n + 1) tau, so only tau <= ub / (3n + 1) can beat it — a window, not an approximation. */
int oob_exact_template(int L, int M, const double *fwd, const double *bwd, int n, double ub, int32_t *stages_out,
                       int32_t *S_out, double *dp_value_out) {
    if (L < 1 || M < 1 || M > 63 || n < 1 || n > L) return 2;
    ctx_t c;
    c.L = L; c.M = M; c.n = n; c.G = n * M;
    c.t = (double *)calloc((size_t)(L + 1) * (L + 1) * (M + 1), sizeof(double));
    size_t nt = 0;
    double *taus = (double *)malloc(sizeof(double) * (size_t)L * (L + 1) / 2 * M + 1);
    for (int u = 0; u < L; ++u)
        for (int d = 1; d <= M; ++d) {
            double s = 0.0;
            for (int v = u + 1; v <= L; ++v) {
                s = s + (fwd[(size_t)(v - 1) * M + d - 1] + bwd[(size_t)(v - 1) * M + d - 1]);
                c.t[((size_t)u * (L + 1) + v) * (M + 1) + d] = s;
                taus[nt++] = s;
            }
        }
    qsort(taus, nt, sizeof(double), cmp_d);
    size_t nu = 0;
    const double tau_max = ub > 0.0 ? ub / (3.0 * n + 1.0) * (1.0 + 1e-12) : INFINITY;
    for (size_t i = 0; i < nt; ++i)
        if ((nu == 0 || taus[i] != taus[nu - 1]) && taus[i] <= tau_max) taus[nu++] = taus[i];
    const size_t W = (size_t)c.G + 1;
    double best = INFINITY;
    double best_tau = 0.0;
#pragma omp parallel
    {
        double *pre = (double *)malloc(sizeof(double) * (size_t)(L + 1) * W);
        double *suf = (double *)malloc(sizeof(double) * (size_t)(L + 1) * W);
        double lb = INFINITY, lt = 0.0;
#pragma omp for schedule(dynamic, 4)
        for (long i = 0; i < (long)nu; ++i) {
            const double tau = taus[i];
            dps(&c, tau, pre, suf, NULL, NULL);
            for (int a = 0; a < L; ++a)
                for (int m = 0; m < c.G; ++m) {
                    const double p = pre[a * W + m];
                    if (p == INFINITY) continue;
                    for (int d = 1; d <= M && (m % M) + d <= M; ++d)
                        for (int b = a + 1; b <= L; ++b) {
                            const double t = T(&c, a, b, d);
                            if (t > tau) break;
                            if (t != tau) continue;
                            const double v = p + suf[b * W + m + d] + 4.0 * tau;
                            if (v < lb || (v == lb && tau < lt)) { lb = v; lt = tau; }
                        }
                }
        }
#pragma omp critical
        {
            if (lb < best || (lb == best && lt < best_tau)) { best = lb; best_tau = lt; }
        }
        free(pre);
        free(suf);
    }
    int rc = 1;
    if (best < INFINITY) {
        /* reconstruct for best_tau: the first (a, m, d, b) reaching the optimum */
        double *pre = (double *)malloc(sizeof(double) * (size_t)(L + 1) * W);
        double *suf = (double *)malloc(sizeof(double) * (size_t)(L + 1) * W);
        int *pp = (int *)malloc(sizeof(int) * (size_t)(L + 1) * W);
        int *sp = (int *)malloc(sizeof(int) * (size_t)(L + 1) * W);
        dps(&c, best_tau, pre, suf, pp, sp);
        int fa = -1, fm = 0, fd = 0, fb = 0;
        for (int a = 0; a < L && fa < 0; ++a)
            for (int m = 0; m < c.G && fa < 0; ++m) {
                if (pre[a * W + m] == INFINITY) continue;
                for (int d = 1; d <= M && (m % M) + d <= M && fa < 0; ++d)
                    for (int b = a + 1; b <= L; ++b) {
                        const double t = T(&c, a, b, d);
                        if (t > best_tau) break;
                        if (t != best_tau) continue;
                        if (pre[a * W + m] + suf[b * W + m + d] + 4.0 * best_tau == best) {
                            fa = a; fm = m; fd = d; fb = b;
                            break;
                        }
                    }
            }
        if (fa >= 0) {
            int32_t tmp[4 * 1024];
            int ns = 0;
            /* prefix stages, walked backwards */
            int l = fa, m = fm;
            while (l > 0) {
                const int code = pp[l * W + m], l0 = code / 64, d = code % 64;
                tmp[4 * ns + 0] = l0; tmp[4 * ns + 1] = l; tmp[4 * ns + 2] = d; tmp[4 * ns + 3] = (m - d) / M;
                ++ns;
                l = l0; m -= d;
            }
            int S = 0;
            for (int i = ns - 1; i >= 0; --i, ++S) memcpy(stages_out + 4 * S, tmp + 4 * i, 4 * sizeof(int32_t));
            stages_out[4 * S + 0] = fa; stages_out[4 * S + 1] = fb; stages_out[4 * S + 2] = fd;
            stages_out[4 * S + 3] = fm / M;
            ++S;
            l = fb; m = fm + fd;
            while (l < L) {
                const int code = sp[l * W + m], l2 = code / 64, d = code % 64;
                stages_out[4 * S + 0] = l; stages_out[4 * S + 1] = l2; stages_out[4 * S + 2] = d;
                stages_out[4 * S + 3] = m / M;
                ++S;
                l = l2; m += d;
            }
            *S_out = S;
            if (dp_value_out) *dp_value_out = best;
            rc = 0;
        }
        free(pre); free(suf); free(pp); free(sp);
    }
    free(taus);
    free(c.t);
    return rc;
}
