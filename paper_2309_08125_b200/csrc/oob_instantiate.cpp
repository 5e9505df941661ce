// Pipeline instantiation (Eq.5, PAPER §4.2.1) and batch distribution (Eq.6,
// §4.2.2) on the host, over a template set produced by the CUDA DP.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>
#include <cstdint>
#include <limits>
#include <string>
#include <unordered_set>
#include <vector>

#include "oob_internal.h"

using namespace oob;

namespace {

// ---------------------------------------------------------------- Eq.6 exact solver
// Minimise sum_i (N_i T_i - mean)^2 with sum N_i = K, N_i >= 1 (DESIGN.md "Batch
// distribution").  Pipelines with equal T form a group g (value tau_g, c_g members); at an
// optimum their counts differ by at most 1, so a group is described by its total M_g.
// For a fixed mean mu the problem is separable convex in M_g and solved by greedy
// marginals delta_g(M) = tau_g^2 (2 floor(M / c_g) + 1) - 2 mu tau_g; sweeping mu from
// -inf to +inf moves single units from smaller-tau to larger-tau groups at the crossing
// points, visiting every allocation that is optimal for some mu.  The global optimum is
// optimal for mu = its own mean, so the best true objective among visited allocations is
// exact.
struct Group {
    double tau;
    int64_t c;
    int64_t Mg;
    std::vector<int> members;
};

double group_objective(const std::vector<Group> &gs, int64_t x) {
    double sum = 0.0;
    for (auto &g : gs) sum += (double)g.Mg * g.tau;
    const double mean = sum / (double)x;
    double obj = 0.0;
    for (auto &g : gs) {
        const int64_t q = g.Mg / g.c, r = g.Mg % g.c;
        const double hi = (double)(q + 1) * g.tau - mean, lo = (double)q * g.tau - mean;
        obj += (double)r * hi * hi + (double)(g.c - r) * lo * lo;
    }
    return obj;
}

inline double marginal(const Group &g, int64_t M) {   // phi(M+1) - phi(M), without tau^2
    return (double)(2 * (M / g.c) + 1);
}

// A (nullable): per-pipeline fill/drain overhead a_i of iteration_ms = a_i + N_b,i t*_i.
// Eq.6 has several minimizers when pipelines share T; inside a group of equal T the extra
// microbatches go to the members with the smaller a_i (then the lower index), which gives the
// minimizer with the smallest plan iteration time (reading R29).
void distribute_exact(const double *T, int x, int64_t K, int64_t *nb, double *obj_out, const double *A = nullptr) {
    std::vector<Group> gs;
    {
        std::vector<int> idx(x);
        for (int i = 0; i < x; ++i) idx[i] = i;
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return T[a] < T[b]; });
        for (int i : idx) {
            if (gs.empty() || gs.back().tau != T[i]) gs.push_back({T[i], 0, 0, {}});
            gs.back().c++;
            gs.back().members.push_back(i);
        }
    }
    for (auto &g : gs)
        std::sort(g.members.begin(), g.members.end(), [&](int a, int b) {
            if (A && A[a] != A[b]) return A[a] < A[b];
            return a < b;
        });
    for (auto &g : gs) g.Mg = g.c;
    gs[0].Mg += K - x;
    std::vector<int64_t> best_M(gs.size());
    double best = group_objective(gs, x);
    for (size_t i = 0; i < gs.size(); ++i) best_M[i] = gs[i].Mg;
    double mu_cur = -std::numeric_limits<double>::infinity();
    for (;;) {
        double best_mu = std::numeric_limits<double>::infinity();
        int bs = -1, bt = -1;
        for (size_t s = 0; s < gs.size(); ++s) {
            if (gs[s].Mg <= gs[s].c) continue;
            const double ds = gs[s].tau * gs[s].tau * marginal(gs[s], gs[s].Mg - 1);
            for (size_t t = s + 1; t < gs.size(); ++t) {
                const double dt = gs[t].tau * gs[t].tau * marginal(gs[t], gs[t].Mg);
                double mu = (dt - ds) / (2.0 * (gs[t].tau - gs[s].tau));
                if (mu < mu_cur) mu = mu_cur;     // rounding guard: never move backwards
                if (mu < best_mu) { best_mu = mu; bs = (int)s; bt = (int)t; }
            }
        }
        if (bs < 0) break;
        mu_cur = best_mu;
        gs[bs].Mg--;
        gs[bt].Mg++;
        const double o = group_objective(gs, x);
        if (o < best) {
            best = o;
            for (size_t i = 0; i < gs.size(); ++i) best_M[i] = gs[i].Mg;
        }
    }
    for (size_t gi = 0; gi < gs.size(); ++gi) {
        const Group &g = gs[gi];
        const int64_t q = best_M[gi] / g.c, r = best_M[gi] % g.c;
        for (size_t k = 0; k < g.members.size(); ++k) nb[g.members[k]] = q + ((int64_t)k < r ? 1 : 0);
    }
    if (obj_out) {
        // objective of the final assignment, per pipeline (Eq.6 as written)
        double sum = 0.0;
        for (int i = 0; i < x; ++i) sum += (double)nb[i] * T[i];
        const double mean = sum / x;
        double o = 0.0;
        for (int i = 0; i < x; ++i) {
            const double d = (double)nb[i] * T[i] - mean;
            o += d * d;
        }
        *obj_out = o;
    }
}

}  // namespace

extern "C" int64_t oob_recommend_batch(int32_t x, int32_t b, int64_t B) {
    if (x < 1) x = 1;
    if (b < 1) b = 1;
    int64_t Bp = std::max<int64_t>(B, (int64_t)x * b);
    if (Bp % b) Bp += b - Bp % b;
    return Bp;
}

extern "C" oob_status oob_distribute_batch(const double *T, int32_t x, int64_t B, int32_t b,
                                           int64_t *nb_out, double *objective_out,
                                           int64_t *recommended_out) {
    if (!T || !nb_out) return fail(OOB_E_INVALID, "oob_distribute_batch: NULL argument");
    if (x < 1 || b < 1 || B < 1) return fail(OOB_E_INVALID, "need x >= 1, microbatch >= 1, B >= 1");
    for (int i = 0; i < x; ++i)
        if (!(std::isfinite(T[i]) && T[i] > 0.0)) return fail(OOB_E_INVALID, "per-microbatch time must be positive");
    if (B % b != 0 || B / b < x) {
        if (recommended_out) *recommended_out = oob_recommend_batch(x, b, B);
        return fail(OOB_E_BATCH, "global batch cannot be distributed: B % b != 0 or B/b < pipelines");
    }
    distribute_exact(T, x, B / b, nb_out, objective_out);
    if (recommended_out) *recommended_out = B;
    return OOB_OK;
}

// ---------------------------------------------------------------- Eq.5
namespace {

// Count of X (sizes n_lo..n_hi, sum x_i n_i = N, sum x_i >= f+1), saturating at INT64_MAX.
// ok (nullable): ok[i] = 0 excludes the template of size n_lo + i (infeasible under stage masks).
int64_t count_sets(int n_lo, int n_hi, int N, int f, const char *ok = nullptr) {
    const int C = f + 2;   // pipeline count buckets 0..f+1 (f+1 = "at least f+1")
    std::vector<double> cnt((size_t)(N + 1) * C, 0.0);   // double: counts can exceed 2^64
    cnt[0] = 1.0;
    for (int n = n_lo; n <= n_hi; ++n) {
        if (ok && !ok[n - n_lo]) continue;
        for (int t = n; t <= N; ++t)
            for (int c = 0; c < C; ++c) {
                const double v = cnt[(size_t)(t - n) * C + c];
                if (v == 0.0) continue;
                cnt[(size_t)t * C + std::min(c + 1, C - 1)] += v;
            }
    }
    const double r = cnt[(size_t)N * C + (C - 1)];
    return r >= 9.2e18 ? INT64_MAX : (int64_t)r;
}

struct InstCtx {
    const oob_template *tpl;   // [p]
    int p, n_lo, N, f;
    int64_t B;
    int b;
    int64_t max_enum, evaluated = 0, distributable = 0;
    int min_pipes_fail = INT32_MAX;
    bool capped = false;
    std::vector<int32_t> x, best_x;
    std::vector<int64_t> best_nb, nb;
    std::vector<double> T, A;
    double best_thr = -1.0, best_iter = 0.0;
    int64_t best_pipes = 0;
};

double plan_iter_lower_bound(const oob_template *tpl, int p, const std::vector<int32_t> &x, int64_t K);

void evaluate(InstCtx &c) {
    int64_t pipes = 0;
    for (int i = 0; i < c.p; ++i) pipes += c.x[i];
    if (pipes < c.f + 1) return;
    c.evaluated++;
    const int64_t K = c.B / c.b;
    if (c.B % c.b != 0 || K < pipes) {
        c.min_pipes_fail = std::min<int64_t>(c.min_pipes_fail, pipes);
        return;
    }
    // bound first: no distribution of K microbatches over X beats B / (water level); skip
    // X when even that cannot reach the best throughput found (exact: ties are kept)
    if (c.best_thr > 0 && (double)c.B / plan_iter_lower_bound(c.tpl, c.p, c.x, K) < c.best_thr * (1.0 - 1e-12)) {
        c.distributable++;
        return;
    }
    c.T.clear();
    c.A.clear();
    for (int i = 0; i < c.p; ++i)
        for (int k = 0; k < c.x[i]; ++k) {
            const oob_template &t = c.tpl[i];
            c.T.push_back(t.tstar_ms);
            c.A.push_back(t.t1_ms + t.t3_ms - (double)(t.num_stages - t.kstar + 1) * t.tstar_ms);
        }
    c.nb.assign(pipes, 0);
    distribute_exact(c.T.data(), (int)pipes, K, c.nb.data(), nullptr, c.A.data());
    c.distributable++;
    double iter = 0.0;
    int64_t pi = 0;
    for (int i = 0; i < c.p; ++i)
        for (int k = 0; k < c.x[i]; ++k, ++pi) {
            const oob_template &t = c.tpl[i];
            // iteration_ms(N_b) = T1 + (N_b - S + k* - 1) t* + T3 (Eq.2 with the real N_b; no
            // negative steady phase below the pipeline fill: reading R30)
            const int64_t steady = std::max<int64_t>(0, c.nb[pi] - t.num_stages + t.kstar - 1);
            const double it = (t.t1_ms + (double)steady * t.tstar_ms) + t.t3_ms;
            iter = std::max(iter, it);
        }
    const double thr = (double)c.B / iter;
    bool better = false;
    if (thr > c.best_thr) better = true;
    else if (thr == c.best_thr) {
        if (pipes < c.best_pipes) better = true;
        else if (pipes == c.best_pipes && c.x < c.best_x) better = true;
    }
    if (better) {
        c.best_thr = thr; c.best_iter = iter; c.best_pipes = pipes;
        c.best_x = c.x; c.best_nb = c.nb;
    }
}

// DFS over x_{p-1} .. x_0 (the recursion of Eq.5: either no more of template p', or one
// more of it), stopping after max_enum feasible sets.
void dfs(InstCtx &c, int i, int rem) {
    if (c.capped) return;
    if (i < 0) {
        if (rem == 0) {
            if (c.evaluated >= c.max_enum) { c.capped = true; return; }
            evaluate(c);
        }
        return;
    }
    const int n = c.n_lo + i;
    const int kmax = c.tpl[i].num_stages > 0 ? rem / n : 0;   // infeasible template (masks): never used
    for (int k = 0; k <= kmax; ++k) {
        c.x[i] = k;
        dfs(c, i - 1, rem - k * n);
        if (c.capped) break;
    }
    c.x[i] = 0;
}

// Candidates when Eq.5's list is too long to enumerate (cfg4: 2.2e19 sets).  With the
// batch balanced, a plan's iteration time is about K / R + overhead, R = sum_i x_i / t*_i
// (the pipelines' total microbatch rate) and overhead = max over used templates of the
// fill/drain term T1 + T3 - (S - k* + 1) t*.  Unbounded knapsacks over nodes (exactly N
// used) maximise R:
//   (1) for every overhead threshold (templates sorted by it), among the templates under
//       it, with >= f+1 pipelines (saturating pipeline-count bucket 0..f+1);
//   (2) among all templates, for every exact pipeline count c = f+1 .. min(K, N/n0) (few
//       microbatches per pipeline make the integer split matter; c <= K keeps the batch
//       distributable).
// Every candidate is then scored exactly (Eq.6 + iteration time) like an enumerated set.
// Candidates for every node count t in [t_lo, N] from one set of knapsack DPs over 0..N
// (out[t - t_lo]); knapsack_candidates(.., N, ..) = the list for N alone.
std::vector<std::vector<std::vector<int32_t>>> knapsack_candidates_range(const oob_template *tpl, int p, int n_lo,
                                                                         int t_lo, int N, int f, int64_t K,
                                                                         int kb_per_count) {
    std::vector<int> order(p);
    std::vector<double> over(p), rate(p);
    std::vector<char> feas(p, 1);
    for (int i = 0; i < p; ++i) {
        order[i] = i;
        feas[i] = tpl[i].num_stages > 0;
        rate[i] = 1.0 / tpl[i].tstar_ms;
        over[i] = tpl[i].t1_ms + tpl[i].t3_ms - (double)(tpl[i].num_stages - tpl[i].kstar + 1) * tpl[i].tstar_ms;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return over[a] < over[b]; });
    const double NEG = -std::numeric_limits<double>::infinity();
    std::vector<double> dp;
    std::vector<int32_t> from;
    const int nT = N - t_lo + 1;
    std::vector<std::vector<std::vector<int32_t>>> outs((size_t)std::max(0, nT));
    std::vector<std::unordered_set<std::string>> seen((size_t)std::max(0, nT));   // dedupe per target
    auto push = [&](int T, const std::vector<int32_t> &x) {
        std::string key(reinterpret_cast<const char *>(x.data()), x.size() * sizeof(int32_t));
        if (seen[(size_t)(T - t_lo)].insert(std::move(key)).second) outs[(size_t)(T - t_lo)].push_back(x);
    };
    // knapsack over the allowed templates with C count buckets (saturating or exact)
    auto run = [&](const std::vector<char> &allowed, int C, bool saturate) {
        dp.assign((size_t)(N + 1) * C, NEG);
        from.assign((size_t)(N + 1) * C, 0);
        dp[0] = 0.0;
        for (int t = 1; t <= N; ++t)
            for (int i = 0; i < p; ++i) {
                if (!allowed[i] || !feas[i]) continue;
                const int n = n_lo + i;
                if (n > t) break;
                for (int c = 0; c < C; ++c) {
                    const double v = dp[(size_t)(t - n) * C + c];
                    if (v == NEG) continue;
                    const int c2 = saturate ? std::min(c + 1, C - 1) : c + 1;
                    if (c2 >= C) continue;
                    const double w = v + rate[i];
                    double &d = dp[(size_t)t * C + c2];
                    if (w > d) { d = w; from[(size_t)t * C + c2] = i | (c << 16); }
                }
            }
    };
    auto add = [&](int C, int c0) {
        for (int T = t_lo; T <= N; ++T) {
            int c = c0;
            if (dp[(size_t)T * C + c] == NEG) continue;
            std::vector<int32_t> x(p, 0);
            int t = T;
            while (t > 0) {
                const int32_t fr = from[(size_t)t * C + c];
                const int i = fr & 0xFFFF;
                x[i]++;
                t -= n_lo + i;
                c = fr >> 16;
            }
            push(T, x);
        }
    };
    std::vector<char> allowed(p, 0);
    for (int th = 0; th < p; ++th) {                       // (1)
        allowed[order[th]] = 1;
        if (th + 1 < p && over[order[th + 1]] == over[order[th]]) continue;
        run(allowed, f + 2, true);
        add(f + 2, f + 1);
    }
    // (3) (near-)homogeneous sets: q or q-1, q-2 pipelines of one template plus at most one
    // pipeline of the size that uses the remaining nodes (equal pipelines balance exactly)
    for (int T = t_lo; T <= N; ++T)
        for (int i = 0; i < p; ++i) {
            const int n = n_lo + i, q = T / n;
            if (!feas[i]) continue;
            for (int k = 0; k <= 2 && q - k >= 1; ++k) {
                const int R = T - (q - k) * n;
                if (R != 0 && (R < n_lo || R >= n_lo + p || !feas[R - n_lo])) continue;
                if ((q - k) + (R ? 1 : 0) < f + 1) continue;
                std::vector<int32_t> x(p, 0);
                x[i] += q - k;
                if (R) x[R - n_lo] += 1;
                push(T, x);
            }
        }
    // (2) with the KB best rates per (nodes, count) state, so near-optimal sets whose
    // integer batch split is better also get scored
    const int64_t cmax = std::min<int64_t>(K, N / n_lo);
    if (cmax >= f + 1 && kb_per_count > 0) {
        constexpr int KB = 4;
        const int kb_out = std::min(KB, kb_per_count);
        const int C = (int)cmax + 1;
        struct E { double v; int32_t i, c, r; };      // value, template, previous count, previous rank
        std::vector<E> kb((size_t)(N + 1) * C * KB, E{NEG, -1, 0, 0});
        auto at = [&](int t, int c, int r) -> E & { return kb[((size_t)t * C + c) * KB + r]; };
        at(0, 0, 0).v = 0.0;
        for (int t = 1; t <= N; ++t)
            for (int c = 1; c < C; ++c) {
                E best[KB];
                for (int r = 0; r < KB; ++r) best[r] = E{NEG, -1, 0, 0};
                for (int i = 0; i < p; ++i) {
                    const int n = n_lo + i;
                    if (n > t) break;
                    if (!feas[i]) continue;
                    for (int r = 0; r < KB; ++r) {
                        const E &prev = at(t - n, c - 1, r);
                        if (prev.v == NEG) break;
                        const E cand{prev.v + rate[i], i, c - 1, r};
                        if (cand.v <= best[KB - 1].v) continue;
                        bool dup = false;                // the same multiset reached in another order
                        for (int k = 0; k < KB; ++k) dup = dup || best[k].v == cand.v;
                        if (dup) continue;
                        int k = KB - 1;
                        while (k > 0 && best[k - 1].v < cand.v) { best[k] = best[k - 1]; --k; }
                        best[k] = cand;
                    }
                }
                for (int r = 0; r < KB; ++r) at(t, c, r) = best[r];
            }
        for (int T = t_lo; T <= N; ++T)
            for (int c = f + 1; c < C; ++c)
                for (int r0 = 0; r0 < kb_out; ++r0) {
                    if (at(T, c, r0).v == NEG) break;
                    std::vector<int32_t> x(p, 0);
                    int t = T, cc = c, r = r0;
                    while (t > 0) {
                        const E &e = at(t, cc, r);
                        x[e.i]++;
                        t -= n_lo + e.i;
                        cc = e.c;
                        r = e.r;
                    }
                    push(T, x);
                }
    }
    return outs;
}

std::vector<std::vector<int32_t>> knapsack_candidates(const oob_template *tpl, int p, int n_lo, int N, int f,
                                                      int64_t K) {
    return knapsack_candidates_range(tpl, p, n_lo, N, N, f, K, 4)[0];
}

// Lower bound of the iteration time (max_i T1 + (N_b,i - S + k* - 1) t* + T3 = a_i + N_b,i t_i)
// of ANY plan on exactly Np nodes distributing K microbatches (N_b,i >= 1): for tau = its
// iteration time, K = sum N_b,i <= sum_i (tau - a_i) / t_i <= Np max_{i in X} (tau - a_i) / (t_i n_i),
// and tau >= T1_i + T3_i for every used i (the steady phase is never negative, R30); so
// tau >= min_j max(T1_j + T3_j, a_j + K t_j n_j / Np).
double iter_lower_bound(const oob_template *tpl, int p, int n_lo, int Np, int64_t K) {
    double lb = std::numeric_limits<double>::infinity();
    for (int j = 0; j < p; ++j) {
        const oob_template &t = tpl[j];
        if (t.num_stages < 1) continue;          // infeasible template (stage masks)
        const double a = t.t1_ms + t.t3_ms - (double)(t.num_stages - t.kstar + 1) * t.tstar_ms;
        const double v = std::max(t.t1_ms + t.t3_ms, a + (double)K * t.tstar_ms * (double)(n_lo + j) / (double)Np);
        lb = std::min(lb, v);
    }
    return lb;
}

// Lower bound of the iteration time of plan x (any distribution, N_b,i >= 1 real): the
// water level tau with sum_i (tau - a_i) / t_i = K, and at least max_i (T1_i + T3_i) (the
// clamped steady phase, R30, keeps every pipeline at or above its fill + drain).
double plan_iter_lower_bound(const oob_template *tpl, int p, const std::vector<int32_t> &x, int64_t K) {
    double R = 0.0, A = 0.0, floor_ = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < p; ++i) {
        if (!x[i]) continue;
        const oob_template &t = tpl[i];
        const double a = t.t1_ms + t.t3_ms - (double)(t.num_stages - t.kstar + 1) * t.tstar_ms;
        R += (double)x[i] / t.tstar_ms;
        A += (double)x[i] * a / t.tstar_ms;
        floor_ = std::max(floor_, t.t1_ms + t.t3_ms);
    }
    return std::max(floor_, ((double)K + A) / R);
}

}  // namespace

extern "C" oob_status oob_count_sets(int32_t n_lo, int32_t n_hi, int32_t N, int32_t f, int64_t *out) {
    if (!out || n_lo < 1 || n_hi < n_lo || N < 0 || f < 0) return fail(OOB_E_INVALID, "oob_count_sets: bad argument");
    *out = count_sets(n_lo, n_hi, N, f);
    return OOB_OK;
}

extern "C" oob_status oob_instantiate(const oob_template_set *set, int32_t profile, int32_t N, int32_t f,
                                      int64_t B, int32_t b, int64_t max_enum, int32_t *counts_out,
                                      int64_t *nb_out, int32_t max_pipelines, int32_t *num_pipelines_out,
                                      double *thr_out, double *iter_out, int64_t *num_feasible_out,
                                      int64_t *rec_out) {
    if (!set || !counts_out || !nb_out || !num_pipelines_out)
        return fail(OOB_E_INVALID, "oob_instantiate: NULL argument");
    if (profile < 0 || profile >= set->num_profiles) return fail(OOB_E_INVALID, "oob_instantiate: bad profile");
    if (f < 0 || b < 1 || B < 1) return fail(OOB_E_INVALID, "oob_instantiate: need f >= 0, b >= 1, B >= 1");
    const int p = set->n_hi - set->n_lo + 1;
    if ((int64_t)N < (int64_t)(f + 1) * set->n_lo) return fail(OOB_E_INFEASIBLE, "insufficient nodes for f+1 replicas");
    InstCtx c;
    c.tpl = &set->templates[(size_t)profile * p];
    c.p = p; c.n_lo = set->n_lo; c.N = N; c.f = f; c.B = B; c.b = b;
    c.max_enum = max_enum > 0 ? max_enum : 1000000;
    c.x.assign(p, 0);
    std::vector<char> ok(p);
    for (int i = 0; i < p; ++i) ok[i] = c.tpl[i].num_stages > 0;
    const int64_t total = count_sets(set->n_lo, set->n_hi, N, f, ok.data());
    if (num_feasible_out) *num_feasible_out = total;
    if (total == 0) return fail(OOB_E_INFEASIBLE, "no feasible pipeline set for this node count");
    if (total <= c.max_enum) {
        dfs(c, p - 1, N);                  // exact: every feasible X (Eq.5)
    } else {
        c.capped = true;                   // too many: knapsack candidates, scored exactly
        for (const auto &x : knapsack_candidates(c.tpl, p, c.n_lo, N, f, B / b)) {
            c.x = x;
            evaluate(c);
        }
    }
    if (c.best_thr < 0) {
        if (rec_out) *rec_out = oob_recommend_batch(c.min_pipes_fail == INT32_MAX ? f + 1 : c.min_pipes_fail, b, B);
        return fail(OOB_E_BATCH, "no feasible set can distribute the global batch");
    }
    if (c.best_pipes > max_pipelines) return fail(OOB_E_NOMEM, "max_pipelines too small for the chosen plan");
    for (int i = 0; i < p; ++i) counts_out[i] = c.best_x[i];
    for (int64_t i = 0; i < c.best_pipes; ++i) nb_out[i] = c.best_nb[i];
    *num_pipelines_out = (int32_t)c.best_pipes;
    if (thr_out) *thr_out = c.best_thr;
    if (iter_out) *iter_out = c.best_iter;
    if (rec_out) *rec_out = B;
    if (c.capped) return fail(OOB_E_TOO_MANY, "more than max_enumerated feasible sets; plan is the best knapsack candidate");
    return OOB_OK;
}

// Plans for every node count N' in [n_min, n_max] (the instantiation for
// whatever number of nodes survives).  Exhaustive (Eq.5 + Eq.6) where the feasible sets
// number <= max_enum; above it, the knapsack candidates of every N' come from one set of DPs
// over 0..n_max and are scored exactly in decreasing order of their own relaxation bound
// until no remaining candidate can beat the best.  upper_bound_out certifies the result: no
// plan of N' nodes reaches a higher throughput (B / iter_lower_bound).
extern "C" oob_status oob_instantiate_all(const oob_template_set *set, int32_t profile, int32_t n_min, int32_t n_max,
                                          int32_t f, int64_t B, int32_t b, int64_t max_enum, int32_t *counts_out,
                                          double *thr_out, double *ub_out, int32_t *exact_out, int32_t *status_out) {
    if (!set || !counts_out || !thr_out || !ub_out || !exact_out || !status_out)
        return fail(OOB_E_INVALID, "oob_instantiate_all: NULL argument");
    if (profile < 0 || profile >= set->num_profiles) return fail(OOB_E_INVALID, "oob_instantiate_all: bad profile");
    if (f < 0 || b < 1 || B < 1 || n_min > n_max) return fail(OOB_E_INVALID, "oob_instantiate_all: bad argument");
    const int p = set->n_hi - set->n_lo + 1;
    const oob_template *tpl = &set->templates[(size_t)profile * p];
    const int64_t K = B / b;
    if (max_enum <= 0) max_enum = 1000000;
    const int lo = std::max<int>(n_min, (f + 1) * set->n_lo);
    std::vector<char> ok(p);
    for (int i = 0; i < p; ++i) ok[i] = tpl[i].num_stages > 0;
    // candidates of every capped N' from one set of knapsack DPs (only when some N' needs them)
    std::vector<std::vector<std::vector<int32_t>>> cands;
    const int c_lo = std::max(lo, n_min);
    for (int Np = c_lo; Np <= n_max; ++Np)
        if (count_sets(set->n_lo, set->n_hi, Np, f, ok.data()) > max_enum) {
            cands = knapsack_candidates_range(tpl, p, set->n_lo, c_lo, n_max, f, K, 4);
            break;
        }
    // the node counts are independent: host threads over N' (each its own context)
    auto solve = [&](int Np) {
        const int k = Np - n_min;
        int32_t *cnt = counts_out + (size_t)k * p;
        std::fill(cnt, cnt + p, 0);
        thr_out[k] = 0.0;
        ub_out[k] = 0.0;
        exact_out[k] = 0;
        status_out[k] = OOB_OK;
        const int64_t total = Np < lo ? 0 : count_sets(set->n_lo, set->n_hi, Np, f, ok.data());
        if (total == 0) {
            status_out[k] = OOB_E_INFEASIBLE;
            return;
        }
        InstCtx c;
        c.tpl = tpl; c.p = p; c.n_lo = set->n_lo; c.N = Np; c.f = f; c.B = B; c.b = b;
        c.max_enum = max_enum;
        c.x.assign(p, 0);
        if (total <= max_enum) {
            dfs(c, p - 1, Np);
            exact_out[k] = 1;
        } else {
            const auto &list = cands[(size_t)(Np - c_lo)];
            std::vector<std::pair<double, size_t>> order;
            for (size_t i = 0; i < list.size(); ++i)
                order.emplace_back(plan_iter_lower_bound(tpl, p, list[i], K), i);
            std::sort(order.begin(), order.end());
            for (const auto &o : order) {
                // no remaining candidate can beat the best found (1e-12: rounding of the bound)
                if (c.best_thr > 0 && (double)B / o.first < c.best_thr * (1.0 - 1e-12)) break;
                c.x = list[o.second];
                evaluate(c);
            }
        }
        if (c.best_thr < 0) { status_out[k] = OOB_E_BATCH; return; }
        for (int i = 0; i < p; ++i) cnt[i] = c.best_x[i];
        thr_out[k] = c.best_thr;
        ub_out[k] = exact_out[k] ? c.best_thr : std::max(c.best_thr, (double)B / iter_lower_bound(tpl, p, set->n_lo, Np, K));
    };
    const int nthr = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), n_max - n_min + 1));
    std::atomic<int> next(n_min);
    std::vector<std::thread> pool;
    for (int t = 0; t < nthr; ++t)
        pool.emplace_back([&]() {
            for (int Np; (Np = next.fetch_add(1)) <= n_max;) solve(Np);
        });
    for (auto &th : pool) th.join();
    return OOB_OK;
}