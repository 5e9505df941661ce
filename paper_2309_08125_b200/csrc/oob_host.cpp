// Host side of the C ABI: errors, profiles (arrays + SPEC JSON), node specification,
// template-set assembly around the CUDA DP engine, Eq.5 instantiation and Eq.6 batch
// distribution (PAPER §4.1.1, §4.2).  See include/oobleck_plan.h for the contract.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "oob_internal.h"

extern char **environ;

namespace oob {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
oob_status fail(oob_status s, const std::string &msg) {
    set_error(msg);
    return s;
}

// ------------------------------------------------------------------ tiny JSON reader
// Enough JSON for the SPEC S:99 profile format: objects, arrays, strings, numbers,
// true/false/null.  Numbers are parsed with strtod (round-trips %.17g and hex floats).
struct JVal {
    enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
    double num = 0;
    bool b = false;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal *get(const std::string &k) const {
        for (auto &kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JParser {
    const char *p, *end;
    std::string err;
    void ws() { while (p < end && std::isspace((unsigned char)*p)) ++p; }
    bool parse(JVal &v, int depth = 0) {
        if (depth > 64) { err = "nesting too deep"; return false; }
        ws();
        if (p >= end) { err = "unexpected end of input"; return false; }
        char c = *p;
        if (c == '{') {
            ++p; v.kind = JVal::OBJ;
            ws();
            if (p < end && *p == '}') { ++p; return true; }
            for (;;) {
                ws();
                JVal key;
                if (p >= end || *p != '"' || !parse_str(key.str)) { if (err.empty()) err = "expected key"; return false; }
                ws();
                if (p >= end || *p != ':') { err = "expected ':'"; return false; }
                ++p;
                JVal val;
                if (!parse(val, depth + 1)) return false;
                v.obj.emplace_back(key.str, std::move(val));
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == '}') { ++p; return true; }
                err = "expected ',' or '}'"; return false;
            }
        }
        if (c == '[') {
            ++p; v.kind = JVal::ARR;
            ws();
            if (p < end && *p == ']') { ++p; return true; }
            for (;;) {
                JVal val;
                if (!parse(val, depth + 1)) return false;
                v.arr.push_back(std::move(val));
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == ']') { ++p; return true; }
                err = "expected ',' or ']'"; return false;
            }
        }
        if (c == '"') { v.kind = JVal::STR; return parse_str(v.str); }
        if (!std::strncmp(p, "true", std::min<size_t>(4, end - p)) && end - p >= 4) { p += 4; v.kind = JVal::BOOL; v.b = true; return true; }
        if (!std::strncmp(p, "false", std::min<size_t>(5, end - p)) && end - p >= 5) { p += 5; v.kind = JVal::BOOL; return true; }
        if (!std::strncmp(p, "null", std::min<size_t>(4, end - p)) && end - p >= 4) { p += 4; v.kind = JVal::NUL; return true; }
        // number
        std::string tok;
        while (p < end && (std::isalnum((unsigned char)*p) || *p == '-' || *p == '+' || *p == '.')) tok += *p++;
        if (tok.empty()) { err = std::string("unexpected character '") + c + "'"; return false; }
        char *q = nullptr;
        v.num = std::strtod(tok.c_str(), &q);
        if (!q || *q) { err = "bad number '" + tok + "'"; return false; }
        v.kind = JVal::NUM;
        return true;
    }
    bool parse_str(std::string &out) {
        ++p;  // opening quote
        while (p < end && *p != '"') {
            if (*p == '\\') {
                ++p;
                if (p >= end) break;
                char e = *p++;
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': out += '?'; p += std::min<ptrdiff_t>(4, end - p); break;
                    default: out += e;
                }
            } else {
                out += *p++;
            }
        }
        if (p >= end) { err = "unterminated string"; return false; }
        ++p;
        return true;
    }
};

static bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

}  // namespace oob

using namespace oob;

// ==================================================================== errors
extern "C" const char *oob_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *oob_status_string(oob_status s) {
    switch (s) {
        case OOB_OK: return "OOB_OK";
        case OOB_E_PARSE: return "OOB_E_PARSE";
        case OOB_E_INVALID: return "OOB_E_INVALID";
        case OOB_E_INFEASIBLE: return "OOB_E_INFEASIBLE";
        case OOB_E_BATCH: return "OOB_E_BATCH";
        case OOB_E_TOO_MANY: return "OOB_E_TOO_MANY";
        case OOB_E_CUDA: return "OOB_E_CUDA";
        case OOB_E_NCCL: return "OOB_E_NCCL";
        case OOB_E_NOMEM: return "OOB_E_NOMEM";
    }
    return "OOB_E_UNKNOWN";
}

// ==================================================================== profiles
extern "C" oob_status oob_profile_from_arrays(int32_t L, int32_t M, const double *fwd,
                                              const double *bwd, const int64_t *state_bytes,
                                              oob_profile **out) {
    if (!out) return fail(OOB_E_INVALID, "oob_profile_from_arrays: out is NULL");
    *out = nullptr;
    if (L < 1) return fail(OOB_E_INVALID, "empty model (L < 1)");
    if (L > 1023) return fail(OOB_E_INVALID, "L > 1023 is not supported");
    if (M < 1 || M > 64) return fail(OOB_E_INVALID, "gpus_per_node must be in 1..64");
    if (!fwd || !bwd) return fail(OOB_E_INVALID, "fwd_ms/bwd_ms is NULL");
    for (int64_t i = 0; i < (int64_t)L * M; ++i)
        if (!finite_pos(fwd[i]) || !finite_pos(bwd[i]))
            return fail(OOB_E_INVALID, "non-positive or non-finite time at layer " +
                                           std::to_string(i / M) + ", d=" + std::to_string(i % M + 1));
    auto *p = new (std::nothrow) oob_profile();
    if (!p) return fail(OOB_E_NOMEM, "out of memory");
    p->L = L; p->M = M;
    p->fwd.assign(fwd, fwd + (size_t)L * M);
    p->bwd.assign(bwd, bwd + (size_t)L * M);
    p->state_bytes.assign(L, 0);
    p->act_bytes.assign(L, 0);
    if (state_bytes) p->state_bytes.assign(state_bytes, state_bytes + L);
    *out = p;
    return OOB_OK;
}

extern "C" oob_status oob_load_profile(const char *path, oob_profile **out) {
    if (!out || !path) return fail(OOB_E_INVALID, "oob_load_profile: NULL argument");
    *out = nullptr;
    std::ifstream in(path, std::ios::binary);
    if (!in) return fail(OOB_E_PARSE, std::string("cannot open ") + path);
    std::stringstream ss;
    ss << in.rdbuf();
    std::string text = ss.str();
    JParser jp{text.data(), text.data() + text.size(), {}};
    JVal root;
    if (!jp.parse(root)) return fail(OOB_E_PARSE, "profile JSON: " + jp.err);
    jp.ws();
    if (jp.p != jp.end) return fail(OOB_E_PARSE, "profile JSON: trailing characters");
    if (root.kind != JVal::OBJ) return fail(OOB_E_PARSE, "profile JSON: top level must be an object");
    const JVal *jm = root.get("gpus_per_node");
    const JVal *jl = root.get("layers");
    if (!jm || jm->kind != JVal::NUM) return fail(OOB_E_INVALID, "missing gpus_per_node");
    if (!jl || jl->kind != JVal::ARR) return fail(OOB_E_INVALID, "missing layers array");
    const int M = (int)jm->num;
    const int L = (int)jl->arr.size();
    if (L == 0) return fail(OOB_E_INVALID, "empty model");
    if (M < 1 || M > 64 || (double)M != jm->num) return fail(OOB_E_INVALID, "gpus_per_node must be an integer in 1..64");
    std::vector<double> fwd((size_t)L * M), bwd((size_t)L * M);
    std::vector<int64_t> state(L, 0), act(L, 0);
    for (int l = 0; l < L; ++l) {
        const JVal &ly = jl->arr[l];
        if (ly.kind != JVal::OBJ) return fail(OOB_E_PARSE, "layer " + std::to_string(l) + " is not an object");
        const JVal *f = ly.get("fwd_ms"), *b = ly.get("bwd_ms");
        if (!f || !b || f->kind != JVal::OBJ || b->kind != JVal::OBJ)
            return fail(OOB_E_INVALID, "layer " + std::to_string(l) + ": missing fwd_ms/bwd_ms");
        for (int d = 1; d <= M; ++d) {
            const JVal *fv = f->get(std::to_string(d)), *bv = b->get(std::to_string(d));
            if (!fv || !bv || fv->kind != JVal::NUM || bv->kind != JVal::NUM)
                return fail(OOB_E_INVALID, "layer " + std::to_string(l) + ": missing device-count entry d=" + std::to_string(d));
            fwd[(size_t)l * M + d - 1] = fv->num;
            bwd[(size_t)l * M + d - 1] = bv->num;
        }
        if (const JVal *s = ly.get("state_bytes"); s && s->kind == JVal::NUM) state[l] = (int64_t)s->num;
        if (const JVal *a = ly.get("activation_bytes_per_sample"); a && a->kind == JVal::NUM) act[l] = (int64_t)a->num;
    }
    oob_profile *p = nullptr;
    oob_status st = oob_profile_from_arrays(L, M, fwd.data(), bwd.data(), state.data(), &p);
    if (st != OOB_OK) return st;
    p->act_bytes = act;
    if (const JVal *mb = root.get("microbatch_reference"); mb && mb->kind == JVal::NUM) p->microbatch_reference = (int32_t)mb->num;
    *out = p;
    return OOB_OK;
}

extern "C" void oob_profile_free(oob_profile *p) { delete p; }
extern "C" int32_t oob_profile_layers(const oob_profile *p) { return p ? p->L : 0; }
extern "C" int32_t oob_profile_gpus_per_node(const oob_profile *p) { return p ? p->M : 0; }
extern "C" oob_status oob_profile_costs(const oob_profile *p, double *fwd, double *bwd, int64_t *state_bytes) {
    if (!p) return fail(OOB_E_INVALID, "oob_profile_costs: NULL profile");
    if (fwd) std::copy(p->fwd.begin(), p->fwd.end(), fwd);
    if (bwd) std::copy(p->bwd.begin(), p->bwd.end(), bwd);
    if (state_bytes) std::copy(p->state_bytes.begin(), p->state_bytes.end(), state_bytes);
    return OOB_OK;
}

extern "C" oob_status oob_min_nodes(const oob_profile *p, int32_t nodes, int64_t gpu_mem,
                                    double util, int32_t spg, int32_t *n0_out) {
    if (!p || !n0_out) return fail(OOB_E_INVALID, "oob_min_nodes: NULL argument");
    if (util <= 0.0) util = 0.8;
    if (util > 1.0) return fail(OOB_E_INVALID, "util must be in (0, 1]");
    if (spg <= 0) spg = 1;
    if (gpu_mem <= 0) return fail(OOB_E_INVALID, "gpu_mem_bytes must be positive");
    long double total = 0;
    for (int l = 0; l < p->L; ++l) total += (long double)p->state_bytes[l] + (long double)spg * p->act_bytes[l];
    long double slice = (long double)p->M * gpu_mem * util;
    long double q = total / slice;
    int64_t n0 = (int64_t)std::ceil((double)q);
    if (n0 < 1) n0 = 1;
    if (nodes > 0 && n0 > nodes) return fail(OOB_E_INFEASIBLE, "model does not fit on the cluster");
    *n0_out = (int32_t)n0;
    return OOB_OK;
}

extern "C" oob_status oob_node_sizes(int32_t N, int32_t f, int32_t n0, int32_t L, int32_t *n_lo,
                                     int32_t *n_hi) {
    if (!n_lo || !n_hi) return fail(OOB_E_INVALID, "oob_node_sizes: NULL argument");
    if (f < 0 || n0 < 1 || L < 1) return fail(OOB_E_INVALID, "need f >= 0, n0 >= 1, L >= 1");
    if ((int64_t)N < (int64_t)(f + 1) * n0) return fail(OOB_E_INFEASIBLE, "cannot maintain f+1 replicas");
    if (n0 > L) return fail(OOB_E_INFEASIBLE, "too few layers for node count");
    *n_lo = n0;
    *n_hi = std::min<int32_t>(N - f * n0, L);
    return OOB_OK;
}

// ==================================================================== template sets
extern "C" oob_status oob_template_set_from_packed(const void *h_packed, const oob_dp_info *info,
                                                   oob_template_set **out) {
    if (!h_packed || !info || !out) return fail(OOB_E_INVALID, "oob_template_set_from_packed: NULL argument");
    *out = nullptr;
    const int p = info->n_hi - info->n_lo + 1;
    auto *s = new (std::nothrow) oob_template_set();
    if (!s) return fail(OOB_E_NOMEM, "out of memory");
    s->L = info->L; s->M = info->M; s->n_lo = info->n_lo; s->n_hi = info->n_hi;
    s->num_profiles = info->num_profiles;
    s->templates.resize((size_t)info->num_profiles * p);
    s->stages.resize((size_t)info->num_profiles * p * info->L);
    const unsigned char *base = (const unsigned char *)h_packed;
    for (int pr = 0; pr < info->num_profiles; ++pr) {
        for (int i = 0; i < p; ++i) {
            const size_t t = (size_t)pr * p + i;
            const PackedHeader *h = (const PackedHeader *)(base + t * info->packed_template_bytes);
            const int32_t *st = (const int32_t *)(h + 1);
            if (h->status == 3 && h->S == 0) {   // no allowed mapping (stage masks, reading R31)
                oob_template &tv = s->templates[t];
                tv.nodes = h->nodes; tv.num_stages = 0; tv.kstar = 0; tv.reserved = 0;
                tv.t1_ms = h->T1; tv.t2_ms = h->T2; tv.t3_ms = h->T3; tv.tstar_ms = h->tstar; tv.iter_ms = h->iter;
                tv.stages = &s->stages[t * info->L];
                continue;
            }
            if (h->S < 1 || h->S > info->L || h->status != 0) {
                const std::string where = " (profile " + std::to_string(pr) + ", template " + std::to_string(i) + ")";
                const int code = h->status;
                delete s;
                if (code == 2)
                    return fail(OOB_E_CUDA, "wavefront pipeline wait timed out (GPU shared with other work?): "
                                            "the DP table is incomplete" + where);
                if (code == 4)
                    return fail(OOB_E_CUDA, "exact solver: bottleneck stage list overflow" + where);
                return fail(OOB_E_CUDA, "corrupt packed template" + where);
            }
            oob_template &tv = s->templates[t];
            tv.nodes = h->nodes; tv.num_stages = h->S; tv.kstar = h->kstar; tv.reserved = 0;
            tv.t1_ms = h->T1; tv.t2_ms = h->T2; tv.t3_ms = h->T3; tv.tstar_ms = h->tstar; tv.iter_ms = h->iter;
            oob_stage *dst = &s->stages[t * info->L];
            for (int j = 0; j < h->S; ++j) {
                dst[j].layer_begin = st[5 * j + 0];
                dst[j].layer_end = st[5 * j + 1];
                dst[j].gpus = st[5 * j + 2];
                dst[j].node = st[5 * j + 3];
                dst[j].gpu_offset = st[5 * j + 4];
            }
            tv.stages = dst;
        }
    }
    *out = s;
    return OOB_OK;
}

extern "C" int32_t oob_template_set_profiles(const oob_template_set *s) { return s ? s->num_profiles : 0; }
extern "C" int32_t oob_template_count(const oob_template_set *s, int32_t profile) {
    if (!s || profile < 0 || profile >= s->num_profiles) return 0;
    return s->n_hi - s->n_lo + 1;
}
extern "C" oob_status oob_template_get(const oob_template_set *s, int32_t profile, int32_t i,
                                       oob_template *view) {
    if (!s || !view) return fail(OOB_E_INVALID, "oob_template_get: NULL argument");
    const int p = s->n_hi - s->n_lo + 1;
    if (profile < 0 || profile >= s->num_profiles || i < 0 || i >= p)
        return fail(OOB_E_INVALID, "oob_template_get: index out of range");
    *view = s->templates[(size_t)profile * p + i];
    return OOB_OK;
}
extern "C" void oob_template_set_free(oob_template_set *s) { delete s; }

// Plans (host geometry + unit queues, a few ms to build at cfg4) are cached across
// oob_generate_templates calls, keyed by shape, device and the OOB_DP_* plan switches; a
// plan is taken out of the cache while in use, so concurrent calls never share one.
namespace {
struct PlanCache {
    std::mutex mu;
    std::vector<std::pair<std::string, oob_dp_plan *>> plans;   // most recent last
};
PlanCache &plan_cache() {
    static PlanCache *c = new PlanCache();   // never destroyed: no CUDA calls at exit
    return *c;
}
std::string plan_key(int L, int M, int n_lo, int n_hi, int P, int dev) {
    std::string k = std::to_string(L) + "," + std::to_string(M) + "," + std::to_string(n_lo) + "," +
                    std::to_string(n_hi) + "," + std::to_string(P) + "," + std::to_string(dev);
    // every plan-time switch: all OOB_DP_* variables of the environment (sorted), so a
    // plan built under other settings is never reused
    std::vector<std::string> kv;
    for (char **e = environ; e && *e; ++e)
        if (std::strncmp(*e, "OOB_DP_", 7) == 0) kv.emplace_back(*e);
    std::sort(kv.begin(), kv.end());
    for (const std::string &x : kv) k += "|" + x;
    return k;
}
oob_dp_plan *take_plan(const std::string &key) {
    PlanCache &c = plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    for (size_t i = c.plans.size(); i-- > 0;)
        if (c.plans[i].first == key) {
            oob_dp_plan *p = c.plans[i].second;
            c.plans.erase(c.plans.begin() + (long)i);
            return p;
        }
    return nullptr;
}
void give_plan(const std::string &key, oob_dp_plan *p) {
    PlanCache &c = plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.plans.emplace_back(key, p);
    while (c.plans.size() > 4) {
        oob_dp_plan_free(c.plans.front().second);
        c.plans.erase(c.plans.begin());
    }
}
}  // namespace

extern "C" oob_status oob_generate_templates(const oob_profile *const *profiles, int32_t num_profiles,
                                             const oob_plan_opts *opts, oob_template_set **out) {
    if (!profiles || !opts || !out || num_profiles < 1)
        return fail(OOB_E_INVALID, "oob_generate_templates: NULL argument or num_profiles < 1");
    *out = nullptr;
    const int L = profiles[0] ? profiles[0]->L : 0;
    const int M = profiles[0] ? profiles[0]->M : 0;
    for (int i = 0; i < num_profiles; ++i) {
        if (!profiles[i]) return fail(OOB_E_INVALID, "NULL profile");
        if (profiles[i]->L != L || profiles[i]->M != M)
            return fail(OOB_E_INVALID, "all profiles of a batch must share L and M");
    }
    if (opts->gpus_per_node != M)
        return fail(OOB_E_INVALID, "opts.gpus_per_node does not match the profile");
    if (opts->exact && (opts->tp_pow2 || opts->stage_mem_bytes > 0.0))
        return fail(OOB_E_INVALID, "opts.exact does not support stage masks");
    int n0 = opts->n0;
    if (n0 <= 0) {
        for (int i = 0; i < num_profiles; ++i) {
            int32_t v = 0;
            oob_status st = oob_min_nodes(profiles[i], opts->nodes, opts->gpu_mem_bytes, opts->util,
                                          opts->samples_per_gpu, &v);
            if (st != OOB_OK) return st;
            n0 = std::max(n0, (int)v);
        }
    }
    int32_t n_lo = 0, n_hi = 0;
    oob_status st = oob_node_sizes(opts->nodes, opts->f, n0, L, &n_lo, &n_hi);
    if (st != OOB_OK) return st;

    cudaError_t e;
    if (opts->device >= 0) {
        e = cudaSetDevice(opts->device);
        if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    cudaStream_t stream = (cudaStream_t)opts->stream;
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess)
        return fail(OOB_E_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    // multi-GPU: with a communicator of world > 1, one profile is planned by
    // every rank with its wavefronts split across the ranks; a batch of profiles is split into
    // contiguous blocks (rank r plans its block) and one all-gather assembles every rank's
    // packed template sets.  Every rank passes the same profiles and receives the whole set.
    const int world = (opts->comm && opts->world > 1) ? opts->world : 1;
    const int rank = world > 1 ? opts->rank : 0;
    if (world > 1 && (rank < 0 || rank >= world)) return fail(OOB_E_INVALID, "opts.rank out of range");
    const bool shard_one = world > 1 && num_profiles == 1;
    int first = 0, count = num_profiles, per_rank = num_profiles;
    if (world > 1 && !shard_one) {
        const int base = num_profiles / world, extra = num_profiles % world;
        first = rank * base + std::min(rank, extra);
        count = base + (rank < extra ? 1 : 0);
        per_rank = base + (extra ? 1 : 0);
    }
    const int plan_P = std::max(1, count);
    std::string key = plan_key(L, M, n_lo, n_hi, plan_P, dev);
    if (shard_one) key += "|comm" + std::to_string((uintptr_t)opts->comm) + "," + std::to_string(world) + "," +
                          std::to_string(rank);
    oob_dp_plan *plan = take_plan(key);
    if (!plan) {
        st = oob_dp_plan_create(L, M, n_lo, n_hi, plan_P, &plan);
        if (st != OOB_OK) return st;
        if (shard_one && (st = oob_dp_set_comm(plan, opts->comm, world, rank)) != OOB_OK) {
            oob_dp_plan_free(plan);
            return st;
        }
    }
    struct Return {
        std::string key;
        oob_dp_plan *p;
        ~Return() { give_plan(key, p); }
    } plan_guard{key, plan};
    oob_dp_info info;
    oob_dp_plan_info(plan, &info);

    const size_t prof_bytes = sizeof(double) * (size_t)L * M;
    const size_t gather_bytes = (world > 1 && !shard_one) ? (size_t)world * per_rank * info.packed_profile_bytes : 0;
    const bool masked_mem = opts->stage_mem_bytes > 0.0;
    const size_t sb_bytes = masked_mem ? align_up_host(sizeof(double) * (size_t)L * plan_P) : 0;
    size_t own_bytes = align_up_host(2 * prof_bytes * plan_P) + align_up_host(std::max<size_t>(
                                                                   info.packed_bytes, (size_t)per_rank * info.packed_profile_bytes)) +
                       align_up_host(gather_bytes) + sb_bytes;
    void *ws = opts->workspace;
    size_t ws_bytes = opts->workspace_bytes;
    void *own = nullptr;
    if (!ws) ws_bytes = 0;
    // inputs + packed output (+ the gathered sets) live after the DP workspace (caller's or ours)
    size_t need = align_up_host(info.workspace_bytes) + own_bytes;
    if (!ws || ws_bytes < need) {
        if (ws && ws_bytes > 0 && ws_bytes < need)
            return fail(OOB_E_NOMEM, "opts.workspace too small: need " + std::to_string(need) + " bytes");
        e = cudaMalloc(&own, need);
        if (e != cudaSuccess) return fail(OOB_E_NOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
        ws = own;
        ws_bytes = need;
    }
    std::unique_ptr<void, void (*)(void *)> own_guard(own, [](void *q) { if (q) cudaFree(q); });
    unsigned char *wsb = (unsigned char *)ws;
    double *d_fwd = (double *)(wsb + align_up_host(info.workspace_bytes));
    double *d_bwd = d_fwd + (size_t)L * M * plan_P;
    unsigned char *d_packed = (unsigned char *)d_fwd + align_up_host(2 * prof_bytes * plan_P);
    unsigned char *d_gather = d_packed + align_up_host(std::max<size_t>(info.packed_bytes,
                                                                        (size_t)per_rank * info.packed_profile_bytes));
    double *d_sb = masked_mem ? (double *)(d_gather + align_up_host(gather_bytes)) : nullptr;
    std::vector<double> h_sb;
    if (masked_mem) {   // per-layer stage bytes (reading R31): state + samples_per_gpu x activations
        const int spg = opts->samples_per_gpu > 0 ? opts->samples_per_gpu : 1;
        h_sb.resize((size_t)L * plan_P);
        for (int i = 0; i < plan_P; ++i) {
            const oob_profile *pf = profiles[count > 0 ? first + i : 0];
            for (int l = 0; l < L; ++l)
                h_sb[(size_t)i * L + l] = (double)pf->state_bytes[l] + (double)spg * (double)pf->act_bytes[l];
        }
        e = cudaMemcpyAsync(d_sb, h_sb.data(), sizeof(double) * h_sb.size(), cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("H2D stage bytes: ") + cudaGetErrorString(e));
    }
    st = oob_dp_set_stage_masks(plan, opts->tp_pow2, d_sb, masked_mem ? opts->stage_mem_bytes : 0.0);
    if (st != OOB_OK) return st;
    // H2D of this rank's profile costs (one copy per array per profile; a rank without
    // profiles plans a copy of profile 0 and discards it)
    for (int i = 0; i < plan_P; ++i) {
        const oob_profile *pf = profiles[count > 0 ? first + i : 0];
        e = cudaMemcpyAsync(d_fwd + (size_t)i * L * M, pf->fwd.data(), prof_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_bwd + (size_t)i * L * M, pf->bwd.data(), prof_bytes, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("H2D profile: ") + cudaGetErrorString(e));
    }
    st = oob_dp_run(plan, d_fwd, d_bwd, ws, info.workspace_bytes, d_packed, stream);
    oob_dp_set_stage_masks(plan, 0, nullptr, 0.0);   // the cached plan carries no masks to other calls
    if (st != OOB_OK) return st;
    // exact optimum (oob_exact_run): the recursion's templates bound the search, the exact
    // ones overwrite them in place
    void *ex_ws = nullptr;
    std::unique_ptr<void, void (*)(void *)> ex_guard(nullptr, [](void *q) { if (q) cudaFree(q); });
    if (opts->exact) {
        size_t ex_bytes = 0;
        if ((st = oob_exact_workspace_bytes(L, M, n_lo, n_hi, plan_P, &ex_bytes)) != OOB_OK) return st;
        if ((e = cudaMalloc(&ex_ws, ex_bytes)) != cudaSuccess)
            return fail(OOB_E_NOMEM, std::string("cudaMalloc exact workspace: ") + cudaGetErrorString(e));
        ex_guard.reset(ex_ws);
        st = oob_exact_run(L, M, n_lo, n_hi, plan_P, d_fwd, d_bwd, d_packed, ex_ws, ex_bytes, d_packed, stream);
        if (st != OOB_OK) return st;
    }
    if (world == 1 || shard_one) {
        std::vector<unsigned char> host(info.packed_bytes);
        e = cudaMemcpyAsync(host.data(), d_packed, info.packed_bytes, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("DP run / D2H: ") + cudaGetErrorString(e));
        return oob_template_set_from_packed(host.data(), &info, out);
    }
    // batched sweep across ranks: one NCCL all-gather of the per-rank blocks (padded to
    // per_rank profiles), then the blocks in rank order are the profiles in order
    const size_t blk = (size_t)per_rank * info.packed_profile_bytes;
    st = nccl_allgather_bytes(opts->comm, d_packed, d_gather, blk, gather_bytes, world, stream);
    if (st != OOB_OK) return st;
    std::vector<unsigned char> host(gather_bytes);
    e = cudaMemcpyAsync(host.data(), d_gather, gather_bytes, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("DP run / all-gather / D2H: ") + cudaGetErrorString(e));
    std::vector<unsigned char> whole((size_t)num_profiles * info.packed_profile_bytes);
    for (int r = 0, pos = 0; r < world; ++r) {
        const int cnt = num_profiles / world + (r < num_profiles % world ? 1 : 0);
        std::memcpy(whole.data() + (size_t)pos * info.packed_profile_bytes, host.data() + (size_t)r * blk,
                    (size_t)cnt * info.packed_profile_bytes);
        pos += cnt;
    }
    oob_dp_info all = info;
    all.num_profiles = num_profiles;
    all.packed_bytes = whole.size();
    return oob_template_set_from_packed(whole.data(), &all, out);
}
