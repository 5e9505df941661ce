// Dynamic reconfiguration over a template set (PAPER §5; Appendix B,
// P:984-1006): an execution state of pipelines instantiated from the templates, updated on
// node failures by simple reinstantiation, node borrowing and pipeline merging (§5.1),
// followed by batch redistribution (§5.2, Eq.6), the copy plan of missing layers
// and the per-layer synchronisation groups of §6.1.  Host C++;
// the readings where the paper is silent are DESIGN.md §10 (R21-R28).
#include <algorithm>
#include <map>
#include <memory>
#include <new>
#include <set>
#include <string>
#include <vector>

#include "oob_internal.h"

struct oob_exec {
    int32_t f = 0, b = 1, n_lo = 0, n_hi = 0, L = 0, profile = 0;
    int64_t B = 0;
    int64_t max_enumerated = 0;
    std::vector<std::vector<oob_stage>> stages;   // [n - n_lo]: template of n nodes
    std::vector<double> tstar;                    // [n - n_lo]
    const oob_template_set *set = nullptr;        // borrowed (replans only)
    std::vector<int64_t> layer_bytes;             // [L]
    std::vector<std::vector<int32_t>> pipes;      // node ids per pipeline (template = size)
    std::vector<int64_t> nb;                      // microbatches per pipeline (Eq.6)
    std::vector<oob_action> actions;              // of the last reconfiguration
    std::vector<oob_transfer> transfers;          // of the last reconfiguration
};

namespace {

using namespace oob;

// node id -> layers it holds (its stages in its pipeline's template)
std::map<int32_t, std::set<int32_t>> owned(const oob_exec &x) {
    std::map<int32_t, std::set<int32_t>> own;
    for (const auto &nodes : x.pipes) {
        for (const oob_stage &s : x.stages[nodes.size() - x.n_lo]) {
            auto &ls = own[nodes[s.node]];
            for (int32_t l = s.layer_begin; l < s.layer_end; ++l) ls.insert(l);
        }
    }
    return own;
}

// Eq.6 over the current pipelines (reading R26)
oob_status redistribute(oob_exec &x, int64_t *recommended) {
    std::vector<double> T;
    for (const auto &nodes : x.pipes) T.push_back(x.tstar[nodes.size() - x.n_lo]);
    x.nb.assign(T.size(), 0);
    return oob_distribute_batch(T.data(), (int32_t)T.size(), x.B, x.b, x.nb.data(), nullptr, recommended);
}

oob_action act(int32_t kind, int32_t a, int32_t b, int32_t nodes) {
    oob_action r;
    r.kind = kind; r.a = a; r.b = b; r.nodes = nodes;
    return r;
}

}  // namespace

extern "C" oob_status oob_exec_create(const oob_template_set *set, int32_t profile, int32_t f,
                                      int64_t global_batch, int32_t microbatch, const int32_t *counts,
                                      const int32_t *node_ids, int32_t num_nodes, const int64_t *layer_bytes,
                                      oob_exec **out) {
    if (!set || !counts || !node_ids || !out) return fail(OOB_E_INVALID, "oob_exec_create: NULL argument");
    *out = nullptr;
    const int p = oob_template_count(set, profile);
    if (p < 1) return fail(OOB_E_INVALID, "oob_exec_create: profile out of range");
    if (f < 0 || microbatch < 1 || global_batch < 1) return fail(OOB_E_INVALID, "need f >= 0, b >= 1, B >= 1");
    auto *x = new (std::nothrow) oob_exec();
    if (!x) return fail(OOB_E_NOMEM, "out of memory");
    std::unique_ptr<oob_exec> guard(x);
    x->set = set; x->profile = profile; x->f = f; x->B = global_batch; x->b = microbatch;
    for (int i = 0; i < p; ++i) {
        oob_template t;
        oob_status st = oob_template_get(set, profile, i, &t);
        if (st != OOB_OK) return st;
        if (t.num_stages < 1)   // reinstantiation assumes every size n_lo..n_hi has a template
            return fail(OOB_E_INVALID, "oob_exec_create: the template set has an infeasible size (stage masks)");
        if (i == 0) x->n_lo = t.nodes;
        x->n_hi = t.nodes;
        x->stages.emplace_back(t.stages, t.stages + t.num_stages);
        x->tstar.push_back(t.tstar_ms);
        x->L = t.stages[t.num_stages - 1].layer_end;
    }
    x->layer_bytes.assign(x->L, 0);
    if (layer_bytes) x->layer_bytes.assign(layer_bytes, layer_bytes + x->L);
    int pos = 0;
    std::set<int32_t> seen;
    for (int i = 0; i < p; ++i) {
        if (counts[i] < 0) return fail(OOB_E_INVALID, "negative pipeline count");
        for (int c = 0; c < counts[i]; ++c) {
            const int n = x->n_lo + i;
            if (pos + n > num_nodes) return fail(OOB_E_INVALID, "counts need more nodes than given");
            x->pipes.emplace_back(node_ids + pos, node_ids + pos + n);
            for (int k = pos; k < pos + n; ++k)
                if (!seen.insert(node_ids[k]).second) return fail(OOB_E_INVALID, "duplicate node id");
            pos += n;
        }
    }
    if (pos != num_nodes) return fail(OOB_E_INVALID, "counts do not use every node");
    if ((int)x->pipes.size() < f + 1) return fail(OOB_E_INFEASIBLE, "fewer than f+1 pipelines");
    int64_t rec = 0;
    oob_status st = redistribute(*x, &rec);
    if (st != OOB_OK) return st;
    *out = guard.release();
    return OOB_OK;
}

extern "C" void oob_exec_free(oob_exec *x) { delete x; }

extern "C" int32_t oob_exec_num_pipelines(const oob_exec *x) { return x ? (int32_t)x->pipes.size() : 0; }

extern "C" oob_status oob_exec_pipeline(const oob_exec *x, int32_t i, int32_t *nodes_out, int32_t max_nodes,
                                        int32_t *num_nodes, int64_t *nb) {
    if (!x || !num_nodes) return fail(OOB_E_INVALID, "oob_exec_pipeline: NULL argument");
    if (i < 0 || i >= (int32_t)x->pipes.size()) return fail(OOB_E_INVALID, "oob_exec_pipeline: index out of range");
    const auto &nodes = x->pipes[i];
    *num_nodes = (int32_t)nodes.size();
    if (nodes_out) {
        if (max_nodes < (int32_t)nodes.size()) return fail(OOB_E_NOMEM, "oob_exec_pipeline: nodes_out too small");
        std::copy(nodes.begin(), nodes.end(), nodes_out);
    }
    if (nb) *nb = x->nb[i];
    return OOB_OK;
}

extern "C" oob_status oob_exec_fail(oob_exec *x, const int32_t *failed, int32_t num_failed,
                                    int64_t *recommended_batch_out) {
    if (!x || (!failed && num_failed > 0) || num_failed < 0) return fail(OOB_E_INVALID, "oob_exec_fail: bad argument");
    std::set<int32_t> fset(failed, failed + num_failed);
    std::set<int32_t> alive;
    for (const auto &nodes : x->pipes) alive.insert(nodes.begin(), nodes.end());
    for (int32_t n : fset)
        if (!alive.count(n)) return fail(OOB_E_INVALID, "oob_exec_fail: unknown or already failed node " + std::to_string(n));
    const auto before = owned(*x);
    const int64_t survivors = (int64_t)alive.size() - (int64_t)fset.size();
    x->actions.clear();
    x->transfers.clear();
    if (survivors < (int64_t)(x->f + 1) * x->n_lo)                    // R25: checkpoint and exit
        return fail(OOB_E_INFEASIBLE, "fewer than (f+1) n0 nodes survive: cannot keep f+1 replicas (checkpoint and exit)");
    std::vector<std::vector<int32_t>> pipes;
    std::vector<int> affected;
    for (size_t i = 0; i < x->pipes.size(); ++i) {
        std::vector<int32_t> keep;
        for (int32_t n : x->pipes[i])
            if (!fset.count(n)) keep.push_back(n);
        if (keep.size() != x->pipes[i].size()) affected.push_back((int)i);
        pipes.push_back(std::move(keep));
    }
    std::vector<char> live(pipes.size(), 1);
    std::vector<oob_action> acts;
    std::stable_sort(affected.begin(), affected.end(), [&](int a, int b) {   // R21
        return pipes[a].size() != pipes[b].size() ? pipes[a].size() < pipes[b].size() : a < b;
    });
    const int n0 = x->n_lo;
    for (int i : affected) {
        if (!live[i]) continue;
        if (pipes[i].empty()) {
            live[i] = 0;
            acts.push_back(act(OOB_ACT_REMOVE, i, -1, 0));
            continue;
        }
        if ((int)pipes[i].size() >= x->n_lo && (int)pipes[i].size() <= x->n_hi) {   // R22
            acts.push_back(act(OOB_ACT_REINSTANTIATE, i, -1, (int32_t)pipes[i].size()));
            continue;
        }
        while ((int)pipes[i].size() < n0) {                                         // R23
            int j = -1;
            for (size_t k = 0; k < pipes.size(); ++k)
                if (live[k] && (int)k != i && (int)pipes[k].size() > n0 &&
                    (j < 0 || pipes[k].size() > pipes[j].size()))
                    j = (int)k;
            if (j < 0) break;
            pipes[i].push_back(pipes[j].back());
            pipes[j].pop_back();
            acts.push_back(act(OOB_ACT_BORROW, j, i, 0));
        }
        while ((int)pipes[i].size() < n0) {                                         // R24
            int j = -1;
            for (size_t k = 0; k < pipes.size(); ++k)
                if (live[k] && (int)k != i && (j < 0 || pipes[k].size() < pipes[j].size())) j = (int)k;
            if (j < 0) return fail(OOB_E_INFEASIBLE, "no pipeline to merge with");
            pipes[i].insert(pipes[i].end(), pipes[j].begin(), pipes[j].end());
            live[j] = 0;
            acts.push_back(act(OOB_ACT_MERGE, i, j, 0));
        }
        if ((int)pipes[i].size() > x->n_hi)
            return fail(OOB_E_INFEASIBLE, "merged pipeline of " + std::to_string(pipes[i].size()) +
                                              " nodes exceeds the largest template (Appendix B premise: n_hi >= 2 n0 - 1)");
        acts.push_back(act(OOB_ACT_REINSTANTIATE, i, -1, (int32_t)pipes[i].size()));
    }
    std::vector<std::vector<int32_t>> next;
    for (size_t i = 0; i < pipes.size(); ++i)
        if (live[i]) next.push_back(pipes[i]);
    if ((int)next.size() < x->f + 1) {                                              // R28: instantiate afresh
        std::vector<int32_t> nodes;
        for (const auto &p : next) nodes.insert(nodes.end(), p.begin(), p.end());
        std::sort(nodes.begin(), nodes.end());
        const int p = x->n_hi - x->n_lo + 1;
        std::vector<int32_t> counts(p, 0);
        std::vector<int64_t> nbv(nodes.size() + 1);
        int32_t npipes = 0;
        double thr = 0, it = 0;
        int64_t nfeas = 0, rec = 0;
        oob_status st = oob_instantiate(x->set, x->profile, (int32_t)nodes.size(), x->f, x->B, x->b,
                                        x->max_enumerated, counts.data(), nbv.data(), (int32_t)nbv.size(), &npipes,
                                        &thr, &it, &nfeas, &rec);
        if (st != OOB_OK && st != OOB_E_TOO_MANY) return st;
        next.clear();
        size_t pos = 0;
        for (int i = 0; i < p; ++i)
            for (int c = 0; c < counts[i]; ++c) {
                next.emplace_back(nodes.begin() + pos, nodes.begin() + pos + x->n_lo + i);
                pos += x->n_lo + i;
            }
        acts.push_back(act(OOB_ACT_REPLAN, (int32_t)next.size(), -1, 0));
    }
    std::vector<std::vector<int32_t>> prev;
    prev.swap(x->pipes);
    x->pipes = next;
    // copy plan (reading R27)
    const auto after = owned(*x);
    std::map<int32_t, int64_t> sent;
    std::vector<oob_transfer> tr;
    for (const auto &kv : after) {
        const int32_t node = kv.first;
        const auto bi = before.find(node);
        for (int32_t layer : kv.second) {
            if (bi != before.end() && !fset.count(node) && bi->second.count(layer)) continue;
            int32_t donor = -1;
            for (const auto &ow : before) {
                if (fset.count(ow.first) || !ow.second.count(layer)) continue;
                if (donor < 0 || sent[ow.first] < sent[donor]) donor = ow.first;
            }
            if (donor < 0) {       // the state is left as it was
                x->pipes.swap(prev);
                return fail(OOB_E_INFEASIBLE, "layer " + std::to_string(layer) +
                                                  " has no surviving copy: unrecoverable (PAPER P:257-263)");
            }
            sent[donor]++;
            oob_transfer t;
            t.layer = layer; t.donor = donor; t.receiver = node; t.reserved = 0;
            t.bytes = x->layer_bytes[layer];
            tr.push_back(t);
        }
    }
    x->actions = acts;
    x->transfers = tr;
    int64_t rec = 0;
    oob_status st = redistribute(*x, &rec);                                          // R26
    if (recommended_batch_out) *recommended_batch_out = rec;
    return st;
}

extern "C" int32_t oob_exec_num_actions(const oob_exec *x) { return x ? (int32_t)x->actions.size() : 0; }
extern "C" oob_status oob_exec_action(const oob_exec *x, int32_t i, oob_action *out) {
    if (!x || !out || i < 0 || i >= (int32_t)x->actions.size()) return fail(OOB_E_INVALID, "oob_exec_action: bad argument");
    *out = x->actions[i];
    return OOB_OK;
}
extern "C" int32_t oob_exec_num_transfers(const oob_exec *x) { return x ? (int32_t)x->transfers.size() : 0; }
extern "C" oob_status oob_exec_transfer(const oob_exec *x, int32_t i, oob_transfer *out) {
    if (!x || !out || i < 0 || i >= (int32_t)x->transfers.size())
        return fail(OOB_E_INVALID, "oob_exec_transfer: bad argument");
    *out = x->transfers[i];
    return OOB_OK;
}

extern "C" oob_status oob_exec_sync_group(const oob_exec *x, int32_t layer, int32_t *pipelines_out,
                                          int32_t *stages_out, int32_t max_entries, int32_t *count) {
    if (!x || !count) return fail(OOB_E_INVALID, "oob_exec_sync_group: NULL argument");
    if (layer < 0 || layer >= x->L) return fail(OOB_E_INVALID, "oob_exec_sync_group: layer out of range");
    int32_t n = 0;
    for (size_t p = 0; p < x->pipes.size(); ++p) {
        const auto &st = x->stages[x->pipes[p].size() - x->n_lo];
        for (size_t s = 0; s < st.size(); ++s)
            if (st[s].layer_begin <= layer && layer < st[s].layer_end) {
                if (n < max_entries) {
                    if (pipelines_out) pipelines_out[n] = (int32_t)p;
                    if (stages_out) stages_out[n] = (int32_t)s;
                }
                ++n;
            }
    }
    *count = n;
    return n <= max_entries ? OOB_OK : fail(OOB_E_NOMEM, "oob_exec_sync_group: output too small");
}
