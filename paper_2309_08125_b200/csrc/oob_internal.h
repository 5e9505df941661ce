// Internal declarations shared by the host planner (C++) and the CUDA DP engine.
// Nothing here is part of the C ABI (include/oobleck_plan.h is).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "oobleck_plan.h"

namespace oob {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string &msg);
oob_status fail(oob_status s, const std::string &msg);

inline size_t align_up_host(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- DP index geometry
// Cell universe and HBM layout:
//  allocation index a:  0..M-2 -> I(a+1) (GPUs inside one node), M-1+q-1 -> W(q) (whole
//  nodes).  lo(a) = q for W(q) else 1; gpus(a) = q*M for W(q) else r.
//  A cell (S', u, v, a) exists iff lo(a) <= S' <= hi(a, v-u) = min(v-u, gpus(a)) and
//  a is in A(l): all I(r), and W(q) for q <= Q_l (Q_L = n_hi, else max(1, n_hi-1)).
//  Cells of one wavefront l = v-u are laid out per range start u (a "slab" of cells(l)
//  cells), inside a slab by allocation then S'.  Global cell index
//     base[l] + u*cells[l] + off[l*A + a] + (S' - lo(a)).
// Cells of padding after each wavefront's cells: no 32-byte sector of the cell, shadow or
// argmin table holds cells of two wavefronts, and a streamed row's read-ahead (<= 96 cells)
// never reaches the next wavefront (pipelined waves may still be producing it).
constexpr int64_t WAVE_PAD = 128;

struct Geometry {
    int L = 0, M = 0, n_lo = 0, n_hi = 0, A = 0;
    std::vector<int32_t> Q;          // [L+1]
    std::vector<int32_t> cells;      // [L+1] cells per slab of length l
    std::vector<int64_t> base;       // [L+2] first cell of wavefront l
    std::vector<int32_t> off;        // [(L+1)*A] offset of alloc a in a slab of length l, -1 if empty
    std::vector<int64_t> wave_splits;   // [L+1] feasible splits of wavefront l (all u)
    std::vector<int64_t> wave_cells;    // [L+1] cells of wavefront l (all u)
    int64_t total_cells = 0;         // cells of the table universe (reported)
    int64_t table_cells = 0;         // per-profile table stride: the waves plus WAVE_PAD cells after each
    int64_t total_splits = 0;

    bool is_whole(int a) const { return a >= M - 1; }
    int alloc_n(int a) const { return is_whole(a) ? a - (M - 1) + 1 : a + 1; }
    int lo(int a) const { return is_whole(a) ? alloc_n(a) : 1; }
    int gpus(int a) const { return is_whole(a) ? alloc_n(a) * M : alloc_n(a); }
    int hi(int a, int l) const { int g = gpus(a); return l < g ? l : g; }
    int idx_I(int r) const { return r - 1; }
    int idx_W(int q) const { return (M - 1) + q - 1; }
};

// Builds the geometry; returns false (and sets the error) on bad arguments.
bool build_geometry(int L, int M, int n_lo, int n_hi, Geometry &g);

// ncclAllGather of `bytes` per rank (oob_dist.cpp)
oob_status nccl_allgather_bytes(void *comm, const void *send, void *recv, size_t bytes, size_t recv_cap,
                                int world, void *stream);

// ---------------------------------------------------------------- packed templates
// Device output record, see oob_dp_run in oobleck_plan.h.
struct PackedHeader {
    int32_t nodes, S, kstar, status;
    double T1, T2, T3, tstar, iter;
    double pad;
};
static_assert(sizeof(PackedHeader) == 64, "packed header is 64 bytes");

inline size_t packed_template_bytes(int L) {
    size_t b = sizeof(PackedHeader) + (size_t)L * 5 * sizeof(int32_t);
    return (b + 63) / 64 * 64;
}

}  // namespace oob

// Opaque handle definitions (C ABI types).
struct oob_profile {
    int32_t L = 0, M = 0;
    int32_t microbatch_reference = 1;
    std::vector<double> fwd, bwd;        // [L][M]
    std::vector<int64_t> state_bytes;    // [L]
    std::vector<int64_t> act_bytes;      // [L]
};

struct oob_template_set {
    int32_t L = 0, M = 0, n_lo = 0, n_hi = 0, num_profiles = 0;
    std::vector<oob_template> templates;   // [num_profiles * p]
    std::vector<oob_stage> stages;         // [num_profiles * p * L]
};
