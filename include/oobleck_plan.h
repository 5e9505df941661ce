/*
 * oobleck_plan.h — C ABI of the B200-native Oobleck pipeline-template planner.
 *
 * The library (paper_2309_08125_b200/liboobleck_plan.so) implements the planning path of
 * Oobleck (arXiv 2309.08125, §4): pipeline-template generation — the memoized
 * divide-and-conquer GPU-stage mapping of §4.1.2 (Eqs.1-4) run for every
 * template node count of the node specification (§4.1.1) — as sm_100a CUDA
 * kernels, plus the host-side instantiation (Eq.5, §4.2.1) and batch
 * distribution (Eq.6, §4.2.2) that consume the template set.
 *
 * Conventions
 *  - Every function returns an oob_status (OOB_OK = 0) unless stated; on failure a
 *    human-readable message is available from oob_last_error() (thread-local, valid until
 *    the next call on the same thread).  No C++ exception crosses this boundary.
 *  - "host" pointers are ordinary CPU memory; "device" pointers are CUDA global memory on
 *    the current device (e.g. torch tensors' data_ptr()).  Streams are cudaStream_t passed
 *    as void* (NULL = legacy default stream).
 *  - Opaque handles (oob_profile, oob_template_set, oob_dp_plan) are created and freed by
 *    the library.  Profiles and template sets are immutable after creation and may be
 *    shared read-only across threads.  An oob_dp_plan must not be used concurrently.
 *  - Per-layer costs are milliseconds, binary64, row-major [L][M]: element [l*M + d-1] is
 *    the cost of layer l on d GPUs of one node (F_{l,d} and B_{l,d}).
 *  - Arithmetic contract: all DP arithmetic is IEEE binary64, round-to-nearest, without
 *    FMA contraction, in the operation order stated in DESIGN.md; results are bit-identical
 *    to oracle/ (tests/).
 */
#ifndef OOBLECK_PLAN_H
#define OOBLECK_PLAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OOB_OK = 0,
    OOB_E_PARSE = 1,       /* malformed profile JSON */
    OOB_E_INVALID = 2,     /* bad argument: empty model, non-positive time, missing d, L>1023 */
    OOB_E_INFEASIBLE = 3,  /* N < (f+1) n0; n0 > L */
    OOB_E_BATCH = 4,       /* B % b != 0 or B/b < pipelines; see recommended */
    OOB_E_TOO_MANY = 5,    /* Eq.5 enumeration exceeded max_enumerated (plan is best-so-far) */
    OOB_E_CUDA = 6,        /* CUDA runtime/launch failure */
    OOB_E_NCCL = 7,        /* collective failure (oob_nccl_*, oob_dp_run with a communicator) */
    OOB_E_NOMEM = 8        /* host allocation or workspace too small */
} oob_status;

typedef struct oob_profile oob_profile;
typedef struct oob_template_set oob_template_set;
typedef struct oob_dp_plan oob_dp_plan;

/* One pipeline stage of a template: layers [layer_begin, layer_end) on
 * `gpus` GPUs of node `node` (0..n-1, template-local), starting at GPU `gpu_offset`. */
typedef struct {
    int32_t layer_begin, layer_end, gpus, node, gpu_offset;
} oob_stage;

/* A pipeline template.  T1/T2/T3 per Eqs.1-3 at N_b = 4S,
 * kstar = 0-based index of the slowest stage, tstar_ms its F+B, iter_ms = (T1+T2)+T3.
 * `stages` borrows from the owning oob_template_set. */
typedef struct {
    int32_t nodes, num_stages, kstar, reserved;
    double t1_ms, t2_ms, t3_ms, tstar_ms, iter_ms;
    const oob_stage *stages;
} oob_template;

/* Options of oob_generate_templates. */
typedef struct {
    int32_t nodes;              /* N: initial node count */
    int32_t gpus_per_node;      /* M; must equal every profile's M */
    int32_t f;                  /* fault-tolerance threshold */
    int32_t n0;                 /* smallest template; <= 0: derive with oob_min_nodes */
    int64_t gpu_mem_bytes;      /* used only when n0 <= 0 */
    double util;                /* usable memory fraction when n0 <= 0 (0: default 0.8) */
    int32_t samples_per_gpu;    /* activation multiplier when n0 <= 0 (0: default 1) */
    int32_t device;             /* CUDA device ordinal (< 0: current device) */
    void *stream;               /* cudaStream_t for all device work (NULL: default) */
    void *workspace;            /* optional caller-owned device memory (NULL: library
                                   allocates and frees it inside the call) */
    size_t workspace_bytes;     /* size of `workspace` (>= oob_dp_plan_info.workspace_bytes) */
    void *comm;                 /* optional ncclComm_t of `world` ranks (oob_nccl_comm_create),
                                   borrowed; NULL or world <= 1: this GPU only */
    int32_t world, rank;        /* ranks of `comm` and this process's rank */
    int32_t tp_pow2;            /* stage mask: GPU counts per stage powers of two (R31) */
    double stage_mem_bytes;     /* > 0: stage mask sum_l (state_bytes_l + samples_per_gpu *
                                   act_bytes_l) / d <= stage_mem_bytes (R31); 0: none */
    int32_t exact;              /* 1: return the EXACT optimum of the 1F1B objective per template
                                   (oob_exact_run, bounded by the recursion's own templates);
                                   0: the paper's recursion (default).  Not with stage masks. */
} oob_plan_opts;

/* ------------------------------------------------------------------ errors */
const char *oob_last_error(void);
const char *oob_status_string(oob_status s);

/* ------------------------------------------------------------------ profiles */
/* Parse the profile JSON of SPEC S:99:
 *  {"gpus_per_node": M, "microbatch_reference": b, "layers": [{"name": s, "state_bytes": i,
 *   "activation_bytes_per_sample": i, "fwd_ms": {"1": f, ..., "M": f}, "bwd_ms": {...}}]}
 * Errors: OOB_E_PARSE (syntax), OOB_E_INVALID (no layers, missing d entry, time <= 0). */
oob_status oob_load_profile(const char *json_path, oob_profile **out);

/* Profile from host arrays fwd_ms/bwd_ms [L][M] (copied); state_bytes [L] may be NULL.
 * Errors: OOB_E_INVALID (L < 1, L > 1023, M < 1, M > 64, non-finite or non-positive time). */
oob_status oob_profile_from_arrays(int32_t L, int32_t M, const double *fwd_ms,
                                   const double *bwd_ms, const int64_t *state_bytes,
                                   oob_profile **out);
void oob_profile_free(oob_profile *p);
int32_t oob_profile_layers(const oob_profile *p);
int32_t oob_profile_gpus_per_node(const oob_profile *p);
/* Copy the profile's costs into caller-owned host arrays fwd_ms/bwd_ms [L][M] (either may be
 * NULL) and state_bytes [L] (may be NULL).  Errors: OOB_E_INVALID. */
oob_status oob_profile_costs(const oob_profile *p, double *fwd_ms, double *bwd_ms, int64_t *state_bytes);

/* SPEC min_nodes (P:335 gives no formula; DESIGN reading R5):
 * n0 = ceil((sum state_bytes + samples_per_gpu * sum act_bytes) / (M * gpu_mem * util)).
 * Errors: OOB_E_INFEASIBLE when the model does not fit on `nodes` nodes. */
oob_status oob_min_nodes(const oob_profile *p, int32_t nodes, int64_t gpu_mem_bytes,
                         double util, int32_t samples_per_gpu, int32_t *n0_out);

/* Node specification: sizes n0 .. min(N - f n0, L) (reading R4).
 * Writes n_lo/n_hi.  Errors: OOB_E_INFEASIBLE if N < (f+1) n0 or n0 > L. */
oob_status oob_node_sizes(int32_t nodes, int32_t f, int32_t n0, int32_t layers,
                          int32_t *n_lo, int32_t *n_hi);

/* ------------------------------------------------------------------ template generation
 * For every profile and every size n in the node specification, one template: the
 * argmin over S in n..min(L, nM) of the memoized recursion T(S, 0, L, W(n))
 * (Eqs.1-4).  Runs on the GPU (sm_100a): host arrays are copied to the device, the DP
 * wavefronts run, the packed templates are copied back.  `profiles` are num_profiles
 * handles with identical L and M (batched sweep).
 * Multi-GPU (opts.comm with world > 1; every rank calls with the same profiles and options
 * on its own device, and every rank receives the whole template set, bit-identical to one
 * GPU): num_profiles == 1 splits each large wavefront's W-cell work across the ranks (one
 * all-gather of partial argmins per such wavefront, see oob_dp_set_comm); num_profiles > 1
 * gives rank r the contiguous block of profiles [r*B + min(r, E), ...) (B = num/world,
 * E = num%world, the first E ranks one extra), planned independently, then one
 * ncclAllGather of the packed blocks.  Errors: OOB_E_INVALID, OOB_E_INFEASIBLE,
 * OOB_E_CUDA, OOB_E_NCCL, OOB_E_NOMEM. */
oob_status oob_generate_templates(const oob_profile *const *profiles, int32_t num_profiles,
                                  const oob_plan_opts *opts, oob_template_set **out);
int32_t oob_template_set_profiles(const oob_template_set *s);
int32_t oob_template_count(const oob_template_set *s, int32_t profile);
/* Fills *view for template i (size n = n_lo + i) of `profile`; view->stages borrows. */
oob_status oob_template_get(const oob_template_set *s, int32_t profile, int32_t i,
                            oob_template *view);
void oob_template_set_free(oob_template_set *s);

/* ------------------------------------------------------------------ device-resident DP
 * The same computation on inputs already in device memory (the hot path timed by
 * bench.py).  A plan holds the index geometry for (L, M, n_lo, n_hi, num_profiles).
 *   d_fwd, d_bwd: device float64 [num_profiles][L][M]
 *   d_workspace : device memory of >= info.workspace_bytes (caller-owned, e.g. torch)
 *   d_packed    : device memory of >= info.packed_bytes receiving the packed templates:
 *     per profile p, template i: a 64-byte header
 *       {int32 nodes, S, kstar, status; double T1, T2, T3, tstar, iter}
 *     followed by L records {int32 layer_begin, layer_end, gpus, node, gpu_offset};
 *     stride info.packed_template_bytes, profile stride info.packed_profile_bytes.
 * Kernels are enqueued on `stream`; the call returns without synchronizing.  The W-cell
 * kernel screens splits with a binary32 round-down lower bound and re-evaluates every
 * candidate in binary64 (never drops a winner or a tie).  For a single
 * profile the wavefront kernels are programmatic dependent launches that synchronise
 * through counters in the workspace (they may overlap each other, never the caller's
 * other work on `stream`: the last kernel, the template extraction, waits for all of
 * them); the workspace must not be shared by concurrent runs.  Its contents need not
 * persist between runs: every run re-initialises the accumulators and counters it uses,
 * and the plan's read-only index geometry lives in plan-owned device memory (allocated and
 * uploaded on the first run on each device, freed by oob_dp_plan_free).  A plan is sized
 * for the SM count of the device current at oob_dp_plan_create; running it on a device
 * with another SM count returns OOB_E_INVALID.  A timed-out pipeline wait (a GPU shared
 * with other work) marks the packed templates (status 2): oob_template_set_from_packed
 * then returns OOB_E_CUDA.  Diagnostic environment switches read at oob_dp_plan_create
 * (OOB_DP_PIPE=0, OOB_DP_FUSE=0, OOB_DP_KERNEL=v1, ...) select equivalent variants with
 * identical results; the effective ones are reported in oob_dp_info. */
typedef struct {
    int32_t L, M, n_lo, n_hi, num_profiles, wavefronts;
    int64_t cells_per_profile;      /* DP cells in the table universe */
    int64_t splits_per_profile;     /* feasible split evaluations (the roofline unit) */
    int64_t kernel_launches;        /* device kernels launched per oob_dp_run */
    size_t workspace_bytes;
    size_t packed_template_bytes, packed_profile_bytes, packed_bytes;
    /* effective plan switches (identical results in every combination) */
    int32_t kernel;                 /* 2 = tiled W-cell kernel, 1 = thread-per-cell fallback */
    int32_t pipelined;              /* wavefronts as programmatic dependent launches */
    int32_t fused;                  /* finalize + next wave's in-node cells inside k_wave_w */
    int32_t seeded;                 /* wavefronts whose accumulators start from seed splits */
    int32_t chunk_max, refresh, small_pairs;
    int32_t num_sms;                /* SMs of the device the plan was built for */
    int32_t world;                  /* ranks sharing the wavefronts (oob_dp_set_comm) */
    int32_t warp_waves;             /* batched wavefronts run one warp per (profile, range) */
    int32_t small_range;            /* wavefronts whose in-node cells run one warp per (profile, range) */
    int32_t exchange;               /* sharded plans: 1 = partials exchanged inside k_wave_w over
                                       NVLink peer memory, 2 = ncclAllGather + k_fin per wave,
                                       3 = virtual shards (device copies); 0 = not sharded */
} oob_dp_info;

oob_status oob_dp_plan_create(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi,
                              int32_t num_profiles, oob_dp_plan **out);
void oob_dp_plan_free(oob_dp_plan *plan);
oob_status oob_dp_plan_info(const oob_dp_plan *plan, oob_dp_info *out);
oob_status oob_dp_run(oob_dp_plan *plan, const double *d_fwd, const double *d_bwd,
                      void *d_workspace, size_t workspace_bytes, void *d_packed, void *stream);
/* Stage masks (variants the paper is silent on, DESIGN reading R31): a
 * stage of layers [u, v) on d GPUs of one node is allowed only if d is a power of two
 * (pow2_tp != 0) and, when d_stage_bytes (device float64 [num_profiles][L], borrowed until
 * the plan's runs complete) is non-NULL, sum_{l=u}^{v-1} stage_bytes[l] / d <= mem_cap_bytes.
 * A disallowed stage is infinite like one spanning nodes; a size with no allowed
 * mapping gives an infeasible template (num_stages = 0, costs +inf; packed status 3).
 * pow2_tp = 0 with d_stage_bytes = NULL: no masks (the paper's method).  Errors: OOB_E_INVALID. */
oob_status oob_dp_set_stage_masks(oob_dp_plan *plan, int32_t pow2_tp, const double *d_stage_bytes,
                                  double mem_cap_bytes);
/* Optional CUDA-event timing of the wavefront kernel (the dominant kernel): when enabled,
 * oob_dp_run records events around each wavefront launch on `stream`; oob_dp_kernel_time
 * returns the summed elapsed ms and number of launches since the last reset (it
 * synchronizes on the recorded events). */
oob_status oob_dp_set_timing(oob_dp_plan *plan, int32_t enable);
oob_status oob_dp_kernel_time(oob_dp_plan *plan, double *ms_out, int64_t *launches_out,
                              int32_t reset);
/* ------------------------------------------------------------------ multi-GPU (one profile)
 * Single-profile sharding across `world` GPUs of one box: every rank calls
 * oob_dp_run on the same profile with the same plan geometry; the W-cell splits of every
 * large wavefront are divided across ranks (rank r takes units r, r+world, ... of each
 * range's unit queue) and the per-rank partial argmins (16 bytes per output) are exchanged
 * so every rank finalizes the whole wavefront with the same lexicographic minimum: every
 * rank ends with the same table and packed templates (bit-identical to world = 1).
 *   oob_nccl_unique_id : rank 0 creates the id (OOB_NCCL_ID_BYTES bytes), the caller
 *                        broadcasts it (e.g. torch.distributed);
 *   oob_nccl_comm_create: every rank, on its CUDA device (`device` < 0: current);
 *   oob_dp_set_comm    : attach the communicator to a plan (comm = NULL, world = 1: detach);
 *                        the plan's workspace grows by world x (largest wavefront partial):
 *                        re-read oob_dp_plan_info afterwards.  The communicator is borrowed.
 *                        Collective (every rank, same order).  By default the partial
 *                        argmins are exchanged INSIDE the wavefront kernel through NVLink
 *                        peer memory: the call allocates a plan-owned exchange buffer and
 *                        maps every rank's (cudaIpc handles all-gathered over `comm`), the
 *                        wavefronts stay pipelined, and every rank must then run the plan the
 *                        same number of times (the peer counters are per run; a rank that
 *                        skips a run makes the others' waits time out -> OOB_E_CUDA).
 *                        OOB_DP_SHARDX=nccl selects one ncclAllGather + finalize launch per
 *                        sharded wavefront instead.
 * Errors: OOB_E_INVALID, OOB_E_NCCL, OOB_E_CUDA. */
#define OOB_NCCL_ID_BYTES 128
oob_status oob_nccl_unique_id(void *id_out);
oob_status oob_nccl_comm_create(const void *id, int32_t world, int32_t rank, int32_t device, void **comm_out);
void oob_nccl_comm_destroy(void *comm);
oob_status oob_dp_set_comm(oob_dp_plan *plan, void *comm, int32_t world, int32_t rank);
/* ncclAllGather of `bytes_per_rank` bytes per rank: d_recv[r * bytes_per_rank ...] receives
 * rank r's d_send (device buffers, enqueued on `stream`).  Used to assemble packed
 * template sets of batched sweeps.  Errors: OOB_E_INVALID, OOB_E_NCCL. */
oob_status oob_nccl_allgather(void *comm, const void *d_send, void *d_recv, size_t bytes_per_rank,
                              void *stream);
/* Virtual shards (test mode of the single-profile sharding on ONE GPU):
 * oob_dp_set_virtual_shards(plan, world) makes the plan split each large wavefront's units
 * across `world` virtual ranks exactly as oob_dp_set_comm does; oob_dp_run_virtual then
 * runs every virtual rank on the current device — per wavefront each rank's k_wave_w over
 * its own workspace d_ws[r] (>= info.workspace_bytes after the call; re-read it), then
 * device copies in place of the all-gather, then each rank's finalize — and writes rank r's
 * packed templates to d_packed[r].  Every rank's output must equal a 1-GPU run.  world = 1
 * restores a plain plan.  Errors: OOB_E_INVALID, OOB_E_NOMEM, OOB_E_CUDA. */
oob_status oob_dp_set_virtual_shards(oob_dp_plan *plan, int32_t world);
oob_status oob_dp_run_virtual(oob_dp_plan *plan, const double *d_fwd, const double *d_bwd,
                              void *const *d_workspace, size_t workspace_bytes,
                              void *const *d_packed, void *stream);

/* ------------------------------------------------------------------ exact optimum
 * The paper's recursion (Eqs.1-4) keeps one argmin per memo cell of the
 * sub-problem's own objective, which is a heuristic for the parent: it can
 * miss the minimum of the closed form T1 + (3S - 1 + k*) t* + T3 (P:381-386, P:424-429,
 * N_b = 4S) over all mappings.  oob_exact_run returns that minimum for every template size
 * n_lo..n_hi: for each distinct stage time tau (the bottleneck t*), the stages before the
 * first bottleneck cost t + 4 tau each and those after it 2t + 3 tau, two shortest paths over
 * (layer boundary, GPUs) solved on the device; the best over tau and bottleneck placements
 * is the optimum (derivation in csrc/oob_exact.cu).  Ties: smallest total,
 * then smallest tau, then the first (layer, GPU) placement; stage costs summed left to
 * right (reading R12).  No stage masks.
 *   d_fwd, d_bwd   : device float64 [num_profiles][L][M] (as oob_dp_run)
 *   d_packed_ub    : device packed templates of the same shape (oob_dp_run's output) whose
 *                    totals bound the search (only tau <= iter / (3n + 1) can win), or NULL
 *                    for an unbounded search (every stage time; slower)
 *   d_workspace    : >= oob_exact_workspace_bytes (same shape, current device); its first 8
 *                    bytes receive the number of (profile, tau) tasks solved (uint64)
 *   d_packed_out   : packed templates in oob_dp_run's layout (status 0; 3 = no mapping; 4 =
 *                    an internal list overflowed: every template of the run is marked and
 *                    oob_template_set_from_packed fails with OOB_E_CUDA); may be d_packed_ub
 *                    (each bound is read before any output is written)
 * Enqueued on `stream`, no synchronisation.  Errors: OOB_E_INVALID (shape: 1 <= n_lo <=
 * n_hi <= L <= 1023, M <= 64, n_hi * M <= ~21,000), OOB_E_NOMEM (workspace), OOB_E_CUDA. */
oob_status oob_exact_workspace_bytes(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi,
                                     int32_t num_profiles, size_t *bytes);
oob_status oob_exact_run(int32_t L, int32_t M, int32_t n_lo, int32_t n_hi, int32_t num_profiles,
                         const double *d_fwd, const double *d_bwd, const void *d_packed_ub,
                         void *d_workspace, size_t workspace_bytes, void *d_packed_out,
                         void *stream);

/* Build a template set from a HOST copy of the packed output (d_packed copied back). */
oob_status oob_template_set_from_packed(const void *h_packed, const oob_dp_info *info,
                                        oob_template_set **out);

/* ------------------------------------------------------------------ instantiation (Eq.5)
 * Best plan for `nodes` available nodes: enumerate every X with
 * sum x_i n_i = N' and sum x_i >= f+1 (Eq.5), distribute the batch for each (Eq.6), and
 * keep the highest throughput B / max_i iteration_ms(N_b,i) (iteration_ms = T1 +
 * max(0, N_b - S + k* - 1) t* + T3, reading R30); Eq.6 ties (equal T_i): the
 * minimizer with the smallest iteration time (R29); ties: fewer pipelines, then lexicographically
 * smallest counts.
 *  counts_out   : caller-owned int32 [oob_template_count] — x_i per template
 *  nb_out       : caller-owned int64 [max_pipelines] — N_b per pipeline, pipelines ordered
 *                 by template index; *num_pipelines_out receives sum x_i
 *  throughput_out, iter_ms_out: of the chosen plan (samples per ms, ms)
 *  num_feasible_out: number of feasible X (saturates at INT64_MAX)
 * max_enumerated <= 0 means 1e6.  Errors: OOB_E_INFEASIBLE (N' < (f+1) n0 or no X),
 * OOB_E_BATCH (no X can be distributed; *recommended_batch_out is set), OOB_E_TOO_MANY
 * (more than max_enumerated X, e.g. 2.2e19 at 512 nodes: not enumerated; the outputs hold
 * the best, scored exactly as above, of the knapsack candidates — for each fill/drain
 * overhead threshold, the X of maximum total microbatch rate sum x_i / t*_i among the
 * templates under it — a heuristic, reading R20), OOB_E_NOMEM (max_pipelines too small). */
oob_status oob_instantiate(const oob_template_set *set, int32_t profile, int32_t nodes,
                           int32_t f, int64_t global_batch, int32_t microbatch,
                           int64_t max_enumerated, int32_t *counts_out, int64_t *nb_out,
                           int32_t max_pipelines, int32_t *num_pipelines_out,
                           double *throughput_out, double *iter_ms_out,
                           int64_t *num_feasible_out, int64_t *recommended_batch_out);

/* Plans for every node count N' = n_min .. n_max in one call (the instantiation for any
 * number of surviving nodes).  Per N' (index k = N' - n_min): counts_out
 * [k * template_count + i] = x_i of the chosen plan, throughput_out[k] (samples per ms),
 * upper_bound_out[k] = a CERTIFIED upper bound of the best throughput of any plan on N'
 * nodes (equal to throughput_out when exact_out[k] = 1: Eq.5 enumerated exhaustively,
 * <= max_enumerated sets), status_out[k] = OOB_OK, OOB_E_INFEASIBLE (N' < (f+1) n0 or no
 * set) or OOB_E_BATCH (B not distributable).  Above max_enumerated the knapsack candidates
 * of every N' (one set of DPs over 0..n_max) are scored exactly in decreasing order of their
 * own relaxation bound until none can beat the best; the bound of N' is
 * B / min_j max(T1_j + T3_j, a_j + K t*_j n_j / N') with a_j = T1 + T3 - (S - k* + 1) t*
 * (DESIGN.md §8).  Caller-owned outputs of (n_max - n_min + 1) entries.  Errors:
 * OOB_E_INVALID. */
oob_status oob_instantiate_all(const oob_template_set *set, int32_t profile, int32_t n_min,
                               int32_t n_max, int32_t f, int64_t global_batch, int32_t microbatch,
                               int64_t max_enumerated, int32_t *counts_out, double *throughput_out,
                               double *upper_bound_out, int32_t *exact_out, int32_t *status_out);

/* Number of X satisfying Eq.5's Requirements 1-2 for sizes n_lo..n_hi (saturating). */
oob_status oob_count_sets(int32_t n_lo, int32_t n_hi, int32_t nodes, int32_t f,
                          int64_t *count_out);

/* ------------------------------------------------------------------ batch distribution (Eq.6)
 * Exact integer minimiser of sum_i (N_b,i T_i - mean)^2 s.t. sum_i N_b,i b = B,
 * N_b,i >= 1 (reading R18), T_i = per-microbatch time of pipeline i (reading
 * R19: the slowest stage's F+B).  per_microbatch_ms: host [x]; nb_out: caller-owned
 * int64 [x]; objective_out may be NULL.  Errors: OOB_E_INVALID (x < 1, b < 1, T_i <= 0),
 * OOB_E_BATCH (B % b != 0 or B/b < x; *recommended_batch_out = smallest distributable
 * B' >= B, P:549-551 / SPEC S:247-255). */
oob_status oob_distribute_batch(const double *per_microbatch_ms, int32_t x,
                                int64_t global_batch, int32_t microbatch, int64_t *nb_out,
                                double *objective_out, int64_t *recommended_batch_out);
int64_t oob_recommend_batch(int32_t x, int32_t microbatch, int64_t global_batch);

/* ------------------------------------------------------------------ dynamic reconfiguration
 * An execution state: pipelines instantiated from a template set, each an ordered
 * list of node ids (template stage i runs on the pipeline's node stages[i].node), with the
 * Eq.6 microbatches of every pipeline.  On node failures (oob_exec_fail) the affected
 * pipelines are repaired by the three steps of PAPER §5.1 — simple
 * reinstantiation from the template of the surviving node count; borrowing nodes from
 * pipelines that can yield (more than n0 nodes), largest first, the donor giving its last
 * node; merging with the smallest other pipeline (Appendix B guarantees a template of the
 * merged size) — processed in ascending surviving size; if whole pipelines failed and fewer
 * than f+1 remain, the survivors are instantiated afresh (oob_instantiate's plan).  Then the
 * batch is redistributed (§5.2, Eq.6, global batch unchanged), the copy plan of missing
 * layers is built (every (node, layer) newly needed, from the surviving previous owner with
 * the fewest transfers so far, ties: lowest node id) and the per-layer synchronisation
 * groups of §6.1 follow from the pipelines.  Readings R21-R28.
 * The template set is borrowed and must outlive the state.  Errors of oob_exec_fail:
 * OOB_E_INVALID (unknown or already failed node), OOB_E_INFEASIBLE (fewer than (f+1) n0
 * survivors: checkpoint and exit; or a layer with no surviving copy, P:257-263;
 * or a merged size above the largest template), OOB_E_BATCH (the pipelines are rebuilt but B
 * cannot be distributed over them; *recommended_batch_out is set). */
typedef struct oob_exec oob_exec;
enum { OOB_ACT_REINSTANTIATE = 1, OOB_ACT_BORROW = 2, OOB_ACT_MERGE = 3, OOB_ACT_REMOVE = 4, OOB_ACT_REPLAN = 5 };
/* reinstantiate: pipeline a (index before the call) -> template of `nodes` nodes;
 * borrow: one node from pipeline a to pipeline b; merge: pipeline b's nodes appended to a;
 * remove: pipeline a lost every node; replan: a = new pipeline count. */
typedef struct {
    int32_t kind, a, b, nodes;
} oob_action;
typedef struct {
    int32_t layer, donor, receiver, reserved;
    int64_t bytes;                  /* layer_bytes[layer] given at creation (0 if none) */
} oob_transfer;

/* counts: caller [template_count] pipelines per template size n_lo + i; node_ids: the
 * sum(counts_i * n_i) nodes, assigned in order (template order, pipelines consecutive);
 * layer_bytes: [L] model-state bytes per layer or NULL.  Errors: OOB_E_INVALID,
 * OOB_E_INFEASIBLE (fewer than f+1 pipelines), OOB_E_BATCH. */
oob_status oob_exec_create(const oob_template_set *set, int32_t profile, int32_t f,
                           int64_t global_batch, int32_t microbatch, const int32_t *counts,
                           const int32_t *node_ids, int32_t num_nodes, const int64_t *layer_bytes,
                           oob_exec **out);
void oob_exec_free(oob_exec *state);
int32_t oob_exec_num_pipelines(const oob_exec *state);
/* nodes_out: caller [max_nodes] (may be NULL); *nb = the pipeline's microbatches. */
oob_status oob_exec_pipeline(const oob_exec *state, int32_t i, int32_t *nodes_out, int32_t max_nodes,
                             int32_t *num_nodes, int64_t *nb);
oob_status oob_exec_fail(oob_exec *state, const int32_t *failed, int32_t num_failed,
                         int64_t *recommended_batch_out);
/* actions and copy transfers of the last oob_exec_fail, in the order they were taken */
int32_t oob_exec_num_actions(const oob_exec *state);
oob_status oob_exec_action(const oob_exec *state, int32_t i, oob_action *out);
int32_t oob_exec_num_transfers(const oob_exec *state);
oob_status oob_exec_transfer(const oob_exec *state, int32_t i, oob_transfer *out);
/* Sync group of `layer` (§6.1): for every pipeline p, the stage holding the layer —
 * entries (pipelines_out[k], stages_out[k]), *count = number of pipelines. */
oob_status oob_exec_sync_group(const oob_exec *state, int32_t layer, int32_t *pipelines_out,
                               int32_t *stages_out, int32_t max_entries, int32_t *count);

#ifdef __cplusplus
}
#endif
#endif /* OOBLECK_PLAN_H */
