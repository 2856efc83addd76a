/*
 * topopt_b200 — C ABI of the B200 DC N-1 MapElites engine.
 *
 * Drop-in boundary for the reference's hot path (arxiv/paper_2605_10128,
 * /root/reference/proj). The reference exposes a C++ API only; every entry
 * point below names the reference interface it replaces (file:line) and keeps
 * its argument meaning and error behaviour. Conventions:
 *   - plain pointers and sizes, caller-owned host buffers, context-owned device
 *     memory; no C++ types and no exceptions cross this boundary;
 *   - every call returns a tg_status; tg_last_error() holds the message of the
 *     most recent failure on the calling thread; statuses mirror
 *     include/topopt/errors.hpp:9-34 (ParseError ... IoError);
 *   - calls on one context are serialized on one CUDA stream, matching
 *     run_optimizer's single-threaded use of a DcContext (qd_optimizer.cpp:344).
 * See INTEGRATION.md for the reference-side shim that binds these symbols.
 */
#ifndef TOPOPT_B200_H
#define TOPOPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tg_status {
  TG_OK = 0,
  TG_PARSE_ERROR = 1,            /* errors.hpp:9-12  ParseError */
  TG_VALIDATION_ERROR = 2,       /* errors.hpp:14-17 ValidationError */
  TG_ISLANDED_CONTINGENCY = 3,   /* errors.hpp:19-22 IslandedContingency */
  TG_SINGULAR_SYSTEM = 4,        /* errors.hpp:24-27 SingularSystem */
  TG_CONFIG_ERROR = 5,           /* errors.hpp:29-31 ConfigError */
  TG_IO_ERROR = 6,               /* errors.hpp:33-35 IoError */
  TG_CUDA_ERROR = 7,             /* device failure (no CPU fallback exists) */
  TG_CAPACITY_ERROR = 8          /* a candidate exceeded a compile-time capacity */
} tg_status;

typedef struct tg_grid tg_grid;           /* host network model (GridModel) */
typedef struct tg_actionset tg_actionset; /* host action encoding (ActionSet) */
typedef struct tg_context tg_context;     /* device-resident DcContext */

/* ---- plain-data network description (replaces const GridModel&,
 *      grid_model.hpp:80-127); arrays are read during tg_context_create only ---- */
typedef struct tg_grid_desc {
  int32_t n_nodes, n_branches, n_injections, slack;
  const int32_t* branch_from;       /* [n_branches] node index */
  const int32_t* branch_to;
  const double* branch_x;           /* series reactance, p.u. (> 0) */
  const double* branch_limit;       /* MW */
  const uint8_t* branch_in_service;
  const int32_t* injection_node;    /* [n_injections] */
  const double* injection_net_mw;   /* Injection::net_mw(), grid_model.hpp:45 */
  int32_t n_contingencies;
  const int32_t* cont_branch_ptr;   /* [n_contingencies+1] CSR */
  const int32_t* cont_branch;
  const int32_t* cont_inj_ptr;      /* [n_contingencies+1] CSR */
  const int32_t* cont_inj;
  int32_t n_substations;
  const int32_t* sub_node;          /* [n_substations] switchable node */
  const int32_t* sub_term_ptr;      /* [n_substations+1] CSR over terminals */
  const int32_t* term_kind;         /* 0 branch from-end, 1 branch to-end, 2 injection */
  const int32_t* term_element;      /* branch or injection index */
  int32_t n_busbar_outages;
  const int32_t* bo_substation;     /* [n_busbar_outages] */
  const int32_t* bo_busbar;         /* busbar index within the substation */
  const int32_t* bo_implied_ptr;    /* [n_busbar_outages+1] default implied branches, grid_model.cpp:217-227 */
  const int32_t* bo_implied;
  /* Timestep extension (not in the reference, whose GridModel has one injection
   * vector, grid_model.hpp:36-46): n_timesteps >= 1 injection profiles; the
   * evaluation runs every profile and sums lambda_o / lambda_c / lambda_c0 /
   * lambda_b and the per-contingency energies over them (islanded at any
   * timestep = islanded). n_timesteps <= 1 (injection_net_mw_t NULL) is the
   * reference's single-vector evaluation. */
  int32_t n_timesteps;
  const double* injection_net_mw_t; /* [n_timesteps][n_injections] net MW */
} tg_grid_desc;

/* ---- plain-data action encoding (replaces const ActionSet&, importer.hpp:28-35).
 *      Actions of one substation must be contiguous (station_ranges). ---- */
typedef struct tg_actionset_desc {
  int32_t n_actions;
  const int32_t* action_substation;     /* [n_actions] */
  const int32_t* action_lambda_r;       /* Action::reassignment_distance */
  const int32_t* action_group_ptr;      /* [n_actions+1] into action_group */
  const uint8_t* action_group;          /* per terminal of the station: 1 = moves to the new node */
  const int32_t* action_busbar_ptr;     /* [n_actions+1] into action_implied_ptr (one slot per busbar) */
  const int32_t* action_implied_ptr;    /* implied branches per (action, busbar), grid_model.cpp:229-242 */
  const int32_t* action_implied;
  int32_t n_disconnectables;
  const int32_t* disconnectables;       /* branch indices, ascending */
} tg_actionset_desc;

/* DcConfig, dc_engine.hpp:16-23 (threads is accepted and ignored on the GPU). */
typedef struct tg_dc_config {
  double islanding_penalty_mw;
  int32_t worst_k;
  double weight_c0;
  double weight_c;
  int32_t fitness_variant;
  int32_t threads;
} tg_dc_config;

/* ScoreVector, dc_engine.hpp:25-39, for n candidates (SoA, caller-owned, length n
 * except worst_* which are [n][worst_k]). Any pointer may be NULL. */
typedef struct tg_scores {
  double* lambda_o;
  int32_t* lambda_c;
  int32_t* lambda_c0;
  double* lambda_b;
  int32_t* lambda_d;
  int32_t* lambda_s;
  int32_t* lambda_r;
  double* fitness;
  uint8_t* islanded;
  int32_t* worst_idx;     /* contingency index, -1 padded */
  double* worst_energy;
  int32_t* worst_n;
  int32_t* islanded_outages;        /* FlowResult::islanded_outages */
  int32_t* islanded_busbar_outages; /* FlowResult::islanded_busbar_outages */
} tg_scores;

/* QdConfig, qd_optimizer.hpp:15-32 */
typedef struct tg_qd_config {
  int32_t n_a, n_d, batch_size, iters_per_epoch, cell_capacity;
  double mutation_mean;
  double p_action[4];
  double p_disc[4];
  double p_crossover_parent1;
  int32_t d_max, s_max, r_max;
  uint64_t seed;
  int64_t max_evaluations;
  double max_seconds;
  /* Lane RNG (extension): 0 = replay of the reference's per-lane
   * std::mt19937_64 + libstdc++ distributions (qd_optimizer.cpp:377-383; bit
   * for bit), 1 = counter-based Philox4x32-10 keyed by the same lane seed
   * (stateless draws, same distributions; not the reference's stream). */
  int32_t rng;
} tg_qd_config;

/* One archive entry of a RepertoireSnapshot (qd_optimizer.hpp:83-95). */
typedef struct tg_snapshot_view {
  int32_t epoch;
  int64_t evaluations;
  double best_fitness;
  int32_t final_snapshot;
  int32_t n_entries;
  int32_t n_slots;                  /* n_a + n_d */
  const int32_t* cell;              /* [n_entries] */
  const int32_t* genome;            /* [n_entries][n_slots] */
  const double* fitness;
  const double* lambda_o;
  const int32_t* lambda_c;
  const int32_t* lambda_c0;
  const double* lambda_b;
  const int32_t* lambda_d;
  const int32_t* lambda_s;
  const int32_t* lambda_r;
  const int32_t* worst_idx;         /* [n_entries][worst_k] */
  const double* worst_energy;
  const int32_t* worst_n;
  int32_t worst_k;
} tg_snapshot_view;

/* SnapshotSink, qd_optimizer.hpp:100: invoked on the calling thread after each epoch. */
typedef void (*tg_snapshot_cb)(const tg_snapshot_view* snap, void* user);

typedef struct tg_opt_stats {
  int64_t evaluations;   /* OptimizerStats, qd_optimizer.hpp:102-107 */
  int32_t epochs;
  int32_t n_trace;       /* fitness_trace entries written to the caller's arrays */
} tg_opt_stats;

const char* tg_last_error(void);
const char* tg_version(void);

/* ---- host-side model and import (the engine's own loaders) ---- */
/* load_grid / grid_from_json_text, grid_model.hpp:130-131 */
tg_status tg_grid_from_json(const char* text, size_t len, tg_grid** out);
void tg_grid_destroy(tg_grid* grid);
/* grid_to_json_text, grid_model.cpp:423-485 (the canonical dump; free with tg_free) */
tg_status tg_grid_to_json(const tg_grid* grid, char** text_out);
/* grid_content_hash, grid_model.cpp:494-503: FNV-1a of the canonical dump, the
 * key of the action cache (importer.cpp:407-479) */
tg_status tg_grid_content_hash(const tg_grid* grid, uint64_t* hash);
/* Branch id string of branch e (grid_model.hpp:37 Branch::id); valid while the grid lives. NULL if e is out of range. */
const char* tg_grid_branch_id(const tg_grid* grid, int32_t e);
/* build_ptdf, importer.cpp:358-401 (PTDFMatrix::sensitivities): computed on
 * `device` from the device inverse of B_red; out [n_branches][n_nodes]
 * row-major, slack column and out-of-service rows zero. SingularSystem on a
 * disconnected grid. */
tg_status tg_build_ptdf(const tg_grid* grid, int device, double* out);
/* fills a desc whose arrays point into the grid object (valid while it lives) */
tg_status tg_grid_describe(const tg_grid* grid, tg_grid_desc* out);
/* build_action_set, importer.hpp:80 (EnumerationConfig seed/cap, importer.hpp:68-71) */
tg_status tg_actionset_build(const tg_grid* grid, uint64_t seed, int64_t cap, tg_actionset** out);
/* build_action_set with the islanding validation of every candidate split
 * (validate_action_islanding, importer.cpp:314-339) on `device`: one CTA per split
 * (BFS connectivity + bridges by tree-path covering); same action ids as
 * tg_actionset_build. */
tg_status tg_actionset_build_device(const tg_grid* grid, uint64_t seed, int64_t cap, int device, tg_actionset** out);
/* load_action_set / save_action_set, importer.hpp:91-94 (JSON text in memory) */
tg_status tg_actionset_from_json(const tg_grid* grid, const char* text, size_t len, tg_actionset** out);
tg_status tg_actionset_to_json(const tg_actionset* set, const tg_grid* grid, char** text_out); /* free with tg_free */
void tg_actionset_destroy(tg_actionset* set);
tg_status tg_actionset_describe(const tg_actionset* set, const tg_grid* grid, tg_actionset_desc* out);
void tg_free(void* p);

/* ---- DcContext (dc_engine.hpp:95-150) ---- */
/* DcContext::DcContext, dc_engine.cpp:80-145: base factorization on `device`,
 * action busbar tables, pre-optimization score. SingularSystem on a
 * disconnected grid. */
tg_status tg_context_create(const tg_grid_desc* grid, const tg_actionset_desc* actions, const tg_dc_config* config,
                            int device, tg_context** out);
void tg_context_destroy(tg_context* ctx);
/* DcContext::evaluate_batch, dc_engine.cpp:439-468 (and ::evaluate for n=1):
 * genomes [n][n_a+n_d] (-1 = empty slot). batch_size pads like the reference
 * (padding is evaluated and dropped). Optional FlowResult outputs
 * (dc_engine.hpp:41-48), NULL to skip: base_flows/max_contingency/max_busbar
 * [n][n_branches], outage_energy [n][n_contingencies]. */
tg_status tg_evaluate_batch(tg_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                            int32_t batch_size, tg_scores* out, double* base_flows, double* max_contingency,
                            double* max_busbar, double* outage_energy);
/* Same batch with genomes and scores already in device memory (no host copies). */
tg_status tg_evaluate_batch_device(tg_context* ctx, const int32_t* d_genomes, int32_t n, int32_t n_a, int32_t n_d,
                                   tg_scores* d_out);
/* DcContext::pre_optimization_score / lambda_b_pre, dc_engine.hpp:112-113 */
tg_status tg_pre_score(tg_context* ctx, tg_scores* out, double* lambda_b_pre);

/* ---- MapElites loop (qd_optimizer.hpp:116-118) ---- */
/* run_optimizer, qd_optimizer.cpp:344-417: device-resident loop; mutation,
 * crossover, evaluation and archive insert stay on the GPU, one snapshot D2H
 * per epoch. stop is polled before every iteration. fitness_trace arrays may be
 * NULL; trace_cap bounds them. ConfigError as the reference. */
tg_status tg_optimizer_run(tg_context* ctx, const tg_qd_config* cfg, tg_snapshot_cb cb, void* user,
                           const volatile int32_t* stop, tg_opt_stats* stats, int64_t* trace_evaluations,
                           double* trace_best, int32_t trace_cap);
/* Step-wise form of the same loop (what run_optimizer does between snapshots):
 * begin = validate + seed the archive (1 evaluation); step = enqueue n
 * generations asynchronously (one CUDA graph launch each, no host sync);
 * fetch = synchronize and copy the archive out as a snapshot view. */
tg_status tg_qd_begin(tg_context* ctx, const tg_qd_config* cfg);
tg_status tg_qd_step(tg_context* ctx, int32_t n_iters);
tg_status tg_qd_fetch(tg_context* ctx, int32_t final_snapshot, tg_snapshot_view* out);
/* Lockstep halves of one generation (parity replay, qd_optimizer.cpp:377-401):
 * offspring = the current iteration's lanes (mutation / crossover from the
 * archive, no evaluation); insert = Repertoire::insert of caller-provided
 * scores for those lanes in lane order, then the iteration counter advances. */
tg_status tg_qd_offspring(tg_context* ctx, int32_t* genomes_out);
tg_status tg_qd_insert(tg_context* ctx, const int32_t* genomes, const tg_scores* scores);
/* Archive of the last run as a snapshot view (valid until the next call). */
tg_status tg_archive_export(tg_context* ctx, tg_snapshot_view* out);
/* Repertoire::insert replay (qd_optimizer.cpp:281-303) on the device archive:
 * resets an archive for cfg and inserts n (genome, score) pairs in order.
 * inserted[n] (optional) receives Repertoire::insert's return value. */
tg_status tg_archive_replay(tg_context* ctx, const tg_qd_config* cfg, const int32_t* genomes, int32_t n,
                            const tg_scores* scores, uint8_t* inserted);
/* ---- island exchange (no reference counterpart: the reference runs one
 * population, qd_optimizer.cpp:344-417; SURVEY.md 8(e) island mode) ----
 * blob_bytes = size of one island's archive blob (fixed for a cfg; after
 * tg_qd_begin). pack writes this archive into the DEVICE buffer d_blob, merge
 * reads n_islands consecutive blobs from the DEVICE buffer d_blobs (e.g. the
 * output of an NCCL allgather), clears the cells and re-inserts every entry in
 * (island, cell, position) order with Repertoire::insert semantics
 * (qd_optimizer.cpp:281-303): islands merging the same blobs end with
 * identical archives. Both are enqueued on tg_context_stream(ctx); the caller
 * orders its collective on that stream. The iteration counter is kept. */
tg_status tg_archive_blob_bytes(tg_context* ctx, int64_t* bytes);
tg_status tg_archive_pack(tg_context* ctx, void* d_blob);
tg_status tg_archive_merge(tg_context* ctx, const void* d_blobs, int32_t n_islands);
/* ---- batch-sharded generation (SURVEY.md 8(e) parity mode): one
 * run_optimizer iteration (qd_optimizer.cpp:376-401) split so that G ranks
 * share one population: every rank runs generation_begin (the same offspring
 * on every rank: lane seeds depend only on (seed, iteration, lane)), evaluates
 * its lane slice, packs it (device blob, scores_blob_bytes(hi - lo)), the
 * slices are allgathered and unpacked, and generation_end inserts all lanes in
 * lane order and advances the iteration: the archive is bit-identical to a
 * one-GPU run. All calls are enqueued on tg_context_stream(ctx). */
tg_status tg_qd_generation_begin(tg_context* ctx);
tg_status tg_qd_evaluate_lanes(tg_context* ctx, int32_t lo, int32_t hi);
tg_status tg_qd_scores_blob_bytes(tg_context* ctx, int32_t n, int64_t* bytes);
tg_status tg_qd_scores_pack(tg_context* ctx, int32_t lo, int32_t hi, void* d_blob);
tg_status tg_qd_scores_unpack(tg_context* ctx, int32_t lo, int32_t hi, const void* d_blob);
tg_status tg_qd_generation_end(tg_context* ctx);
/* ---- native NCCL exchange (host/islands.cpp): one context
 * per process / GPU, ncclAllGather on the context's stream between the
 * engine's kernels (no host sync, no torch). NCCL is loaded at run time
 * (dlopen libnccl.so.2); without it these return TG_CUDA_ERROR.
 * unique_id: ncclGetUniqueId (128 bytes) on one rank, distributed by the
 * caller out of band; create: ncclCommInitRank on the context's device (call
 * on every rank, collectively). exchange = tg_archive_pack -> allgather ->
 * tg_archive_merge (after tg_qd_begin). step: n generations of this island
 * with an exchange after every merge_every-th (0 = never). shard_step: n
 * batch-sharded generations of ONE population (batch_size = the QdConfig's,
 * divisible by world): generation_begin, this rank's lane slice, score-slice
 * allgather + unpack, generation_end; the archive equals a one-GPU run. */
typedef struct tg_islands tg_islands;
tg_status tg_islands_unique_id(uint8_t* id /* [128] */);
tg_status tg_islands_create(tg_context* ctx, const uint8_t* id, int32_t rank, int32_t world, tg_islands** out);
void tg_islands_destroy(tg_islands* islands);
tg_status tg_islands_exchange(tg_islands* islands);
tg_status tg_islands_step(tg_islands* islands, int32_t n, int32_t merge_every);
tg_status tg_islands_shard_step(tg_islands* islands, int32_t n, int32_t batch_size);
/* descriptor_to_cell, qd_optimizer.cpp:12-17 */
int32_t tg_descriptor_to_cell(int32_t lambda_d, int32_t lambda_s, int32_t lambda_r, const tg_qd_config* cfg);
/* Device mutation / crossover of single lanes with the reference RNG stream
 * (mt19937_64 + libstdc++ distributions, qd_optimizer.cpp:202-277).
 * parents [n][n_slots], seeds [n]: one lane per entry. */
tg_status tg_mutate_lanes(tg_context* ctx, const tg_qd_config* cfg, const int32_t* parents, const uint64_t* seeds,
                          int32_t n, int32_t* children);
tg_status tg_crossover_lanes(tg_context* ctx, const tg_qd_config* cfg, const int32_t* parents1,
                             const int32_t* parents2, const uint64_t* seeds, int32_t n, int32_t* children);

/* ---- snapshot hand-off to the AC stage ----
 * SnapshotChannel, channel.hpp:15-79: single-producer single-consumer queue of
 * RepertoireSnapshots; a bounded channel never blocks the producer, when full
 * the oldest non-final snapshot is dropped; capacity 0 = unbounded.
 * tg_channel_sink, a callback of type tg_snapshot_cb with user = the channel, copies each
 * snapshot of tg_optimizer_run into the channel, so the DC loop feeds the AC
 * consumer thread with no caller code in between (pipeline.cpp:354-366).
 * pop: blocking waits until a snapshot arrives or the channel is closed and
 * drained; returns 1 with *out valid until the next pop / destroy on this
 * channel, 0 when none. */
typedef struct tg_channel tg_channel;
tg_channel* tg_channel_create(int64_t capacity);
void tg_channel_destroy(tg_channel* ch);
void tg_channel_push(tg_channel* ch, const tg_snapshot_view* snap); /* deep copy */
void tg_channel_sink(const tg_snapshot_view* snap, void* channel);
void tg_channel_close(tg_channel* ch);
int32_t tg_channel_pop(tg_channel* ch, int32_t blocking, tg_snapshot_view* out);
int64_t tg_channel_pending(tg_channel* ch);
int64_t tg_channel_dropped(tg_channel* ch);

/* ---- counters and timing for the benchmark contract ---- */
void* tg_context_stream(tg_context* ctx);   /* the context's cudaStream_t (for caller-side events) */
/* Enables/disables CUDA-event timing of the fused sweep on evaluate calls and
 * returns (then resets) the accumulated milliseconds and launch count. */
tg_status tg_sweep_timing(tg_context* ctx, int32_t enable, double* total_ms, int64_t* launches);
/* (branch row, candidate pair, contingency tile) blocks of the sweep since the
 * last call: offered, passing the per-row bound (first FMA computed), fully
 * computed (passing the per-element bound), holding at least one overload. */
tg_status tg_sweep_rows(tg_context* ctx, int64_t* computed, int64_t* offered, int64_t* overloaded, int64_t* partial);
/* Chunk-level skip statistics of the chunked scores-only sweep since the last
 * call: (candidate, tile, 32-row chunk) tests run and chunks that failed the
 * bound (their rows went to the row-level stages). Resets the counters. */
tg_status tg_sweep_chunks(tg_context* ctx, int64_t* tested, int64_t* hot);
/* Low-rank update size of each candidate of the last evaluated batch (-1 = not swept). */
tg_status tg_batch_ranks(tg_context* ctx, int32_t n, int32_t* ranks);
/* Measured FP64 FMA throughput of `device` (TFLOP/s) from a DFMA microbenchmark. */
tg_status tg_fp64_peak(int device, double* tflops);
tg_status tg_context_info(tg_context* ctx, int64_t* values, int32_t n_values); /* see capi.cu */
int64_t tg_kernel_launches(tg_context* ctx);  /* engine kernels launched so far */

/* ---- AC validation: batched Newton-Raphson on the device.
 * Replaces AcNetwork / AcValidator (ac_validator.hpp:18-140, ac_validator.cpp:26-495):
 * every (genome, contingency) case is one CTA running the reference's polar
 * Newton-Raphson from a flat start (dense Jacobian, LU with partial pivoting),
 * in shared memory for small networks, in a per-CTA HBM scratch slot otherwise. */
typedef struct tg_ac_context tg_ac_context;

/* AcConfig, ac_validator.hpp:18-26 */
typedef struct tg_ac_config {
  double tolerance_pu;               /* 1e-6 */
  int32_t max_iterations;            /* 30 */
  int32_t worst_k_nonconverged;      /* q = 2 */
  double nonconverged_fraction;      /* 0.05 */
  int32_t similarity_distance;       /* 1   (host-side eliminate) */
  double dominance_fitness_frac;     /* 0.01 (host-side eliminate) */
  double improvement_threshold_frac; /* 0.05 (host-side eliminate) */
} tg_ac_config;

/* RejectionReason, ac_validator.hpp:63-71 */
typedef enum tg_ac_reason {
  TG_AC_NONE = 0,
  TG_AC_NONCONVERGENCE = 1,
  TG_AC_OVERLOAD_NOT_IMPROVED = 2,
  TG_AC_CRITICAL_COUNT_INCREASED = 3,
  TG_AC_ELIMINATED_SIMILAR = 4,
  TG_AC_ELIMINATED_DOMINATED = 5,
  TG_AC_ELIMINATED_BELOW_THRESHOLD = 6
} tg_ac_reason;

/* Baseline metrics of the unchanged grid (AcValidator::AcValidator, ac_validator.cpp:313-343). */
typedef struct tg_ac_baseline {
  double lambda_o;          /* baseline_lambda_o() */
  int32_t critical_count;   /* baseline_critical_count() */
  uint8_t base_converged;
  double base_energy;
  double pre_fitness;       /* DcContext::pre_optimization_score().fitness */
} tg_ac_baseline;

/* AcCaseResult per case (ac_validator.hpp:28-36) plus overload_energy /
 * critical_count (ac_validator.cpp:274-288). Any pointer may be NULL;
 * loading_mva is [n_cases][n_branches], vm_pu / va_rad [n_cases][n_nodes + n_a]. */
typedef struct tg_ac_case_out {
  uint8_t* converged;
  int32_t* iterations;
  double* overload_energy;
  int32_t* critical_count;
  double* loading_mva;
  double* vm_pu;
  double* va_rad;
} tg_ac_case_out;

/* AcValidator(grid, actions, dc, config): device tables + the baseline (base case and
 * every contingency of the unchanged grid) computed on `device`. cfg NULL = defaults.
 * dc supplies the pre-optimization DC fitness (may be NULL: 0). */
tg_status tg_ac_context_create(const tg_grid* grid, const tg_actionset* actions, tg_context* dc,
                               const tg_ac_config* cfg, int device, tg_ac_context** out);
void tg_ac_context_destroy(tg_ac_context* ctx);
/* baseline values; case_converged / case_energy: [n_contingencies] or NULL */
tg_status tg_ac_baseline_get(tg_ac_context* ctx, tg_ac_baseline* out, uint8_t* case_converged, double* case_energy);
/* AcNetwork(grid, apply_genome(genome)).run_case(k) for a batch of cases
 * (ac_validator.cpp:26-272): case i solves genome case_genome[i] under contingency
 * case_contingency[i] (-1 = base case). genomes: [n_genomes][n_a + n_d], -1 = empty slot. */
tg_status tg_ac_run_cases(tg_ac_context* ctx, const int32_t* genomes, int32_t n_genomes, int32_t n_a, int32_t n_d,
                          const int32_t* case_genome, const int32_t* case_contingency, int32_t n_cases,
                          tg_ac_case_out* out);
/* AcValidator::worst_k_check for n genomes at once (ac_validator.cpp:399-425): base case
 * plus each genome's DC worst contingencies worst_idx[i][0 .. worst_n[i]); reason[i] = tg_ac_reason. */
tg_status tg_ac_worst_k_check(tg_ac_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                              const int32_t* worst_idx, const int32_t* worst_n, int32_t worst_stride, int32_t* reason);
/* AcValidator::full_validation for n genomes at once (ac_validator.cpp:427-473): base case
 * and every contingency; reason / accepted / ac_lambda_o per genome (accepted, ac_lambda_o may be NULL). */
tg_status tg_ac_full_validation(tg_ac_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                                int32_t* reason, uint8_t* accepted, double* ac_lambda_o);
int64_t tg_ac_kernel_launches(tg_ac_context* ctx);  /* AC kernels launched so far */

#ifdef __cplusplus
}
#endif

#endif /* TOPOPT_B200_H */
