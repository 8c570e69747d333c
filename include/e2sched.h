/*
 * e2sched.h — C-ABI drop-in boundary for Preble's E2 global-scheduler hot path.
 *
 * Every entry point here replaces one public member of the reference's
 * kvsched::GlobalScheduler (proj/include/kvsched/global_scheduler.hpp) or the
 * free function load_cost (proj/include/kvsched/cost_model.hpp:87-89), with
 * plain pointers and sizes instead of C++ types.  Three libraries implement
 * this exact header:
 *
 *   paper_2407_00023_b200/libe2sched.so  the product: device-resident radix
 *                                        tree + sm_100a kernels (CUDA)
 *   oracle/_ref/libe2ref.so              test-only: the unmodified reference
 *                                        sources behind a shim
 *   oracle/libe2oracle.so                test-only: plain-C restatement
 *
 * Semantics follow the reference one call at a time: a batched call
 * (e2_replay*) is defined as the equivalent sequence of single calls in
 * arrival order.  Handles are single-writer and not reentrant, exactly like
 * the reference.
 *
 * Error model (reference exceptions -> codes; the C++ wrapper e2sched.hpp
 * rethrows the same exception types):
 *   E2_OK                 success
 *   E2_ERR_CONFIG         kvsched::ConfigError   (global_scheduler.cpp:8-15, 27-37)
 *   E2_ERR_NO_ADMISSIBLE  kvsched::NoAdmissibleGpu (global_scheduler.cpp:80-83)
 *   E2_ERR_SIM            kvsched::SimError      (global_scheduler.cpp:149-155,
 *                                                 prefix_tree.cpp:74,123-125,188)
 *   E2_ERR_CUDA           device/runtime failure (product only)
 *   E2_ERR_ARG            invalid argument / capacity (boundary only)
 * On error, e2_last_error() returns the message.  State mutations that the
 * reference performs before throwing (redirect upkeep, window pruning,
 * tree_reads) are preserved, as in the reference.
 */
#ifndef E2SCHED_H
#define E2SCHED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define E2_OK 0
#define E2_ERR_CONFIG 1
#define E2_ERR_NO_ADMISSIBLE 2
#define E2_ERR_SIM 3
#define E2_ERR_CUDA 4
#define E2_ERR_ARG 5

/* Instances (the reference's GpuIds) supported by one handle: the caching
 * set of a node is a 64-bit mask. */
#define E2_MAX_GPUS 64

/* kvsched::SchedulerConfig (global_scheduler.hpp:18-27). */
typedef struct {
  double history_window_ms;   /* H */
  double th_bal;              /* rebalance trigger ratio */
  double imbal_ratio;         /* decode-pressure threshold */
  int64_t priority_groups;    /* P (validated only; local scheduler) */
  int64_t kv_capacity_tokens; /* per instance */
  int64_t default_output_len; /* avg-output fallback */
} e2_sched_cfg;

/* kvsched::TimeModel (cost_model.hpp:12-17). */
typedef struct {
  double prefill_base_ms;      /* c0 */
  double prefill_per_token_ms; /* c1 */
  double decode_per_token_ms;  /* c2 */
  double iteration_base_ms;    /* c3 */
} e2_time_model;

/* kvsched::GlobalPolicy (global_scheduler.hpp:29-36). */
#define E2_MODE_PREFIX_AWARE 0
#define E2_MODE_ROUND_ROBIN 1
typedef struct {
  int32_t mode;
  int32_t rebalance;
  int32_t autoscale;
  int32_t pd_balance;
} e2_policy;

/* kvsched::Branch (global_scheduler.hpp:38-43). */
#define E2_BRANCH_EXPLOIT 0
#define E2_BRANCH_EXPLORE 1
#define E2_BRANCH_DECODE_PRESSURE 2
#define E2_BRANCH_ROUND_ROBIN 3

/* kvsched::GpuCandidateCost + CostBreakdown (global_scheduler.hpp:47-50,
 * cost_model.hpp:73-82).  total = (L + M) + P, exactly as total_ms(). */
typedef struct {
  int32_t gpu;
  int32_t eviction_infeasible;
  double current_load_ms; /* L */
  double eviction_ms;     /* M */
  double prefill_ms;      /* P */
} e2_cost;

/* kvsched::Decision (global_scheduler.hpp:53-64) plus matched_len, the
 * decide()-time longest-prefix match (global_scheduler.cpp:94), which the
 * reference computes but does not return. */
typedef struct {
  int64_t request;
  int32_t branch;
  int32_t gpu;
  int32_t redirected;
  int32_t pre_redirect_gpu;
  int32_t n_costs;     /* entries written to the cost array, evaluation order */
  int32_t has_ratios;  /* decode_ratios populated (explore path) */
  int64_t cached_len;
  int64_t missed_len;
  int64_t missed_on_chosen;
  int64_t matched_len;
} e2_decision;

/* kvsched::GlobalStats (global_scheduler.hpp:85-94). */
typedef struct {
  int64_t exploit;
  int64_t explore;
  int64_t decode_pressure;
  int64_t round_robin;
  int64_t redirected;
  int64_t rebalance_installs;
  int64_t autoscale_events;
  int64_t tree_reads;
} e2_stats;

typedef struct e2_handle e2_handle;

/* GlobalScheduler(int n_gpus, const SchedulerConfig&, const TimeModel&,
 * const GlobalPolicy&)  — global_scheduler.hpp:101-102, .cpp:27-37. */
int e2_create(int32_t n_gpus, const e2_sched_cfg* cfg, const e2_time_model* model,
              const e2_policy* policy, e2_handle** out);
void e2_destroy(e2_handle* h);
/* Return h to its just-created state, keeping its allocations (bench steps). */
int e2_reset(e2_handle* h);
/* Product only: enqueue all device work of h on `stream` (a cudaStream_t);
 * NULL restores the handle's own stream. */
int e2_set_stream(e2_handle* h, void* stream);
/* Message of the last failed call on h (or of the last failed e2_create
 * when h is NULL). */
const char* e2_last_error(const e2_handle* h);
/* Implementation tag: "b200", "reference", "oracle". */
const char* e2_backend(void);

/* Decision schedule_request(const Request&, SimTime) — global_scheduler.cpp:177-192.
 * costs: room for n_gpus + 1 entries (may be NULL);
 * ratios: room for n_gpus doubles (may be NULL). */
int e2_schedule(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int64_t request_id,
                double arrival_ms, double now, e2_decision* out, e2_cost* costs, double* ratios);
/* Decision decide(const Request&, SimTime) — global_scheduler.cpp:76-158. */
int e2_decide(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int64_t request_id,
              double now, e2_decision* out, e2_cost* costs, double* ratios);

/* Simulator callbacks — global_scheduler.cpp:340-369. */
int e2_note_admitted(e2_handle* h, int64_t request_id, double now);
int e2_note_prefill_cached(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int32_t gpu,
                           double now);
/* note_eviction(EvictedRange{seq, tail_len}, gpu, now) */
int e2_note_eviction(e2_handle* h, const int32_t* seq, int64_t seq_len, int64_t tail_len,
                     int32_t gpu, double now);
int e2_note_finished(e2_handle* h, int64_t request_id, double now, int64_t output_len);

/* Queries — global_scheduler.cpp:39-47, 371-373; prefix_tree.cpp:395-398. */
int e2_decode_ratio(e2_handle* h, int32_t gpu, double* out);
int e2_gpu_load_ms(e2_handle* h, int32_t gpu, double now, double* out);
int e2_prune_dead_nodes(e2_handle* h, double now, int64_t* removed);
int e2_cached_tokens(e2_handle* h, int32_t gpu, int64_t* out);
int e2_node_count(e2_handle* h, int64_t* out); /* excludes the root */
/* redirects(): out[g] = target or -1. */
int e2_redirects(e2_handle* h, int32_t* out);
int e2_get_stats(e2_handle* h, e2_stats* out);
/* load_cost(mirror(), window(gpu), gpu, kv_capacity, missed, model, now)
 * — cost_model.cpp:75-100, as the fidelity probes call it
 * (reference_scheduler.cpp:409-420). */
int e2_load_cost(e2_handle* h, int32_t gpu, int64_t missed_tokens, double now, e2_cost* out);
/* Read-only MatchResult of mirror().match(seq) — prefix_tree.cpp:116-120.
 * per_gpu: room for n_gpus extents (0 when absent). */
int e2_match(e2_handle* h, const int32_t* seq, int64_t len, int64_t* matched_len,
             int64_t* cached_len, int64_t* per_gpu);

/* Mirror export — prefix_tree.cpp:436-461 (export_nodes), depth-first in
 * child-token order, index 0 = root.  Hits are exported as the in-window
 * count at `now` (what debug_dump prints) rather than raw lazily-pruned
 * deques, whose contents depend on read history. */
typedef struct {
  uint64_t id;
  uint64_t parent_id;
  int64_t edge_off; /* into the tokens buffer */
  int64_t edge_len;
  uint64_t caching_mask;     /* bit g = cached on g */
  uint64_t last_access_mask; /* bit g = last_access[g] present */
  int64_t pin_count;
} e2_node;
/* Phase 1: sizes.  Phase 2: fill (nodes[n_nodes], tokens[n_tokens],
 * last_access[n_nodes*n_gpus], hits[n_nodes*n_gpus]); any may be NULL. */
int e2_export_size(e2_handle* h, int64_t* n_nodes, int64_t* n_tokens);
int e2_export(e2_handle* h, double now, e2_node* nodes, int32_t* tokens, double* last_access,
              int64_t* hits);
/* debug_dump(now, horizon) — prefix_tree.cpp:411-455. Writes up to cap bytes
 * (NUL-terminated) and the full length to *needed. */
int e2_debug_dump(e2_handle* h, double now, char* buf, size_t cap, size_t* needed);

/* Window contents after pruning at now (snapshot(), global_scheduler.cpp:375-394). */
int e2_window_sizes(e2_handle* h, int32_t gpu, double now, int64_t* n_scheduled,
                    int64_t* n_completed, int64_t* inflight_cached, int64_t* inflight_prompt);
/* snapshot(now).gpus[gpu].scheduled / .completed — global_scheduler.cpp:384-389,
 * LoadWindow::snapshot_scheduled/completed (cost_model.cpp:55-63): the
 * entries after pruning at now, oldest first, sized by e2_window_sizes.
 * Any pointer may be NULL. */
int e2_window_entries(e2_handle* h, int32_t gpu, double now, double* sched_t, int64_t* sched_missed,
                      int64_t* sched_est, double* comp_t, int64_t* comp_out);
/* snapshot(now).nodes[i].hits — export_nodes (prefix_tree.cpp:436-448) hit
 * stamps in e2_export's node order, gpu-minor, each list oldest first; list
 * (i, g) holds e2_export's hits[i*G+g] stamps.  Only in-window stamps
 * (t >= now - history_window_ms): what every read of the reference sees
 * after its lazy prune (prefix_tree.cpp:37-43); the reference's raw deques
 * may still hold older ones.  *n_stamps = total; stamps may be NULL. */
int e2_export_hit_stamps(e2_handle* h, double now, double* stamps, int64_t cap, int64_t* n_stamps);

/* ---------------------------------------------------------------------------
 * Batched trace driver.  The reference's own throughput loop
 * (tests/acceptance_main.cpp:367-416, criterion 7) generalised:
 *
 *   for i in arrival order:
 *     now = max(now, arrival[i])
 *     while prune_interval_ms > 0 and next_tick <= now:
 *       prune_dead_nodes(next_tick); next_tick += prune_interval_ms
 *     d = schedule_request(r_i, now)
 *     if prefill_cached: note_prefill_cached(p_i, d.gpu, now)
 *     eviction == FIFO_TAIL: push (i, |p_i| - trunk_len) on fifo[d.gpu];
 *        while cached_tokens(d.gpu) > high_water and fifo[d.gpu] nonempty:
 *          pop (k, tail); note_eviction({p_k, tail}, d.gpu, now)
 *     eviction == MIRROR_LRU: if cached_tokens(d.gpu) > high_water:
 *          plan = mirror.plan_eviction(d.gpu, cached - high_water, {}, true)
 *          ranges = [{path_tokens(e.node), e.tokens} for e in plan]
 *          for r in ranges: note_eviction(r, d.gpu, now)
 *     if i >= finish_lag: note_finished(id[i - lag], now, output_len[i - lag])
 *
 * Results are identical to issuing those calls one by one.
 * ------------------------------------------------------------------------- */
#define E2_EVICT_NONE 0
#define E2_EVICT_FIFO_TAIL 1
#define E2_EVICT_MIRROR_LRU 2
typedef struct {
  int32_t eviction;
  int32_t prefill_cached;
  int64_t trunk_len;
  int64_t high_water;
  int64_t finish_lag;
  int64_t batch; /* requests per device batch (0 = implementation default) */
  /* > 0: before a request at `now`, prune_dead_nodes(T) for every tick
   * T = k * prune_interval_ms (k = 1, 2, ...) with T <= now, in order — the
   * simulator's RebalanceTick cadence (simulator.cpp:217-229, H/2). */
  double prune_interval_ms;
} e2_driver_cfg;

/* Host buffers: tokens (CSR, offsets[n+1]), ids, arrivals, output_lens.
 * out[n]; costs: NULL or n*(n_gpus+1); ratios: NULL or n*n_gpus.
 * *n_done = requests fully processed (== n on success). */
int e2_replay(e2_handle* h, const int32_t* tokens, const int64_t* offsets, const int64_t* ids,
              const double* arrivals, const int64_t* output_lens, int64_t n,
              const e2_driver_cfg* drv, e2_decision* out, e2_cost* costs, double* ratios,
              int64_t* n_done);

/* Product only: same as e2_replay but every array is a DEVICE pointer that
 * stays resident, and all work is enqueued on `stream` (a cudaStream_t). */
int e2_replay_device(e2_handle* h, const int32_t* d_tokens, const int64_t* d_offsets,
                     const int64_t* d_ids, const double* d_arrivals,
                     const int64_t* d_output_lens, int64_t n, const e2_driver_cfg* drv,
                     e2_decision* d_out, e2_cost* d_costs, double* d_ratios, void* stream,
                     int64_t* n_done);

/* ---------------------------------------------------------------------------
 * Sharded replay (product only).  The reference scheduler is
 * single-threaded and has no counterpart: this is the multi-GPU form of the
 * batched replay above (acceptance_main.cpp:367-416 generalised).  Every rank
 * holds a replica of the tree and the whole trace in its own HBM.  Per batch:
 *   all ranks: e2_shard_next (the batch bounds; identical on every rank),
 *              e2_shard_match on the rank's contiguous slice [lo, lo+cnt)
 *              (K1), writing a summary slice of 16 + per*row_bytes bytes;
 *   caller:    gathers the world's slices, rank-major, to rank 0 (NCCL);
 *   rank 0:    e2_shard_commit (leader rounds + the serial decide/commit
 *              pass + the state delta vs what the replicas hold), then
 *              e2_shard_delta_copy into a device buffer of delta_bytes;
 *   caller:    broadcasts the delta from rank 0 (NCCL);
 *   replicas:  e2_shard_apply.  After it every replica's tree, LRU, windows
 *              and counters equal rank 0's byte for byte.
 * The loop ends when e2_shard_next returns nb == 0 (also after a failed
 * batch: e2_shard_end then returns the batch's error on every rank).
 * Decisions/costs are written on rank 0 only (device pointers).
 * ------------------------------------------------------------------------- */
int e2_shard_begin(e2_handle* h, const int32_t* d_tokens, const int64_t* d_offsets, const int64_t* d_ids,
                   const double* d_arrivals, const int64_t* d_output_lens, int64_t n, const e2_driver_cfg* drv,
                   e2_decision* d_out, e2_cost* d_costs, double* d_ratios, int32_t rank, int32_t world);
int e2_shard_next(e2_handle* h, int64_t* b0, int64_t* nb, int64_t* row_bytes);
int e2_shard_match(e2_handle* h, int64_t lo, int64_t cnt, void* d_slice);
int e2_shard_commit(e2_handle* h, const void* d_gathered, int64_t per, int64_t* delta_bytes);
int e2_shard_delta_copy(e2_handle* h, void* d_dst);
int e2_shard_apply(e2_handle* h, const void* d_delta, int64_t bytes);
int e2_shard_end(e2_handle* h, int64_t* n_done);
/* Order-independent digest of every replicated state region plus the hot
 * counters (n_out = regions + 1 values): equal digests on every rank after
 * each e2_shard_apply is the replication invariant the tests check.  Does not
 * mutate the state (unlike an export, which brings hit windows current). */
int e2_state_digest(e2_handle* h, uint64_t* out, int32_t cap, int32_t* n_out);

/* Streamed traces (product only): with `on`, each e2_replay / e2_replay_device
 * call continues the previous one as if the chunks were one trace — the
 * driver clock is kept and the note_finished calls of the previous chunk's
 * last finish_lag requests fall in the next chunk where a single replay
 * makes them (config 5 is streamed in chunks).  Decisions of
 * the concatenated chunks equal one replay of the concatenation.  Mirror-LRU
 * and no-eviction drivers only.  e2_reset starts a new stream. */
int e2_replay_set_continue(e2_handle* h, int32_t on);

/* Product only: per-kernel device time (ms) and launch counts accumulated
 * since the last reset, for the bench's roofline (kernel ids below). */
#define E2_K_MATCH 0  /* K1 batched prefix match */
#define E2_K_GROUP 1  /* intra-batch LCP leader rounds */
#define E2_K_COMMIT 2 /* serial decide+commit replay */
#define E2_K_OTHER 3
#define E2_K_COUNT 4
typedef struct {
  double ms[E2_K_COUNT];
  int64_t launches[E2_K_COUNT];
  int64_t match_bytes;    /* algorithmic bytes of K1 */
  int64_t match_requests; /* requests K1 walked */
  int64_t group_retries;  /* leader-round restarts after a grouping-hash collision */
  int64_t delta_bytes;    /* sharded replay (rank 0): state-delta bytes exported */
  int64_t delta_chunks;   /* sharded replay (rank 0): 64-byte chunks in those deltas */
} e2_profile;
int e2_profile_get(e2_handle* h, e2_profile* out);
int e2_profile_reset(e2_handle* h, int32_t enable_timing);

/* ---------------------------------------------------------------------------
 * Synthetic trace generation (input only).  Archetypes of workload.cpp:133-194
 * plus the shapes SURVEY.md 8(d) adds for configs 3-5.  Identical token
 * content to kvsched::generate for the reference archetypes.
 * ------------------------------------------------------------------------- */
#define E2_ARCH_CUSTOM 0
#define E2_ARCH_TOOLBENCH 1
#define E2_ARCH_EMBODIED 2
#define E2_ARCH_PROGRAMMING 3
#define E2_ARCH_VIDEO_QA 4
#define E2_ARCH_DOC_QA 5
#define E2_ARCH_TREE_OF_THOUGHT 6 /* new: deep branching (config 4) */
typedef struct {
  int32_t archetype;
  int32_t zipf; /* popularity: 0 uniform, 1 zipf */
  int64_t request_count;
  int64_t system_prompt_len;
  int64_t branch_count;
  int64_t branch_len;     /* fixed trunk length (grouped) */
  int64_t branch_len_max; /* >branch_len: per-trunk U[branch_len, max] (config 3) */
  double zipf_s;
  int64_t unique_min, unique_max;
  int64_t output_min, output_max;
  double requests_per_group;
  double chain_mean_len;
  int64_t observation_len;
  int64_t fanout; /* tree-of-thought */
  int64_t depth;  /* tree-of-thought */
} e2_workload_spec;
/* archetype_default(a) — workload.cpp:133-194. */
void e2_workload_default(int32_t archetype, e2_workload_spec* out);
/* Phase 1 (tokens == NULL): counts. Phase 2: fill. Arrivals: Poisson at
 * rps with seed arrival_seed (workload.cpp:486-497); ids 1..n. */
int e2_generate(const e2_workload_spec* spec, uint64_t seed, double rps, uint64_t arrival_seed,
                int64_t* n_requests, int64_t* n_tokens, int32_t* tokens, int64_t* offsets,
                int64_t* ids, double* arrivals, int64_t* output_lens);

/* ---------------------------------------------------------------------------
 * Corpus / trace files and the corpus study (workload.cpp:329-601; SURVEY 8(f)
 * row 4).  Host-side input tooling.  Two-phase reads: pass NULL buffers to
 * get the sizes.  Parse errors return E2_ERR_ARG with the reference's
 * "<what> line N: ..." message in e2_last_error(NULL).
 * ------------------------------------------------------------------------- */
/* write_corpus_file: "id [arrival %.3f] tok... output_len" per line;
 * arrivals may be NULL (none written) or per-line via has_arrival. */
int e2_corpus_write(const char* path, const int32_t* tokens, const int64_t* offsets, const int64_t* ids,
                    const double* arrivals, const int32_t* has_arrival, const int64_t* output_lens, int64_t n);
/* read_corpus_file. */
int e2_corpus_read(const char* path, int64_t* n, int64_t* n_tokens, int32_t* tokens, int64_t* offsets,
                   int64_t* ids, double* arrivals, int32_t* has_arrival, int64_t* output_lens);
/* read_trace_file: CSV with a header row, rows stably sorted by arrival. */
int e2_trace_read(const char* path, int64_t* n, double* arrival_s, int64_t* prompt_len, int64_t* output_len);
/* synthesize_from_trace: toolbench-shaped prompts of the trace's lengths in
 * arrival order, ids 1..n, arrivals in ms. */
int e2_synthesize_from_trace(const e2_workload_spec* content, uint64_t seed, const double* arrival_s,
                             const int64_t* prompt_len, const int64_t* output_len, int64_t n, int64_t* n_tokens,
                             int32_t* tokens, int64_t* offsets, int64_t* ids, double* arrivals_ms,
                             int64_t* output_lens);
typedef struct {
  int64_t count;
  double mean, p50, p99, min, max;
} e2_dist; /* DistStats (workload.hpp:113-120) */
typedef struct {
  int64_t requests;
  int64_t total_prompt_tokens;
  int64_t total_output_tokens;
  int64_t total_shared_tokens;
  double shared_token_fraction;
  double mean_request_shared_fraction;
  double mean_prompt_output_ratio;
  e2_dist prompt_len;
  e2_dist output_len;
  int64_t key_portion_count;
  double mean_key_portion_len;
  e2_dist requests_per_shared_sequence;
} e2_study; /* StudyReport (workload.hpp:126-141) */
/* analyze: the infinite-cache corpus study (workload.cpp:530-601). */
int e2_analyze(const int32_t* tokens, const int64_t* offsets, const int64_t* output_lens, int64_t n, e2_study* out);

#ifdef __cplusplus
}
#endif

#endif /* E2SCHED_H */
