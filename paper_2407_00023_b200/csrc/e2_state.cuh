// e2_state.cuh — HBM layout of one scheduler handle.
//
// Radix tree (reference: prefix_tree.hpp:20-39, prefix_tree.cpp):
//   * node pool, slot-indexed SoA.  NodeHdr (32 B) is what a walk touches:
//     creation id, edge = [edge_off, edge_off+edge_len) in the token arena,
//     parent slot, first edge token, start depth.  Edges never copy tokens:
//     they point into the arena that holds every prompt seen.
//   * per-(slot, instance) arrays [slot*G + g]: last_access, windowed hit
//     counter, cached-child count; per-slot 64-bit caching / last_access
//     presence masks.
//   * one global open-addressing child table keyed (parent_slot<<32 | token).
//   * SPLIT KEEPS THE SLOT ON THE LOWER HALF: split_node (prefix_tree.cpp:
//     122-154) gives the prefix the old id and the suffix a new id and the
//     children.  Here the existing slot becomes the suffix (new id, keeps its
//     children and their table keys) and a fresh slot takes the prefix (old
//     id), so a split rewrites two table entries instead of rekeying every
//     child, and any "node ending at depth d" slot stays valid forever.
// Per-instance LRU index (prefix_tree.hpp:199-201): a paged ordered set of
// (last_access bits, id) keys, 32 keys per page so one lane owns one key.
// Load windows (cost_model.hpp:29-71): per-instance rings + integer sums.
#pragma once

#include "e2_common.cuh"

namespace e2 {

struct NodeHdr {
  u64 id;        // creation order (reference NodeId)
  i64 edge_off;  // token arena offset of the edge
  u32 edge_len;  // 0 only for the root and for removed slots
  u32 parent;    // slot, kNil for the root
  i32 first_tok; // arena[edge_off]
  u32 depth;     // tokens on the root path before this edge
};

constexpr u64 kEmptyKey = ~0ull;
constexpr u64 kTombKey = ~0ull - 1;
constexpr i64 kNoInflight = INT64_MIN;
constexpr int kPage = 32;  // LRU keys per page

// Error codes mirrored from e2sched.h.
constexpr i32 kErrConfig = 1;
constexpr i32 kErrNoAdmissible = 2;
constexpr i32 kErrSim = 3;
constexpr i32 kErrCapacity = 5;

// Reasons (for the host-side message).
enum ErrWhy : i32 {
  kWhyNone = 0,
  kWhyPromptTooLong,
  kWhyNotContiguous,
  kWhyEmptyInsert,
  kWhyCccUnderflow,
  kWhyNodeCap,
  kWhyTableFull,
  kWhyPageCap,
  kWhyDirCap,
  kWhyWindowCap,
  kWhyInflightCap,
  kWhyScratchCap,
  kWhyWalk,
  kWhySplitBounds,
  kWhyFifoCap,
};

enum StatIdx : int {
  kStExploit = 0,
  kStExplore,
  kStPressure,
  kStRoundRobin,
  kStRedirected,
  kStInstalls,
  kStAutoscale,
  kStTreeReads,
};

struct Cfg {
  i32 G;
  i32 mode;  // 0 prefix-aware, 1 round robin
  i32 rebalance, autoscale, pd_balance;
  i32 pad;
  double H, th_bal, imbal;
  i64 cap, default_out;
  double c0, c1, c2, c3;
};

// State the serial replay keeps in shared memory while it runs (the single
// writer); mirrored to HBM between launches.
struct Hot {
  i64 cached_tokens[kMaxG];
  i64 inflight_cached[kMaxG];
  i64 inflight_prompt[kMaxG];
  i32 redirect[kMaxG];
  u64 ws_head[kMaxG], ws_tail[kMaxG];
  i64 ws_missed_sum[kMaxG], ws_missed_nz[kMaxG];
  u64 wc_head[kMaxG], wc_tail[kMaxG];
  i64 wc_output_sum[kMaxG];
  u32 dir_head[kMaxG], dir_n[kMaxG];
  u64 fifo_head[kMaxG], fifo_tail[kMaxG];
  u64 next_id;
  i64 node_count;
  u32 slots_used;
  u32 pages_used;
  u32 free_top;
  u32 pad0;
  i64 rr_next;
  i64 stats[8];
  i64 inflight_n;
  double drv_now;  // driver clock: now = max(now, arrival)
  i32 err, why;
  i64 err_req;  // request index / op index that failed
  i64 done;     // ops fully processed in the last launch
};

struct Dev {
  Cfg cfg;
  const i32* tok;  // token arena
  // nodes
  u32 node_cap;
  u32 pad1;
  NodeHdr* hdr;
  u64* cmask;
  u64* lamask;
  i32* nchild;
  double* la;
  i32* hits;
  i32* ccc;
  // child table
  u64* ck;
  u32* cv;
  u64 ct_mask;
  // windows
  u64 wcap;  // power of two per instance
  double* ws_t;
  i64* ws_missed;
  i64* ws_est;
  u32* ws_slot;
  double* wc_t;
  i64* wc_out;
  // LRU
  u32 dcap;  // directory ring per instance (power of two)
  u32 page_cap;
  u32* dir_page;
  u64* dir_la;
  u64* dir_id;
  u64* pg_la;
  u64* pg_id;
  u32* pg_slot;
  i32* pg_n;
  u32* free_pages;
  // inflight map
  u64 inf_mask;
  i64* inf_key;
  i32* inf_gpu;
  i64* inf_cached;
  i64* inf_prompt;
  double* inf_arr;
  u64* inf_root;
  // driver FIFO (criterion-7 eviction)
  u64 fcap;
  i64* fifo_req;
  i64* fifo_tail;
  // scratch: per instance plan work lists, serial victim list
  u32 scap;
  u32 vcap;
  u32* scr_slot;
  i64* scr_val;
  u64* scr_la;
  u64* scr_id;
  u32* vic_slot;
  i64* vic_tok;
  Hot* hot_g;
};

}  // namespace e2
