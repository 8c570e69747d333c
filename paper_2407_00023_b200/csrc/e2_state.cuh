// e2_state.cuh — HBM layout of one scheduler handle.
//
// Radix tree (reference: prefix_tree.hpp:20-39, prefix_tree.cpp):
//   * node pool of fixed-stride records (AoS): a 64-byte header (creation id,
//     edge = [edge_off, edge_off+edge_len) in the token arena, parent slot,
//     first edge token, start depth, caching / last_access-presence masks,
//     child count) followed by per-instance last_access[G], windowed hit
//     counters[G] and cached-child counts[G].  One record is one or a few
//     coalesced warp loads; the serial kernel keeps hot records in a
//     shared-memory cache (e2_tree.cuh).  Edges never copy tokens: they point
//     into the arena that holds every prompt seen.
//   * one global open-addressing child table keyed (parent_slot<<32 | token),
//     16-byte entries so a 32-lane probe returns key and child together.
//   * SPLIT KEEPS THE SLOT ON THE LOWER HALF: split_node (prefix_tree.cpp:
//     122-154) gives the prefix the old id and the suffix a new id and the
//     children.  Here the existing slot becomes the suffix (new id, keeps its
//     children and their table keys) and a fresh slot takes the prefix (old
//     id), so a split rewrites two table entries instead of rekeying every
//     child, and any "node ending at depth d" slot stays valid forever.
// Per-instance LRU index (prefix_tree.hpp:199-201): a paged ordered set of
// (last_access bits, id) keys, 32 keys per page so one lane owns one key; a
// per-instance directory ring of 32-byte entries {page, count, max key}.
// Load windows (cost_model.hpp:29-71): per-instance rings + integer sums.
#pragma once

#include "e2_common.cuh"

namespace e2 {

struct NodeRec {
  u64 id;         // creation order (reference NodeId)
  i64 edge_off;   // token arena offset of the edge
  u32 edge_len;   // 0 only for the root and for removed slots
  u32 parent;     // slot, kNil for the root
  i32 first_tok;  // arena[edge_off]
  u32 depth;      // tokens on the root path before this edge
  u64 cmask;      // bit g: cached on instance g
  u64 lamask;     // bit g: last_access[g] entry exists
  i32 nchild;
  u32 ctpos;  // position of this node's own child-table entry (its parent's key for it), or kCtInline
  // One child is kept inline (first token, slot; in_slot 0 = none, the root
  // is never a child): a lookup reads the parent's header first and probes
  // the hashed table only for its other children.  Splits link the suffix
  // here and new leaves land here whenever the parent has none, so chains,
  // fresh split prefixes and single-child nodes never touch the table.
  i32 in_tok;
  u32 in_slot;
  // followed by: double la[G]; i32 hits[G]; i32 ccc[G];
};
static_assert(sizeof(NodeRec) == 64, "node header must stay 64 bytes");

E2_HDX constexpr u32 rec_stride(int G) { return (u32)(((64 + 16 * G) + 127) / 128 * 128); }
E2_HDX double* rla(NodeRec* r) { return (double*)((char*)r + 64); }
E2_HDX i32* rhits(NodeRec* r, int G) { return (i32*)((char*)r + 64 + 8 * G); }
E2_HDX i32* rccc(NodeRec* r, int G) { return (i32*)((char*)r + 64 + 12 * G); }
E2_HDX const double* rla(const NodeRec* r) { return (const double*)((const char*)r + 64); }
E2_HDX const i32* rhits(const NodeRec* r, int G) { return (const i32*)((const char*)r + 64 + 8 * G); }
E2_HDX const i32* rccc(const NodeRec* r, int G) { return (const i32*)((const char*)r + 64 + 12 * G); }

struct CtEntry {
  u64 key;
  u32 val;
  u32 pad;
};

struct DirEntry {
  u32 page;
  i32 cnt;
  u64 max_la;
  u64 max_id;
  u64 pad;
};

struct InfRec {
  i64 key;
  i32 gpu;
  i32 pad;
  i64 cached;
  i64 prompt;
  double arr;
  u64 root;
  u64 pad2;
};

static_assert(sizeof(InfRec) % 8 == 0, "inflight records are copied as 8-byte words");

struct WinEnt {
  double t;
  i64 missed;
  i64 est;
  u32 slot;  // tail slot of the committed prompt
  u32 plen;  // levels of its path in the instance's path log (kNil: not logged)
};

struct CompEnt {
  double t;
  i64 out;
};

constexpr u32 kCtInline = 0xfffffffeu;  // ctpos: the node is its parent's inline child
constexpr u64 kEmptyKey = ~0ull;
constexpr u64 kTombKey = ~0ull - 1;
constexpr i64 kNoInflight = INT64_MIN;
constexpr int kPage = 32;   // LRU keys per page
constexpr int kPathHint = 1024;  // initial K1 hint stride (path slots per request, kNil-terminated)
constexpr int kMaxHint = 16384;  // largest hint stride the host grows to
#ifndef E2_MAX_PATH
#define E2_MAX_PATH 512  // 1024 measured slower: the larger scratch takes shared memory from L1
#endif
constexpr int kMaxPath = E2_MAX_PATH;  // path levels a request keeps in shared memory
constexpr u32 kXPath = 1u << 16;  // deeper levels: global overflow (DEV.xp_*)

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
  i32 gtop;  // power of two >= min(G, 32): xor-reduction span over per-instance lanes
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
  u64 ws_done[kMaxG];     // window entries whose hit stamps were already undone
  double ws_head_t[kMaxG];  // time of the oldest scheduled entry
  i64 ws_missed_sum[kMaxG], ws_missed_nz[kMaxG];
  u64 wc_head[kMaxG], wc_tail[kMaxG];
  double wc_head_t[kMaxG];
  i64 wc_output_sum[kMaxG];
  u32 dir_head[kMaxG], dir_n[kMaxG];
  u64 fifo_head[kMaxG], fifo_tail[kMaxG];
  u64 pl_head[kMaxG], pl_tail[kMaxG];  // path-log ring positions
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
  u64 phase_cycles[48];  // E2_PHASES builds: clock64 per replay phase
  u64 phase_last, phase_last1;
};
static_assert(sizeof(Hot) % 8 == 0, "Hot is copied as u64 words");

struct Dev {
  Cfg cfg;
  const i32* tok;  // token arena
  // nodes
  u32 node_cap;
  u32 rs;  // record stride (bytes)
  char* rec;
  // child table
  CtEntry* ct;
  u64 ct_mask;
  // windows
  u64 wcap;  // power of two per instance
  WinEnt* win;
  CompEnt* comp;
  // path log: per instance ring of the slots of each window entry's root
  // path (top-down), so expiring hit stamps are undone level-parallel
  u64 pcap;  // power of two per instance
  u32* plog;
  // LRU
  u32 dcap;  // directory ring per instance (power of two)
  u32 page_cap;
  DirEntry* dir;
  u64* pg_la;
  u64* pg_id;
  u32* pg_slot;
  u32* free_pages;
  // inflight map
  u64 inf_mask;
  InfRec* inf;
  // driver FIFO (criterion-7 eviction) and per-request tail slots
  u64 fcap;
  i64* fifo_req;
  i64* fifo_tail;
  u32* req_tail;  // replay: node ending at |p_r| after request r's commit
  // scratch: per instance plan work lists, serial victim list
  u32 scap;
  u32 vcap;
  u32* scr_slot;
  i64* scr_val;
  u64* scr_la;
  u64* scr_id;
  u32* vic_slot;
  i64* vic_tok;
  // path levels >= kMaxPath of the request being processed
  u32* xp_slot;
  u32* xp_m;
  u64* xp_cm;
  u64* xp_la0;
  u32* xp_flag;
  Hot* hot_g;
};

E2_HDX NodeRec* grec(const Dev& d, u32 s) { return (NodeRec*)(d.rec + (u64)s * d.rs); }

}  // namespace e2
