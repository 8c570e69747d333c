// e2_kernels.cuh — kernel bodies: the serial replay/op warp, K1 match, and
// the leader-round grouping.  Included once by e2_lib.cu.
#pragma once

#include "e2_engine.cuh"
#include "e2_match.cuh"
#include "e2sched.h"

namespace e2 {

enum OpKind : i32 {
  OP_SCHEDULE = 1,
  OP_DECIDE,
  OP_PREFILL,
  OP_EVICT,
  OP_FINISHED,
  OP_LOAD_COST,
  OP_GPU_LOAD,
  OP_MATCH,
  OP_EXPIRE_ALL,
  OP_WINDOW,
  OP_INFLIGHT_GET,
  OP_PRUNE_DEAD,
  OP_MARK_NODE,      // autoscale: mark_cached_node(slot, gpu, now)
  OP_MARK_SUBTREE,   // autoscale: mark_cached_subtree
  OP_UNCACHE_SUBTREE // autoscale: uncache_subtree
};

struct OpDesc {
  i32 kind;
  i32 gpu;
  i64 off;  // arena offset of the sequence
  i64 len;
  i64 L;    // matched length from K1
  i64 x;    // tail_len / missed / output_len / slot
  i64 id;
  double now;
  double arr;
};

struct ApiOut {
  e2_decision dec;
  e2_cost costs[kMaxG + 1];
  double ratios[kMaxG];
  i64 ext[kMaxG];
  double v;
  i64 i0, i1, i2, i3;
  u64 u0;
};

struct SerialArgs {
  i32 kind;  // 0 replay batch, 1 api op
  i32 eviction, prefill;
  i32 no_prefetch;  // pipelined replay: warp 2 idles (dev comparisons)
  i64 base, n;
  const i64* off;
  const i64* len;
  const i64* ids;
  const double* arr;
  const i64* outl;
  const i64* L;     // batch-local
  const i64* S;     // batch-local K1 snapshot match lengths
  const i64* lead;  // batch-local in-batch leader (LCP = L) or -1
  u32* hint;        // batch-local K1 path hints [n][hstride]; a committed request's row is
                    // rewritten with its committed path (the hints of its in-batch followers)
  i32 hstride;
  i32 pad2;
  e2_decision* dec;
  e2_cost* costs;
  double* ratios;
  i64 trunk, hw, lag;
  OpDesc op;
  ApiOut* out;
};

// Bring every instance's window and hit counters current at `now`
// (export / dump / dead-node removal read hits for all instances).  Warp-wide.
E2_D void expire_all(double now) {
  const int G = DEV.cfg.G;
  for (int g = lane(); g < G; g += kWidth) win_prune(g, now);
  wsync();
  for (int g = 0; g < G; ++g) hits_catchup(g);
}

E2_D void write_decision(const Scr* s, const Dec& r, i64 req_id, e2_decision* dec,
                         e2_cost* costs, double* ratios) {
  const int G = DEV.cfg.G;
  const bool cost_path = (r.branch == 0 || r.branch == 1) && DEV.cfg.mode == 0;
  const int nc = cost_path ? s->n_costs : 0;
  if (lane0()) {
    dec->request = req_id;
    dec->branch = r.branch;
    dec->gpu = r.gpu;
    dec->redirected = r.redirected;
    dec->pre_redirect_gpu = r.pre;
    dec->n_costs = nc;
    dec->has_ratios = r.has_ratios;
    dec->cached_len = r.cached_len;
    dec->missed_len = r.missed_len;
    dec->missed_on_chosen = r.moc;
    dec->matched_len = r.matched;
  }
  if (costs) {
    for (int i = lane(); i < nc; i += kWidth) {
      e2_cost c;
      c.gpu = s->cgpu[i];
      c.eviction_infeasible = s->cinf[i];
      c.current_load_ms = s->cL[i];
      c.eviction_ms = s->cM[i];
      c.prefill_ms = s->cP[i];
      costs[i] = c;
    }
  }
  if (ratios && r.has_ratios) {
    for (int g = lane(); g < G; g += kWidth) ratios[g] = s->ratios[g];
  }
  wsync();
}

// Dead-node removal (prefix_tree.cpp:357-378): a node goes when it is
// uncached, childless and has no in-window hit on any instance; repeat until
// a fixpoint (the reference removes bottom-up in one DFS).  Warp-wide.
E2_D i64 prune_dead() {
  const int G = DEV.cfg.G;
  i64 removed = 0;
  bool again = true;
  while (again) {
    again = false;
    const u32 used = HOT.slots_used;
    for (u32 b = 1; b < used; b += 32) {
      u32 m = vote(32, [&](int j) {
        const u32 sl = b + (u32)j;
        if (sl >= used) return false;
        const NodeRec* r = npeek(sl);
        if (r->edge_len == 0 || r->cmask != 0 || r->nchild != 0) return false;
        for (int g = 0; g < G; ++g)
          if (rhits(r, G)[g] != 0) return false;
        return true;
      });
      wsync();
      while (m) {
        const int j = ffs32(m);
        m &= m - 1;
        const u32 v = b + (u32)j;
        NodeRec* rv = nget(v);
        const u32 par = rv->parent;
        const i32 ft = rv->first_tok;
        wsync();
        if (lane0()) {
          rv->edge_len = 0;
          rv->parent = kNil;
          ndirty(rv);
          HOT.node_count--;
        }
        wsync();
        child_erase_at(rv->ctpos, par, ft);
        NodeRec* rp = nget(par);
        if (lane0()) {
          rp->nchild -= 1;
          ndirty(rp);
        }
        wsync();
        removed++;
        again = true;
      }
    }
  }
  return removed;
}

// Subtree walks for autoscale replication (global_scheduler.cpp:299-338):
// children are found by scanning parents (rare path).
E2_D void subtree_apply(u32 root, int g, double now, bool mark) {
  u32 top = 0;
  if (lane0()) DEV.vic_slot[0] = root;
  wsync();
  top = 1;
  u32 order = 0;
  // collect the subtree (breadth-first) into vic_slot, then apply
  while (order < top) {
    const u32 p = DEV.vic_slot[order++];
    const u32 used = HOT.slots_used;
    for (u32 b = 1; b < used; b += 32) {
      const u32 m = vote(32, [&](int j) {
        const u32 sl = b + (u32)j;
        if (sl >= used) return false;
        const NodeRec* r = npeek(sl);
        return r->edge_len > 0 && r->parent == p;
      });
      wsync();
      if (top + (u32)popc32(m) > DEV.vcap) {  // the host sizes vic_slot from its tree copy first
        if (lane0()) set_err(kErrCapacity, kWhyScratchCap);
        return;
      }
      if (lane0()) {
        u32 mm = m, t = top;
        while (mm) {
          DEV.vic_slot[t++] = b + (u32)ffs32(mm);
          mm &= mm - 1;
        }
      }
      wsync();
      top += (u32)popc32(m);
    }
  }
  if (mark) {
    for (u32 i = 0; i < top; ++i) {
      const u32 v = DEV.vic_slot[i];
      if (v == kRoot) continue;
      set_cached(v, g);
      touch_la(v, g, now);
    }
  } else {
    for (u32 i = top; i-- > 0;) {  // children before parents
      const u32 v = DEV.vic_slot[i];
      if (v != kRoot) clear_cached(v, g);
    }
  }
}

// dL: the matched length K1 left on the device (used when op.L < 0, so a
// per-call API op needs no host round trip between the match and the op).
// op.L == kMatchInline: match the sequence here first (one warp, K1's
// match_one with its path hints), so a per-call op is a single launch.
constexpr i64 kMatchInline = -2;
E2_D void api_op(Scr* s, const OpDesc& op0, const u32* hint, int nh, ApiOut* out, const i64* dL = nullptr) {
  OpDesc op = op0;
  if (op.L == kMatchInline) {
    const MatchRes m = match_one(DEV.tok + op.off, op.len, (u32*)hint, nh);
    op.L = m.S;
    wsync();
  } else if (op.L < 0) {
    op.L = dL ? dL[0] : 0;
  }
  const int G = DEV.cfg.G;
  if (lane0()) s->loads_ok = 0;
  wsync();
  const i32* seq = DEV.tok + op.off;
  switch (op.kind) {
    case OP_SCHEDULE:
    case OP_DECIDE: {
      const bool commit_it = op.kind == OP_SCHEDULE;
      if (commit_it && DEV.cfg.mode == 0 && DEV.cfg.rebalance && G > 1) update_redirects(s, op.now);
      Walk w;
      Dec r = decide(s, seq, op.len, op.L, hint, nh, op.L, op.now, w);
      if (!r.ok) return;
      if (commit_it) {
        commit(op.off, op.len, op.L, w, r, op.id, op.arr, op.now, false, s);
        if (HOT.err) return;
        count_stats(r);
      }
      write_decision(s, r, op.id, &out->dec, out->costs, out->ratios);
      break;
    }
    case OP_PREFILL: {
      if (DEV.cfg.mode != 0 || op.len == 0) break;
      Walk w = walk_known(seq, op.L, hint, nh, s->ext);
      if (!w.ok) {
        if (lane0()) set_err(kErrSim, kWhyWalk);
        wsync();
        return;
      }
      u32 tail = ensure_path(op.off, op.len, op.L, w);
      if (tail == kNil || HOT.err) return;
      mark_cached_chain(tail, op.gpu, op.now);
      break;
    }
    case OP_EVICT: {
      if (DEV.cfg.mode != 0) break;
      i64 f = uncache_suffix(seq, op.len, op.L, op.x, op.gpu);
      if (lane0()) out->i0 = f;
      wsync();
      break;
    }
    case OP_FINISHED:
      note_finished(op.id, op.now, op.x);
      break;
    case OP_LOAD_COST: {
      cost_prepare(op.gpu, op.x, op.now);
      if (lane0()) {
        CostOut c = cost_for(op.gpu, op.x, op.now);
        out->costs[0].gpu = op.gpu;
        out->costs[0].eviction_infeasible = c.inf ? 1 : 0;
        out->costs[0].current_load_ms = c.L;
        out->costs[0].eviction_ms = c.M;
        out->costs[0].prefill_ms = c.P;
      }
      wsync();
      break;
    }
    case OP_GPU_LOAD: {
      if (lane0()) out->v = win_load(op.gpu, op.now);
      wsync();
      break;
    }
    case OP_MATCH: {
      Walk w = walk_known(seq, op.L, hint, nh, s->ext);
      for (int g = lane(); g < G; g += kWidth) out->ext[g] = ((w.present >> g) & 1ull) ? s->ext[g] : 0;
      if (lane0()) {
        out->i0 = op.L;
        out->i1 = w.cached_len;
      }
      wsync();
      break;
    }
    case OP_EXPIRE_ALL:
      expire_all(op.now);
      break;
    case OP_WINDOW: {
      if (lane0()) {
        win_prune(op.gpu, op.now);
        out->i0 = (i64)(HOT.ws_tail[op.gpu] - HOT.ws_head[op.gpu]);
        out->i1 = (i64)(HOT.wc_tail[op.gpu] - HOT.wc_head[op.gpu]);
        out->i2 = HOT.inflight_cached[op.gpu];
        out->i3 = HOT.inflight_prompt[op.gpu];
      }
      wsync();
      break;
    }
    case OP_INFLIGHT_GET: {
      if (lane0()) {
        bool found;
        u64 i = inf_find(op.id, found);
        out->i0 = found ? 1 : 0;
        if (found) {
          out->u0 = DEV.inf[i].root;
          out->v = DEV.inf[i].arr;
          out->i1 = DEV.inf[i].gpu;
        }
      }
      wsync();
      break;
    }
    case OP_PRUNE_DEAD: {
      expire_all(op.now);
      i64 rm = prune_dead();
      if (lane0()) out->i0 = rm;
      wsync();
      break;
    }
    case OP_MARK_NODE: {
      u32 v = (u32)op.x;
      if (v != kRoot) {
        set_cached(v, op.gpu);
        touch_la(v, op.gpu, op.now);
      }
      break;
    }
    case OP_MARK_SUBTREE:
      subtree_apply((u32)op.x, op.gpu, op.now, true);
      break;
    case OP_UNCACHE_SUBTREE:
      subtree_apply((u32)op.x, op.gpu, op.now, false);
      break;
    default:
      break;
  }
}

#ifndef E2_DEFER_LRU
#define E2_DEFER_LRU true  // the path's LRU re-indexing runs on warp 1 beside the rest of the commit
#endif
#define PHASE_T0() PHASE_MARK(15)
#define PHASE(i) PHASE_MARK(i)

// One request of the generalised criterion-7 loop (e2sched.h, e2_replay),
// split at the points where the two-warp pipeline hands over:
//   pre   now + redirect upkeep                  (reads the load windows)
//   main  decide + commit (+ note_prefill_cached) (the tree, the LRU of g)
//   post  stats, decision record, note_finished   (windows, inflight map)
//   evict the driver's eviction notices on g      (LRU of g, cmask, splits)
// evict(i) commutes with post(i) and pre(i+1): it touches no window or
// inflight state, so the pipelined replay runs it on a second warp while the
// first warp continues; main(i+1) waits for it (it reads what evict wrote).

E2_D double replay_pre(Scr* s, const SerialArgs& a, i64 li) {
  const int G = DEV.cfg.G;
  const i64 r = a.base + li;
  PHASE_T0();
  const double now = max_(HOT.drv_now, a.arr[r]);
  if (lane0()) {
    HOT.drv_now = now;
    s->loads_ok = 0;
  }
  wsync();
  if (DEV.cfg.mode == 0 && DEV.cfg.rebalance && G > 1) update_redirects(s, now);
  PHASE(0);
  return now;
}

// spec_w: a speculative decide of this request already validated by the
// pipeline (its Walk and Scr path are current), or null.
E2_D bool replay_main(Scr* s, const SerialArgs& a, i64 li, double now, Dec& dec, const Walk* spec_w = nullptr,
                      bool defer_lru = false, bool defer_inflight = false, volatile long long* fix_flag = nullptr) {
  const i64 r = a.base + li;
  const i64 off = a.off[r], n = a.len[r];
  const i32* seq = DEV.tok + off;
  Walk w;
  if (spec_w) {
    w = *spec_w;
  } else {
    dec = decide(s, seq, n, a.L[li], a.hint + li * a.hstride, a.hstride, a.S[li], now, w, false,
                 a.lead ? a.lead + li : nullptr, a.hint);
  }
  if (!dec.ok) return false;
  PHASE(1);
  const bool fuse = a.prefill && DEV.cfg.mode == 0;  // note_prefill_cached(p, d.gpu, now) folded in
  const u32 tail = commit(off, n, a.L[li], w, dec, a.ids[r], a.arr[r], now, fuse, s, defer_lru, defer_inflight,
                          fix_flag, li + 1);
  if (HOT.err) return false;
  PHASE(2);
  if (lane0()) DEV.req_tail[r] = tail;
  // this request's hint row now holds its committed path: the hints of the
  // later requests of the batch that extend it (leader rounds)
  const int D = s->cpath;
  if (D >= 0) {
    u32* row = a.hint + li * a.hstride;
    const int nw = min_(D, a.hstride - 1);
    for (int l = lane(); l <= nw; l += kWidth) row[l] = l < nw ? PSLOT(s, l) : kNil;
  }
  wsync();
  PHASE(36);  // hint row
  return true;
}

E2_D void replay_out(const Scr* s, const SerialArgs& a, i64 li, const Dec& dec) {
  const int G = DEV.cfg.G;
  const i64 r = a.base + li;
  count_stats(dec);
  write_decision(s, dec, a.ids[r], a.dec + r, a.costs ? a.costs + r * (G + 1) : nullptr,
                 a.ratios ? a.ratios + r * G : nullptr);
}

E2_D void replay_finish(const SerialArgs& a, i64 li, double now) {
  const i64 r = a.base + li;
  if (li + a.base >= a.lag) {
    const i64 k = r - a.lag;
    note_finished(a.ids[k], now, a.outl[k]);
  }
  PHASE(5);
}

E2_D void replay_evict(const SerialArgs& a, i64 li, int g) {
  const i64 r = a.base + li;
  if (a.eviction == E2_EVICT_FIFO_TAIL) {
    if (lane0()) {
      u64 t = HOT.fifo_tail[g];
      u64 i = (u64)g * DEV.fcap + (t & (DEV.fcap - 1));
      if (t - HOT.fifo_head[g] >= DEV.fcap) set_err(kErrCapacity, kWhyFifoCap);
      DEV.fifo_req[i] = r;
      DEV.fifo_tail[i] = a.len[r] - a.trunk;
      HOT.fifo_tail[g] = t + 1;
    }
    wsync();
    while (HOT.cached_tokens[g] > a.hw && HOT.fifo_head[g] < HOT.fifo_tail[g] && !HOT.err) {
      u64 i = (u64)g * DEV.fcap + (HOT.fifo_head[g] & (DEV.fcap - 1));
      const i64 k = DEV.fifo_req[i], tl = DEV.fifo_tail[i];
      wsync();
      if (lane0()) HOT.fifo_head[g]++;
      wsync();
      if (DEV.cfg.mode == 0) uncache_tail(DEV.req_tail[k], a.len[k], tl, g);
    }
  } else if (a.eviction == E2_EVICT_MIRROR_LRU) {
    const i64 cached = HOT.cached_tokens[g];
    if (cached > a.hw && DEV.cfg.mode == 0) evict_lru(g, cached - a.hw);
  }
  PHASE(4);
}

// Sequential replay (one warp; the host emulation).
E2_D void replay_seq(Scr* s, const SerialArgs& a) {
  i64 i = 0;
  for (; i < a.n; ++i) {
    const double now = replay_pre(s, a, i);
    Dec dec;
    if (replay_main(s, a, i, now, dec) && !HOT.err) {
      replay_out(s, a, i, dec);
      PHASE(3);
      replay_finish(a, i, now);
      if (!HOT.err) replay_evict(a, i, dec.gpu);
    }
    if (HOT.err) {
      if (lane0()) HOT.err_req = a.base + i;
      wsync();
      break;
    }
  }
  if (lane0()) HOT.done = i;
  wsync();
}

#if E2_WARP
// Two-warp pipelined replay.  Warp 0 runs pre/main/post; warp 1 runs evict
// of the previous request meanwhile.  Named barrier 1: warp 1 finished its
// evict (warp 0 may read the tree/LRU/cmask it wrote); barrier 2: warp 0
// committed request i and published (i, gpu) — warp 1 may start evict(i).
struct Pipe {
  i64 li;
  i32 g;
  i32 stop;
  Dec dec;
  Scr* s;  // the request's scratch (path, costs): double-buffered by warp 0
  // request being committed: its inflight record + note_finished of its step
  // are applied by warp 1 once warp 0 raises `ready` (= request index + 1)
  volatile long long ready;
  volatile long long books_done;  // warp 3: bookkeeping of requests [0, books_done) applied
  volatile long long fix_ready;   // warp 0: request fix_ready-1's path is updated (LRU fixes may start)
  volatile long long commit_done; // warp 0: request commit_done-1 is fully committed (FIFO driver)
  volatile long long w1_fixed;    // warp 1: done with the scratch of requests < w1_fixed (out + fixes)
  i32 c_ok;                       // the request handed to warp 1 commits (else warp 1 does not evict)
  const Scr* fs;                  // that request's scratch (deferred LRU fixes)
  i32 fg;                         // and instance
  i64 c_id, c_cached, c_n;
  u64 c_root;
  double c_arr, c_now;
  i32 c_g, c_defer;
};

#ifndef E2_WAIT_NS
#define E2_WAIT_NS 32  // back-off of the hand-off polls (0: spin)
#endif
E2_D void wait_pause() {
  if (E2_WAIT_NS > 0) __nanosleep(E2_WAIT_NS);
}

// bar.sync is the .aligned barrier: the whole warp must arrive converged,
// and the flag polls before it let lanes leave their loops on different
// iterations (compute-sanitizer synccheck), so reconverge first.
// While warp 0 waits at barrier 1: L1 prefetches for the commit of the
// request it just decided speculatively — the per-instance parts of the
// path's records (last_access, hits, cached-child counts: the path update
// reads them) and the edge token at the split point (ensure_path).
E2_D void prefetch_commit(const Scr* s, const Walk& w) {
  const int np = min_(s->npath, kMaxPath);
  const u32 rs = DEV.rs;
  for (int l = lane(); l < np; l += kWidth) {
    const char* rec = (const char*)grec(PSLOT(s, l));
    if (rs > 128) pf(rec + 128);
    if (rs > 256) pf(rec + 256);
  }
  if (lane0() && w.ok && w.last != kRoot) {
    const NodeRec* r = npeek(w.last);
    if (w.last_m < (i64)r->edge_len) pf(DEV.tok + r->edge_off + w.last_m);
  }
}

E2_D void bar_pair(int id) {
  __syncwarp();
  asm volatile("barrier.sync %0, 64;" ::"r"(id) : "memory");
}

// Flag hand-offs between the pipeline's warps (shared memory): the writer
// stores its data, fences (__threadfence_block) and then raises a volatile
// flag; the reader polls the flag and fences again before reading the data
// (acquire), then reconverges.
E2_D void acquire_after_poll() {
  __threadfence_block();
  wsync();
}

// Warp 0, after barrier 1: did the eviction that ran beside a speculative
// decide touch any node of the decided path?
E2_D bool spec_conflict(const Scr* s) {
  const u32 nt = g_ntouch;
  if (nt > kTouchCap) return true;
  const int np = s->npath;
  if (np < 0) return true;
  bool hit = false;
  for (int l = lane(); l < np; l += kWidth) {
    const u32 v = PSLOT(s, l);
    for (u32 j = 0; j < nt; ++j) hit |= g_touch[j] == v;
  }
  return any(hit);
}

// Warp 2 (optional): an L1 prefetcher running one request ahead of warp 0.
// It only issues prefetches for addresses the next request will probably
// touch — its hint-path records, the prompt token at L and the child-table
// window of the leaf it will insert, the inflight slots of its insert and of
// the note_finished of its step, each instance's window head and LRU head
// victim — so a race with the writers can only cost a useless prefetch.
__shared__ volatile long long g_pf_cur;
__shared__ volatile int g_pf_stop;


E2_D void prefetch_request(const SerialArgs& a, i64 j) {
  const int G = DEV.cfg.G;
  const i64 r = a.base + j;
  const i64 off = a.off[r], n = a.len[r], L = a.L[j];
  const u32* row = a.hint + j * a.hstride;
  const u32 c = row[lane()];
  const u32 nilm = ballot(c == kNil);
  const int nh = nilm ? ffs32(nilm) : 32;
  if (lane() < nh && c < DEV.node_cap) {
    const char* rec = (const char*)grec(c);
    pf(rec);
    if (DEV.rs > 128) pf(rec + 128);
  }
  const u32 last = nh > 0 ? shfl(c, nh - 1) : kRoot;
  if (L < n) {
    const i32 t = DEV.tok[off + L];
    const u64 b = mix64(ckey(last, t)) & DEV.ct_mask;
    if (lane() < 4) pf(&DEV.ct[(b + 8 * lane()) & DEV.ct_mask]);
  }
  if (lane() == 4) {
    const u64 h = mix64((u64)a.ids[r]) & DEV.inf_mask;
    pf(&DEV.inf[h]);
    pf(&DEV.inf[(h + 2) & DEV.inf_mask]);
  }
  if (lane() == 5 && j + a.base >= a.lag) {
    const u64 h = mix64((u64)a.ids[r - a.lag]) & DEV.inf_mask;
    pf(&DEV.inf[h]);
    pf(&DEV.inf[(h + 2) & DEV.inf_mask]);
  }
  if (lane() == 6 && a.lead) {
    const i64 ld = a.lead[j];  // in-batch leader: its committed path row
    if (ld >= 0) pf(a.hint + ld * a.hstride);
  }
  for (int g = lane(); g < G; g += kWidth) {
    pf(&DEV.win[wslot(g, HOT.ws_head[g])]);
    pf(&DEV.comp[wslot(g, HOT.wc_head[g])]);
    if (HOT.dir_n[g] > 0) {
      const DirEntry e = DEV.dir[dring(g, 0)];
      if (e.page < DEV.page_cap) {
        const u64 pi = (u64)e.page * kPage;
        pf(&DEV.pg_la[pi]);
        pf(&DEV.pg_la[pi + 16]);
        pf(&DEV.pg_id[pi]);
        pf(&DEV.pg_id[pi + 16]);
        // the first two LRU victims and their parents
        for (int q = 0; q < 2 && q < e.cnt; ++q) {
          const u32 v = DEV.pg_slot[pi + q];
          if (v < DEV.node_cap) {
            const char* rec = (const char*)grec(v);
            pf(rec);
            pf(rec + 128);
            const NodeRec* rv = (const NodeRec*)rec;
            const u32 p = rv->parent;
            if (p < DEV.node_cap) pf(grec(p));
          }
        }
      }
      const DirEntry t = DEV.dir[dring(g, HOT.dir_n[g] - 1)];
      if (t.page < DEV.page_cap && t.cnt < kPage) {
        const u64 ti = (u64)t.page * kPage + t.cnt;  // where the next fresh key lands
        pf(&DEV.pg_la[ti]);
        pf(&DEV.pg_id[ti]);
        pf(&DEV.pg_slot[ti]);
      }
    }
  }
}

#ifndef E2_PF_SLEEP
#define E2_PF_SLEEP 4000  // ns between polls of warp 0's progress
#endif
#ifndef E2_PF_AHEAD
#define E2_PF_AHEAD 2
#endif
constexpr int kPfAhead = E2_PF_AHEAD;  // requests prefetched ahead of warp 0

E2_D void prefetch_loop(const SerialArgs& a) {
  i64 done = -1;
  while (!g_pf_stop) {
    const i64 cur = g_pf_cur;
    const i64 want = min_<i64>(cur + kPfAhead, a.n - 1);
    if (done >= want) {
      __nanosleep(E2_PF_SLEEP);
      continue;
    }
    done = max_<i64>(done + 1, cur + 1);
    prefetch_request(a, done);
  }
}

// Warp 3 (bookkeeping): for each request warp 0 hands off (`ready`), its
// inflight record, note_finished of its step, then the next request's `now`
// and redirect upkeep; publishes `books_done`.  Touches only the load
// windows, the inflight map/sums, redirects and the next request's scratch
// loads — state no other warp writes meanwhile (warp 0 inserts into the
// tree, warp 1 writes the decision record or evicts).
E2_D void books_loop(Scr* s2, const SerialArgs& a, Pipe* pp) {
  for (i64 ci = 0;; ++ci) {
    while (pp->ready != ci + 1 && !*(volatile i32*)&pp->stop) wait_pause();
    acquire_after_poll();
    if (pp->ready != ci + 1) break;
    if (pp->c_defer) inflight_insert(pp->c_id, pp->c_g, pp->c_cached, pp->c_n, pp->c_arr, pp->c_root);
    replay_finish(a, ci, pp->c_now);
    // the next request's `now` and redirect upkeep: its windows are final
    // (this step's scheduled entry was appended before `ready`)
    if (pp->c_defer && ci + 1 < a.n) {
      Scr* sn = s2 + ((ci + 1) & 1);
      const double nn = replay_pre(sn, a, ci + 1);
      if (lane0()) sn->pre_now = nn;
      wsync();
    }
    if (lane0()) {
      __threadfence_block();
      pp->books_done = ci + 1;
    }
    wsync();
  }
}

E2_D void replay_pipe(Scr* s2, const SerialArgs& a, Pipe* pp) {
  if ((threadIdx.x >> 5) == 2) {
    if (!a.no_prefetch) prefetch_loop(a);
    return;
  }
  if ((threadIdx.x >> 5) == 3) {
    books_loop(s2, a, pp);
    return;
  }
  if ((threadIdx.x >> 5) == 1) {
    // warp 1: LRU fixes + evictions of request i between barriers 2 and 1;
    // its decision record between barriers 1 and 2 of the next request
    // (beside warp 0's commit), when warp 0 writes the other scratch buffer
    bool have = false;
    i64 pli = 0;
    Dec pdec;
    const Scr* psb = nullptr;
    PHASE_MARK1(23);
    // the evictions of request ci start as soon as warp 0's path update of
    // ci is done (the LRU fixes before them); the rest of warp 0's commit
    // (path log, window slot, hint row) touches nothing an eviction reads.
    // The criterion-7 FIFO driver reads request ci's tail slot, written at
    // the very end of the commit: there the evictions wait for commit_done.
    const bool early = a.eviction != E2_EVICT_FIFO_TAIL;
    for (i64 ci = 0;; ++ci) {
      bar_pair(1);
      PHASE_MARK1(23);  // waiting
      if (have) replay_out(psb, a, pli, pdec);
      PHASE_MARK1(22);  // decision record
      // wait for warp 0's path update of ci; meanwhile apply its deferred
      // re-keying of a split suffix (lane 0 reads the flags: warp-uniform)
      for (;;) {
        u32 st = 0;
        if (lane0())
          st = (pp->fix_ready == ci + 1 ? 1u : 0u) | (*(volatile i32*)&pp->stop ? 2u : 0u) |
               (g_rkd.pending ? 4u : 0u);
        st = shfl(st, 0);
        if (st & 4u) {
          rekey_deferred();
          continue;
        }
        if (st & 3u) break;
        wait_pause();
      }
      acquire_after_poll();
      PHASE_MARK1(31);  // waiting for warp 0's path update
      bool go = pp->fix_ready == ci + 1 && !*(volatile i32*)&pp->stop;
      if (go && pp->fs->fix_D > 0) path_lru_fix(pp->fs, pp->fs->fix_D, pp->fg);
      PHASE_MARK1(20);  // LRU fixes
      if (lane0()) {
        __threadfence_block();
        pp->w1_fixed = ci + 1;  // warp 0 may reuse the scratch buffers
      }
      wsync();
      if (go && !early) {
        while (pp->commit_done != ci + 1 && !*(volatile i32*)&pp->stop) wait_pause();
        acquire_after_poll();
        go = pp->commit_done == ci + 1;
      }
      if (!go || !pp->c_ok || *(volatile i32*)&HOT.err) {
        if (shfl((u32)g_rkd.pending, 0)) rekey_deferred();  // keep the LRU index consistent
        if (g_ctd.pending) {  // the failing request's leaf: keep the table consistent
          child_insert(g_ctd.parent, g_ctd.tok, g_ctd.child);
          if (lane0()) g_ctd.pending = 0;
          wsync();
        }
        break;
      }
      if (lane0()) g_ntouch = 0;
      wsync();
      if (g_ctd.pending) {  // warp 0's deferred child-table insert of request ci's leaf
        child_insert(g_ctd.parent, g_ctd.tok, g_ctd.child);
        if (lane0()) g_ctd.pending = 0;
        wsync();
      }
      const Scr* sb = pp->s;
      pli = pp->li;
      pdec = pp->dec;
      psb = sb;
      have = true;
      replay_evict(a, pp->li, pp->g);
      PHASE_MARK1(21);  // evictions
    }
    bar_pair(2);  // final rendezvous: warp 0 waits for the last decision record
    return;
  }
  i64 i = 0, fail = -1;
  bool pre_done = false;  // warp 1 ran this request's replay_pre
  for (; i < a.n; ++i) {
    Scr* s = s2 + (i & 1);  // warp 1 reads the other buffer (request i-1) meanwhile
    if (lane0()) g_pf_cur = i;
    // warp 3 applied request i-1's bookkeeping (and, if deferred, prepared
    // this request's `now` and loads)
    if (i > 0) {
      while (pp->books_done < i) wait_pause();
      acquire_after_poll();
      PHASE(30);  // waiting for warp 3's bookkeeping
      // warp 1 finished reading the scratch this request reuses (request
      // i-2's decision record, request i-1's LRU fixes)
      while (pp->w1_fixed < i) wait_pause();
      acquire_after_poll();
      PHASE(18);  // waiting for warp 1's LRU fixes / decision record
    }
    const double now = pre_done ? s->pre_now : replay_pre(s, a, i);
    // decide speculatively while warp 1 evicts for request i-1
    Dec dec;
    Walk w;
    const bool specd = i > 0;
    if (specd) {
      const i64 r = a.base + i;
      dec = decide(s, DEV.tok + a.off[r], a.len[r], a.L[i], a.hint + i * a.hstride, a.hstride, a.S[i], now, w, true,
                   a.lead ? a.lead + i : nullptr, a.hint);
    }
    if (specd && !s->spec_bad && s->spec_walked) prefetch_commit(s, w);  // only after a complete walk
    PHASE(1);
    bar_pair(1);
    PHASE(16);  // waiting for the previous request's eviction
    if (HOT.err) {  // evict(i-1) failed
      fail = i - 1;
      break;
    }
    bool ok;
    const bool walked = specd && s->spec_walked;
    const bool conflict = walked && spec_conflict(s);
    if (conflict) PHASE_COUNT(43);  // the eviction touched the decided path
    bool valid = specd && !s->spec_bad && !conflict;
    if (valid) {
      if (DEV.cfg.mode == 0 && lane0()) HOT.stats[kStTreeReads]++;
      wsync();
      PHASE(34);  // validation
    } else {
      PHASE_COUNT(17);  // speculation redone (keeping its walk when the path is untouched)
      const i64 r = a.base + i;
      dec = decide(s, DEV.tok + a.off[r], a.len[r], a.L[i], a.hint + i * a.hstride, a.hstride, a.S[i], now, w, false,
                   a.lead ? a.lead + i : nullptr, a.hint, walked && !conflict);
    }
    // hand the inflight record (prefix root known before the insert: the
    // first matched level keeps its id through a split at L; with nothing
    // matched it is the new leaf, id next_id) and this step's note_finished
    // to warp 1, which applies them beside this warp's tree insert
    {
      const i64 r = a.base + i;
      const i64 L = a.L[i];
      const bool defer = dec.ok && DEV.cfg.mode == 0 && a.len[r] > 0 && s->npath >= 0 && (L == 0 || s->npath > 0);
      u64 root = 0;
      if (defer) root = L > 0 ? nget(PSLOT(s, 0))->id : HOT.next_id;
      if (dec.ok && lane0()) {
        pp->c_id = a.ids[r];
        pp->c_g = dec.gpu;
        pp->c_cached = dec.cached_len;
        pp->c_n = a.len[r];
        pp->c_arr = a.arr[r];
        pp->c_root = root;
        pp->c_now = now;
        pp->c_defer = defer ? 1 : 0;
        if (defer) {
          // the scheduled-window entry first: warp 1's redirect upkeep of
          // the next request reads the windows (commit fills in its slot
          // and path-log length)
          s->widx = HOT.ws_tail[dec.gpu];
          win_add_sched(dec.gpu, now, dec.moc, DEV.cfg.default_out, kNil, kNil);
          s->win_done = 1;
        }
        __threadfence_block();
        if (defer) pp->ready = i + 1;
      }
      wsync();
      pre_done = defer && i + 1 < a.n;
      PHASE(35);  // hand-off
      if (lane0()) {
        pp->fs = s;
        pp->fg = dec.gpu;
        s->fix_D = 0;  // nothing to re-index unless path_update_par defers it
        // what warp 1 needs for this request's decision record and evictions
        pp->li = i;
        pp->g = dec.gpu;
        pp->dec = dec;
        pp->s = s;
        pp->c_ok = dec.ok ? 1 : 0;
      }
      wsync();
      ok = dec.ok && replay_main(s, a, i, now, dec, &w, E2_DEFER_LRU, defer, E2_DEFER_LRU ? &pp->fix_ready : nullptr);
      // commits that raised no hand-off (no level-parallel path update, round
      // robin, a failed decide): release warp 1 with nothing to re-index
      if (lane0() && pp->fix_ready != i + 1) {
        __threadfence_block();
        pp->fix_ready = i + 1;
      }
      wsync();
      // not deferred (round robin, very deep paths): the commit wrote the
      // inflight record itself; only then may warp 1 apply note_finished
      if (dec.ok && !defer) {
        if (lane0()) {
          __threadfence_block();
          pp->ready = i + 1;
        }
        wsync();
      }
    }
    if (!ok || HOT.err) {
      fail = i;
      break;
    }
    if (lane0()) {
      __threadfence_block();
      pp->commit_done = i + 1;
    }
    wsync();
    PHASE(37);
  }
  if (fail < 0) bar_pair(1);  // wait for the last evict
  if (HOT.err && fail < 0) fail = a.n - 1;  // the last evict failed
  if (lane0()) {
    __threadfence_block();
    pp->stop = 1;
    g_pf_stop = 1;
  }
  wsync();
  bar_pair(2);
  if (lane0()) {
    HOT.done = fail < 0 ? a.n : fail;
    if (fail >= 0) HOT.err_req = a.base + fail;
  }
  wsync();
}
#endif

E2_D void serial_body(Scr* s, const SerialArgs& a, void* pipe = nullptr) {
  if (thread0()) HOT.done = 0;
  wsync();
  if (a.kind == 0) {
#if E2_WARP
    if (pipe) {
      replay_pipe(s, a, (Pipe*)pipe);
      nflush();
      return;
    }
#endif
    replay_seq(s, a);
  } else {
    api_op(s, a.op, a.hint, a.hstride, a.out, a.L);
    if (lane0()) HOT.done = HOT.err ? 0 : 1;
    wsync();
  }
  nflush();
}

}  // namespace e2
