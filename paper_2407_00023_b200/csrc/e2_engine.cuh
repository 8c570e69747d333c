// e2_engine.cuh — the serial E2 semantics (decide + commit + callbacks +
// batched driver) executed by one warp over the HBM-resident state.
//
// Every operation reproduces one reference call with identical state
// effects; floating point uses explicit round-to-nearest intrinsics in the
// reference's operation order.  Token comparisons never happen here: every
// walk is given its matched length (and K1's path hints) by the batched
// match kernels (e2_match.cuh), so a walk costs no child-table probe when
// the hinted path is still current.
#pragma once

#include "e2_tree.cuh"

namespace e2 {

// Warp-shared per-decision scratch (shared memory on device).
struct Scr {
  double loads[kMaxG];
  double ratios[kMaxG];
  i64 ext[kMaxG];
  i32 cgpu[kMaxG + 1];
  i32 cinf[kMaxG + 1];
  double cL[kMaxG + 1], cM[kMaxG + 1], cP[kMaxG + 1];
  i32 n_costs;
  i32 loads_ok;  // loads[] hold load_ms at this request's `now` (update_redirects ran)
  i32 spec_bad;  // a speculative decide gave up (see decide)
  i32 spec_walked;  // ... after a complete walk that probed no table (reusable if the path is untouched)
  i32 fix_D;     // path levels whose LRU fixes path_update_par deferred (0: none)
  i32 cpath;     // levels of the committed path in pslot (-1: not recorded)
  i32 win_done;  // the scheduled-window entry was appended before the commit (pipelined replay)
  u64 widx;      // its ring position: commit fills in the tail slot and path-log length
  double pre_now;  // this request's `now`, computed by replay_pre on the other warp
  i32 npath;  // levels recorded by walk_par (-1: path too deep, sequential fallback)
  // the request's root path, top-down (walk_par / commit)
  u32 pslot[kMaxPath + 1];
  u32 pm[kMaxPath];  // tokens matched in the level
  u64 pcm[kMaxPath];  // caching mask of the level
  u64 pla0[kMaxPath + 1];  // path_update: old last_access bits
  u32 pflag[kMaxPath + 1];  // path_update: bit0 newly cached, bit1 leaf before, bit2 leaf after, bit3 key moved
};

// Per-level path arrays: levels [0, kMaxPath) in shared memory (Scr),
// deeper ones in the handle's global overflow; max depth kMaxPath + kXPath.
#define PSLOT(s, i) (*((i) < kMaxPath ? &(s)->pslot[(i)] : &DEV.xp_slot[(i)-kMaxPath]))
#define PM(s, i) (*((i) < kMaxPath ? &(s)->pm[(i)] : &DEV.xp_m[(i)-kMaxPath]))
#define PCM(s, i) (*((i) < kMaxPath ? &(s)->pcm[(i)] : &DEV.xp_cm[(i)-kMaxPath]))
#define PLA0(s, i) (*((i) < kMaxPath ? &(s)->pla0[(i)] : &DEV.xp_la0[(i)-kMaxPath]))
#define PFLAG(s, i) (*((i) < kMaxPath ? &(s)->pflag[(i)] : &DEV.xp_flag[(i)-kMaxPath]))
constexpr int kPathLevels = kMaxPath + (int)kXPath;

// Result of a node-level walk with a known matched length.
struct Walk {
  u32 last;        // deepest node touched (kRoot when nothing matched)
  i64 last_m;      // tokens matched inside `last`
  i64 cached_len;  // Σ spans cached somewhere (prefix_tree.cpp:104-106)
  u64 present;     // gpus with a per_gpu_matched_len entry (first span's set)
  bool ok;
};

// ---------------------------------------------------------------------------
// Load windows — LoadWindow (cost_model.cpp:20-73).  Single-lane.
// ---------------------------------------------------------------------------
E2_HD u64 wslot(int g, u64 i) { return (u64)g * DEV.wcap + (i & (DEV.wcap - 1)); }

constexpr double kInf = __builtin_huge_val();

// prune (cost_model.cpp:31-42): inclusive horizon, t >= now - H survives.
// Hit stamps of pruned entries are undone lazily (hits_catchup).
E2_HD void win_prune(int g, double now) {
  const double cutoff = dsub(now, DEV.cfg.H);
  if (HOT.ws_head_t[g] < cutoff) {
    u64 hd = HOT.ws_head[g];
    const u64 tl = HOT.ws_tail[g];
    double t = HOT.ws_head_t[g];
    while (hd < tl && t < cutoff) {
      const i64 m = DEV.win[wslot(g, hd)].missed;
      HOT.ws_missed_sum[g] -= m;
      if (m > 0) HOT.ws_missed_nz[g] -= 1;
      hd++;
      t = hd < tl ? DEV.win[wslot(g, hd)].t : kInf;
    }
    HOT.ws_head[g] = hd;
    HOT.ws_head_t[g] = t;
  }
  if (HOT.wc_head_t[g] < cutoff) {
    u64 ch = HOT.wc_head[g];
    const u64 ct = HOT.wc_tail[g];
    double t = HOT.wc_head_t[g];
    while (ch < ct && t < cutoff) {
      HOT.wc_output_sum[g] -= DEV.comp[wslot(g, ch)].out;
      ch++;
      t = ch < ct ? DEV.comp[wslot(g, ch)].t : kInf;
    }
    HOT.wc_head[g] = ch;
    HOT.wc_head_t[g] = t;
  }
}

// load_ms (cost_model.cpp:65-73) — prefill folded from integer sums, decode
// = count * (c2 * avg_output).
E2_HD double win_load(int g, double now) {
  win_prune(g, now);
  const Cfg& c = DEV.cfg;
  const i64 nsched = (i64)(HOT.ws_tail[g] - HOT.ws_head[g]);
  const i64 ncomp = (i64)(HOT.wc_tail[g] - HOT.wc_head[g]);
  const double prefill = dadd(dmul(c.c0, i2d(HOT.ws_missed_nz[g])), dmul(c.c1, i2d(HOT.ws_missed_sum[g])));
  const double avg = ncomp == 0 ? i2d(c.default_out) : ddiv(i2d(HOT.wc_output_sum[g]), i2d(ncomp));
  const double decode = dmul(i2d(nsched), dmul(c.c2, avg));
  return dadd(prefill, decode);
}

E2_HD bool win_add_sched(int g, double now, i64 missed, i64 est, u32 tail, u32 plen) {
  const u64 t = HOT.ws_tail[g];
  if (t - HOT.ws_done[g] >= DEV.wcap) {
    set_err(kErrCapacity, kWhyWindowCap);
    return false;
  }
  WinEnt e;
  e.t = now;
  e.missed = missed;
  e.est = est;
  e.slot = tail;
  e.plen = plen;
  DEV.win[wslot(g, t)] = e;
  if (t == HOT.ws_head[g]) HOT.ws_head_t[g] = now;
  HOT.ws_tail[g] = t + 1;
  HOT.ws_missed_sum[g] += missed;
  if (missed > 0) HOT.ws_missed_nz[g] += 1;
  return true;
}

E2_HD bool win_add_comp(int g, double now, i64 out) {
  const u64 t = HOT.wc_tail[g];
  if (t - HOT.wc_head[g] >= DEV.wcap) {
    set_err(kErrCapacity, kWhyWindowCap);
    return false;
  }
  CompEnt e;
  e.t = now;
  e.out = out;
  DEV.comp[wslot(g, t)] = e;
  if (t == HOT.wc_head[g]) HOT.wc_head_t[g] = now;
  HOT.wc_tail[g] = t + 1;
  HOT.wc_output_sum[g] += out;
  return true;
}

// hits(n, g) counts in-window requests placed on g whose prompt passes
// through n.  Undo the stamps of requests that left g's
// window since the last catch-up.  A logged entry's path (top-down slots
// at commit) is decremented level-parallel; splits since then inserted
// prefix nodes above some logged slots (they copied the stamp), found as
// the parent chain between consecutive logged slots.  Unlogged entries walk
// the parent chain from their tail slot.  Warp-wide.
E2_DNI void hits_catchup_one(int g);

E2_DNI void hits_catchup(int g) {
  const int G = DEV.cfg.G;
#if E2_WARP
  // Several expired entries per warp step: consecutive entries' logged paths
  // are contiguous in the path-log ring, so lane l takes ring position
  // pl_head + l and the group undoes up to kWidth levels in one pass (the
  // decrements are atomic: the group's paths share their upper nodes).
  constexpr int kGroup = 8;
  while (HOT.ws_done[g] < HOT.ws_head[g]) {
    const u64 d0 = HOT.ws_done[g];
    const int avail = (int)min_<u64>(HOT.ws_head[g] - d0, (u64)kGroup);
    u32 plen = kNil;
    if (lane() < avail) plen = DEV.win[wslot(g, d0 + (u64)lane())].plen;
    // take entries while they are logged and their levels fit the warp
    u32 take = 0, total = 0;
    for (int j = 0; j < avail; ++j) {
      const u32 pj = shfl(plen, j);
      if (pj == kNil || total + pj > (u32)kWidth) break;
      total += pj;
      take++;
    }
    if (take == 0) {
      // an unlogged entry, or one path longer than a warp: one entry, as below
      hits_catchup_one(g);
      continue;
    }
    // lane l: its entry's first level?  (exclusive prefix sums of plen)
    bool first = false;
    {
      u32 acc = 0;
      for (u32 j = 0; j < take; ++j) {
        if ((u32)lane() == acc) first = true;
        acc += shfl(plen, (int)j);
      }
    }
    const u64 h0 = HOT.pl_head[g], pmask = DEV.pcap - 1;
    const u32* ring = DEV.plog + (u64)g * DEV.pcap;
    if ((u32)lane() < total) {
      const u32 v = ring[(h0 + (u64)lane()) & pmask];
      const u32 up = first ? kRoot : ring[(h0 + (u64)lane() - 1) & pmask];
      NodeRec* r = npoke(v);
      atomicAdd(&rhits(r, G)[g], -1);
      // prefix halves a split inserted above v since the commit
      for (u32 p = r->parent; p != up && p != kRoot && p != kNil;) {
        NodeRec* rp = npoke(p);
        atomicAdd(&rhits(rp, G)[g], -1);
        p = rp->parent;
      }
    }
    wsync();
    if (lane0()) {
      HOT.pl_head[g] = h0 + total;
      HOT.ws_done[g] = d0 + take;
    }
    wsync();
  }
#else
  while (HOT.ws_done[g] < HOT.ws_head[g]) hits_catchup_one(g);
#endif
}

// One expired window entry of instance g: undo its hit stamps.
E2_DNI void hits_catchup_one(int g) {
  const int G = DEV.cfg.G;
  {
    const WinEnt e = DEV.win[wslot(g, HOT.ws_done[g])];
    if (e.plen != kNil) {
      const u64 h0 = HOT.pl_head[g], pmask = DEV.pcap - 1;
      const u32* ring = DEV.plog + (u64)g * DEV.pcap;
      for (u32 b = 0; b < e.plen; b += kWidth) {
        const u32 i = b + (u32)lane();
        if (i < e.plen) {
          const u32 v = ring[(h0 + i) & pmask];
          const u32 up = i == 0 ? kRoot : ring[(h0 + i - 1) & pmask];
          NodeRec* r = npoke(v);
          rhits(r, G)[g] -= 1;
          for (u32 p = r->parent; p != up && p != kRoot && p != kNil;) {
            NodeRec* rp = npoke(p);
            rhits(rp, G)[g] -= 1;
            p = rp->parent;
          }
        }
      }
      wsync();
      if (lane0()) HOT.pl_head[g] = h0 + e.plen;
    } else {
      for (u32 n = e.slot; n != kRoot && n != kNil;) {
        NodeRec* r = nget(n);
        const u32 p = r->parent;
        if (lane0()) {
          rhits(r, G)[g] -= 1;
          ndirty(r);
        }
        wsync();
        n = p;
      }
    }
    if (lane0()) HOT.ws_done[g]++;
    wsync();
  }
}

// Append a committed path (top-down slots) to g's path log; returns the
// logged length, or kNil when the ring has no room (the entry then falls
// back to the parent-chain walk).  Warp-wide.
E2_DNI u32 plog_append(Scr* s, int D, int g) {
  const u64 t = HOT.pl_tail[g];
  if (D < 0 || DEV.pcap == 0 || t + (u64)D - HOT.pl_head[g] > DEV.pcap) return kNil;
  u32* ring = DEV.plog + (u64)g * DEV.pcap;
  for (int i = lane(); i < D; i += kWidth) ring[(t + (u64)i) & (DEV.pcap - 1)] = PSLOT(s, i);
  wsync();
  if (lane0()) HOT.pl_tail[g] = t + (u64)D;
  wsync();
  return (u32)D;
}

E2_HD double prefill_time(const Cfg& c, i64 missed) {
  if (missed <= 0) return 0.0;
  return dadd(c.c0, dmul(c.c1, i2d(missed)));
}

// ---------------------------------------------------------------------------
// Eviction planning — PrefixTree::plan_eviction (prefix_tree.cpp:273-308).
// Single-lane, read-only on the tree (npeek); per-instance scratch holds the
// surfaced-parent work list (sorted) and the simulated cached-child counts.
// visit(slot, tokens) is called per plan entry in plan order.
// Returns freed tokens.
// ---------------------------------------------------------------------------
template <typename Visit>
E2_HD i64 plan_eviction(int g, i64 need, bool partial, Visit&& visit) {
  if (need <= 0) return 0;
  const int G = DEV.cfg.G;
  const u32 half = DEV.scap / 2;
  u32* s_slot = DEV.scr_slot + (u64)g * DEV.scap;  // [0,half): surfaced list, [half,scap): sim ccc
  u64* s_la = DEV.scr_la + (u64)g * DEV.scap;
  u64* s_id = DEV.scr_id + (u64)g * DEV.scap;
  i64* s_val = DEV.scr_val + (u64)g * DEV.scap;
  u32 ns = 0, nsurf_head = 0, nsim = 0;
  // simulated cached-child counts of the parents met so far: the first kLin
  // in a list (short plans: a few L1-resident compares), the rest in an
  // open-addressing table keyed (plan generation << 32 | slot), so keys of
  // earlier plans read as empty and the table needs no clearing
  constexpr u32 kLin = 16;
  const u64 tmask = (u64)((DEV.scap - half) / 2) - 1;  // table entries: a power of two below scap - half - kLin
  u64 gen = 0;  // taken when the table is first used by this plan
  const u32 nd = HOT.dir_n[g];
  u32 k = 0, j = 0, page = kNil;
  i32 pcnt = 0;
  if (nd > 0) {
    const DirEntry e = DEV.dir[dring(g, 0)];
    page = e.page;
    pcnt = e.cnt;
  }
  i64 freed = 0;
  while (freed < need) {
    const bool have_a = page != kNil;
    const bool have_b = nsurf_head < ns;
    if (!have_a && !have_b) break;
    u32 v;
    bool take_b = false;
    if (have_a && have_b) {
      const u64 ai = (u64)page * kPage + j;
      take_b = kless(s_la[nsurf_head], s_id[nsurf_head], DEV.pg_la[ai], DEV.pg_id[ai]);
    } else {
      take_b = have_b;
    }
    if (take_b) {
      v = s_slot[nsurf_head++];
    } else {
      v = DEV.pg_slot[(u64)page * kPage + j];
      if (++j >= (u32)pcnt) {
        j = 0;
        if (++k < nd) {
          const DirEntry e = DEV.dir[dring(g, k)];
          page = e.page;
          pcnt = e.cnt;
        } else {
          page = kNil;
        }
      }
    }
    const NodeRec* rv = npeek(v);
    const i64 tok = rv->edge_len;
    const i64 remaining = need - freed;
    if (partial && tok > remaining) {
      visit(v, remaining, rv);
      freed += remaining;
      break;
    }
    visit(v, tok, rv);
    freed += tok;
    const u32 p = rv->parent;
    if (p != kNil && p != kRoot) {
      const NodeRec* rp = npeek(p);
      if (!rcached(rp, g)) continue;
      const u32 nlin = min_(nsim, kLin);
      u64 xi = 0;
      while (xi < nlin && s_slot[half + xi] != p) ++xi;
      bool found = xi < nlin;
      if (!found && nsim >= kLin) {
        if (gen == 0) gen = ++s_la[half];  // this instance's plan counter (s_la's upper half is unused)
        const u64 key = (gen << 32) | (u64)p;
        u64 h = mix64((u64)p) & tmask;
        for (;;) {
          const u64 kk = s_id[half + kLin + h];
          if (kk == key || (kk >> 32) != gen) break;  // found, or a free entry (another plan's key)
          h = (h + 1) & tmask;
        }
        xi = kLin + h;
        found = s_id[half + xi] == key;
        if (!found) {
          if ((u64)(nsim - kLin) * 2 >= tmask + 1) {
            set_err(kErrCapacity, kWhyScratchCap);
            break;
          }
          s_id[half + xi] = key;
        }
      }
      i64 c;
      if (found) {
        c = s_val[half + xi] - 1;
      } else {
        c = (i64)rccc(rp, G)[g] - 1;
        if (nsim < kLin) s_slot[half + nsim] = p;  // xi == nsim: the list's next entry
        nsim++;
      }
      s_val[half + xi] = c;
      if (c == 0) {
        // sorted insert into the pending part of the surfaced list
        if (ns >= half) {
          set_err(kErrCapacity, kWhyScratchCap);
          break;
        }
        const u64 pla = dbits(rla(rp)[g]), pid = rp->id;
        u32 pos = ns;
        while (pos > nsurf_head && kless(pla, pid, s_la[pos - 1], s_id[pos - 1])) {
          s_la[pos] = s_la[pos - 1];
          s_id[pos] = s_id[pos - 1];
          s_slot[pos] = s_slot[pos - 1];
          --pos;
        }
        s_la[pos] = pla;
        s_id[pos] = pid;
        s_slot[pos] = p;
        ns++;
      }
    }
  }
  return freed;
}

// load_cost (cost_model.cpp:75-100).  Single-lane; when need > 0 the
// caller has run hits_catchup(g) (cost_prepare).
struct CostOut {
  double L, M, P;
  bool inf;
};

E2_HD CostOut cost_for(int g, i64 missed, double now, const Scr* s = nullptr) {
  CostOut o;
  // update_redirects already computed load_ms(g, now) this request; nothing
  // touches the windows between it and the cost evaluation
  o.L = (s && s->loads_ok) ? s->loads[g] : win_load(g, now);
  o.P = prefill_time(DEV.cfg, missed);
  o.M = 0.0;
  o.inf = false;
  const i64 free_tokens = DEV.cfg.cap - HOT.cached_tokens[g];
  const i64 need = missed - free_tokens;
  if (need > 0) {
    const i64 total = (i64)(HOT.ws_tail[g] - HOT.ws_head[g]);  // scheduled_count (already pruned)
    const Cfg& c = DEV.cfg;
    const int G = c.G;
    double M = 0.0;
    const i64 freed = plan_eviction(g, need, false, [&](u32, i64 tok, const NodeRec* rv) {
      if (total > 0) {
        const double nj = ddiv(i2d(rhits(rv, G)[g]), i2d(total));
        M = dadd(M, dmul(prefill_time(c, tok), nj));
      }
    });
    o.M = M;
    o.inf = freed < need;
  }
  return o;
}

// Warp-wide: make g's windowed hit counters current before a cost with an
// eviction term is evaluated.
E2_DNI void cost_prepare(int g, i64 missed, double now) {
  if (lane0()) win_prune(g, now);
  wsync();
  if (missed - (DEV.cfg.cap - HOT.cached_tokens[g]) > 0) hits_catchup(g);
}

// Warp-wide, for every instance in `set` (missed = n - ext[g]): prune its
// window and, only where the eviction term will be evaluated (need > 0),
// bring its hit counters current.
E2_DNI void cost_prepare_set(const Scr* s, u64 set, i64 n, double now) {
  const int G = DEV.cfg.G;
  u64 needm = 0;
  for (int b = 0; b < G; b += kWidth) {
    const int g = b + lane();
    bool need = false;
    if (g < G && ((set >> g) & 1ull)) {
      win_prune(g, now);
      need = (n - s->ext[g]) - (DEV.cfg.cap - HOT.cached_tokens[g]) > 0 && HOT.ws_done[g] < HOT.ws_head[g];
    }
    needm |= (u64)ballot(need) << b;
  }
  wsync();
  for (u64 m = needm; m; m &= m - 1) hits_catchup(ffs64(m));
}

// ---------------------------------------------------------------------------
// Walks (warp-wide).  `L` = matched length of the sequence against the
// current tree, from the batched match; prefix_tree.cpp:79-114.  `hint`
// holds K1's path slots (may be stale after in-batch splits; validated).
// ---------------------------------------------------------------------------
E2_DNI Walk walk_known(const i32* seq, i64 L, const u32* hint, int nhint, i64* ext) {
  Walk w;
  w.last = kRoot;
  w.last_m = 0;
  w.cached_len = 0;
  w.present = 0;
  w.ok = true;
  const int G = DEV.cfg.G;
  for (int g = lane(); g < G; g += kWidth) ext[g] = 0;
  u64 alive = 0;
  bool first_span = true;
  i64 pos = 0;
  u32 cur = kRoot;
  int level = 0;
  bool live = hint != nullptr;  // hints end at K1's kNil terminator
  while (pos < L) {
    const i32 t = seq[pos];
    u32 ch = kNil;
    const NodeRec* r = nullptr;
    if (live && level < nhint) {
      const u32 c = hint[level];
      if (c != kNil) {
        r = nget(c);
        if (r->parent == cur && r->first_tok == t && r->edge_len > 0) ch = c;
      } else {
        live = false;
      }
    }
    if (ch == kNil) {
      note_probe();
      ch = child_lookup(cur, t);
      if (ch == kNil) {
        w.ok = false;
        break;
      }
      r = nget(ch);
    }
    const i64 len = r->edge_len;
    const i64 m = min_(len, L - pos);
    const u64 cm = r->cmask;
    if (first_span) {
      alive = cm;
      w.present = cm;
      first_span = false;
    } else {
      alive &= cm;
    }
    for (int g = lane(); g < G; g += kWidth)
      if ((alive >> g) & 1ull) ext[g] += m;
    if (cm != 0) w.cached_len += m;
    pos += m;
    cur = ch;
    w.last = ch;
    w.last_m = m;
    level++;
    if (m < len) break;
  }
  wsync();
  return w;
}

#if E2_WARP
E2_D i64 warp_incl_sum(i64 v) {
  for (int o = 1; o < 32; o <<= 1) {
    const i64 u = (i64)__shfl_up_sync(0xffffffffu, (long long)v, o);
    if (lane() >= o) v += u;
  }
  return v;
}
E2_D i64 warp_sum(i64 v) {
  for (int o = 16; o; o >>= 1) v += (i64)__shfl_xor_sync(0xffffffffu, (long long)v, o);
  return v;
}
#endif

// Walk with a known matched length, level-parallel (warp-wide): 32 hinted
// levels are loaded and validated at once (parent chain, first token,
// position from a prefix sum of edge lengths); levels without a valid hint
// fall back to one child-table probe each.  Records the path top-down in
// s->pslot/pm/pcm and derives the per-gpu extents and cached_len from it
// (prefix_tree.cpp:79-114).  s->npath = -1 when the path exceeds kMaxPath:
// the caller then uses the sequential walk.
// hS: K1's snapshot match length.  A hinted slot is on this prompt's path
// only while its (current) start lies below hS: the last hint may be a node
// K1 matched only partially, whose slot now holds the part past hS.
// Leader hints: the committed path of the request's in-batch leader (LCP =
// L), used past the point where its own K1 hints end (bound L instead of
// hS).  lead points at the request's leader index (-1: none); the leader's
// row is hint_rows + leader * nhint.  Read only when needed.
E2_DNI Walk walk_par(const i32* seq, i64 L, const u32* hint, int nhint, Scr* s, i64 hS,
                     const i64* lead = nullptr, const u32* hint_rows = nullptr) {
  const u32* hint2 = nullptr;
  Walk w;
  w.last = kRoot;
  w.last_m = 0;
  w.cached_len = 0;
  w.present = 0;
  w.ok = true;
  const int G = DEV.cfg.G;
  int np = 0, hi = 0;  // path levels recorded, hints consumed
  i64 pos = 0;
  u32 cur = kRoot;
  bool fast = hint != nullptr;
  bool done = false;
  constexpr u32 kFull = kWidth == 32 ? 0xffffffffu : 1u;
  while (pos < L && !done) {
    if (np >= kPathLevels) {
      if (lane0()) s->npath = -1;
      wsync();
      w.ok = false;
      return w;
    }
    if (fast && hi < nhint) {
      // kWidth hinted levels at once, one per lane
      const int k = lane(), lvl = hi + k;
      const u32 c = lvl < nhint ? hint[lvl] : kNil;
      // K1 terminates the hint list with kNil; nothing after it is read
      const u32 nilm = ballot(c == kNil);
      const bool in = k < (nilm ? ffs32(nilm) : kWidth) && np + k < kPathLevels;
      u32 par = kNil;
      i64 len = 0, pk = 0;
      u64 cm = 0;
      if (in) {
        const NodeRec* r = npeek(c);
        par = r->parent;
        len = r->edge_len;
        cm = r->cmask;
        pk = r->depth;
      }
      // A hint is K1's node for this very prompt.  If its parent is still
      // the previous level's node, no split has cut the chain since K1, so
      // the edge still starts at its stored depth and its first token is
      // the prompt's (K1 followed the child table with it): no token load.
      u32 prev = shfl_up1(c);
      if (k == 0) prev = cur;
      const bool ok = in && par == prev && len > 0 && pk < hS;
      const u32 okm = ballot(ok);
      const int nvalid = (okm == kFull) ? kWidth : ffs32(~okm);
      const u32 lastm = ballot(ok && pk + len >= L) & (nvalid == 32 ? 0xffffffffu : ((1u << nvalid) - 1));
      const int used = lastm ? ffs32(lastm) + 1 : nvalid;
      if (used > 0) {
        const i64 m = min_(len, L - pk);
        if (k < used) {
          PSLOT(s, np + k) = c;
          PM(s, np + k) = (u32)m;
          PCM(s, np + k) = cm;
        }
        const u32 lc = shfl(c, used - 1);
        const i64 lm = shfl(m, used - 1), lp = shfl(pk, used - 1), ll = shfl(len, used - 1);
        wsync();
        np += used;
        hi += used;
        pos = lp + lm;
        cur = lc;
        w.last = lc;
        w.last_m = lm;
        if (lastm) done = true;  // reached L (or the match ends inside this edge)
        if (lm < ll) done = true;
        PHASE_MARK(38);  // walk: hinted levels
        continue;
      }
      // The next hint does not hang off `cur`.  Splits since K1 keep every
      // hinted slot on the path (the slot keeps the suffix, whose end is
      // unchanged) and insert the prefix halves above it: climb from the
      // hint's parent to `cur` and take the inserted nodes as levels.
      const bool in0 = shfl((int)in, 0) != 0;
      const u32 p0 = shfl(par, 0);
      const i64 l0 = shfl(len, 0);
      if (!in0 || l0 == 0 || p0 == cur || p0 == kNil) {
        if (lead && !hint2) {
          const i64 ld = *lead;
          hint2 = ld >= 0 ? hint_rows + ld * (i64)nhint : hint;
        }
        if (hint2 && hint != hint2) {
          // switch to the leader's committed path: its entries starting at or
          // after `pos` continue this prompt's path (both share [0, L))
          hint = hint2;
          hS = L;
          // the leader's path is top-down with strictly increasing depths:
          // resume at its first entry starting at or after `pos` (the count
          // of entries starting below it), kWidth entries per step
          int idx = 0;
          for (int b0 = 0; b0 < nhint - 1; b0 += kWidth) {
            const int j = b0 + lane();
            bool below = false;
            if (j < nhint - 1) {
              const u32 c2 = hint[j];
              below = c2 != kNil && (i64)npeek(c2)->depth < pos;
            }
            const u32 bm = ballot(below);
            const int run = (bm == kFull) ? kWidth : ffs32(~bm);
            idx = b0 + run;
            if (run < kWidth) break;
          }
          hi = min_(idx, nhint - 1);
          PHASE_MARK(39);  // walk: switch to the leader's committed path
          continue;
        }
        fast = false;
        continue;
      }
      int nc = 0;
      u32 x = p0;
      while (x != cur && x != kRoot && x != kNil && np + nc < kPathLevels) {
        if (lane0()) PSLOT(s, np + nc) = x;
        nc++;
        x = npeek(x)->parent;
      }
      wsync();
      if (x != cur || nc == 0) {
        fast = false;
        continue;
      }
      // the chain was recorded bottom-up: reverse it in place, then take its
      // levels top-down, kWidth per step, while they start below hS
      for (int j = lane(); j < nc / 2; j += kWidth) {
        const u32 t0 = PSLOT(s, np + j), t1 = PSLOT(s, np + nc - 1 - j);
        PSLOT(s, np + j) = t1;
        PSLOT(s, np + nc - 1 - j) = t0;
      }
      wsync();
      for (int c0 = 0; c0 < nc && !done;) {
        const int j = c0 + k, chunk = min_(nc - c0, kWidth);
        u32 v = kNil;
        i64 vl = 0, vp = 0;
        u64 vc = 0;
        if (k < chunk) {
          v = PSLOT(s, np + k);
          const NodeRec* r = npeek(v);
          vl = r->edge_len;
          vc = r->cmask;
          vp = r->depth;
        }
        (void)j;
        const u32 okc = ballot(k < chunk && vp < hS);
        const int nvc = (okc == kFull) ? kWidth : ffs32(~okc);
        if (nvc == 0) {
          fast = false;
          break;
        }
        const u32 lastc = ballot(k < nvc && vp + vl >= L);
        const int usedc = lastc ? ffs32(lastc) + 1 : nvc;
        const i64 mc = min_(vl, L - vp);
        if (k < usedc) {
          PM(s, np + k) = (u32)mc;
          PCM(s, np + k) = vc;
        }
        const u32 lc = shfl(v, usedc - 1);
        const i64 lm = shfl(mc, usedc - 1), lp = shfl(vp, usedc - 1), ll = shfl(vl, usedc - 1);
        wsync();
        np += usedc;
        c0 += usedc;
        pos = lp + lm;
        cur = lc;
        w.last = lc;
        w.last_m = lm;
        if (lastc) done = true;
        if (lm < ll) done = true;
        if (usedc < chunk) break;  // a chain node starts past hS: re-evaluated next pass
      }
      PHASE_MARK(40);  // walk: climb across splits
      continue;
    }
    // no usable hint: one child-table probe per level
    const i32 t = seq[pos];
    PHASE_COUNT(12);
    note_probe();
    const u32 ch = child_lookup(cur, t);
    if (ch == kNil) {
      w.ok = false;
      break;
    }
    const NodeRec* r = nget(ch);
    const i64 len = r->edge_len;
    const i64 m = min_(len, L - pos);
    const u64 cm = r->cmask;
    if (lane0()) {
      PSLOT(s, np) = ch;
      PM(s, np) = (u32)m;
      PCM(s, np) = cm;
    }
    wsync();
    np++;
    pos += m;
    cur = ch;
    w.last = ch;
    w.last_m = m;
    if (m < len) break;
  }
  PHASE_MARK(41);  // walk: child-table probes
  if (lane0()) s->npath = np;
  wsync();
  if (!w.ok) return w;
  // extents: a gpu accumulates while every level so far is cached on it;
  // entries exist for the gpus caching the first span
  w.present = np > 0 ? PCM(s, 0) : 0;
#if E2_WARP
  if (np <= 8 && G <= 32) {
    // shallow path: lane g walks the levels itself (no scans); every lane
    // also sums cached_len redundantly, so no reduction is needed
    i64 e = 0, cl = 0;
    bool alive = lane() < G && ((w.present >> lane()) & 1ull);
    for (int l = 0; l < np; ++l) {
      const u64 cm = s->pcm[l];
      const i64 m = (i64)s->pm[l];
      alive = alive && ((cm >> lane()) & 1ull);
      if (alive) e += m;
      if (cm != 0) cl += m;
    }
    if (lane() < G) s->ext[lane()] = e;
    w.cached_len = cl;
    wsync();
    return w;
  }
  // level-parallel: alive_l = AND of pcm[0..l] (monotone), P_l = matched
  // tokens through level l; gpu g's extent is P at the last level where it
  // is alive, written by the lane of the level where it drops out.
  for (int g = lane(); g < G; g += kWidth) s->ext[g] = 0;
  wsync();
  {
    u64 carry = ~0ull;
    i64 pcarry = 0;
    for (int b = 0; b < np; b += kWidth) {
      const int l = b + lane();
      const bool in = l < np;
      u64 v = in ? PCM(s, l) : ~0ull;
      for (int o = 1; o < 32; o <<= 1) {
        const u64 u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane() >= o) v &= u;
      }
      v &= carry;
      const i64 P = pcarry + warp_incl_sum(in ? (i64)PM(s, l) : 0);
      const u64 dn = __shfl_down_sync(0xffffffffu, v, 1);
      const u64 an = (l + 1 < np) ? (lane() < 31 ? dn : (v & PCM(s, l + 1))) : 0ull;
      if (in)
        for (u64 d = v & ~an; d; d &= d - 1) s->ext[ffs64(d)] = P;
      carry = shfl(v, 31);
      pcarry = shfl(P, 31);
    }
  }
  wsync();
#else
  for (int g = lane(); g < G; g += kWidth) {
    i64 e = 0;
    if ((w.present >> g) & 1ull)
      for (int l = 0; l < np && ((PCM(s, l) >> g) & 1ull); ++l) e += PM(s, l);
    s->ext[g] = e;
  }
#endif
  i64 cl = 0;
  for (int l = lane(); l < np; l += kWidth)
    if (PCM(s, l) != 0) cl += (i64)PM(s, l);
#if E2_WARP
  cl = warp_sum(cl);
#endif
  w.cached_len = cl;
  wsync();
  return w;
}

// path_update over the recorded path (s->pslot[0..D), top-down), one lane
// per node: same final state as the sequential path_update.  Nodes whose
// LRU membership or key changes are re-indexed afterwards, serially.
// Warp-wide.
// The LRU re-indexing of the path, after path_update_par (deferred variant:
// run by the eviction warp of the pipelined replay before its eviction).
E2_DNI void fix_level(const Scr* s, int i, int g);
E2_DNI void path_lru_fix(const Scr* s, int D, int g) {
  // the flagged levels (usually the last one or two) found kWidth at a time
  for (int b = 0; b < D; b += kWidth) {
    u32 m = ballot(b + lane() < D && (PFLAG(s, b + lane()) & 8u));
    while (m) {
      const int i = b + ffs32(m);
      m &= m - 1;
      fix_level(s, i, g);
    }
  }
}

E2_DNI void fix_level(const Scr* s, int i, int g) {
  {
    const u32 f = PFLAG(s, i);
    const u32 v = PSLOT(s, i);
    const NodeRec* r = nget(v);
    const u64 id = r->id, la1 = dbits(rla(r)[g]);
    if (f & 2u) lru_erase(g, PLA0(s, i), id);
    if (f & 4u) lru_insert(g, la1, id, v);
  }
}

// defer: leave the LRU re-indexing to path_lru_fix (s->fix_D = D).
#if E2_WARP
#ifndef E2_PF_CHUNKS
#define E2_PF_CHUNKS 3
#endif
constexpr int kPfChunks = E2_PF_CHUNKS;
// the lines of a path record the path update reads and writes on g
E2_D void pf_path_rec(u32 v, int g, int G) {
  if (v >= DEV.node_cap) return;
  const char* r = (const char*)grec(v);
  pf(r);
  pf(r + 64 + 8 * g);
  pf(r + 64 + 8 * G + 4 * g);
  pf(r + 64 + 12 * G + 4 * g);
}
#endif

E2_DNI u64 path_update_par(Scr* s, int D, int g, double now, bool mark, bool defer = false) {
  const int G = DEV.cfg.G;
  // the parent's cached-child count uses its child's "newly cached" flag:
  // one lane per level, the child's flag from the next lane (one pass) when
  // the path fits a warp, else from a first pass through shared memory
  const bool onepass = E2_WARP && D <= kWidth;
  if (!onepass) {
#if E2_WARP
    // deep paths: the first kPfChunks chunks' record lines in flight at once,
    // then each chunk prefetches the one kPfChunks ahead
    for (int i = lane(); i < D && i < kPfChunks * kWidth; i += kWidth) pf_path_rec(PSLOT(s, i), g, G);
#endif
    for (int i = lane(); i < D; i += kWidth) {
#if E2_WARP
      if (i + kPfChunks * kWidth < D) pf_path_rec(PSLOT(s, i + kPfChunks * kWidth), g, G);
#endif
      const NodeRec* r = npeek(PSLOT(s, i));
      PFLAG(s, i) = (mark && !rcached(r, g)) ? 1u : 0u;
    }
    wsync();
  }
  i64 add = 0;
  u32 any = 0;
  u64 id0 = 0;
#if E2_WARP
  if (!onepass)
    for (int i = lane(); i < D && i < kPfChunks * kWidth; i += kWidth) pf_path_rec(PSLOT(s, i), g, G);
#endif
  for (int b = 0; b < D; b += kWidth) {
    const int i = b + lane();
    const bool in = i < D;
#if E2_WARP
    if (!onepass && i + kPfChunks * kWidth < D) pf_path_rec(PSLOT(s, i + kPfChunks * kWidth), g, G);
#endif
    NodeRec* r = in ? npoke(PSLOT(s, i)) : nullptr;
    const bool was = in && rcached(r, g);
    bool newly, inc;
    if (onepass) {
      newly = in && mark && !was;
      inc = (shfl_down1((int)newly) != 0) && i + 1 < D;
    } else {
      newly = in && (PFLAG(s, i) & 1u);
      inc = in && i + 1 < D && (PFLAG(s, i + 1) & 1u);
    }
    if (i == 0) id0 = r->id;
    if (!in) continue;
    const i32 ccc0 = rccc(r, G)[g];
    const i32 ccc1 = ccc0 + (inc ? 1 : 0);
    const double la0 = rla(r)[g];
    const double la1 = now > la0 ? now : la0;
    const bool leaf0 = was && ccc0 == 0;
    const bool leaf1 = (was || mark) && ccc1 == 0;
    const bool moved = dbits(la0) != dbits(la1);
    rhits(r, G)[g] += 1;
    r->lamask |= (1ull << g);
    rla(r)[g] = la1;
    if (inc) rccc(r, G)[g] = ccc1;
    if (newly) {
      r->cmask |= (1ull << g);
      add += r->edge_len;
    }
    const bool fix = (leaf0 && (!leaf1 || moved)) || (leaf1 && (!leaf0 || moved));
    PLA0(s, i) = dbits(la0);
    PFLAG(s, i) = (newly ? 1u : 0u) | (leaf0 ? 2u : 0u) | (leaf1 ? 4u : 0u) | (fix ? 8u : 0u);
    any |= fix ? 1u : 0u;
#if E2_WARP
    // the next requests' walks and decides re-read these lines: bring them
    // back into L1 (A/B on one box: C4 +2.2 %, C2 +3 %; the same after a
    // split or a new leaf was slower, profiles/r2_ab.md)
    pf(r);
    pf(rla(r) + g);
#endif
  }
#if E2_WARP
  add = warp_sum(add);
  any = ballot(any != 0) ? 1u : 0u;
  id0 = shfl(id0, 0);
#endif
  wsync();
  if (lane0()) HOT.cached_tokens[g] += add;
  wsync();
  if (D > 0 && (PFLAG(s, 0) & 1u)) {  // a first-level node became cached: root count
    NodeRec* r = nget(kRoot);
    if (lane0()) rccc(r, G)[g] += 1;
    wsync();
  }
  if (defer) {
    if (lane0()) s->fix_D = any ? D : 0;
    wsync();
  } else if (any) {
    path_lru_fix(s, D, g);
  }
  return D > 0 ? id0 : 0;
}

// ensure_path (prefix_tree.cpp:156-185) given the walk of the same sequence.
// Returns the node whose edge ends exactly at |seq| (kNil on error).
E2_DNI u32 ensure_path(i64 seq_off, i64 n, i64 L, const Walk& w) {
  u32 cur = (L == 0) ? kRoot : w.last;
  if (L > 0 && w.last_m < (i64)nget(w.last)->edge_len) {
    cur = split_node(w.last, (u32)w.last_m);
    if (cur == kNil) return kNil;
  }
  if (L == n) return cur;
  return new_leaf(cur, seq_off + L, (u32)(n - L), (u32)L);
}

// ---------------------------------------------------------------------------
// Redirect upkeep — update_redirects (global_scheduler.cpp:194-219).  Warp-wide.
// ---------------------------------------------------------------------------
E2_DNI void update_redirects(Scr* s, double now) {
  const int G = DEV.cfg.G;
  const double th = DEV.cfg.th_bal;
  for (int g = lane(); g < G; g += kWidth) s->loads[g] = win_load(g, now);
  wsync();
  // expiry: each redirect's check reads only the loads (lane per source)
  for (int src = lane(); src < G; src += kWidth) {
    const int dst = HOT.redirect[src];
    if (dst >= 0 && s->loads[src] <= dmul(th, s->loads[dst])) HOT.redirect[src] = -1;
  }
  // hi / lo: first index of the max / min (strict > / < scans from 0)
  int hi = 0, lo = 0;
#if E2_WARP
  {
    int ih = -1, il = -1;
    double vh = 0, vl = 0;
    for (int g = lane(); g < G; g += kWidth) {
      const double v = s->loads[g];
      if (ih < 0 || v > vh) { vh = v; ih = g; }
      if (il < 0 || v < vl) { vl = v; il = g; }
    }
    // lanes [0, gtop) hold every instance (g and g+32 share a lane): an
    // xor butterfly over gtop lanes, then lane 0's answer to all
    for (int o = DEV.cfg.gtop >> 1; o; o >>= 1) {
      const double wh = __shfl_xor_sync(0xffffffffu, vh, o), wl = __shfl_xor_sync(0xffffffffu, vl, o);
      const int jh = __shfl_xor_sync(0xffffffffu, ih, o), jl = __shfl_xor_sync(0xffffffffu, il, o);
      if (jh >= 0 && (ih < 0 || wh > vh || (wh == vh && jh < ih))) { vh = wh; ih = jh; }
      if (jl >= 0 && (il < 0 || wl < vl || (wl == vl && jl < il))) { vl = wl; il = jl; }
    }
    hi = shfl(ih, 0);
    lo = shfl(il, 0);
  }
#else
  for (int g = 1; g < G; ++g) {
    if (s->loads[g] > s->loads[hi]) hi = g;
    if (s->loads[g] < s->loads[lo]) lo = g;
  }
#endif
  wsync();
  if (lane0()) {
    if (!(hi == lo || !(s->loads[hi] > dmul(th, s->loads[lo])))) {
      if (HOT.redirect[hi] != lo) {
        HOT.redirect[hi] = lo;
        HOT.stats[kStInstalls]++;
      }
    }
    s->loads_ok = 1;
  }
  wsync();
}

// pick_min_cost (global_scheduler.cpp:54-74) over s->c*[0, n): the first
// index with the minimum total among the feasible candidates, else among all.
// Device: one lane per candidate and a (total, index) warp reduction.
E2_HD int pick_min(const Scr* s, int n) {
#if E2_WARP
  int bf = -1, ba = -1;  // best feasible / best overall candidate index
  double tf = 0, ta = 0;
  for (int i = lane(); i < n; i += kWidth) {
    const double t = dadd(dadd(s->cL[i], s->cM[i]), s->cP[i]);
    if (!s->cinf[i] && (bf < 0 || t < tf)) { tf = t; bf = i; }
    if (ba < 0 || t < ta) { ta = t; ba = i; }
  }
  // candidates sit in lanes [0, top), top = pow2 >= min(n, 32)
  int top = 1;
  while (top < n && top < 32) top <<= 1;
  const bool anyf = any(bf >= 0);
  for (int o = top >> 1; o; o >>= 1) {
    if (anyf) {
      const double uf = __shfl_xor_sync(0xffffffffu, tf, o);
      const int jf = __shfl_xor_sync(0xffffffffu, bf, o);
      if (jf >= 0 && (bf < 0 || uf < tf || (uf == tf && jf < bf))) { tf = uf; bf = jf; }
    } else {
      const double ua = __shfl_xor_sync(0xffffffffu, ta, o);
      const int ja = __shfl_xor_sync(0xffffffffu, ba, o);
      if (ja >= 0 && (ba < 0 || ua < ta || (ua == ta && ja < ba))) { ta = ua; ba = ja; }
    }
  }
  const int b = shfl(anyf ? bf : ba, 0);
  return b >= 0 ? s->cgpu[b] : -1;
#else
  int best = -1;
  double bt = 0;
  for (int i = 0; i < n; ++i) {
    if (s->cinf[i]) continue;
    const double t = dadd(dadd(s->cL[i], s->cM[i]), s->cP[i]);
    if (best < 0 || t < bt) {
      best = s->cgpu[i];
      bt = t;
    }
  }
  if (best >= 0) return best;
  for (int i = 0; i < n; ++i) {
    const double t = dadd(dadd(s->cL[i], s->cM[i]), s->cP[i]);
    if (best < 0 || t < bt) {
      best = s->cgpu[i];
      bt = t;
    }
  }
  return best;
#endif
}

struct Dec {
  i32 branch, gpu, redirected, pre;
  i64 cached_len, missed_len, moc, matched;
  i32 has_ratios;
  i32 ok;  // 0 = error raised
};

E2_HD void put_cost(Scr* s, int idx, int g, const CostOut& c) {
  s->cgpu[idx] = g;
  s->cL[idx] = c.L;
  s->cM[idx] = c.M;
  s->cP[idx] = c.P;
  s->cinf[idx] = c.inf ? 1 : 0;
}

// decide (global_scheduler.cpp:76-158).  Warp-wide.  Fills s->c* and
// s->ratios; w receives the walk for a following commit.
// Warp-wide: does any instance in `set` need the eviction term
// (missed - free > 0) for this prompt?
E2_D bool any_need(const Scr* s, u64 set, i64 n) {
  bool need = false;
  for (int g = lane(); g < DEV.cfg.G; g += kWidth)
    if ((set >> g) & 1ull) need |= (n - s->ext[g]) - (DEV.cfg.cap - HOT.cached_tokens[g]) > 0;
  return any(need);
}

// decide (global_scheduler.cpp:76-158).  Warp-wide.  Fills s->c* and
// s->ratios; w receives the walk for a following commit.
//
// spec: run concurrently with the eviction warp (two-warp replay).  The
// decide then changes no shared state and gives up (s->spec_bad) instead of
// raising an error or evaluating an eviction term (which reads the LRU and
// hit counters the eviction is changing); the caller validates the result
// against the nodes the eviction touched and redoes it when needed.  With no
// eviction term, the cost of instance g depends on the eviction only through
// need = missed - (cap - cached_tokens[g]) <= 0, which an eviction (cached
// tokens only decrease) cannot turn positive.
// reuse_walk: the walk of a speculative decide of this request that gave up
// later (an eviction term was due) and whose path the concurrent eviction
// did not touch: w and s's path/extents are current, the walk is skipped.
E2_D Dec decide(Scr* s, const i32* seq, i64 n, i64 L, const u32* hint, int nhint, i64 hS, double now, Walk& w,
                  bool spec = false, const i64* lead = nullptr, const u32* hint_rows = nullptr,
                  bool reuse_walk = false) {
  Dec r;
  r.branch = 1;
  r.gpu = -1;
  r.redirected = 0;
  r.pre = -1;
  r.cached_len = 0;
  r.missed_len = 0;
  r.moc = 0;
  r.matched = L;
  r.has_ratios = 0;
  r.ok = 1;
  const int G = DEV.cfg.G;
  if (lane0()) {
    s->n_costs = 0;
    s->spec_bad = 0;
    if (!reuse_walk) s->spec_walked = 0;
  }
  wsync();
#define SPEC_FAIL()           \
  do {                        \
    PHASE_COUNT(42);          \
    if (lane0()) s->spec_bad = 1; \
    wsync();                  \
    r.ok = 0;                 \
    return r;                 \
  } while (0)
  if (n > DEV.cfg.cap) {
    if (spec) SPEC_FAIL();
    if (lane0()) set_err(kErrNoAdmissible, kWhyPromptTooLong);
    wsync();
    r.ok = 0;
    return r;
  }
  if (DEV.cfg.mode == 1) {
    r.branch = 3;
    r.gpu = (i32)(HOT.rr_next % G);
    r.missed_len = n;
    r.moc = n;
    r.matched = 0;
    return r;
  }
  if (!spec && lane0()) HOT.stats[kStTreeReads]++;  // a validated speculative decide is counted by the caller
  wsync();
  PHASE_MARK(32);
  if (!reuse_walk) {
#if E2_WARP
    if (lane0()) g_probed = 0;
    wsync();
#endif
    w = walk_par(seq, L, hint, nhint, s, hS, lead, hint_rows);
    if (!w.ok && s->npath < 0) {
      if (spec) SPEC_FAIL();
      w = walk_known(seq, L, hint, nhint, s->ext);
    }
    PHASE_MARK(6);
#if E2_WARP
    if (spec && g_probed) SPEC_FAIL();  // the table may lack the previous leaf's entry yet
#endif
    if (spec && w.ok && lane0()) s->spec_walked = 1;
    wsync();
  }
  if (!w.ok) {
    if (spec) SPEC_FAIL();
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    r.ok = 0;
    return r;
  }
  // per_gpu_matched_len entries exist only for gpus caching the first span
  for (int g = lane(); g < G; g += kWidth)
    if (!((w.present >> g) & 1ull)) s->ext[g] = 0;
  wsync();
  r.cached_len = w.cached_len;
  r.missed_len = n - w.cached_len;
  if (r.missed_len < r.cached_len) {
    r.branch = 0;
    i64 best = 0;
    u64 cand = 0;
#if E2_WARP
    {
      i64 mine = 0;
      for (int g = lane(); g < G; g += kWidth)
        if ((w.present >> g) & 1ull) mine = max_(mine, s->ext[g]);
      for (int o = DEV.cfg.gtop >> 1; o; o >>= 1) mine = max_(mine, (i64)__shfl_xor_sync(0xffffffffu, (long long)mine, o));
      best = shfl(mine, 0);
      for (int b = 0; b < G; b += 32) {
        const int g = b + lane();
        const bool c = g < G && ((w.present >> g) & 1ull) && s->ext[g] == best;
        cand |= (u64)ballot(c) << b;
      }
    }
#else
    for (u64 m = w.present; m; m &= m - 1) best = max_(best, s->ext[ffs64(m)]);
    for (u64 m = w.present; m; m &= m - 1) {
      const int g = ffs64(m);
      if (s->ext[g] == best) cand |= (1ull << g);
    }
#endif
    PHASE_MARK(33);
    if (spec && any_need(s, cand, n)) SPEC_FAIL();
    cost_prepare_set(s, cand, n, now);
    PHASE_MARK(7);
    for (int g = lane(); g < G; g += kWidth) {
      if ((cand >> g) & 1ull) {
        const int idx = popc64(cand & ((1ull << g) - 1));
        put_cost(s, idx, g, cost_for(g, n - s->ext[g], now, s));
      }
    }
    wsync();
    int nc = popc64(cand);
    int gpu = pick_min(s, nc);
    if (gpu >= 0 && HOT.redirect[gpu] >= 0 && HOT.redirect[gpu] != gpu) {
      const int t = HOT.redirect[gpu];
      int ti = -1;
      for (int i = 0; i < nc; ++i)
        if (s->cgpu[i] == t) ti = i;
      if (ti < 0) {
        if (spec && any_need(s, 1ull << t, n)) SPEC_FAIL();
        cost_prepare(t, n - s->ext[t], now);
        if (lane0()) put_cost(s, nc, t, cost_for(t, n - s->ext[t], now, s));
        wsync();
        ti = nc;
        nc++;
      }
      if (!s->cinf[ti]) {
        r.redirected = 1;
        r.pre = gpu;
        gpu = t;
      }
    }
    if (lane0()) s->n_costs = nc;
    wsync();
    r.gpu = gpu;
    PHASE_MARK(8);
  } else {
    r.has_ratios = 1;
    for (int g = lane(); g < G; g += kWidth) {
      const i64 ip = HOT.inflight_prompt[g];
      s->ratios[g] = ip <= 0 ? 0.0 : ddiv(i2d(HOT.inflight_cached[g]), i2d(ip));
    }
    wsync();
    int max_g = -1;
    double max_r = -1.0;
    for (int g = 0; g < G; ++g) {
      if (s->ratios[g] > max_r) {
        max_r = s->ratios[g];
        max_g = g;
      }
    }
    if (DEV.cfg.pd_balance && max_r > DEV.cfg.imbal) {
      r.branch = 2;
      r.gpu = max_g;
    } else {
      r.branch = 1;
      const u64 all = G == 64 ? ~0ull : ((1ull << G) - 1);
      if (spec && any_need(s, all, n)) SPEC_FAIL();
      PHASE_MARK(46);  // explore: ratios
      cost_prepare_set(s, all, n, now);
      PHASE_MARK(44);  // explore: window prune + hit catch-up
      for (int g = lane(); g < G; g += kWidth) put_cost(s, g, g, cost_for(g, n - s->ext[g], now, s));
      wsync();
      PHASE_MARK(45);  // explore: every instance's cost
      if (lane0()) s->n_costs = G;
      wsync();
      r.gpu = pick_min(s, G);
    }
  }
  if (!spec && HOT.err) {
    r.ok = 0;
    return r;
  }
  if (r.gpu < 0 || r.gpu >= G) {
    if (spec) SPEC_FAIL();
    if (lane0()) set_err(kErrSim, kWhyNotContiguous);
    wsync();
    r.ok = 0;
    return r;
  }
  r.moc = n - s->ext[r.gpu];
  return r;
#undef SPEC_FAIL
}

// ---------------------------------------------------------------------------
// Inflight map: request id -> placement (global_scheduler.hpp:129-135).
// Single-lane; linear probing with backward-shift deletion; 64-byte records.
// ---------------------------------------------------------------------------
E2_HD u64 inf_find(i64 id, bool& found) {
  u64 i = mix64((u64)id) & DEV.inf_mask;
  for (u64 k = 0; k <= DEV.inf_mask; ++k, i = (i + 1) & DEV.inf_mask) {
    const i64 key = DEV.inf[i].key;
    if (key == kNoInflight) {
      found = false;
      return i;
    }
    if (key == id) {
      found = true;
      return i;
    }
  }
  found = false;
  return ~0ull;
}

E2_HD void inf_erase_at(u64 i) {
  u64 j = i;
  for (;;) {
    j = (j + 1) & DEV.inf_mask;
    const InfRec rj = DEV.inf[j];
    if (rj.key == kNoInflight) break;
    const u64 home = mix64((u64)rj.key) & DEV.inf_mask;
    // move j into the hole at i if home is not cyclically in (i, j]
    const bool in_range = (i <= j) ? (home > i && home <= j) : (home > i || home <= j);
    if (!in_range) {
      DEV.inf[i] = rj;
      i = j;
    }
  }
  DEV.inf[i].key = kNoInflight;
}

// One bottom-up pass over the committed path: record_hit on every node
// (prefix_tree.cpp:45-51, via insert :193-196) and, when `mark`,
// mark_cached_path's set_cached + last_access update (:200-213) for the
// same gpu and time.  In the batched driver note_prefill_cached follows the
// commit immediately, so both passes are applied together; the LRU index is
// a set, so moving each node once from its initial to its final
// (membership, key) equals the reference's erase/insert sequence.  A node's
// cached-child count is read before its child's increment is applied.
// Returns the first-level node id.  Warp-wide.
E2_DNI u64 path_update(u32 tail, int g, double now, bool mark) {
  const int G = DEV.cfg.G;
  bool inc = false;  // the previous (child) node became cached on g
  u64 first_id = 0;
  u32 v = tail;
  while (v != kRoot) {
    NodeRec* r = nget(v);
    const u32 p = r->parent;
    const u64 id = r->id;
    const bool was = rcached(r, g);
    const i32 ccc0 = rccc(r, G)[g];
    const i32 ccc1 = ccc0 + (inc ? 1 : 0);
    const double la0 = rla(r)[g];
    const double la1 = now > la0 ? now : la0;
    const bool newly = mark && !was;
    const bool leaf0 = was && ccc0 == 0;
    const bool leaf1 = (was || mark) && ccc1 == 0;
    first_id = id;
    if (lane0()) {
      rhits(r, G)[g] += 1;
      r->lamask |= (1ull << g);
      rla(r)[g] = la1;
      if (inc) rccc(r, G)[g] = ccc1;
      if (newly) {
        r->cmask |= (1ull << g);
        HOT.cached_tokens[g] += r->edge_len;
      }
    }
    wsync();
    const bool moved = dbits(la0) != dbits(la1);
    if (leaf0 && (!leaf1 || moved)) lru_erase(g, dbits(la0), id);
    if (leaf1 && (!leaf0 || moved)) lru_insert(g, dbits(la1), id, v);
    inc = newly;
    v = p;
  }
  if (inc) {  // set_cached on a first-level node also counts on the root
    NodeRec* r = nget(kRoot);
    if (lane0()) rccc(r, G)[g] += 1;
    wsync();
  }
  return first_id;
}

// commit (global_scheduler.cpp:160-175), optionally fused with the
// driver's note_prefill_cached (see path_update).  Warp-wide.  Returns the
// tail slot.
// defer_inflight: the inflight sums and record are left to the caller
// (the pipelined replay's second warp, inflight_insert).
// fix_flag: raised (to fix_val) as soon as the path's deferred LRU
// re-indexing may start (s_path->fix_D), before the path log is written.
E2_DNI u32 commit(i64 seq_off, i64 n, i64 L, const Walk& w, const Dec& r, i64 req_id, double arrival,
                  double now, bool mark, Scr* s_path, bool defer_lru = false, bool defer_inflight = false,
                  volatile long long* fix_flag = nullptr, long long fix_val = 0) {
  const bool win_done = s_path && s_path->win_done;
  if (s_path && lane0()) {
    s_path->fix_D = 0;
    s_path->cpath = -1;
    s_path->win_done = 0;
  }
  wsync();
  if (DEV.cfg.mode == 1) {
    if (lane0()) HOT.rr_next++;
    wsync();
    return kNil;
  }
  if (n == 0) {
    if (lane0()) set_err(kErrSim, kWhyEmptyInsert);
    wsync();
    return kNil;
  }
  PHASE_MARK(2);
  const u32 tail = ensure_path(seq_off, n, L, w);
  PHASE_MARK(9);
  if (tail == kNil || HOT.err) return kNil;
  const int g = r.gpu;
  u64 root_id;
  int D = s_path ? s_path->npath : -1;
  if (D >= 0) {
    // the path after ensure_path: the split prefix (or the last level)
    // ends at L; a new leaf is appended when L < n
    const u32 at_L = (L == n) ? tail : (L > 0 ? nget(tail)->parent : kNil);
    if (L > 0 && D > 0) {
      if (lane0()) PSLOT(s_path, D - 1) = at_L;
      wsync();
    }
    if (L < n) {
      if (D + 1 > kPathLevels) {
        D = -1;
      } else {
        if (lane0()) PSLOT(s_path, D) = tail;
        wsync();
        D++;
      }
    }
  }
  u32 plen = kNil;
  if (D >= 0) {
    if (lane0()) s_path->cpath = D;
    // levels past kMaxPath live in the single global overflow: not deferrable
    root_id = path_update_par(s_path, D, g, now, mark, defer_lru && D <= kMaxPath);
    if (fix_flag) {
      if (lane0()) {
        fence_block();
        *fix_flag = fix_val;
      }
      wsync();
    }
    PHASE_MARK(10);
    plen = plog_append(s_path, D, g);
  } else {
    root_id = path_update(tail, g, now, mark);
  }
  if (defer_inflight) {
    if (lane0()) {
      if (win_done) {
        // appended early (window_early): hit expiry reads these two fields
        WinEnt* e = &DEV.win[wslot(g, s_path->widx)];
        e->slot = tail;
        e->plen = plen;
      } else {
        win_add_sched(g, now, r.moc, DEV.cfg.default_out, tail, plen);
      }
    }
    wsync();
    return tail;
  }
  if (lane0()) {
    win_add_sched(g, now, r.moc, DEV.cfg.default_out, tail, plen);
    HOT.inflight_cached[g] += r.cached_len;
    HOT.inflight_prompt[g] += n;
    bool found;
    const u64 i = inf_find(req_id, found);
    if (i == ~0ull) {
      set_err(kErrCapacity, kWhyInflightCap);
    } else {
      if (!found) {
        HOT.inflight_n++;
        if ((u64)HOT.inflight_n * 2 > DEV.inf_mask + 1) set_err(kErrCapacity, kWhyInflightCap);
      }
      InfRec e;
      e.key = req_id;
      e.gpu = g;
      e.pad = 0;
      e.cached = r.cached_len;
      e.prompt = n;
      e.arr = arrival;
      e.root = root_id;
      e.pad2 = 0;
      DEV.inf[i] = e;
    }
  }
  wsync();
  return tail;
}

// The inflight half of commit (global_scheduler.cpp:172-174): sums and the
// id -> placement record.  root_id is the first-level node of the committed
// path.  Warp-wide (single-lane work).
E2_DNI void inflight_insert(i64 req_id, int g, i64 cached_len, i64 n, double arrival, u64 root_id) {
  if (lane0()) {
    HOT.inflight_cached[g] += cached_len;
    HOT.inflight_prompt[g] += n;
    bool found;
    const u64 i = inf_find(req_id, found);
    if (i == ~0ull) {
      set_err(kErrCapacity, kWhyInflightCap);
    } else {
      if (!found) {
        HOT.inflight_n++;
        if ((u64)HOT.inflight_n * 2 > DEV.inf_mask + 1) set_err(kErrCapacity, kWhyInflightCap);
      }
      InfRec e;
      e.key = req_id;
      e.gpu = g;
      e.pad = 0;
      e.cached = cached_len;
      e.prompt = n;
      e.arr = arrival;
      e.root = root_id;
      e.pad2 = 0;
      DEV.inf[i] = e;
    }
  }
  wsync();
}

// Stats (global_scheduler.cpp:183-189).
E2_D void count_stats(const Dec& r) {
  if (lane0()) {
    HOT.stats[r.branch == 0 ? kStExploit : r.branch == 1 ? kStExplore : r.branch == 2 ? kStPressure : kStRoundRobin]++;
    if (r.redirected) HOT.stats[kStRedirected]++;
  }
  wsync();
}

// mark_cached_path bottom-up part (prefix_tree.cpp:203-211) from a known tail.
E2_DNI void mark_cached_chain(u32 tail, int g, double now) {
  for (u32 v = tail; v != kRoot;) {
    set_cached(v, g);
    touch_la(v, g, now);
    v = nget(v)->parent;
  }
}

// note_finished (global_scheduler.cpp:361-369).  Warp-wide.
E2_DNI void note_finished(i64 id, double now, i64 out) {
  if (lane0()) {
    bool found;
    const u64 i = inf_find(id, found);
    if (found) {
      const InfRec e = DEV.inf[i];
      win_add_comp(e.gpu, now, out);
      HOT.inflight_cached[e.gpu] -= e.cached;
      HOT.inflight_prompt[e.gpu] -= e.prompt;
      inf_erase_at(i);
      HOT.inflight_n--;
    }
  }
  wsync();
}

// Clear [start, end) of the root path ending at `bottom`, deepest first
// (the second half of uncache_suffix, prefix_tree.cpp:262-270).  The node
// containing `start` has already been split there.
E2_DNI i64 clear_range_from(u32 bottom, i64 start, int g) {
  i64 freed = 0;
  for (u32 v = bottom; v != kRoot && v != kNil;) {
    const NodeRec* r = nget(v);
    const i64 v_end = (i64)r->depth + r->edge_len;
    if (v_end <= start) break;
    const u32 p = r->parent;
    if (rcached(r, g)) {
      freed += r->edge_len;
      clear_cached(v, g);
    }
    v = p;
  }
  return freed;
}

// uncache_suffix (prefix_tree.cpp:237-271) for a sequence whose matched
// length M is known.  Warp-wide.  Returns tokens uncached.
E2_DNI i64 uncache_suffix(const i32* seq, i64 n, i64 M, i64 tail_len, int g) {
  if (n == 0 || tail_len <= 0) return 0;
  const i64 end = min_(n, M);
  i64 start = n - tail_len;
  if (start < 0) start = 0;
  if (start >= end) return 0;
  // walk down, aligning splits; `bottom` ends at `end`
  i64 off = 0;
  u32 cur = kRoot, bottom = kNil;
  while (off < end) {
    const u32 ch = child_lookup(cur, seq[off]);
    if (ch == kNil) {
      if (lane0()) set_err(kErrSim, kWhyWalk);
      wsync();
      return 0;
    }
    const i64 len = nget(ch)->edge_len;
    const i64 m = min_(len, M - off);
    u32 node = ch;
    if (m < len) {
      node = split_node(ch, (u32)m);  // keep the part on seq's path
      if (node == kNil) return 0;
    }
    const i64 node_end = off + m;
    if (node_end > start && off < start) {
      // split at start: the slot keeps the suffix, which is the target
      if (split_node(node, (u32)(start - off)) == kNil) return 0;
    }
    bottom = node;
    cur = node;
    off = node_end;
    if (m < len) break;
  }
  return clear_range_from(bottom, start, g);
}

// uncache_suffix for a prompt committed earlier in this replay: its tail
// slot (the node ending at |p|) is stable under splits, so the path is the
// parent chain and no token is read.  Warp-wide.
E2_DNI i64 uncache_tail(u32 tail, i64 n, i64 tail_len, int g) {
  if (n == 0 || tail_len <= 0 || tail == kNil) return 0;
  i64 start = n - tail_len;
  if (start < 0) start = 0;
  if (start >= n) return 0;
  // find the node containing `start` on the chain and split there
  for (u32 v = tail; v != kRoot;) {
    const NodeRec* r = nget(v);
    const i64 dep = r->depth;
    const u32 p = r->parent;
    if (dep <= start) {
      if (dep < start && split_node(v, (u32)(start - dep)) == kNil) return 0;
      break;
    }
    v = p;
  }
  return clear_range_from(tail, start, g);
}

// Partial eviction of the last `tok` tokens of LRU leaf v on g
// (uncache_suffix with the range ending at v's end: split at len-tok, clear
// the suffix).  Net effect on g's LRU index: the leaf key (la, id) stays —
// the prefix keeps v's id and last_access and becomes the leaf — so the
// entry is relabelled to the prefix slot instead of erased and reinserted.
// Other instances caching v see the suffix re-keyed exactly as in split.
// Warp-wide.
E2_DNI void evict_tail(u32 v, i64 tok, int g) {
  const int G = DEV.cfg.G;
  NodeRec* r = nget(v);
  const u32 len = r->edge_len;
  const u64 id0 = r->id, la0 = dbits(rla(r)[g]), cm = r->cmask;
  const bool leaf = rleaf(r, v, g, G);
  // other instances where v is a leaf: split re-keys them (new suffix id)
  PHASE_MARK1(28);
  const u32 q = split_node(v, (u32)(len - tok), false);
  PHASE_MARK1(25);
  if (q == kNil) return;
  const u64 id1 = nget(v)->id;
  for (u64 m = cm & ~(1ull << g); m; m &= m - 1) {
    const int o = ffs64(m);
    const NodeRec* rv = nget(v);
    if (rccc(rv, G)[o] == 0) lru_rekey(o, dbits(rla(rv)[o]), id0, id1, v);
  }
  // clear the suffix on g without touching g's index, then relabel
  r = nget(v);
  if (lane0()) {
    r->cmask &= ~(1ull << g);
    HOT.cached_tokens[g] -= r->edge_len;
  }
  wsync();
  NodeRec* rq = nget(q);
  if (lane0()) rccc(rq, G)[g] -= 1;  // 1 -> 0: the prefix is the leaf now
  wsync();
  if (leaf) lru_relabel(g, la0, id0, q);
}

// Mirror-LRU eviction: plan_eviction(g, over, {}, partial)
// then note_eviction for every entry, ranges built before any is applied.
E2_DNI void evict_lru(int g, i64 over) {
  if (lane0()) {
    u32 nv = 0;
    plan_eviction(g, over, true, [&](u32 v, i64 tok, const NodeRec* rv) {
      if (nv < DEV.vcap) {
        DEV.vic_slot[nv] = v;
        DEV.vic_tok[nv] = tok;
        nv++;
        // a partial victim is split at len - tok: fetch that token early
        if (tok < (i64)rv->edge_len) pf(DEV.tok + rv->edge_off + (rv->edge_len - tok));
      } else {
        set_err(kErrCapacity, kWhyScratchCap);
      }
    });
    DEV.scr_val[(u64)DEV.cfg.G * DEV.scap] = nv;  // count, in the spare scratch word
  }
  wsync();
  PHASE_MARK(11);
  PHASE_MARK1(24);
  const u32 nv = (u32)DEV.scr_val[(u64)DEV.cfg.G * DEV.scap];
  for (u32 i = 0; i < nv && !HOT.err; ++i) {
    const u32 v = DEV.vic_slot[i];
    const i64 tok = DEV.vic_tok[i];
    const i64 len = nget(v)->edge_len;
    if (tok < len) {
      PHASE_COUNT(13);
      evict_tail(v, tok, g);
      PHASE_MARK1(26);
    } else {
      PHASE_COUNT(14);
      clear_cached(v, g);
      PHASE_MARK1(27);
    }
  }
}

}  // namespace e2
