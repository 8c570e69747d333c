// e2_tree.cuh — warp-cooperative radix-tree store, shared-memory node cache
// and per-instance LRU index.
//
// Execution model of the serial kernel: one warp; scalar control logic is
// executed redundantly by every lane on uniform values; all writes to shared
// state go through lane 0 followed by __syncwarp; the cooperative pieces use
// vote/ballot/shuffle.  Functions marked "warp-wide" must be called by all
// lanes with uniform arguments; "single-lane" functions must not contain
// warp collectives.
#pragma once

#include "e2_state.cuh"

namespace e2 {

// ---------------------------------------------------------------------------
// Node cache: 4-way set-associative, write-back, in shared memory.  The
// serial kernel is the only writer of the tree while it runs, so the cache
// is coherent by construction; it is flushed before the kernel exits.
// Pointers returned by nget/nnew are valid until the next nget/nnew.
// ---------------------------------------------------------------------------
constexpr int kWays = 4;

struct NCache {
  u32 nsets;  // power of two
  u32 clock;
  u32 victim;
  u32 pad;
  u32* tag;    // [nsets*kWays], kNil = empty
  u32* tick;   // last use
  u32* dirty;
  char* data;  // [nsets*kWays][rs]
};

// The serial kernel's state lives at fixed addresses: the handle's device
// pointers and config in constant memory (uploaded before every launch), the
// hot scalar state and the node cache in static shared memory.
#if E2_DEVICE_BUILD
__constant__ Dev g_dev;
__shared__ Hot g_hot;
__shared__ NCache g_nc;
#define DEV (::e2::g_dev)
#define HOT (::e2::g_hot)
#define NC (::e2::g_nc)
#else
inline Dev g_dev_h;
inline Hot* g_hot_h = nullptr;
inline NCache g_nc_h;
#define DEV (::e2::g_dev_h)
#define HOT (*::e2::g_hot_h)
#define NC (::e2::g_nc_h)
#endif

E2_HD NodeRec* grec(u32 s) { return (NodeRec*)(DEV.rec + (u64)s * DEV.rs); }

// Two-warp pipelined replay (e2_kernels.cuh): the eviction warp (warp 1)
// records every node whose structure or caching mask it changes, so the
// decision warp can validate a decide it ran concurrently.
constexpr u32 kTouchCap = 64;
#if E2_WARP
__shared__ u32 g_touch[kTouchCap];
__shared__ u32 g_ntouch;
E2_D void touch(u32 v) {
  if (threadIdx.x >= 32 && lane0()) {
    const u32 n = g_ntouch;
    if (n < kTouchCap) g_touch[n] = v;
    g_ntouch = n + 1;
  }
}
#else
E2_HD void touch(u32) {}
#endif

// Deferred child-table inserts (pipelined replay): a new leaf whose parent
// already has its inline child needs a hashed-table entry, i.e. one random
// HBM round trip.  Warp 0 leaves that insert to the eviction warp, which
// performs it first thing after barrier 2, while warp 0 moves on to the next
// speculative decide; a speculative walk that probes the table meanwhile
// gives up (g_probed) and is redone after barrier 1.
#if E2_WARP
struct CtDefer {
  u32 parent, child;
  i32 tok;
  u32 pending;
};
__shared__ CtDefer g_ctd;
// Deferred LRU re-keying of a split's suffix (pipelined replay): the suffix
// is off the committing request's path, so its leaf keys on the instances
// caching it can take the new id on the eviction warp, which does it while
// it waits for warp 0's path update (before its LRU fixes and evictions).
struct RekeyDefer {
  u64 mask;  // instances where the suffix is an LRU leaf
  u64 old_id, new_id;
  u32 slot;
  volatile u32 pending;
};
__shared__ RekeyDefer g_rkd;
__shared__ u32 g_defer_ct;  // warp 0 of the pipelined replay defers
__shared__ u32 g_probed;    // a walk probed the child table
E2_D void note_probe() {
  if (lane0()) g_probed = 1;
}
#else
E2_HD void note_probe() {}
#endif

// E2_PHASES (dev-only instrumented builds): cycles since the previous mark
// are added to phase_cycles[i].  Compiled out of the product.
#if defined(E2_PHASES) && E2_DEVICE_BUILD
#define PHASE_MARK(i)                                          \
  do {                                                         \
    wsync();                                                   \
    const u64 _pn = clock64();                                 \
    if (lane0() && threadIdx.x < 32) {                         \
      HOT.phase_cycles[i] += _pn - HOT.phase_last;             \
      HOT.phase_last = _pn;                                    \
    }                                                          \
    wsync();                                                   \
  } while (0)
// warp 1 of the pipelined replay: slots 20..23
#define PHASE_MARK1(i)                                         \
  do {                                                         \
    wsync();                                                   \
    const u64 _pn = clock64();                                 \
    if (lane0()) {                                             \
      HOT.phase_cycles[i] += _pn - HOT.phase_last1;            \
      HOT.phase_last1 = _pn;                                   \
    }                                                          \
    wsync();                                                   \
  } while (0)
#elif defined(E2_PHASES)
#include <x86intrin.h>
#define PHASE_MARK1(i)
#define PHASE_MARK(i)                                          \
  do {                                                         \
    const u64 _pn = __rdtsc();                                 \
    HOT.phase_cycles[i] += _pn - HOT.phase_last;               \
    HOT.phase_last = _pn;                                      \
  } while (0)
#else
#define PHASE_MARK(i)
#define PHASE_MARK1(i)
#endif
#if defined(E2_PHASES)
#if E2_DEVICE_BUILD
#define PHASE_COUNT(i)                                         \
  do {                                                         \
    if (lane0()) atomicAdd((unsigned long long*)&HOT.phase_cycles[i], 1ull); \
  } while (0)
#else
#define PHASE_COUNT(i)                                         \
  do {                                                         \
    HOT.phase_cycles[i] += 1;                                  \
  } while (0)
#endif
#else
#define PHASE_COUNT(i)
#endif

E2_HD void set_err(i32 code, i32 why) {
  if (HOT.err == 0) {
    HOT.err = code;
    HOT.why = why;
  }
}

E2_HD NodeRec* nentry(u32 w) { return (NodeRec*)(NC.data + (u64)w * DEV.rs); }

// Every resident record is written back on eviction/flush (almost every
// record the serial pass touches is modified anyway), so no dirty tracking.
E2_HD void ndirty(const NodeRec*) {}

#if !defined(E2_SMEM_NODECACHE)
// Default: records are read and written in place in HBM.  The serial kernel
// is the only writer while it runs and its SM's L1 (~180 KB, the carveout
// left by the small static shared state) holds the hot records; measured
// ~9% faster per request than the shared-memory cache below, which is kept
// as an opt-in (-DE2_SMEM_NODECACHE) for comparison.
E2_D NodeRec* nget(u32 s) { return grec(s); }
E2_DNI NodeRec* nnew(u32 s) {
  u64* dst = (u64*)grec(s);
  for (u32 j = (u32)lane(); j < DEV.rs / 8; j += kWidth) dst[j] = 0;
  wsync();
  return grec(s);
}
E2_HD const NodeRec* npeek(u32 s) { return grec(s); }
E2_HD NodeRec* npoke(u32 s) { return grec(s); }
E2_D void nflush() {}
#else
// warp-wide copy of one record (rs bytes, 8-byte words; at most
// rec_stride(kMaxG)/8 = 144 words): every load is issued before the first
// store, so a miss costs one memory latency, not one per 32 words.
E2_D void rcopy(u64* dst, const u64* src, u32 words) {
#if E2_WARP
  constexpr int kPer = (rec_stride(kMaxG) / 8 + 31) / 32;
  u64 v[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const u32 j = (u32)lane() + 32u * k;
    if (j < words) v[k] = src[j];
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const u32 j = (u32)lane() + 32u * k;
    if (j < words) dst[j] = v[k];
  }
#else
  for (u32 j = 0; j < words; ++j) dst[j] = src[j];
#endif
}

// warp-wide: pick the way to (re)use in s's set; write back its record.
E2_DNI u32 nclaim(u32 s) {
  const u32 base = (s & (NC.nsets - 1)) * kWays;
  if (lane0()) {
    u32 best = base;
    for (u32 k = 0; k < (u32)kWays; ++k) {
      const u32 w = base + k;
      if (NC.tag[w] == kNil) {
        best = w;
        break;
      }
      if (NC.tick[w] < NC.tick[best]) best = w;
    }
    NC.victim = best;
  }
  wsync();
  const u32 w = NC.victim;
  const u32 old = NC.tag[w];
  if (old != kNil) rcopy((u64*)grec(old), (const u64*)nentry(w), DEV.rs / 8);
  return w;
}

E2_DNI NodeRec* nget_miss(u32 s) {
  const u32 w = nclaim(s);
  rcopy((u64*)nentry(w), (const u64*)grec(s), DEV.rs / 8);
  wsync();
  if (lane0()) {
    NC.tag[w] = s;
    NC.tick[w] = ++NC.clock;
  }
  wsync();
  return nentry(w);
}

// warp-wide: make node s resident and return its cached record.  Hit path:
// one 4-lane vote; tick/clock are private to lane 0 (only nclaim reads them).
E2_D NodeRec* nget(u32 s) {
  const u32 base = (s & (NC.nsets - 1)) * kWays;
  const u32 hit = vote(kWays, [&](int k) { return NC.tag[base + k] == s; });
  if (hit) {
    const u32 w = base + (u32)ffs32(hit);
    if (lane0()) NC.tick[w] = ++NC.clock;
    return nentry(w);
  }
  return nget_miss(s);
}

// warp-wide: a fresh (zeroed, dirty) record for a newly allocated slot.
E2_DNI NodeRec* nnew(u32 s) {
  const u32 w = nclaim(s);
  u64* dst = (u64*)nentry(w);
  for (u32 j = (u32)lane(); j < DEV.rs / 8; j += kWidth) dst[j] = 0;
  wsync();
  if (lane0()) {
    NC.tag[w] = s;
    NC.tick[w] = ++NC.clock;
  }
  wsync();
  return nentry(w);
}

// single-lane read-only view (cached copy if resident, else HBM).
E2_HD const NodeRec* npeek(u32 s) {
  const u32 base = (s & (NC.nsets - 1)) * kWays;
  for (u32 k = 0; k < (u32)kWays; ++k)
    if (NC.tag[base + k] == s) return nentry(base + k);
  return grec(s);
}

// single-lane writable view: the cached copy if resident, else HBM.  Only
// for phases without cache fills (each lane touching a different node).
E2_HD NodeRec* npoke(u32 s) {
  const u32 base = (s & (NC.nsets - 1)) * kWays;
  for (u32 k = 0; k < (u32)kWays; ++k)
    if (NC.tag[base + k] == s) return nentry(base + k);
  return grec(s);
}

// warp-wide: write every dirty record back.
E2_D void nflush() {
  const u32 n = NC.nsets * kWays;
  for (u32 w = 0; w < n; ++w) {
    if (NC.tag[w] != kNil) rcopy((u64*)grec(NC.tag[w]), (const u64*)nentry(w), DEV.rs / 8);
  }
  wsync();
}

#endif

// single-lane record access inside a lane-0 block (no cache fill): the
// cached copy if resident, else HBM.
E2_HD NodeRec* nget_lane(u32 s) { return npoke(s); }

// ---------------------------------------------------------------------------
// Child table: open addressing, linear probing, key = parent<<32 | token.
// Replaces TreeNode::children (std::map) lookups, prefix_tree.cpp:85, 160.
// ---------------------------------------------------------------------------
E2_HDX u64 ckey(u32 parent, i32 tok) { return ((u64)parent << 32) | (u64)(u32)tok; }

struct Probe {
  u64 pos;   // table index of the key (found) or of the first free slot
  u32 val;
  bool found;
};

// warp-wide (read-only): each step probes 32 consecutive 16-byte entries.
E2_DNI Probe ct_probe(u64 key) {
  u64 b = mix64(key) & DEV.ct_mask;
  u64 first_free = ~0ull;
  for (u64 step = 0; step <= DEV.ct_mask; step += 32, b += 32) {
#if E2_WARP
    const CtEntry e = DEV.ct[(b + lane()) & DEV.ct_mask];
    const u32 hit = ballot(e.key == key);
    const u32 emp = ballot(e.key == kEmptyKey);
    const u32 fr = emp | ballot(e.key == kTombKey);
    if (first_free == ~0ull && fr) first_free = (b + (u64)ffs32(fr)) & DEV.ct_mask;
    if (hit) {
      const int j = ffs32(hit);
      return Probe{(b + (u64)j) & DEV.ct_mask, shfl(e.val, j), true};
    }
    if (emp) return Probe{first_free, 0, false};
#else
    // Scalar: linear probing with early exit.  Same answers as the 32-wide
    // window: no key ever sits past an empty entry of its probe sequence
    // (inserts take the first free entry; erases leave tombstones).
    for (int j = 0; j < 32; ++j) {
      const u64 p = (b + (u64)j) & DEV.ct_mask;
      const CtEntry e = DEV.ct[p];
      if (e.key == key) return Probe{p, e.val, true};
      if (e.key == kEmptyKey || e.key == kTombKey) {
        if (first_free == ~0ull) first_free = p;
        if (e.key == kEmptyKey) return Probe{first_free, 0, false};
      }
    }
#endif
  }
  return Probe{first_free, 0, false};
}

// warp-wide: the inline child first, the table only for the other children
E2_D u32 child_lookup(u32 parent, i32 tok) {
  const NodeRec* r = npeek(parent);
  const u32 is = r->in_slot;
  if (is != 0 && r->in_tok == tok) return is;
  if (r->nchild <= (is != 0 ? 1 : 0)) return kNil;  // no child in the table
  Probe p = ct_probe(ckey(parent, tok));
  return p.found ? p.val : kNil;
}

// warp-wide; key must be absent.  Records the entry's position in the
// child's record (ctpos), so re-pointing or erasing it needs no probe.
E2_DNI bool child_insert(u32 parent, i32 tok, u32 child) {
  NodeRec* rp = nget(parent);
  if (rp->in_slot == 0) {  // the parent's inline child
    wsync();
    if (lane0()) {
      rp->in_tok = tok;
      rp->in_slot = child;
      nget_lane(child)->ctpos = kCtInline;
    }
    wsync();
    return true;
  }
  const u64 key = ckey(parent, tok);
  Probe p = ct_probe(key);
  if (p.found || p.pos == ~0ull) {
    if (lane0()) set_err(kErrCapacity, kWhyTableFull);
    wsync();
    return false;
  }
  wsync();
  if (lane0()) {
    CtEntry e;
    e.key = key;
    e.val = child;
    e.pad = 0;
    DEV.ct[p.pos] = e;
    NodeRec* rc = nget_lane(child);
    rc->ctpos = (u32)p.pos;
  }
  wsync();
  return true;
}

// warp-wide; key must be present.
E2_DNI void child_update(u32 parent, i32 tok, u32 child) {
  NodeRec* rp = nget(parent);
  if (rp->in_slot != 0 && rp->in_tok == tok) {
    wsync();
    if (lane0()) rp->in_slot = child;
    wsync();
    return;
  }
  Probe p = ct_probe(ckey(parent, tok));
  wsync();
  if (lane0()) {
    if (p.found)
      DEV.ct[p.pos].val = child;
    else
      set_err(kErrSim, kWhyWalk);
  }
  wsync();
}

// warp-wide
E2_DNI void child_erase(u32 parent, i32 tok) {
  NodeRec* rp = nget(parent);
  if (rp->in_slot != 0 && rp->in_tok == tok) {
    wsync();
    if (lane0()) {
      rp->in_slot = 0;
      rp->in_tok = 0;
    }
    wsync();
    return;
  }
  Probe p = ct_probe(ckey(parent, tok));
  wsync();
  if (lane0()) {
    if (p.found)
      DEV.ct[p.pos].key = kTombKey;
    else
      set_err(kErrSim, kWhyWalk);
  }
  wsync();
}

// warp-wide: erase the entry at a known position (the node's ctpos);
// falls back to a probe if the position does not hold the key.
E2_DNI void child_erase_at(u32 pos, u32 parent, i32 tok) {
  if (pos == kCtInline) {
    NodeRec* rp = nget(parent);
    wsync();
    if (lane0() && rp->in_tok == tok && rp->in_slot != 0) {
      rp->in_slot = 0;
      rp->in_tok = 0;
    }
    wsync();
    return;
  }
  const u64 key = ckey(parent, tok);
  if ((u64)pos <= DEV.ct_mask && DEV.ct[pos].key == key) {
    if (lane0()) DEV.ct[pos].key = kTombKey;
    wsync();
    return;
  }
  child_erase(parent, tok);
}


// ---------------------------------------------------------------------------
// Per-instance LRU index: ordered set of (last_access bits, id) over LRU
// leaves (cached on g, no cached child on g) — prefix_tree.cpp:14-35.
// ---------------------------------------------------------------------------
E2_HDX bool kless(u64 ala, u64 aid, u64 bla, u64 bid) { return ala < bla || (ala == bla && aid < bid); }

E2_HD u64 dring(int g, u32 k) {
  return (u64)g * DEV.dcap + ((HOT.dir_head[g] + k) & (DEV.dcap - 1));
}

// warp-wide: first directory position whose page max >= key (n if none).
E2_DNI u32 dir_lower_bound(int g, u64 kla, u64 kid) {
  u32 lo = 0, hi = HOT.dir_n[g];
#if E2_WARP
  while (hi > lo) {
    const u32 step = (hi - lo + 31) / 32;
    const u32 J = (hi - lo + step - 1) / step;
    const u32 F = (u32)popc32(vote((int)J, [&](int j) {
      const DirEntry& e = DEV.dir[dring(g, lo + (u32)j * step)];
      return kless(e.max_la, e.max_id, kla, kid);
    }));
    if (F == 0) return lo;
    if (step == 1) return lo + F;
    const u32 newlo = lo + (F - 1) * step + 1;
    const u32 newhi = F < J ? lo + F * step : hi;
    lo = newlo;
    hi = newhi;
  }
  return lo;
#else
  while (lo < hi) {
    u32 mid = lo + (hi - lo) / 2;
    const DirEntry& e = DEV.dir[dring(g, mid)];
    if (kless(e.max_la, e.max_id, kla, kid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
#endif
}

// warp-wide page allocation.
E2_D u32 page_alloc() {
  u32 p = kNil;
  if (HOT.free_top > 0)
    p = DEV.free_pages[HOT.free_top - 1];
  else if (HOT.pages_used < DEV.page_cap)
    p = HOT.pages_used;
  wsync();
  if (lane0()) {
    if (p == kNil)
      set_err(kErrCapacity, kWhyPageCap);
    else if (HOT.free_top > 0)
      HOT.free_top--;
    else
      HOT.pages_used++;
  }
  wsync();
  return p;
}

E2_D void page_free(u32 p) {
  if (lane0()) {
    DEV.free_pages[HOT.free_top] = p;
    HOT.free_top++;
  }
  wsync();
}

// warp-wide: insert a directory entry at position k.
E2_DNI bool dir_insert_at(int g, u32 k, const DirEntry& e) {
  const u32 n = HOT.dir_n[g];
  if (n >= DEV.dcap) {
    if (lane0()) set_err(kErrCapacity, kWhyDirCap);
    wsync();
    return false;
  }
  if (k == 0 && n > 0) {
    if (lane0()) HOT.dir_head[g] = (HOT.dir_head[g] + DEV.dcap - 1) & (DEV.dcap - 1);
    wsync();
  } else {
    // shift [k, n) up by one, highest chunk first
    for (i64 top = (i64)n - 1; top >= (i64)k; top -= kWidth) {
      const i64 pos = top - lane();
      const bool act = pos >= (i64)k;
      DirEntry v;
      if (act) v = DEV.dir[dring(g, (u32)pos)];
      wsync();
      if (act) DEV.dir[dring(g, (u32)pos + 1)] = v;
      wsync();
    }
  }
  if (lane0()) {
    DEV.dir[dring(g, k)] = e;
    HOT.dir_n[g] = n + 1;
  }
  wsync();
  return true;
}

// warp-wide: remove directory position k.
E2_DNI void dir_remove_at(int g, u32 k) {
  const u32 n = HOT.dir_n[g];
  if (k == 0) {
    if (lane0()) HOT.dir_head[g] = (HOT.dir_head[g] + 1) & (DEV.dcap - 1);
  } else {
    for (u32 lo = k + 1; lo < n; lo += kWidth) {
      const u32 pos = lo + (u32)lane();
      const bool act = pos < n;
      DirEntry v;
      if (act) v = DEV.dir[dring(g, pos)];
      wsync();
      if (act) DEV.dir[dring(g, pos - 1)] = v;
      wsync();
    }
  }
  if (lane0()) HOT.dir_n[g] = n - 1;
  wsync();
}

// warp-wide: insert into page p (has room) at directory position k.
E2_DNI void page_insert(int g, u32 k, u32 p, i32 cnt, u64 kla, u64 kid, u32 slot) {
  const u64 base = (u64)p * kPage;
#if E2_WARP
  const int j = lane();
  const bool valid = j < cnt;
  u64 ela = 0, eid = 0;
  u32 es = 0;
  if (valid) {
    ela = DEV.pg_la[base + j];
    eid = DEV.pg_id[base + j];
    es = DEV.pg_slot[base + j];
  }
  const int pos = popc32(ballot(valid && kless(ela, eid, kla, kid)));
  wsync();
  if (valid && j >= pos) {
    DEV.pg_la[base + j + 1] = ela;
    DEV.pg_id[base + j + 1] = eid;
    DEV.pg_slot[base + j + 1] = es;
  }
  if (j == pos) {
    DEV.pg_la[base + j] = kla;
    DEV.pg_id[base + j] = kid;
    DEV.pg_slot[base + j] = slot;
  }
#else
  int pos = 0;
  while (pos < cnt && kless(DEV.pg_la[base + pos], DEV.pg_id[base + pos], kla, kid)) pos++;
  for (int j = cnt - 1; j >= pos; --j) {
    DEV.pg_la[base + j + 1] = DEV.pg_la[base + j];
    DEV.pg_id[base + j + 1] = DEV.pg_id[base + j];
    DEV.pg_slot[base + j + 1] = DEV.pg_slot[base + j];
  }
  DEV.pg_la[base + pos] = kla;
  DEV.pg_id[base + pos] = kid;
  DEV.pg_slot[base + pos] = slot;
#endif
  if (lane0()) {
    DirEntry& e = DEV.dir[dring(g, k)];
    e.cnt = cnt + 1;
    if (pos == cnt) {
      e.max_la = kla;
      e.max_id = kid;
    }
  }
  wsync();
}

// warp-wide
E2_DNI void lru_insert(int g, u64 kla, u64 kid, u32 slot) {
  const u32 n = HOT.dir_n[g];
  if (n > 0) {
    // fast path: strictly after every key (fresh last_access) -> tail page
    const DirEntry t = DEV.dir[dring(g, n - 1)];
    if (kless(t.max_la, t.max_id, kla, kid)) {
      if (t.cnt < kPage) {
        if (lane0()) {
          const u64 i = (u64)t.page * kPage + t.cnt;
          DEV.pg_la[i] = kla;
          DEV.pg_id[i] = kid;
          DEV.pg_slot[i] = slot;
          DirEntry& e = DEV.dir[dring(g, n - 1)];
          e.cnt = t.cnt + 1;
          e.max_la = kla;
          e.max_id = kid;
        }
        wsync();
        return;
      }
      const u32 q = page_alloc();
      if (q == kNil) return;
      DirEntry e;
      e.page = q;
      e.cnt = 1;
      e.max_la = kla;
      e.max_id = kid;
      e.pad = 0;
      if (lane0()) {
        DEV.pg_la[(u64)q * kPage] = kla;
        DEV.pg_id[(u64)q * kPage] = kid;
        DEV.pg_slot[(u64)q * kPage] = slot;
      }
      wsync();
      dir_insert_at(g, n, e);
      return;
    }
  } else {
    const u32 q = page_alloc();
    if (q == kNil) return;
    DirEntry e;
    e.page = q;
    e.cnt = 1;
    e.max_la = kla;
    e.max_id = kid;
    e.pad = 0;
    if (lane0()) {
      DEV.pg_la[(u64)q * kPage] = kla;
      DEV.pg_id[(u64)q * kPage] = kid;
      DEV.pg_slot[(u64)q * kPage] = slot;
    }
    wsync();
    dir_insert_at(g, 0, e);
    return;
  }
  u32 k = dir_lower_bound(g, kla, kid);
  if (k >= n) k = n - 1;
  DirEntry e = DEV.dir[dring(g, k)];
  u32 p = e.page;
  i32 cnt = e.cnt;
  if (cnt >= kPage) {
    // split page p: upper half moves to a new page at k+1
    const u32 q = page_alloc();
    if (q == kNil) return;
    const int half = kPage / 2;
    const u64 bp = (u64)p * kPage, bq = (u64)q * kPage;
    for (int j = lane(); j < half; j += kWidth) {
      DEV.pg_la[bq + j] = DEV.pg_la[bp + half + j];
      DEV.pg_id[bq + j] = DEV.pg_id[bp + half + j];
      DEV.pg_slot[bq + j] = DEV.pg_slot[bp + half + j];
    }
    wsync();
    const u64 nmla = DEV.pg_la[bp + half - 1], nmid = DEV.pg_id[bp + half - 1];
    wsync();
    DirEntry eq;
    eq.page = q;
    eq.cnt = half;
    eq.max_la = e.max_la;
    eq.max_id = e.max_id;
    eq.pad = 0;
    if (lane0()) {
      DirEntry& ep = DEV.dir[dring(g, k)];
      ep.cnt = half;
      ep.max_la = nmla;
      ep.max_id = nmid;
    }
    wsync();
    if (!dir_insert_at(g, k + 1, eq)) return;
    if (kless(nmla, nmid, kla, kid)) {
      p = q;
      k = k + 1;
    }
    cnt = half;
  }
  page_insert(g, k, p, cnt, kla, kid, slot);
}

// warp-wide
E2_DNI void lru_erase(int g, u64 kla, u64 kid) {
  const u32 n = HOT.dir_n[g];
  u32 k;
  const DirEntry h0 = DEV.dir[dring(g, 0)];
  if (n > 0 && !kless(h0.max_la, h0.max_id, kla, kid))
    k = 0;  // fast path: in the head page (LRU victims)
  else
    k = dir_lower_bound(g, kla, kid);
  if (k >= n) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const DirEntry e = k == 0 ? h0 : DEV.dir[dring(g, k)];
  const u32 p = e.page;
  const i32 cnt = e.cnt;
  const u64 base = (u64)p * kPage;
#if E2_WARP
  const int j = lane();
  const bool valid = j < cnt;
  u64 ela = 0, eid = 0;
  u32 es = 0;
  if (valid) {
    ela = DEV.pg_la[base + j];
    eid = DEV.pg_id[base + j];
    es = DEV.pg_slot[base + j];
  }
  const u32 m = ballot(valid && ela == kla && eid == kid);
  if (!m) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const int idx = ffs32(m);
  const u64 pla = shfl(ela, cnt >= 2 ? cnt - 2 : 0);
  const u64 pid = shfl(eid, cnt >= 2 ? cnt - 2 : 0);
  wsync();
  if (valid && j > idx) {
    DEV.pg_la[base + j - 1] = ela;
    DEV.pg_id[base + j - 1] = eid;
    DEV.pg_slot[base + j - 1] = es;
  }
#else
  int idx = -1;
  for (int j = 0; j < cnt; ++j)
    if (DEV.pg_la[base + j] == kla && DEV.pg_id[base + j] == kid) idx = j;
  if (idx < 0) {
    set_err(kErrSim, kWhyWalk);
    return;
  }
  const u64 pla = cnt >= 2 ? DEV.pg_la[base + cnt - 2] : 0;
  const u64 pid = cnt >= 2 ? DEV.pg_id[base + cnt - 2] : 0;
  for (int j = idx + 1; j < cnt; ++j) {
    DEV.pg_la[base + j - 1] = DEV.pg_la[base + j];
    DEV.pg_id[base + j - 1] = DEV.pg_id[base + j];
    DEV.pg_slot[base + j - 1] = DEV.pg_slot[base + j];
  }
#endif
  if (lane0()) {
    DirEntry& er = DEV.dir[dring(g, k)];
    er.cnt = cnt - 1;
    if (cnt - 1 > 0 && idx == cnt - 1) {
      er.max_la = pla;
      er.max_id = pid;
    }
  }
  wsync();
  if (cnt - 1 == 0) {
    page_free(p);
    dir_remove_at(g, k);
  }
}

// warp-wide: the entry with key (kla, kid) now belongs to slot `slot`.
E2_DNI void lru_relabel(int g, u64 kla, u64 kid, u32 slot) {
  const u32 n = HOT.dir_n[g];
  u32 k;
  const DirEntry h0 = DEV.dir[dring(g, 0)];
  if (n > 0 && !kless(h0.max_la, h0.max_id, kla, kid))
    k = 0;
  else
    k = dir_lower_bound(g, kla, kid);
  if (k >= n) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const DirEntry e = k == 0 ? h0 : DEV.dir[dring(g, k)];
  const u64 base = (u64)e.page * kPage;
  const u32 m = vote(e.cnt, [&](int j) { return DEV.pg_la[base + j] == kla && DEV.pg_id[base + j] == kid; });
  wsync();
  if (!m) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
  } else if (lane0()) {
    DEV.pg_slot[base + ffs32(m)] = slot;
  }
  wsync();
}

// warp-wide: the entry (kla, old_id) is re-keyed to (kla, new_id), new_id
// larger than every id in the index (split suffixes take next_id).  When no
// key lies between the two (the usual case: no other leaf shares this
// last_access), the entry keeps its position and only its id and slot
// change; otherwise it is erased and re-inserted.  Same set either way.
E2_DNI void lru_rekey(int g, u64 kla, u64 old_id, u64 new_id, u32 slot) {
  const u32 n = HOT.dir_n[g];
  u32 k;
  const DirEntry h0 = DEV.dir[dring(g, 0)];
  if (n > 0 && !kless(h0.max_la, h0.max_id, kla, old_id))
    k = 0;
  else
    k = dir_lower_bound(g, kla, old_id);
  if (k >= n) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const DirEntry e = k == 0 ? h0 : DEV.dir[dring(g, k)];
  const u64 base = (u64)e.page * kPage;
  const u32 m = vote(e.cnt, [&](int j) { return DEV.pg_la[base + j] == kla && DEV.pg_id[base + j] == old_id; });
  wsync();
  if (!m) {
    if (lane0()) set_err(kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const int idx = ffs32(m);
  bool inplace = true;
  if (idx + 1 < e.cnt) {
    inplace = kless(kla, new_id, DEV.pg_la[base + idx + 1], DEV.pg_id[base + idx + 1]);
  } else if (k + 1 < n) {
    const DirEntry e2 = DEV.dir[dring(g, k + 1)];
    const u64 b2 = (u64)e2.page * kPage;
    inplace = kless(kla, new_id, DEV.pg_la[b2], DEV.pg_id[b2]);
  }
  if (!inplace) {
    lru_erase(g, kla, old_id);
    lru_insert(g, kla, new_id, slot);
    return;
  }
  if (lane0()) {
    DEV.pg_id[base + idx] = new_id;
    DEV.pg_slot[base + idx] = slot;
    if (idx == e.cnt - 1) DEV.dir[dring(g, k)].max_id = new_id;
  }
  wsync();
}

// ---------------------------------------------------------------------------
// Node state helpers (all warp-wide; records via the node cache)
// ---------------------------------------------------------------------------
E2_HD bool rcached(const NodeRec* r, int g) { return (r->cmask >> g) & 1ull; }

E2_HD bool rleaf(const NodeRec* r, u32 s, int g, int G) {
  return s != kRoot && rcached(r, g) && rccc(r, G)[g] == 0;
}

// warp-wide: allocate a fresh slot and its zeroed cached record.
E2_D u32 node_alloc() {
  const u32 s = HOT.slots_used;
  wsync();
  if (s >= DEV.node_cap) {
    if (lane0()) set_err(kErrCapacity, kWhyNodeCap);
    wsync();
    return kNil;
  }
  if (lane0()) HOT.slots_used = s + 1;
  wsync();
  return s;
}

// warp-wide: split_node(s, k) with the slot kept on the suffix — see
// e2_state.cuh.  Returns the new slot holding the prefix (old id).
// Reference: prefix_tree.cpp:122-154.  rekey=false leaves the LRU index to
// the caller (evict_tail: the suffix is uncached right away).
E2_DNI u32 split_node(u32 s, u32 k, bool rekey = true) {
  const int G = DEV.cfg.G;
  NodeRec* rs = nget(s);
  const NodeRec hs = *rs;
  if (k == 0 || k >= hs.edge_len) {
    if (lane0()) set_err(kErrSim, kWhySplitBounds);
    wsync();
    return kNil;
  }
  const u32 q = node_alloc();
  if (q == kNil) return kNil;
  touch(s);
  touch(q);
  const u64 new_id = HOT.next_id;
  const i32 tok_k = DEV.tok[hs.edge_off + k];
  // prefix: copy the whole record (la/hits), then fix header and ccc
#if defined(E2_SMEM_NODECACHE)
  NodeRec* rq = nnew(q);
#else
  NodeRec* rq = grec(q);  // every word is overwritten by the copy below
#endif
  rs = nget(s);
  {
    const u64* src = (const u64*)rs;
    u64* dst = (u64*)rq;
    for (u32 j = (u32)lane(); j < DEV.rs / 8; j += kWidth) dst[j] = src[j];
  }
  wsync();
  if (lane0()) {
    rq->edge_len = k;
    rq->nchild = 1;
    for (int g = 0; g < G; ++g) rccc(rq, G)[g] = ((hs.cmask >> g) & 1ull) ? 1 : 0;
    rs->id = new_id;
    rs->edge_off = hs.edge_off + k;
    rs->edge_len = hs.edge_len - k;
    rs->parent = q;
    rs->first_tok = tok_k;
    rs->depth = hs.depth + k;
    ndirty(rs);
    HOT.next_id = new_id + 1;
    HOT.node_count++;
  }
  wsync();
  // the parent's entry for this edge now leads to the prefix (which copied
  // the record, ctpos included); the suffix hangs under the prefix as its
  // inline child (no table entry)
  if (lane0()) {
    if (hs.ctpos == kCtInline)
      npoke(hs.parent)->in_slot = q;
    else
      DEV.ct[hs.ctpos].val = q;
    rq->in_tok = tok_k;
    rq->in_slot = s;
    rs->ctpos = kCtInline;
  }
  wsync();
  if (!rekey) return q;
  // LRU: the suffix inherits the leaf role under its new id.
#if E2_WARP
  if (g_defer_ct && threadIdx.x < 32 && !g_rkd.pending) {
    if (lane0()) {
      const NodeRec* r = nget(s);
      u64 lm = 0;
      for (u64 m = hs.cmask; m; m &= m - 1) {
        const int g = ffs64(m);
        if (rccc(r, G)[g] == 0) lm |= 1ull << g;
      }
      if (lm) {
        g_rkd.mask = lm;
        g_rkd.old_id = hs.id;
        g_rkd.new_id = new_id;
        g_rkd.slot = s;
        __threadfence_block();
        g_rkd.pending = 1;
      }
    }
    wsync();
    return q;
  }
#endif
  u64 m = hs.cmask;
  while (m) {
    const int g = ffs64(m);
    m &= m - 1;
    const NodeRec* r = nget(s);
    if (rccc(r, G)[g] == 0) lru_rekey(g, dbits(rla(r)[g]), hs.id, new_id, s);
  }
  return q;
}

#if E2_WARP
// The eviction warp: apply a deferred re-keying (see RekeyDefer).
// Warp-uniform caller: g_rkd.pending was seen set (by lane 0).
E2_D void rekey_deferred() {
  __threadfence_block();
  const int G = DEV.cfg.G;
  const u32 s = g_rkd.slot;
  for (u64 m = g_rkd.mask; m; m &= m - 1) {
    const int g = ffs64(m);
    const NodeRec* r = nget(s);
    lru_rekey(g, dbits(rla(r)[g]), g_rkd.old_id, g_rkd.new_id, s);
  }
  wsync();
  if (lane0()) g_rkd.pending = 0;
  wsync();
}
#endif

// warp-wide: new leaf under parent with edge [off, off+len).
E2_DNI u32 new_leaf(u32 parent, i64 off, u32 len, u32 depth) {
  const u32 l = node_alloc();
  if (l == kNil) return kNil;
  const i32 t0 = DEV.tok[off];
  const u64 id = HOT.next_id;
  NodeRec* rl = nnew(l);
  if (lane0()) {
    rl->id = id;
    rl->edge_off = off;
    rl->edge_len = len;
    rl->parent = parent;
    rl->first_tok = t0;
    rl->depth = depth;
    HOT.next_id = id + 1;
    HOT.node_count++;
  }
  wsync();
  NodeRec* rp = nget(parent);
  if (lane0()) {
    rp->nchild += 1;
    ndirty(rp);
  }
  wsync();
#if E2_WARP
  if (g_defer_ct && threadIdx.x < 32 && rp->in_slot != 0) {
    if (lane0()) {
      g_ctd.parent = parent;
      g_ctd.child = l;
      g_ctd.tok = t0;
      g_ctd.pending = 1;
    }
    wsync();
    return l;
  }
#endif
  child_insert(parent, t0, l);
  return l;
}

// warp-wide: set_cached (prefix_tree.cpp:53-63).
E2_DNI void set_cached(u32 s, int g) {
  const int G = DEV.cfg.G;
  if (s == kRoot) return;
  NodeRec* r = nget(s);
  if (rcached(r, g)) return;
  const u32 p = r->parent;
  const u32 len = r->edge_len;
  const u64 sid = r->id;
  wsync();
  if (lane0()) {
    r->cmask |= (1ull << g);
    ndirty(r);
    HOT.cached_tokens[g] += len;
  }
  wsync();
  if (rccc(r, G)[g] == 0) lru_insert(g, dbits(rla(r)[g]), sid, s);
  if (p != kNil) {
    NodeRec* rp = nget(p);
    const bool p_was = rleaf(rp, p, g, G);
    const u64 pla = dbits(rla(rp)[g]), pid = rp->id;
    wsync();
    if (lane0()) {
      rccc(rp, G)[g] += 1;
      ndirty(rp);
    }
    wsync();
    if (p_was) lru_erase(g, pla, pid);
  }
}

// warp-wide: clear_cached (prefix_tree.cpp:65-77).
E2_DNI void clear_cached(u32 s, int g) {
  const int G = DEV.cfg.G;
  NodeRec* r = nget(s);
  if (!rcached(r, g)) return;
  touch(s);
  const u32 p = r->parent;
  const u32 len = r->edge_len;
  if (rleaf(r, s, g, G)) lru_erase(g, dbits(rla(r)[g]), r->id);
  r = nget(s);
  wsync();
  if (lane0()) {
    r->cmask &= ~(1ull << g);
    ndirty(r);
    HOT.cached_tokens[g] -= len;
  }
  wsync();
  if (p != kNil) {
    NodeRec* rp = nget(p);
    const i32 c = rccc(rp, G)[g] - 1;
    wsync();
    if (lane0()) {
      rccc(rp, G)[g] = c;
      ndirty(rp);
      if (c < 0) set_err(kErrSim, kWhyCccUnderflow);
    }
    wsync();
    if (c == 0 && rleaf(rp, p, g, G)) lru_insert(g, dbits(rla(rp)[g]), rp->id, p);
  }
}

// warp-wide: last_access[g] = max(last_access[g], now) with the entry created
// (record_hit / mark_cached_path: prefix_tree.cpp:45-51, 207-210).
E2_DNI void touch_la(u32 s, int g, double now) {
  const int G = DEV.cfg.G;
  NodeRec* r = nget(s);
  const double old = rla(r)[g];
  const bool was = rleaf(r, s, g, G);
  const u64 id = r->id;
  const bool upd = now > old;
  wsync();
  if (lane0()) {
    r->lamask |= (1ull << g);
    if (upd) rla(r)[g] = now;
    ndirty(r);
  }
  wsync();
  if (upd && was) {
    lru_erase(g, dbits(old), id);
    lru_insert(g, dbits(now), id, s);
  }
}

}  // namespace e2
