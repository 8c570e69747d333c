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

struct Ctx {
  Dev d;
  Hot* h;
  NCache* c;
};

E2_HD void set_err(Hot* h, i32 code, i32 why) {
  if (h->err == 0) {
    h->err = code;
    h->why = why;
  }
}

E2_HD NodeRec* nentry(const Ctx& x, u32 w) { return (NodeRec*)(x.c->data + (u64)w * x.d.rs); }

// single-lane: mark the cache entry holding r as modified
E2_HD void ndirty(const Ctx& x, const NodeRec* r) {
  x.c->dirty[(u32)(((const char*)r - x.c->data) / x.d.rs)] = 1;
}

// warp-wide copy of one record (rs bytes, 8-byte words)
E2_D void rcopy(u64* dst, const u64* src, u32 words) {
  for (u32 j = (u32)lane(); j < words; j += kWidth) dst[j] = src[j];
}

// warp-wide: pick the way to (re)use in s's set; write back if dirty.
E2_D u32 nclaim(Ctx& x, u32 s) {
  NCache* c = x.c;
  const u32 base = (s & (c->nsets - 1)) * kWays;
  if (lane0()) {
    u32 best = base;
    for (u32 k = 0; k < (u32)kWays; ++k) {
      const u32 w = base + k;
      if (c->tag[w] == kNil) {
        best = w;
        break;
      }
      if (c->tick[w] < c->tick[best]) best = w;
    }
    c->victim = best;
  }
  wsync();
  const u32 w = c->victim;
  const u32 old = c->tag[w];
  if (old != kNil && c->dirty[w]) rcopy((u64*)grec(x.d, old), (const u64*)nentry(x, w), x.d.rs / 8);
  return w;
}

// warp-wide: make node s resident and return its cached record.
E2_D NodeRec* nget(Ctx& x, u32 s) {
  NCache* c = x.c;
  const u32 base = (s & (c->nsets - 1)) * kWays;
  const u32 hit = vote(kWays, [&](int k) { return c->tag[base + k] == s; });
  if (hit) {
    const u32 w = base + (u32)ffs32(hit);
    wsync();
    if (lane0()) c->tick[w] = ++c->clock;
    wsync();
    return nentry(x, w);
  }
  const u32 w = nclaim(x, s);
  rcopy((u64*)nentry(x, w), (const u64*)grec(x.d, s), x.d.rs / 8);
  wsync();
  if (lane0()) {
    c->tag[w] = s;
    c->tick[w] = ++c->clock;
    c->dirty[w] = 0;
  }
  wsync();
  return nentry(x, w);
}

// warp-wide: a fresh (zeroed, dirty) record for a newly allocated slot.
E2_D NodeRec* nnew(Ctx& x, u32 s) {
  NCache* c = x.c;
  const u32 w = nclaim(x, s);
  u64* dst = (u64*)nentry(x, w);
  for (u32 j = (u32)lane(); j < x.d.rs / 8; j += kWidth) dst[j] = 0;
  wsync();
  if (lane0()) {
    c->tag[w] = s;
    c->tick[w] = ++c->clock;
    c->dirty[w] = 1;
  }
  wsync();
  return nentry(x, w);
}

// single-lane read-only view (cached copy if resident, else HBM).
E2_HD const NodeRec* npeek(const Ctx& x, u32 s) {
  const NCache* c = x.c;
  const u32 base = (s & (c->nsets - 1)) * kWays;
  for (u32 k = 0; k < (u32)kWays; ++k)
    if (c->tag[base + k] == s) return nentry(x, base + k);
  return grec(x.d, s);
}

// warp-wide: write every dirty record back.
E2_D void nflush(Ctx& x) {
  NCache* c = x.c;
  const u32 n = c->nsets * kWays;
  for (u32 w = 0; w < n; ++w) {
    if (c->tag[w] != kNil && c->dirty[w]) rcopy((u64*)grec(x.d, c->tag[w]), (const u64*)nentry(x, w), x.d.rs / 8);
  }
  wsync();
  for (u32 w = (u32)lane(); w < n; w += kWidth) c->dirty[w] = 0;
  wsync();
}

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
E2_D Probe ct_probe(const Dev& d, u64 key) {
  u64 b = mix64(key) & d.ct_mask;
  u64 first_free = ~0ull;
  for (u64 step = 0; step <= d.ct_mask; step += 32, b += 32) {
#if E2_DEVICE_BUILD
    const CtEntry e = d.ct[(b + lane()) & d.ct_mask];
    const u32 hit = ballot(e.key == key);
    const u32 emp = ballot(e.key == kEmptyKey);
    const u32 fr = emp | ballot(e.key == kTombKey);
    if (first_free == ~0ull && fr) first_free = (b + (u64)ffs32(fr)) & d.ct_mask;
    if (hit) {
      const int j = ffs32(hit);
      return Probe{(b + (u64)j) & d.ct_mask, shfl(e.val, j), true};
    }
#else
    u32 hit = 0, emp = 0, fr = 0;
    for (int j = 0; j < 32; ++j) {
      const u64 k = d.ct[(b + j) & d.ct_mask].key;
      if (k == key) hit |= 1u << j;
      if (k == kEmptyKey) emp |= 1u << j;
      if (k == kEmptyKey || k == kTombKey) fr |= 1u << j;
    }
    if (first_free == ~0ull && fr) first_free = (b + (u64)ffs32(fr)) & d.ct_mask;
    if (hit) {
      const u64 p = (b + (u64)ffs32(hit)) & d.ct_mask;
      return Probe{p, d.ct[p].val, true};
    }
#endif
    if (emp) return Probe{first_free, 0, false};
  }
  return Probe{first_free, 0, false};
}

// warp-wide
E2_D u32 child_lookup(const Dev& d, u32 parent, i32 tok) {
  Probe p = ct_probe(d, ckey(parent, tok));
  return p.found ? p.val : kNil;
}

// warp-wide; key must be absent.
E2_D bool child_insert(const Dev& d, Hot* h, u32 parent, i32 tok, u32 child) {
  const u64 key = ckey(parent, tok);
  Probe p = ct_probe(d, key);
  if (p.found || p.pos == ~0ull) {
    if (lane0()) set_err(h, kErrCapacity, kWhyTableFull);
    wsync();
    return false;
  }
  wsync();
  if (lane0()) {
    CtEntry e;
    e.key = key;
    e.val = child;
    e.pad = 0;
    d.ct[p.pos] = e;
  }
  wsync();
  return true;
}

// warp-wide; key must be present.
E2_D void child_update(const Dev& d, Hot* h, u32 parent, i32 tok, u32 child) {
  Probe p = ct_probe(d, ckey(parent, tok));
  wsync();
  if (lane0()) {
    if (p.found)
      d.ct[p.pos].val = child;
    else
      set_err(h, kErrSim, kWhyWalk);
  }
  wsync();
}

// warp-wide
E2_D void child_erase(const Dev& d, Hot* h, u32 parent, i32 tok) {
  Probe p = ct_probe(d, ckey(parent, tok));
  wsync();
  if (lane0()) {
    if (p.found)
      d.ct[p.pos].key = kTombKey;
    else
      set_err(h, kErrSim, kWhyWalk);
  }
  wsync();
}

// ---------------------------------------------------------------------------
// Per-instance LRU index: ordered set of (last_access bits, id) over LRU
// leaves (cached on g, no cached child on g) — prefix_tree.cpp:14-35.
// ---------------------------------------------------------------------------
E2_HDX bool kless(u64 ala, u64 aid, u64 bla, u64 bid) { return ala < bla || (ala == bla && aid < bid); }

E2_HD u64 dring(const Dev& d, const Hot* h, int g, u32 k) {
  return (u64)g * d.dcap + ((h->dir_head[g] + k) & (d.dcap - 1));
}

// warp-wide: first directory position whose page max >= key (n if none).
E2_D u32 dir_lower_bound(const Dev& d, const Hot* h, int g, u64 kla, u64 kid) {
  u32 lo = 0, hi = h->dir_n[g];
#if E2_DEVICE_BUILD
  while (hi > lo) {
    const u32 step = (hi - lo + 31) / 32;
    const u32 J = (hi - lo + step - 1) / step;
    const u32 F = (u32)popc32(vote((int)J, [&](int j) {
      const DirEntry& e = d.dir[dring(d, h, g, lo + (u32)j * step)];
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
    const DirEntry& e = d.dir[dring(d, h, g, mid)];
    if (kless(e.max_la, e.max_id, kla, kid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
#endif
}

// warp-wide page allocation.
E2_D u32 page_alloc(const Dev& d, Hot* h) {
  u32 p = kNil;
  if (h->free_top > 0)
    p = d.free_pages[h->free_top - 1];
  else if (h->pages_used < d.page_cap)
    p = h->pages_used;
  wsync();
  if (lane0()) {
    if (p == kNil)
      set_err(h, kErrCapacity, kWhyPageCap);
    else if (h->free_top > 0)
      h->free_top--;
    else
      h->pages_used++;
  }
  wsync();
  return p;
}

E2_D void page_free(const Dev& d, Hot* h, u32 p) {
  if (lane0()) {
    d.free_pages[h->free_top] = p;
    h->free_top++;
  }
  wsync();
}

// warp-wide: insert a directory entry at position k.
E2_D bool dir_insert_at(const Dev& d, Hot* h, int g, u32 k, const DirEntry& e) {
  const u32 n = h->dir_n[g];
  if (n >= d.dcap) {
    if (lane0()) set_err(h, kErrCapacity, kWhyDirCap);
    wsync();
    return false;
  }
  if (k == 0 && n > 0) {
    if (lane0()) h->dir_head[g] = (h->dir_head[g] + d.dcap - 1) & (d.dcap - 1);
    wsync();
  } else {
    // shift [k, n) up by one, highest chunk first
    for (i64 top = (i64)n - 1; top >= (i64)k; top -= kWidth) {
      const i64 pos = top - lane();
      const bool act = pos >= (i64)k;
      DirEntry v;
      if (act) v = d.dir[dring(d, h, g, (u32)pos)];
      wsync();
      if (act) d.dir[dring(d, h, g, (u32)pos + 1)] = v;
      wsync();
    }
  }
  if (lane0()) {
    d.dir[dring(d, h, g, k)] = e;
    h->dir_n[g] = n + 1;
  }
  wsync();
  return true;
}

// warp-wide: remove directory position k.
E2_D void dir_remove_at(const Dev& d, Hot* h, int g, u32 k) {
  const u32 n = h->dir_n[g];
  if (k == 0) {
    if (lane0()) h->dir_head[g] = (h->dir_head[g] + 1) & (d.dcap - 1);
  } else {
    for (u32 lo = k + 1; lo < n; lo += kWidth) {
      const u32 pos = lo + (u32)lane();
      const bool act = pos < n;
      DirEntry v;
      if (act) v = d.dir[dring(d, h, g, pos)];
      wsync();
      if (act) d.dir[dring(d, h, g, pos - 1)] = v;
      wsync();
    }
  }
  if (lane0()) h->dir_n[g] = n - 1;
  wsync();
}

// warp-wide: insert into page p (has room) at directory position k.
E2_D void page_insert(const Dev& d, Hot* h, int g, u32 k, u32 p, i32 cnt, u64 kla, u64 kid, u32 slot) {
  const u64 base = (u64)p * kPage;
#if E2_DEVICE_BUILD
  const int j = lane();
  const bool valid = j < cnt;
  u64 ela = 0, eid = 0;
  u32 es = 0;
  if (valid) {
    ela = d.pg_la[base + j];
    eid = d.pg_id[base + j];
    es = d.pg_slot[base + j];
  }
  const int pos = popc32(ballot(valid && kless(ela, eid, kla, kid)));
  wsync();
  if (valid && j >= pos) {
    d.pg_la[base + j + 1] = ela;
    d.pg_id[base + j + 1] = eid;
    d.pg_slot[base + j + 1] = es;
  }
  if (j == pos) {
    d.pg_la[base + j] = kla;
    d.pg_id[base + j] = kid;
    d.pg_slot[base + j] = slot;
  }
#else
  int pos = 0;
  while (pos < cnt && kless(d.pg_la[base + pos], d.pg_id[base + pos], kla, kid)) pos++;
  for (int j = cnt - 1; j >= pos; --j) {
    d.pg_la[base + j + 1] = d.pg_la[base + j];
    d.pg_id[base + j + 1] = d.pg_id[base + j];
    d.pg_slot[base + j + 1] = d.pg_slot[base + j];
  }
  d.pg_la[base + pos] = kla;
  d.pg_id[base + pos] = kid;
  d.pg_slot[base + pos] = slot;
#endif
  if (lane0()) {
    DirEntry& e = d.dir[dring(d, h, g, k)];
    e.cnt = cnt + 1;
    if (pos == cnt) {
      e.max_la = kla;
      e.max_id = kid;
    }
  }
  wsync();
}

// warp-wide
E2_D void lru_insert(const Dev& d, Hot* h, int g, u64 kla, u64 kid, u32 slot) {
  const u32 n = h->dir_n[g];
  if (n > 0) {
    // fast path: strictly after every key (fresh last_access) -> tail page
    const DirEntry t = d.dir[dring(d, h, g, n - 1)];
    if (kless(t.max_la, t.max_id, kla, kid)) {
      if (t.cnt < kPage) {
        if (lane0()) {
          const u64 i = (u64)t.page * kPage + t.cnt;
          d.pg_la[i] = kla;
          d.pg_id[i] = kid;
          d.pg_slot[i] = slot;
          DirEntry& e = d.dir[dring(d, h, g, n - 1)];
          e.cnt = t.cnt + 1;
          e.max_la = kla;
          e.max_id = kid;
        }
        wsync();
        return;
      }
      const u32 q = page_alloc(d, h);
      if (q == kNil) return;
      DirEntry e;
      e.page = q;
      e.cnt = 1;
      e.max_la = kla;
      e.max_id = kid;
      e.pad = 0;
      if (lane0()) {
        d.pg_la[(u64)q * kPage] = kla;
        d.pg_id[(u64)q * kPage] = kid;
        d.pg_slot[(u64)q * kPage] = slot;
      }
      wsync();
      dir_insert_at(d, h, g, n, e);
      return;
    }
  } else {
    const u32 q = page_alloc(d, h);
    if (q == kNil) return;
    DirEntry e;
    e.page = q;
    e.cnt = 1;
    e.max_la = kla;
    e.max_id = kid;
    e.pad = 0;
    if (lane0()) {
      d.pg_la[(u64)q * kPage] = kla;
      d.pg_id[(u64)q * kPage] = kid;
      d.pg_slot[(u64)q * kPage] = slot;
    }
    wsync();
    dir_insert_at(d, h, g, 0, e);
    return;
  }
  u32 k = dir_lower_bound(d, h, g, kla, kid);
  if (k >= n) k = n - 1;
  DirEntry e = d.dir[dring(d, h, g, k)];
  u32 p = e.page;
  i32 cnt = e.cnt;
  if (cnt >= kPage) {
    // split page p: upper half moves to a new page at k+1
    const u32 q = page_alloc(d, h);
    if (q == kNil) return;
    const int half = kPage / 2;
    const u64 bp = (u64)p * kPage, bq = (u64)q * kPage;
    for (int j = lane(); j < half; j += kWidth) {
      d.pg_la[bq + j] = d.pg_la[bp + half + j];
      d.pg_id[bq + j] = d.pg_id[bp + half + j];
      d.pg_slot[bq + j] = d.pg_slot[bp + half + j];
    }
    wsync();
    const u64 nmla = d.pg_la[bp + half - 1], nmid = d.pg_id[bp + half - 1];
    wsync();
    DirEntry eq;
    eq.page = q;
    eq.cnt = half;
    eq.max_la = e.max_la;
    eq.max_id = e.max_id;
    eq.pad = 0;
    if (lane0()) {
      DirEntry& ep = d.dir[dring(d, h, g, k)];
      ep.cnt = half;
      ep.max_la = nmla;
      ep.max_id = nmid;
    }
    wsync();
    if (!dir_insert_at(d, h, g, k + 1, eq)) return;
    if (kless(nmla, nmid, kla, kid)) {
      p = q;
      k = k + 1;
    }
    cnt = half;
  }
  page_insert(d, h, g, k, p, cnt, kla, kid, slot);
}

// warp-wide
E2_D void lru_erase(const Dev& d, Hot* h, int g, u64 kla, u64 kid) {
  const u32 n = h->dir_n[g];
  u32 k;
  const DirEntry h0 = d.dir[dring(d, h, g, 0)];
  if (n > 0 && !kless(h0.max_la, h0.max_id, kla, kid))
    k = 0;  // fast path: in the head page (LRU victims)
  else
    k = dir_lower_bound(d, h, g, kla, kid);
  if (k >= n) {
    if (lane0()) set_err(h, kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const DirEntry e = k == 0 ? h0 : d.dir[dring(d, h, g, k)];
  const u32 p = e.page;
  const i32 cnt = e.cnt;
  const u64 base = (u64)p * kPage;
#if E2_DEVICE_BUILD
  const int j = lane();
  const bool valid = j < cnt;
  u64 ela = 0, eid = 0;
  u32 es = 0;
  if (valid) {
    ela = d.pg_la[base + j];
    eid = d.pg_id[base + j];
    es = d.pg_slot[base + j];
  }
  const u32 m = ballot(valid && ela == kla && eid == kid);
  if (!m) {
    if (lane0()) set_err(h, kErrSim, kWhyWalk);
    wsync();
    return;
  }
  const int idx = ffs32(m);
  const u64 pla = shfl(ela, cnt >= 2 ? cnt - 2 : 0);
  const u64 pid = shfl(eid, cnt >= 2 ? cnt - 2 : 0);
  wsync();
  if (valid && j > idx) {
    d.pg_la[base + j - 1] = ela;
    d.pg_id[base + j - 1] = eid;
    d.pg_slot[base + j - 1] = es;
  }
#else
  int idx = -1;
  for (int j = 0; j < cnt; ++j)
    if (d.pg_la[base + j] == kla && d.pg_id[base + j] == kid) idx = j;
  if (idx < 0) {
    set_err(h, kErrSim, kWhyWalk);
    return;
  }
  const u64 pla = cnt >= 2 ? d.pg_la[base + cnt - 2] : 0;
  const u64 pid = cnt >= 2 ? d.pg_id[base + cnt - 2] : 0;
  for (int j = idx + 1; j < cnt; ++j) {
    d.pg_la[base + j - 1] = d.pg_la[base + j];
    d.pg_id[base + j - 1] = d.pg_id[base + j];
    d.pg_slot[base + j - 1] = d.pg_slot[base + j];
  }
#endif
  if (lane0()) {
    DirEntry& er = d.dir[dring(d, h, g, k)];
    er.cnt = cnt - 1;
    if (cnt - 1 > 0 && idx == cnt - 1) {
      er.max_la = pla;
      er.max_id = pid;
    }
  }
  wsync();
  if (cnt - 1 == 0) {
    page_free(d, h, p);
    dir_remove_at(d, h, g, k);
  }
}

// ---------------------------------------------------------------------------
// Node state helpers (all warp-wide; records via the node cache)
// ---------------------------------------------------------------------------
E2_HD bool rcached(const NodeRec* r, int g) { return (r->cmask >> g) & 1ull; }

E2_HD bool rleaf(const NodeRec* r, u32 s, int g, int G) {
  return s != kRoot && rcached(r, g) && rccc(r, G)[g] == 0;
}

// warp-wide: allocate a fresh slot and its zeroed cached record.
E2_D u32 node_alloc(Ctx& x) {
  Hot* h = x.h;
  const u32 s = h->slots_used;
  wsync();
  if (s >= x.d.node_cap) {
    if (lane0()) set_err(h, kErrCapacity, kWhyNodeCap);
    wsync();
    return kNil;
  }
  if (lane0()) h->slots_used = s + 1;
  wsync();
  return s;
}

// warp-wide: split_node(s, k) with the slot kept on the suffix — see
// e2_state.cuh.  Returns the new slot holding the prefix (old id).
// Reference: prefix_tree.cpp:122-154.
E2_D u32 split_node(Ctx& x, u32 s, u32 k) {
  const Dev& d = x.d;
  Hot* h = x.h;
  const int G = d.cfg.G;
  NodeRec* rs = nget(x, s);
  const NodeRec hs = *rs;
  if (k == 0 || k >= hs.edge_len) {
    if (lane0()) set_err(h, kErrSim, kWhySplitBounds);
    wsync();
    return kNil;
  }
  const u32 q = node_alloc(x);
  if (q == kNil) return kNil;
  const u64 new_id = h->next_id;
  const i32 tok_k = d.tok[hs.edge_off + k];
  // prefix: copy the whole record (la/hits), then fix header and ccc
  NodeRec* rq = nnew(x, q);
  rs = nget(x, s);
  {
    const u64* src = (const u64*)rs;
    u64* dst = (u64*)rq;
    for (u32 j = (u32)lane(); j < d.rs / 8; j += kWidth) dst[j] = src[j];
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
    ndirty(x, rs);
    h->next_id = new_id + 1;
    h->node_count++;
  }
  wsync();
  child_update(d, h, hs.parent, hs.first_tok, q);
  child_insert(d, h, q, tok_k, s);
  // LRU: the suffix inherits the leaf role under its new id.
  u64 m = hs.cmask;
  while (m) {
    const int g = ffs64(m);
    m &= m - 1;
    const NodeRec* r = nget(x, s);
    if (rccc(r, G)[g] == 0) {
      const u64 l = dbits(rla(r)[g]);
      lru_erase(d, h, g, l, hs.id);
      lru_insert(d, h, g, l, new_id, s);
    }
  }
  return q;
}

// warp-wide: new leaf under parent with edge [off, off+len).
E2_D u32 new_leaf(Ctx& x, u32 parent, i64 off, u32 len, u32 depth) {
  const Dev& d = x.d;
  Hot* h = x.h;
  const u32 l = node_alloc(x);
  if (l == kNil) return kNil;
  const i32 t0 = d.tok[off];
  const u64 id = h->next_id;
  NodeRec* rl = nnew(x, l);
  if (lane0()) {
    rl->id = id;
    rl->edge_off = off;
    rl->edge_len = len;
    rl->parent = parent;
    rl->first_tok = t0;
    rl->depth = depth;
    h->next_id = id + 1;
    h->node_count++;
  }
  wsync();
  NodeRec* rp = nget(x, parent);
  if (lane0()) {
    rp->nchild += 1;
    ndirty(x, rp);
  }
  wsync();
  child_insert(d, h, parent, t0, l);
  return l;
}

// warp-wide: set_cached (prefix_tree.cpp:53-63).
E2_D void set_cached(Ctx& x, u32 s, int g) {
  const Dev& d = x.d;
  Hot* h = x.h;
  const int G = d.cfg.G;
  if (s == kRoot) return;
  NodeRec* r = nget(x, s);
  if (rcached(r, g)) return;
  const u32 p = r->parent;
  const u32 len = r->edge_len;
  const u64 sid = r->id;
  wsync();
  if (lane0()) {
    r->cmask |= (1ull << g);
    ndirty(x, r);
    h->cached_tokens[g] += len;
  }
  wsync();
  if (rccc(r, G)[g] == 0) lru_insert(d, h, g, dbits(rla(r)[g]), sid, s);
  if (p != kNil) {
    NodeRec* rp = nget(x, p);
    const bool p_was = rleaf(rp, p, g, G);
    const u64 pla = dbits(rla(rp)[g]), pid = rp->id;
    wsync();
    if (lane0()) {
      rccc(rp, G)[g] += 1;
      ndirty(x, rp);
    }
    wsync();
    if (p_was) lru_erase(d, h, g, pla, pid);
  }
}

// warp-wide: clear_cached (prefix_tree.cpp:65-77).
E2_D void clear_cached(Ctx& x, u32 s, int g) {
  const Dev& d = x.d;
  Hot* h = x.h;
  const int G = d.cfg.G;
  NodeRec* r = nget(x, s);
  if (!rcached(r, g)) return;
  const u32 p = r->parent;
  const u32 len = r->edge_len;
  if (rleaf(r, s, g, G)) lru_erase(d, h, g, dbits(rla(r)[g]), r->id);
  r = nget(x, s);
  wsync();
  if (lane0()) {
    r->cmask &= ~(1ull << g);
    ndirty(x, r);
    h->cached_tokens[g] -= len;
  }
  wsync();
  if (p != kNil) {
    NodeRec* rp = nget(x, p);
    const i32 c = rccc(rp, G)[g] - 1;
    wsync();
    if (lane0()) {
      rccc(rp, G)[g] = c;
      ndirty(x, rp);
      if (c < 0) set_err(h, kErrSim, kWhyCccUnderflow);
    }
    wsync();
    if (c == 0 && rleaf(rp, p, g, G)) lru_insert(d, h, g, dbits(rla(rp)[g]), rp->id, p);
  }
}

// warp-wide: last_access[g] = max(last_access[g], now) with the entry created
// (record_hit / mark_cached_path: prefix_tree.cpp:45-51, 207-210).
E2_D void touch_la(Ctx& x, u32 s, int g, double now) {
  const Dev& d = x.d;
  Hot* h = x.h;
  const int G = d.cfg.G;
  NodeRec* r = nget(x, s);
  const double old = rla(r)[g];
  const bool was = rleaf(r, s, g, G);
  const u64 id = r->id;
  const bool upd = now > old;
  wsync();
  if (lane0()) {
    r->lamask |= (1ull << g);
    if (upd) rla(r)[g] = now;
    ndirty(x, r);
  }
  wsync();
  if (upd && was) {
    lru_erase(d, h, g, dbits(old), id);
    lru_insert(d, h, g, dbits(now), id, s);
  }
}

}  // namespace e2
