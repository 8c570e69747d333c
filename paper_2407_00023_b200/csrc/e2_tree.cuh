// e2_tree.cuh — warp-cooperative radix-tree store and per-instance LRU index.
//
// Functions marked "warp-wide" must be called by all 32 lanes with uniform
// arguments (they use ballot/shuffle and lane-0 writes + __syncwarp).
// Functions marked "single-lane" mutate only from the calling lane and must
// not contain warp collectives.
#pragma once

#include "e2_state.cuh"

namespace e2 {

struct Ctx {
  Dev d;   // pointers + config (by value: kernel parameter / host copy)
  Hot* h;  // shared memory while the serial kernel runs
};

E2_HD void set_err(Hot* h, i32 code, i32 why) {
  if (h->err == 0) {
    h->err = code;
    h->why = why;
  }
}

// ---------------------------------------------------------------------------
// Child table: open addressing, linear probing, key = parent<<32 | token.
// Replaces TreeNode::children (std::map) lookups, prefix_tree.cpp:85, 160.
// ---------------------------------------------------------------------------
E2_HDX u64 ckey(u32 parent, i32 tok) { return ((u64)parent << 32) | (u64)(u32)tok; }

struct Probe {
  u64 pos;   // table index of the key (found) or of the first free slot
  bool found;
};

// warp-wide (read-only): each step probes kWidth consecutive slots.
E2_D Probe ct_probe(const Dev& d, u64 key) {
  u64 b = mix64(key) & d.ct_mask;
  u64 first_free = ~0ull;
  for (u64 step = 0; step <= d.ct_mask; step += kWidth, b += kWidth) {
    u64 idx = (b + (u64)lane()) & d.ct_mask;
    u64 k = d.ck[idx];
    u32 hit = ballot(k == key);
    u32 emp = ballot(k == kEmptyKey);
    u32 fr = emp | ballot(k == kTombKey);
    if (first_free == ~0ull && fr) first_free = (b + (u64)ffs32(fr)) & d.ct_mask;
    if (hit) return Probe{(b + (u64)ffs32(hit)) & d.ct_mask, true};
    if (emp) return Probe{first_free, false};
  }
  return Probe{first_free, false};
}

// warp-wide
E2_D u32 child_lookup(const Dev& d, u32 parent, i32 tok) {
  Probe p = ct_probe(d, ckey(parent, tok));
  return p.found ? d.cv[p.pos] : kNil;
}

// warp-wide; key must be absent.
E2_D bool child_insert(const Dev& d, Hot* h, u32 parent, i32 tok, u32 child) {
  u64 key = ckey(parent, tok);
  Probe p = ct_probe(d, key);
  if (p.found || p.pos == ~0ull) {
    if (lane0()) set_err(h, kErrCapacity, kWhyTableFull);
    wsync();
    return false;
  }
  if (lane0()) {
    d.ck[p.pos] = key;
    d.cv[p.pos] = child;
  }
  wsync();
  return true;
}

// warp-wide; key must be present.
E2_D void child_update(const Dev& d, Hot* h, u32 parent, i32 tok, u32 child) {
  Probe p = ct_probe(d, ckey(parent, tok));
  if (lane0()) {
    if (p.found)
      d.cv[p.pos] = child;
    else
      set_err(h, kErrSim, kWhyWalk);
  }
  wsync();
}

// warp-wide
E2_D void child_erase(const Dev& d, Hot* h, u32 parent, i32 tok) {
  Probe p = ct_probe(d, ckey(parent, tok));
  if (lane0()) {
    if (p.found)
      d.ck[p.pos] = kTombKey;
    else
      set_err(h, kErrSim, kWhyWalk);
  }
  wsync();
}

// ---------------------------------------------------------------------------
// Per-instance LRU index: ordered set of (last_access bits, id) over LRU
// leaves (cached on g, no cached child on g) — prefix_tree.cpp:14-35.
// Directory = ring of page ids per instance with each page's max key.
// ---------------------------------------------------------------------------
E2_HDX bool kless(u64 ala, u64 aid, u64 bla, u64 bid) { return ala < bla || (ala == bla && aid < bid); }

E2_HD u32 dring(const Dev& d, const Hot* h, int g, u32 k) {
  return (u32)g * d.dcap + ((h->dir_head[g] + k) & (d.dcap - 1));
}

// warp-wide: first directory position whose page max >= key (n if none).
E2_D u32 dir_lower_bound(const Dev& d, const Hot* h, int g, u64 kla, u64 kid) {
  u32 lo = 0, hi = h->dir_n[g];
#if E2_DEVICE_BUILD
  while (hi > lo) {
    u32 span = hi - lo;
    u32 step = (span + kWidth - 1) / kWidth;
    u32 j = (u32)lane();
    u32 pos = lo + j * step;
    bool valid = pos < hi;
    bool geq = false;
    if (valid) {
      u32 r = dring(d, h, g, pos);
      geq = !kless(d.dir_la[r], d.dir_id[r], kla, kid);
    }
    u32 falses = ballot(valid && !geq);
    u32 F = (u32)popc32(falses);
    if (F == 0) return lo;
    u32 J = (u32)popc32(ballot(valid));
    u32 newlo = lo + (F - 1) * step + 1;
    u32 newhi = F < J ? lo + F * step : hi;
    if (step == 1) return F < J ? lo + F : hi;
    lo = newlo;
    hi = newhi;
  }
  return lo;
#else
  while (lo < hi) {
    u32 mid = lo + (hi - lo) / 2;
    u32 r = dring(d, h, g, mid);
    if (kless(d.dir_la[r], d.dir_id[r], kla, kid))
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

// warp-wide: insert page id at directory position k.
E2_D bool dir_insert_at(const Dev& d, Hot* h, int g, u32 k, u32 page, u64 mla, u64 mid) {
  u32 n = h->dir_n[g];
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
      i64 pos = top - lane();
      u32 pg = 0;
      u64 a = 0, b = 0;
      bool act = pos >= (i64)k;
      if (act) {
        u32 r = dring(d, h, g, (u32)pos);
        pg = d.dir_page[r];
        a = d.dir_la[r];
        b = d.dir_id[r];
      }
      wsync();
      if (act) {
        u32 r = dring(d, h, g, (u32)pos + 1);
        d.dir_page[r] = pg;
        d.dir_la[r] = a;
        d.dir_id[r] = b;
      }
      wsync();
    }
  }
  if (lane0()) {
    u32 r = dring(d, h, g, k);
    d.dir_page[r] = page;
    d.dir_la[r] = mla;
    d.dir_id[r] = mid;
    h->dir_n[g] = n + 1;
  }
  wsync();
  return true;
}

// warp-wide: remove directory position k.
E2_D void dir_remove_at(const Dev& d, Hot* h, int g, u32 k) {
  u32 n = h->dir_n[g];
  if (k == 0) {
    if (lane0()) h->dir_head[g] = (h->dir_head[g] + 1) & (d.dcap - 1);
  } else {
    for (u32 lo = k + 1; lo < n; lo += kWidth) {
      u32 pos = lo + (u32)lane();
      bool act = pos < n;
      u32 pg = 0;
      u64 a = 0, b = 0;
      if (act) {
        u32 r = dring(d, h, g, pos);
        pg = d.dir_page[r];
        a = d.dir_la[r];
        b = d.dir_id[r];
      }
      wsync();
      if (act) {
        u32 r = dring(d, h, g, pos - 1);
        d.dir_page[r] = pg;
        d.dir_la[r] = a;
        d.dir_id[r] = b;
      }
      wsync();
    }
  }
  if (lane0()) h->dir_n[g] = n - 1;
  wsync();
}

// warp-wide: insert (kla, kid) -> slot into page p at the right position
// (page has room).
E2_D void page_insert(const Dev& d, Hot* h, int g, u32 k, u32 p, u64 kla, u64 kid, u32 slot) {
  i32 cnt = d.pg_n[p];
  u64 base = (u64)p * kPage;
#if E2_DEVICE_BUILD
  int j = lane();
  u64 ela = 0, eid = 0;
  u32 es = 0;
  bool valid = j < cnt;
  if (valid) {
    ela = d.pg_la[base + j];
    eid = d.pg_id[base + j];
    es = d.pg_slot[base + j];
  }
  int pos = popc32(ballot(valid && kless(ela, eid, kla, kid)));
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
  if (j == 0) {
    d.pg_n[p] = cnt + 1;
    if (pos == cnt) {
      u32 r = dring(d, h, g, k);
      d.dir_la[r] = kla;
      d.dir_id[r] = kid;
    }
  }
  wsync();
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
  d.pg_n[p] = cnt + 1;
  if (pos == cnt) {
    u32 r = dring(d, h, g, k);
    d.dir_la[r] = kla;
    d.dir_id[r] = kid;
  }
#endif
}

// warp-wide
E2_D void lru_insert(const Dev& d, Hot* h, int g, u64 kla, u64 kid, u32 slot) {
  u32 n = h->dir_n[g];
  if (n == 0) {
    u32 p = page_alloc(d, h);
    if (p == kNil) return;
    if (lane0()) d.pg_n[p] = 0;
    wsync();
    if (!dir_insert_at(d, h, g, 0, p, kla, kid)) return;
    page_insert(d, h, g, 0, p, kla, kid, slot);
    return;
  }
  u32 k = dir_lower_bound(d, h, g, kla, kid);
  bool beyond = (k == n);
  if (beyond) k = n - 1;
  u32 p = d.dir_page[dring(d, h, g, k)];
  i32 cnt = d.pg_n[p];
  if (cnt >= kPage) {
    if (beyond) {  // strictly after every key: open a fresh tail page
      u32 q = page_alloc(d, h);
      if (q == kNil) return;
      if (lane0()) d.pg_n[q] = 0;
      wsync();
      if (!dir_insert_at(d, h, g, n, q, kla, kid)) return;
      page_insert(d, h, g, n, q, kla, kid, slot);
      return;
    }
    // split page p: upper half moves to a new page at k+1
    u32 q = page_alloc(d, h);
    if (q == kNil) return;
    const int half = kPage / 2;
    u64 bp = (u64)p * kPage, bq = (u64)q * kPage;
    for (int j = lane(); j < half; j += kWidth) {
      d.pg_la[bq + j] = d.pg_la[bp + half + j];
      d.pg_id[bq + j] = d.pg_id[bp + half + j];
      d.pg_slot[bq + j] = d.pg_slot[bp + half + j];
    }
    wsync();
    u64 oldmax_la = d.pg_la[bp + kPage - 1], oldmax_id = d.pg_id[bp + kPage - 1];
    u64 newmax_la = d.pg_la[bp + half - 1], newmax_id = d.pg_id[bp + half - 1];
    wsync();
    if (lane0()) {
      d.pg_n[q] = half;
      d.pg_n[p] = half;
      u32 r = dring(d, h, g, k);
      d.dir_la[r] = newmax_la;
      d.dir_id[r] = newmax_id;
    }
    wsync();
    if (!dir_insert_at(d, h, g, k + 1, q, oldmax_la, oldmax_id)) return;
    if (kless(newmax_la, newmax_id, kla, kid)) {
      p = q;
      k = k + 1;
    }
  }
  page_insert(d, h, g, k, p, kla, kid, slot);
}

// warp-wide
E2_D void lru_erase(const Dev& d, Hot* h, int g, u64 kla, u64 kid) {
  u32 n = h->dir_n[g];
  u32 k = dir_lower_bound(d, h, g, kla, kid);
  if (k >= n) {
    if (lane0()) set_err(h, kErrSim, kWhyWalk);
    wsync();
    return;
  }
  u32 p = d.dir_page[dring(d, h, g, k)];
  i32 cnt = d.pg_n[p];
  u64 base = (u64)p * kPage;
#if E2_DEVICE_BUILD
  int j = lane();
  bool valid = j < cnt;
  u64 ela = 0, eid = 0;
  u32 es = 0;
  if (valid) {
    ela = d.pg_la[base + j];
    eid = d.pg_id[base + j];
    es = d.pg_slot[base + j];
  }
  u32 m = ballot(valid && ela == kla && eid == kid);
  if (!m) {
    if (lane0()) set_err(h, kErrSim, kWhyWalk);
    wsync();
    return;
  }
  int idx = ffs32(m);
  // new last key if we removed the max
  u64 pla = shfl(ela, cnt >= 2 ? cnt - 2 : 0);
  u64 pid = shfl(eid, cnt >= 2 ? cnt - 2 : 0);
  wsync();
  if (valid && j > idx) {
    d.pg_la[base + j - 1] = ela;
    d.pg_id[base + j - 1] = eid;
    d.pg_slot[base + j - 1] = es;
  }
  if (j == 0) {
    d.pg_n[p] = cnt - 1;
    if (cnt - 1 > 0 && idx == cnt - 1) {
      u32 r = dring(d, h, g, k);
      d.dir_la[r] = pla;
      d.dir_id[r] = pid;
    }
  }
  wsync();
#else
  int idx = -1;
  for (int j = 0; j < cnt; ++j)
    if (d.pg_la[base + j] == kla && d.pg_id[base + j] == kid) idx = j;
  if (idx < 0) {
    set_err(h, kErrSim, kWhyWalk);
    return;
  }
  for (int j = idx + 1; j < cnt; ++j) {
    d.pg_la[base + j - 1] = d.pg_la[base + j];
    d.pg_id[base + j - 1] = d.pg_id[base + j];
    d.pg_slot[base + j - 1] = d.pg_slot[base + j];
  }
  d.pg_n[p] = cnt - 1;
  if (cnt - 1 > 0 && idx == cnt - 1) {
    u32 r = dring(d, h, g, k);
    d.dir_la[r] = d.pg_la[base + cnt - 2];
    d.dir_id[r] = d.pg_id[base + cnt - 2];
  }
#endif
  if (cnt - 1 == 0) {
    page_free(d, h, p);
    dir_remove_at(d, h, g, k);
  }
}

// ---------------------------------------------------------------------------
// Node state helpers
// ---------------------------------------------------------------------------
E2_HD bool cached_on(const Dev& d, u32 s, int g) { return (d.cmask[s] >> g) & 1ull; }

E2_HD bool lru_leaf(const Dev& d, u32 s, int g) {
  return s != kRoot && cached_on(d, s, g) && d.ccc[(u64)s * d.cfg.G + g] == 0;
}

E2_HD u64 la_bits(const Dev& d, u32 s, int g) { return dbits(d.la[(u64)s * d.cfg.G + g]); }

// warp-wide: bring node s's LRU membership on g up to date after a change.
// was/old_la describe the state before; the index is a set, so applying the
// final-state difference equals the reference's erase/insert sequence.
E2_D void lru_fix(const Dev& d, Hot* h, u32 s, int g, bool was, u64 old_la, u64 old_id) {
  bool now_leaf = lru_leaf(d, s, g);
  u64 nla = la_bits(d, s, g), nid = d.hdr[s].id;
  bool same = was && now_leaf && nla == old_la && nid == old_id;
  if (same) return;
  if (was) lru_erase(d, h, g, old_la, old_id);
  if (now_leaf) lru_insert(d, h, g, nla, nid, s);
}

// warp-wide: allocate a fresh slot (zeroed by the host at growth time).
E2_D u32 node_alloc(const Dev& d, Hot* h) {
  u32 s = h->slots_used;
  wsync();
  if (s >= d.node_cap) {
    if (lane0()) set_err(h, kErrCapacity, kWhyNodeCap);
    wsync();
    return kNil;
  }
  if (lane0()) h->slots_used = s + 1;
  wsync();
  return s;
}

// warp-wide: split_node(s, k) with the slot kept on the suffix — see the
// header comment.  Returns the new slot holding the prefix (old id).
// Reference: prefix_tree.cpp:122-154.
E2_D u32 split_node(const Dev& d, Hot* h, u32 s, u32 k) {
  NodeHdr hs = d.hdr[s];
  if (k == 0 || k >= hs.edge_len) {
    if (lane0()) set_err(h, kErrSim, kWhySplitBounds);
    wsync();
    return kNil;
  }
  u32 q = node_alloc(d, h);
  if (q == kNil) return kNil;
  const int G = d.cfg.G;
  const u64 new_id = h->next_id;
  const i32 tok_k = d.tok[hs.edge_off + k];
  const u64 cm = d.cmask[s];
  wsync();
  if (lane0()) {
    NodeHdr hq;
    hq.id = hs.id;
    hq.edge_off = hs.edge_off;
    hq.edge_len = k;
    hq.parent = hs.parent;
    hq.first_tok = hs.first_tok;
    hq.depth = hs.depth;
    d.hdr[q] = hq;
    NodeHdr ns = hs;
    ns.id = new_id;
    ns.edge_off = hs.edge_off + k;
    ns.edge_len = hs.edge_len - k;
    ns.parent = q;
    ns.first_tok = tok_k;
    ns.depth = hs.depth + k;
    d.hdr[s] = ns;
    d.cmask[q] = cm;
    d.lamask[q] = d.lamask[s];
    d.nchild[q] = 1;
    h->next_id = new_id + 1;
    h->node_count++;
  }
  for (int g = lane(); g < G; g += kWidth) {
    u64 qi = (u64)q * G + g, si = (u64)s * G + g;
    d.la[qi] = d.la[si];
    d.hits[qi] = d.hits[si];
    d.ccc[qi] = ((cm >> g) & 1ull) ? 1 : 0;
  }
  wsync();
  child_update(d, h, hs.parent, hs.first_tok, q);
  child_insert(d, h, q, tok_k, s);
  // LRU: the suffix inherits the leaf role under its new id.
  u64 m = cm;
  while (m) {
    int g = ffs64(m);
    m &= m - 1;
    if (d.ccc[(u64)s * G + g] == 0) {
      u64 l = la_bits(d, s, g);
      lru_erase(d, h, g, l, hs.id);
      lru_insert(d, h, g, l, new_id, s);
    }
  }
  return q;
}

// warp-wide: new leaf under parent with edge [off, off+len).
E2_D u32 new_leaf(const Dev& d, Hot* h, u32 parent, i64 off, u32 len, u32 depth) {
  u32 l = node_alloc(d, h);
  if (l == kNil) return kNil;
  const i32 t0 = d.tok[off];
  const u64 id = h->next_id;
  wsync();
  if (lane0()) {
    NodeHdr hl;
    hl.id = id;
    hl.edge_off = off;
    hl.edge_len = len;
    hl.parent = parent;
    hl.first_tok = t0;
    hl.depth = depth;
    d.hdr[l] = hl;
    d.nchild[parent] += 1;
    h->next_id = id + 1;
    h->node_count++;
  }
  wsync();
  child_insert(d, h, parent, t0, l);
  return l;
}

// warp-wide: set_cached (prefix_tree.cpp:53-63).
E2_D void set_cached(const Dev& d, Hot* h, u32 s, int g) {
  if (s == kRoot || cached_on(d, s, g)) return;
  const int G = d.cfg.G;
  u32 p = d.hdr[s].parent;
  bool p_was = (p != kNil) && lru_leaf(d, p, g);
  u64 p_la = p != kNil ? la_bits(d, p, g) : 0, p_id = p != kNil ? d.hdr[p].id : 0;
  wsync();
  if (lane0()) {
    d.cmask[s] |= (1ull << g);
    h->cached_tokens[g] += d.hdr[s].edge_len;
    if (p != kNil) d.ccc[(u64)p * G + g] += 1;
  }
  wsync();
  if (lru_leaf(d, s, g)) lru_insert(d, h, g, la_bits(d, s, g), d.hdr[s].id, s);
  if (p_was) lru_erase(d, h, g, p_la, p_id);
}

// warp-wide: clear_cached (prefix_tree.cpp:65-77).
E2_D void clear_cached(const Dev& d, Hot* h, u32 s, int g) {
  if (!cached_on(d, s, g)) return;
  const int G = d.cfg.G;
  if (lru_leaf(d, s, g)) lru_erase(d, h, g, la_bits(d, s, g), d.hdr[s].id);
  u32 p = d.hdr[s].parent;
  i32 c = p != kNil ? d.ccc[(u64)p * G + g] - 1 : 0;
  wsync();
  if (lane0()) {
    d.cmask[s] &= ~(1ull << g);
    h->cached_tokens[g] -= d.hdr[s].edge_len;
    if (p != kNil) d.ccc[(u64)p * G + g] = c;
    if (c < 0) set_err(h, kErrSim, kWhyCccUnderflow);
  }
  wsync();
  if (p != kNil && c == 0 && lru_leaf(d, p, g)) lru_insert(d, h, g, la_bits(d, p, g), d.hdr[p].id, p);
}

// warp-wide: last_access[g] = max(last_access[g], now) with the entry created
// (record_hit / mark_cached_path: prefix_tree.cpp:45-51, 207-210).
E2_D void touch_la(const Dev& d, Hot* h, u32 s, int g, double now) {
  const int G = d.cfg.G;
  u64 i = (u64)s * G + g;
  double old = d.la[i];
  bool was = lru_leaf(d, s, g);
  u64 old_bits = dbits(old), id = d.hdr[s].id;
  bool upd = now > old;
  wsync();
  if (lane0()) {
    d.lamask[s] |= (1ull << g);
    if (upd) d.la[i] = now;
  }
  wsync();
  if (upd && was) lru_fix(d, h, s, g, was, old_bits, id);
}

}  // namespace e2
