// e2_match.cuh — K1 batched prefix match + intra-batch leader rounds.
//
// K1: one warp per request walks the batch-start tree: a child-table probe
// per level (32 slots per ballot), then the edge span is compared against the
// prompt 4x32 tokens per step.  Replaces PrefixTree::walk
// (prefix_tree.cpp:79-114) — the token-by-token loop at :91 is the
// reference's hot loop.
//
// Leader rounds: a batch is matched against its start snapshot, so a request
// may also share a longer prefix with an EARLIER request of the same batch
// (SURVEY 7.1 E2/E3).  The true matched length is
//   L_i = max(S_i, max_{j<i in batch} LCP(p_i, p_j))
// since, without dead-node pruning inside a batch, the tree before request i
// holds exactly the prefixes of every earlier prompt.  Requests are grouped
// by their divergence point (same (S+1)-prefix); the lowest index of a group
// is its leader and the others compare against it; the process recurses on
// (leader, LCP, next token) until every request leads its group.  Each
// round is one warp-LCP per active request plus an atomicMin hash grouping.
#pragma once

#include "e2_tree.cuh"

namespace e2 {

// First index in [0, lim) where a and b differ, or lim.  Warp-wide.
E2_D i64 warp_lcp(const i32* a, const i32* b, i64 lim) {
#if E2_DEVICE_BUILD
  const int l = lane();
  for (i64 base = 0; base < lim; base += 4 * kWidth) {
    i32 av[4], bv[4];
    bool in[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      i64 i = base + l + 32 * k;
      in[k] = i < lim;
      av[k] = in[k] ? __ldg(a + i) : 0;
      bv[k] = in[k] ? __ldcs(b + i) : 0;  // prompt side streams (evict-first in L2)
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u32 m = ballot(in[k] && av[k] != bv[k]);
      if (m) return base + 32 * k + ffs32(m);
    }
  }
  return lim;
#else
  i64 i = 0;
  while (i < lim && a[i] == b[i]) ++i;
  return i;
#endif
}

struct MatchRes {
  i64 S;         // matched length against the snapshot
  u32 div_slot;  // node where the walk stopped (kRoot if nothing matched)
  u32 div_m;     // tokens matched inside div_slot
  i64 levels;    // nodes on the matched path
  i64 bytes;     // algorithmic bytes
};

// Warp-wide walk with token comparison; records up to nh path slots.
E2_D MatchRes match_one(const i32* seq, i64 n, u32* path, int nh) {
  MatchRes r;
  r.S = 0;
  r.div_slot = kRoot;
  r.div_m = 0;
  i64 pos = 0, depth = 0;
  u32 cur = kRoot;
  int level = 0;
  while (pos < n) {
    const u32 ch = child_lookup(cur, seq[pos]);
    depth++;
    if (ch == kNil) break;
    const NodeRec* hd = grec(ch);
    const i64 off = hd->edge_off, len = hd->edge_len;
    const i64 lim = min_(len, n - pos);
    // first token equal by construction of the child key
    const i64 m = 1 + warp_lcp(DEV.tok + off + 1, seq + pos + 1, lim - 1);
    if (path && level < nh && lane0()) path[level] = ch;
    level++;
    pos += m;
    cur = ch;
    r.div_slot = ch;
    r.div_m = (u32)m;
    if (m < len) break;
  }
  // kNil-terminated (readers never look past the terminator)
  if (path && level < nh && lane0()) path[level] = kNil;
  r.S = pos;
  r.levels = level;
  // B_match = 4*min(|p|, matched+1) + 4*matched + 32*(depth+1)
  r.bytes = 4 * min_(n, pos + 1) + 4 * pos + 32 * (depth + 1);
  return r;
}

// Grouping table: hash(A,B) -> min request index (batch-local).
E2_HDX u64 gkey(u64 A, u64 B, int round) {
  u64 k = mix64(A ^ mix64(B + 0x9e3779b97f4a7c15ull * (u64)(round + 1)));
  return k | 1ull;  // 0 is the empty marker
}

}  // namespace e2
