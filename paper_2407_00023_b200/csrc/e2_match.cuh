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

#if E2_WARP
// Tokens R..R+3 of the 8-token window (x, y): realigns the tree side's
// 16-byte quads to the prompt's phase (R is the phase difference).
template <int R>
E2_D int4 funnel4(const int4& x, const int4& y) {
  if (R == 0) return x;
  if (R == 1) return make_int4(x.y, x.z, x.w, y.x);
  if (R == 2) return make_int4(x.z, x.w, y.x, y.y);
  return make_int4(x.w, y.x, y.y, y.z);
}

// Valid-token mask of a quad whose element 0 is token t0, tokens [0, lim).
E2_D u32 quad_mask(i64 t0, i64 lim) {
  const i64 hi = lim - t0;
  u32 vm = hi >= 4 ? 0xfu : hi <= 0 ? 0u : ((1u << (u32)hi) - 1u);
  if (t0 < 0) vm &= ~((1u << (u32)(-t0)) - 1u);
  return vm;
}

constexpr int kLcpU = 2;  // quads per lane per side in flight per step (kLcpU*128 tokens)

// b-frame quad q (element k = token 4q+k-sb); a-frame index t+sa = 4(q+dq)+k+R.
template <int R>
E2_D i64 warp_lcp_phase(const int4* A4, const int4* B4, int sb, int dq, i64 lim) {
  const int l = lane();
  const i64 qb_end = (lim + sb + 3) >> 2;
  const i64 qa_end = (lim + sb + dq * 4 + R + 3) >> 2;  // (lim + sa + 3) >> 2
  for (i64 q0 = 0; q0 < qb_end; q0 += kLcpU * 32) {
    int4 bv[kLcpU], xv[kLcpU], zv[kLcpU];
#pragma unroll
    for (int u = 0; u < kLcpU; ++u) {
      const i64 q = q0 + l + 32 * u;
      const i64 qa = q + dq;
      bv[u] = q < qb_end ? __ldcs(B4 + q) : make_int4(0, 0, 0, 0);
      xv[u] = (qa >= 0 && qa < qa_end) ? __ldg(A4 + qa) : make_int4(0, 0, 0, 0);
      if (R != 0) zv[u] = (l == 31 && qa + 1 < qa_end) ? __ldg(A4 + qa + 1) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kLcpU; ++u) {
      int4 av = xv[u];
      if (R != 0) {
        int4 yv;
        yv.x = __shfl_down_sync(0xffffffffu, xv[u].x, 1);
        yv.y = __shfl_down_sync(0xffffffffu, xv[u].y, 1);
        yv.z = __shfl_down_sync(0xffffffffu, xv[u].z, 1);
        yv.w = __shfl_down_sync(0xffffffffu, xv[u].w, 1);
        if (l == 31) yv = zv[u];
        av = funnel4<R>(xv[u], yv);
      }
      const i64 t0 = 4 * (q0 + l + 32 * u) - sb;  // token index of element 0
      u32 mm = (av.x != bv[u].x ? 1u : 0u) | (av.y != bv[u].y ? 2u : 0u) | (av.z != bv[u].z ? 4u : 0u) |
               (av.w != bv[u].w ? 8u : 0u);
      mm &= quad_mask(t0, lim);
      const u32 wm = ballot(mm != 0);
      if (wm) {
        const int f = ffs32(wm);
        const u32 fm = shfl(mm, f);
        return 4 * (q0 + f + 32 * u) - sb + ffs32(fm);
      }
    }
  }
  return lim;
}
#endif

// First index in [0, lim) where a and b differ, or lim.  Warp-wide.
// Device: 128-bit loads on both sides.  The prompt side b streams as aligned
// int4 quads (evict-first in L2: read once); the tree side a (edge tokens,
// shared by many prompts: L1/L2-resident) is read as aligned quads too and
// realigned to b's phase from the lane's quad and its neighbour's (shfl);
// the phase difference is warp-uniform, so each phase has its own loop.
E2_D i64 warp_lcp(const i32* a, const i32* b, i64 lim) {
#if E2_WARP
  if (lim <= 0) return 0;
  const int sb = (int)(((unsigned long long)b >> 2) & 3);
  const int sa = (int)(((unsigned long long)a >> 2) & 3);
  const int4* B4 = (const int4*)(b - sb);
  const int4* A4 = (const int4*)(a - sa);
  const int dd = sa - sb;
  const int dq = dd < 0 ? -1 : 0;
  switch (dd - 4 * dq) {
    case 0: return warp_lcp_phase<0>(A4, B4, sb, dq, lim);
    case 1: return warp_lcp_phase<1>(A4, B4, sb, dq, lim);
    case 2: return warp_lcp_phase<2>(A4, B4, sb, dq, lim);
    default: return warp_lcp_phase<3>(A4, B4, sb, dq, lim);
  }
#else
  i64 i = 0;
  while (i < lim && a[i] == b[i]) ++i;
  return i;
#endif
}

#if E2_WARP
// ---- staged top of the tree (K1, SURVEY north star) -------------------------
// Per batch, k_top_build writes an image of the root's hottest children
// (first token, slot, edge, and the first tokens of each edge) to global
// memory; every K1 block copies it into shared memory with one TMA bulk copy
// (cp.async.bulk + mbarrier complete_tx).  Level 0 of a walk then costs no
// child-table probe and compares the head of its edge from shared memory.
#ifndef E2_TOP_KB
#define E2_TOP_KB 32
#endif
constexpr u32 kTopBytes = E2_TOP_KB * 1024;
constexpr u32 kTopMaxEnt = 254;
constexpr u32 kTopHeadMax = 2048;  // tokens staged per root child at most
struct TopHdr {
  u32 n;      // entries, sorted by first token
  u32 bytes;  // image size (multiple of 16)
  u32 pad[2];
};
struct TopEnt {
  i32 tok;
  u32 slot;
  u32 edge_len;
  u32 head_len;  // tokens staged (edge tokens [0, head_len))
  u32 head_off;  // byte offset of the staged tokens in the image (16-aligned)
  u32 pad;
  i64 edge_off;
};
static_assert(sizeof(TopEnt) == 32, "top entries are 32 bytes");

E2_D u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
E2_D void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
E2_D void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// one 1-D TMA bulk copy global -> shared, completing on `bar`
E2_D void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
E2_D void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TOPW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra TOPW_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Entry of first token t in the staged table (binary search), or -1.
E2_D int top_find(const char* top, i32 t) {
  const TopHdr* h = (const TopHdr*)top;
  const TopEnt* e = (const TopEnt*)(top + 16);
  int lo = 0, hi = (int)h->n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (e[mid].tok < t) lo = mid + 1;
    else hi = mid;
  }
  return (lo < (int)h->n && e[lo].tok == t) ? lo : -1;
}

// First index in [0, lim) where the staged head a (shared memory, 16-byte
// aligned) and the prompt b differ, or lim.  Warp-wide, 128 tokens a step.
E2_D i64 smem_lcp(const i32* a, const i32* b, i64 lim) {
  for (i64 k0 = 0; k0 < lim; k0 += 128) {
    const i64 t0 = k0 + 4 * lane();
    u32 mm = 0;
    if (t0 < lim) {
      const int4 av = *(const int4*)(a + t0);
      const i32 bv[4] = {b[t0], t0 + 1 < lim ? b[t0 + 1] : av.y, t0 + 2 < lim ? b[t0 + 2] : av.z,
                         t0 + 3 < lim ? b[t0 + 3] : av.w};
      mm = (av.x != bv[0] ? 1u : 0u) | (av.y != bv[1] ? 2u : 0u) | (av.z != bv[2] ? 4u : 0u) |
           (av.w != bv[3] ? 8u : 0u);
      mm &= quad_mask(t0, lim) & 0xfu;
    }
    const u32 wm = ballot(mm != 0);
    if (wm) {
      const int f = ffs32(wm);
      return k0 + 4 * f + ffs32(shfl(mm, f));
    }
  }
  return lim;
}
#endif

struct MatchRes {
  i64 S;         // matched length against the snapshot
  u32 div_slot;  // node where the walk stopped (kRoot if nothing matched)
  u32 div_m;     // tokens matched inside div_slot
  i64 levels;    // nodes on the matched path
  i64 bytes;     // algorithmic bytes
};

// Warp-wide walk with token comparison; records up to nh path slots.
// top/ent (K1): the staged table and this prompt's level-0 entry in it (-1:
// not staged, probe the child table).
E2_D MatchRes match_one(const i32* seq, i64 n, u32* path, int nh, const char* top = nullptr, int ent = -1) {
  MatchRes r;
  r.S = 0;
  r.div_slot = kRoot;
  r.div_m = 0;
  i64 pos = 0, depth = 0;
  u32 cur = kRoot;
  int level = 0;
  bool stop = false;
#if E2_WARP
  if (top && ent >= 0 && n > 0) {
    // level 0 from shared memory: the first token equals by the table key
    const TopEnt e = ((const TopEnt*)(top + 16))[ent];
    const i64 len = e.edge_len, lim = min_(len, n);
    const i64 hl = min_((i64)e.head_len, lim);
    i64 m = hl >= 1 ? smem_lcp((const i32*)(top + e.head_off), seq, hl) : 1;
    if (m == max_<i64>(hl, 1) && m < lim) m += warp_lcp(DEV.tok + e.edge_off + m, seq + m, lim - m);
    depth = 1;
    if (path && nh > 0 && lane0()) path[0] = e.slot;
    level = 1;
    pos = m;
    cur = e.slot;
    r.div_slot = e.slot;
    r.div_m = (u32)m;
    stop = m < len;  // the match ends inside the root child
  }
#endif
  while (!stop && pos < n) {
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
