// e2_lib.cu — the product library: kernels for sm_100a + host orchestration
// behind the C ABI of include/e2sched.h.
//
// Build (see __graft_entry__.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared ...
//        -o paper_2407_00023_b200/libe2sched.so
// The same file compiled by g++ with -DE2_HOSTSIM (tests/_build only) runs
// the identical engine on the host with a warp width of 1; that build is a
// test double for the CPU suite and is never shipped.
#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "e2_kernels.cuh"

#if E2_DEVICE_BUILD
#include <cuda_runtime.h>
#endif

using namespace e2;

#if !E2_DEVICE_BUILD
struct uint4 {
  unsigned int x, y, z, w;
};
#endif

// ---------------------------------------------------------------------------
// memory / launch layer
// ---------------------------------------------------------------------------
namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#if E2_DEVICE_BUILD
#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw Fail(E2_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
typedef cudaStream_t Stream;
void* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 8;
  CK(cudaMalloc(&p, n));
  // the handle's stream is non-blocking: finish the zero-fill before any
  // async upload on that stream can land in this buffer
  CK(cudaMemset(p, 0, n));
  CK(cudaDeviceSynchronize());
  return p;
}
void dfree(void* p) {
  if (p) cudaFree(p);
}
void h2d(void* dst, const void* src, size_t n, Stream s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s));
}
void d2h(void* dst, const void* src, size_t n, Stream s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s));
}
void d2d(void* dst, const void* src, size_t n, Stream s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s));
}
void dset(void* p, int v, size_t n, Stream s) {
  if (n) CK(cudaMemsetAsync(p, v, n, s));
}
void ssync(Stream s) { CK(cudaStreamSynchronize(s)); }
#else
typedef int Stream;
void* dalloc(size_t n) {
  if (n == 0) n = 8;
  void* p = calloc(1, n);
  if (!p) throw Fail(E2_ERR_ARG, "host alloc failed");
  return p;
}
void dfree(void* p) { free(p); }
void h2d(void* dst, const void* src, size_t n, Stream) {
  if (n) memcpy(dst, src, n);
}
void d2h(void* dst, const void* src, size_t n, Stream) {
  if (n) memcpy(dst, src, n);
}
void d2d(void* dst, const void* src, size_t n, Stream) {
  if (n) memmove(dst, src, n);
}
void dset(void* p, int v, size_t n, Stream) {
  if (n) memset(p, v, n);
}
void ssync(Stream) {}
#endif

template <typename T>
T* talloc(size_t n) {
  return (T*)dalloc(n * sizeof(T));
}

u64 pow2_at_least(u64 v) {
  u64 p = 1;
  while (p < v) p <<= 1;
  return p;
}

// grow a device array keeping the first `keep` elements, zero-filling the rest
template <typename T>
void grow(T*& p, size_t keep, size_t n, Stream s) {
  T* q = talloc<T>(n);
  if (p && keep) d2d(q, p, keep * sizeof(T), s);
  ssync(s);
  dfree(p);
  p = q;
}

}  // namespace

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
namespace {

constexpr int kMatchWarpsPerBlock = 8;
#ifndef E2_FIRST_BATCH
#define E2_FIRST_BATCH 2048
#endif
constexpr i64 kFirstBatch = E2_FIRST_BATCH;  // replay batch-size ramp start
#ifndef E2_SHORT_FIRST_BATCH
#define E2_SHORT_FIRST_BATCH 256
#endif
// short replays (at most 4 first batches) start the ramp lower: there the
// cold-tree first batch is most of the trace, and K1 launch latency is cheap
// next to hint-less walks
constexpr i64 kShortFirstBatch = E2_SHORT_FIRST_BATCH;
constexpr size_t kScrBytes = (2 * sizeof(Scr) + 127) / 128 * 128;

#if E2_DEVICE_BUILD
// blockDim 32: one warp runs everything; blockDim 64 (replays): the
// two-warp pipeline of e2_kernels.cuh (warp 1 runs the evictions).
// Dynamic shared memory: two Scr buffers (the pipeline alternates them per
// request), then the node-cache arrays (a stub unless E2_SMEM_NODECACHE).
// Block prologue shared by k_serial and k_session: the hot state into shared
// memory (warp 0), the node-cache arrays, the pipeline's flags.
__device__ void serial_prologue(u32 nsets, char* dyn, Scr* ss, Pipe* pipe, bool pipelined) {
  const u32 ne = nsets * kWays;
  if (threadIdx.x < 32) {
    const u64* src = (const u64*)g_dev.hot_g;
    u64* dst = (u64*)&g_hot;
    for (u32 i = threadIdx.x; i < sizeof(Hot) / 8; i += 32) dst[i] = src[i];
  }
  if (threadIdx.x == 0) {
    g_nc.nsets = nsets;
    g_nc.clock = 0;
    g_nc.tag = (u32*)dyn;
    g_nc.tick = g_nc.tag + ne;
    g_nc.dirty = g_nc.tick + ne;
    g_nc.data = dyn + ((3 * ne * 4 + 15) / 16) * 16;
  }
  for (u32 i = threadIdx.x; i < ne && threadIdx.x < 32; i += 32) {
    ((u32*)dyn)[i] = kNil;
    ((u32*)dyn)[ne + i] = 0;
    ((u32*)dyn)[2 * ne + i] = 0;
  }
  if (threadIdx.x == 0) {
    g_ctd.pending = 0;
    g_rkd.pending = 0;
    g_defer_ct = pipelined ? 1u : 0u;  // the pipelined replay only
    g_probed = 0;
    g_pf_cur = -1;
    g_pf_stop = 0;
    if (pipe) {
      pipe->ready = 0;
      pipe->books_done = 0;
      pipe->fix_ready = 0;
      pipe->commit_done = 0;
      pipe->w1_fixed = 0;
      pipe->c_ok = 0;
      pipe->stop = 0;
    }
    ss[0].win_done = ss[1].win_done = 0;
  }
}

__device__ void serial_epilogue() {
  if (threadIdx.x < 32) {
    const u64* src = (const u64*)&g_hot;
    u64* dst = (u64*)g_dev.hot_g;
    for (u32 i = threadIdx.x; i < sizeof(Hot) / 8; i += 32) dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(128, 1) k_serial(SerialArgs a, u32 nsets) {
  __shared__ Pipe pipe;
  extern __shared__ __align__(16) char dyn0[];
  Scr* ss = (Scr*)dyn0;
  serial_prologue(nsets, dyn0 + kScrBytes, ss, &pipe, a.kind == 0 && blockDim.x >= 64);
  __syncthreads();
  serial_body(ss, a, blockDim.x >= 64 ? &pipe : nullptr);
  __syncwarp();  // the warps leave their polling loops lane by lane
  __syncthreads();
  serial_epilogue();
}

// ---- per-call session: a persistent one-warp kernel ------------------------
// The per-call API (e2_schedule, note_*, ...) costs a launch, a hot-state
// round trip through HBM and a stream synchronisation per call when each op
// is its own k_serial launch.  A session keeps one warp resident with the hot
// state in shared memory: the host writes the op (and its prompt tokens) into
// a pinned, device-mapped command block and bumps `seq`; the warp polls it,
// copies the tokens into the arena, runs the same api_op, writes ApiOut and
// the hot state into the mapped result block, fences (system scope) and
// publishes `seq`.  The warp exits on a stop command, on an error, or after
// `idle_ns` without a command (so a device-wide synchronisation elsewhere
// never waits on it for long); the host restarts it on the next op.
struct SessCmd {
  volatile unsigned long long seq;
  i32 stop;
  i32 need_match;
  i64 ntok;
  OpDesc op;
  // prompt tokens follow at kSessTok
};
constexpr size_t kSessTok = (sizeof(SessCmd) + 127) / 128 * 128;
constexpr u32 kSessHdrWords = sizeof(SessCmd) / 8;
static_assert(sizeof(SessCmd) % 8 == 0 && kSessHdrWords <= 32, "one word per lane");
struct SessRes {
  volatile unsigned long long seq;  // last command completed
  u64 pad[15];
  ApiOut api;
  Hot hot;
};

__shared__ Hot g_hot_pub;  // k_session: the hot state as last published to the host
constexpr u32 kSessFirst = 4096;  // token bytes read beside the header

__device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(32, 1) k_session(SessCmd* cmd, SessRes* res, unsigned long long next, u32* hint,
                                                   int hstride, u32 nsets, u64 idle_ns) {
  extern __shared__ __align__(16) char dyn0[];
  Scr* ss = (Scr*)dyn0;
  serial_prologue(nsets, dyn0 + kScrBytes, ss, nullptr, false);
  __syncwarp();
  for (u32 i = lane(); i < sizeof(Hot) / 8; i += 32) ((u64*)&g_hot_pub)[i] = ((const u64*)&g_hot)[i];
  u64 tsum[4] = {res->pad[0], res->pad[1], res->pad[2], res->pad[3]};
  __syncwarp();
  u64 t_idle = gtimer();
  for (;;) {
    u32 got = 0;
    if (lane0()) {
      for (;;) {
        if (cmd->seq == next) {
          got = 1;
          break;
        }
        if (gtimer() - t_idle > idle_ns) break;
        __nanosleep(100);
      }
    }
    got = shfl(got, 0);
    if (!got) break;
    const u64 t0 = gtimer();
    // no acquire fence: the reads below issue after the poll returned the new
    // seq, and the host made the command visible before the seq (x86 TSO +
    // its release fence)
    asm volatile("" ::: "memory");
    // one wave over the link: lane i reads header word i and the first 4 KB
    // of tokens are read speculatively beside it (the block always has room).
    // (A TMA bulk copy from the mapped host block never completes.)
    __shared__ u64 hdr[kSessHdrWords];
    const int4* q = (const int4*)((const char*)cmd + kSessTok);
    int4 v[8];
    u64 hw = 0;
    if (lane() < (int)kSessHdrWords) hw = ((const volatile u64*)cmd)[lane()];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                   : "l"(q + k * 32 + lane()));
    if (lane() < (int)kSessHdrWords) hdr[lane()] = hw;
    __syncwarp();
    const SessCmd* c = (const SessCmd*)hdr;
    if (c->stop) break;
    const OpDesc op = c->op;
    const i64 ntok = c->ntok;
    const bool need_match = c->need_match != 0;
    i32* arena = (i32*)g_dev.tok + op.off;
    const i64 nq = (ntok + 3) / 4;  // whole quads: the arena has tail slack
    for (i64 b = 0;; b += 8 * 32) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const i64 j = b + k * 32 + lane();
        if (j < nq) {
          arena[4 * j] = v[k].x;
          if (4 * j + 1 < ntok) arena[4 * j + 1] = v[k].y;
          if (4 * j + 2 < ntok) arena[4 * j + 2] = v[k].z;
          if (4 * j + 3 < ntok) arena[4 * j + 3] = v[k].w;
        }
      }
      if (b + 8 * 32 >= nq) break;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const i64 j = b + 8 * 32 + k * 32 + lane();
        if (j < nq)
          asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                       : "l"(q + j));
      }
    }
    __syncwarp();
    const u64 t1 = gtimer();
    if (lane0()) HOT.done = 0;
    wsync();
    api_op(ss, op, need_match ? hint : nullptr, hstride, &res->api, nullptr);
    const u64 t2 = gtimer();
    if (lane0()) HOT.done = HOT.err ? 0 : 1;
    wsync();
    nflush();
    {
      // only the words that changed since the last publish (the host keeps
      // the whole block current)
      const u64* src = (const u64*)&g_hot;
      u64* sh = (u64*)&g_hot_pub;
      volatile u64* dst = (volatile u64*)&res->hot;
      for (u32 i = lane(); i < sizeof(Hot) / 8; i += 32) {
        const u64 x = src[i];
        if (x != sh[i]) {
          sh[i] = x;
          dst[i] = x;
        }
      }
    }
    if (lane0()) {
      const u64 t3 = gtimer();
      tsum[0] += t1 - t0;  // command header + tokens
      tsum[1] += t2 - t1;  // the op
      tsum[2] += t3 - t2;  // hot state out
      tsum[3] += 1;
      for (int k = 0; k < 4; ++k) res->pad[k] = tsum[k];
    }
    __threadfence_system();
    __syncwarp();
    if (lane0()) res->seq = next;
    ++next;
    const bool err = HOT.err != 0;
    wsync();
    if (err) break;  // the host stops the session and handles the error on the launch path
    t_idle = gtimer();
  }
  __syncwarp();
  serial_epilogue();
  __threadfence_system();
}

// The staged top image for the next K1 launch (one block): the distinct
// level-0 slots of the previous batch's path rows that are still children of
// the root, most used first, each with the head of its edge while the image
// budget lasts; entries sorted by first token.
constexpr u32 kTopSet = 1024;  // distinct level-0 slots tracked (more: the rest probe the child table)
__global__ void __launch_bounds__(1024) k_top_build(const u32* rows, int hstride, i64 nrows, char* img) {
  __shared__ u32 key[kTopSet];
  __shared__ u32 cnt[kTopSet];
  __shared__ u32 cand[kTopSet], ccnt[kTopSet], rank_[kTopSet], hlen[kTopSet];
  __shared__ u32 ncand;
  for (u32 i = threadIdx.x; i < kTopSet; i += blockDim.x) {
    key[i] = kNil;
    cnt[i] = 0;
  }
  if (threadIdx.x == 0) ncand = 0;
  __syncthreads();
  // a sample of the rows is enough to rank the root's children by use
  const i64 step = nrows > 4096 ? nrows / 4096 : 1;
  for (i64 w = (i64)threadIdx.x * step; w < nrows; w += (i64)blockDim.x * step) {
    const u32 v = rows[w * (i64)hstride];
    if (v == kNil || v == kRoot || v >= g_dev.node_cap) continue;
    u32 h = (u32)(mix64(v) & (kTopSet - 1));
    for (u32 probe = 0; probe < 64; ++probe, h = (h + 1) & (kTopSet - 1)) {
      const u32 prev = atomicCAS(&key[h], kNil, v);
      if (prev == kNil || prev == v) {
        atomicAdd(&cnt[h], 1u);
        break;
      }
    }
  }
  __syncthreads();
  for (u32 i = threadIdx.x; i < kTopSet; i += blockDim.x) {
    const u32 v = key[i];
    if (v == kNil) continue;
    const NodeRec* r = grec(g_dev, v);
    if (r->parent != kRoot || r->edge_len == 0) continue;  // split or pruned since: not a root child now
    const u32 k = atomicAdd(&ncand, 1u);
    cand[k] = v;
    ccnt[k] = cnt[i];
  }
  __syncthreads();
  const u32 nc = ncand;
  // rank by (count desc, slot asc); keep the first kTopMaxEnt
  for (u32 i = threadIdx.x; i < nc; i += blockDim.x) {
    u32 rk = 0;
    for (u32 j = 0; j < nc; ++j) rk += (ccnt[j] > ccnt[i] || (ccnt[j] == ccnt[i] && cand[j] < cand[i])) ? 1u : 0u;
    rank_[i] = rk;
    hlen[i] = min_(grec(g_dev, cand[i])->edge_len, kTopHeadMax) & ~3u;  // whole quads
  }
  __syncthreads();
  const u32 ne = min_(nc, kTopMaxEnt);
  const u32 body = 16 + 32 * kTopMaxEnt;
  TopEnt* ents = (TopEnt*)(img + 16);
  for (u32 i = threadIdx.x; i < nc; i += blockDim.x) {
    if (rank_[i] >= ne) continue;
    // heads in rank order while the budget lasts
    u32 before = 0;
    for (u32 j = 0; j < nc; ++j)
      if (rank_[j] < rank_[i]) before += hlen[j];
    u32 hl = hlen[i];
    if (body + 4 * (before + hl) > kTopBytes) hl = 0;  // over the budget: lookup only
    const u32 hoff = hl ? body + 4 * before : body;
    // position in first-token order among the kept entries
    const NodeRec* r = grec(g_dev, cand[i]);
    const i32 t = r->first_tok;
    u32 pos = 0;
    for (u32 j = 0; j < nc; ++j)
      if (rank_[j] < ne && grec(g_dev, cand[j])->first_tok < t) ++pos;
    TopEnt e;
    e.tok = t;
    e.slot = cand[i];
    e.edge_len = r->edge_len;
    e.head_len = hl;
    e.head_off = hoff;
    e.pad = 0;
    e.edge_off = r->edge_off;
    ents[pos] = e;
  }
  __syncthreads();
  // the heads, every thread of the block per entry
  for (u32 j = 0; j < ne; ++j) {
    const TopEnt e = ents[j];
    for (u32 k = threadIdx.x; k < e.head_len; k += blockDim.x)
      ((i32*)(img + e.head_off))[k] = g_dev.tok[e.edge_off + k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 end = body;
    for (u32 j = 0; j < ne; ++j) end = max_(end, ents[j].head_off + 4 * ents[j].head_len);
    TopHdr* hd = (TopHdr*)img;
    hd->n = ne;
    hd->bytes = min_((end + 15) & ~15u, kTopBytes);
    hd->pad[0] = hd->pad[1] = 0;
  }
}

// Persistent: kMatchBlocksPerSM blocks per SM; each warp takes kTile
// requests at a time from a global counter (fetched one ahead, so the
// atomic's latency hides behind the current match) until the batch is
// drained.  The block first copies the staged top image into shared memory
// (one TMA bulk copy).  A tile's level-0 lookups are deduplicated: lanes
// holding the same first token form a __match_any_sync group and only its
// lowest lane searches the staged table.
#ifndef E2_K1_BLOCKS
#define E2_K1_BLOCKS 4
#endif
constexpr int kMatchBlocksPerSM = E2_K1_BLOCKS;
#ifndef E2_K1_TILE
#define E2_K1_TILE 2
#endif
constexpr int kTile = E2_K1_TILE;  // requests per warp work unit (level-0 lookups deduplicated across them)
__global__ void __launch_bounds__(kMatchWarpsPerBlock * 32, kMatchBlocksPerSM)
    k_match(i64 n, i64 base, const i64* off, const i64* len, i64* S, u32* dslot, u32* dm, u32* path, int hstride,
            unsigned long long* bytes, unsigned int* max_levels, unsigned int* next, const char* top_img) {
  __shared__ __align__(128) char top[kTopBytes];
  __shared__ __align__(8) u64 top_bar;
  const bool staged = top_img != nullptr;
  if (staged) {
    if (threadIdx.x == 0) {
      const u32 tb = ((const TopHdr*)top_img)->bytes;
      mbar_init(&top_bar, 1);
      mbar_expect_tx(&top_bar, tb);
      bulk_g2s(top, top_img, tb, &top_bar);
    }
    __syncthreads();  // the barrier is initialised; each warp waits on it at its first lookup
  }
  bool top_ready = !staged;
  unsigned long long acc = 0;
  unsigned int w = 0;
  if (lane0()) w = atomicAdd(next, (unsigned)kTile);
  w = shfl(w, 0);
  while ((i64)w < n) {
    unsigned int wn = 0;
    if (lane0()) wn = atomicAdd(next, (unsigned)kTile);
    int ent = -1;
    if (staged) {
      const i64 q = (i64)w + lane();
      i32 key = (i32)(0x80000000u | (u32)lane());  // distinct negative sentinels (tokens are >= 0)
      if (lane() < kTile && q < n && len[base + q] > 0) key = g_dev.tok[off[base + q]];
      const u32 grp = __match_any_sync(0xffffffffu, key);
      const int lead = ffs32(grp);
      if (!top_ready) {  // the bulk copy overlapped this warp's first loads
        mbar_wait(&top_bar, 0);
        top_ready = true;
      }
      if (lane() == lead && key >= 0) ent = top_find(top, key);
      ent = shfl(ent, lead);
    }
    for (int t = 0; t < kTile; ++t) {
      const i64 q = (i64)w + t;
      if (q >= n) break;
      const int e = shfl(ent, t);
      const MatchRes m = match_one(g_dev.tok + off[base + q], len[base + q], path + q * hstride, hstride,
                                   staged ? top : nullptr, e);
      if (lane0()) {
        S[q] = m.S;
        dslot[q] = m.div_slot;
        dm[q] = m.div_m;
        if (m.levels >= hstride) atomicMax(max_levels, (unsigned int)min_<i64>(m.levels, 0x7fffffff));
        acc += (unsigned long long)m.bytes;
      }
    }
    w = shfl(wn, 0);
  }
  // algorithmic-byte counter: one global atomic per block
  __shared__ unsigned long long blk_bytes;
  if (threadIdx.x == 0) blk_bytes = 0;
  __syncthreads();
  if (acc) atomicAdd(&blk_bytes, acc);  // the lanes that counted requests
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(bytes, blk_bytes);
}

__device__ __forceinline__ void gtab_insert(u64* tk, u32* tv, u64 mask, u64 key, u32 i) {
  u64 idx = key & mask;
  for (;;) {
    unsigned long long prev = atomicCAS((unsigned long long*)&tk[idx], 0ull, (unsigned long long)key);
    if (prev == 0ull || prev == key) {
      atomicMin(&tv[idx], i);
      return;
    }
    idx = (idx + 1) & mask;
  }
}

__device__ __forceinline__ u32 gtab_find(const u64* tk, const u32* tv, u64 mask, u64 key) {
  u64 idx = key & mask;
  for (;;) {
    u64 k = tk[idx];
    if (k == key) return tv[idx];
    if (k == 0) return kNil;
    idx = (idx + 1) & mask;
  }
}

__global__ void k_group_init(i64 n, i64 base, const i64* off, const i64* len, const i64* S, const u32* dslot,
                             const u32* dm, i32* state, u64* A, u64* B, i64* cand, i64* L, u64* tk, u32* tv,
                             u64 mask, i64* leader, int salt) {
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 r = base + i;
  const i64 s = S[i];
  leader[i] = -1;  // the final leader (LCP = L) of a request extended by the rounds
  if (s >= len[r]) {
    state[i] = 0;
    L[i] = s;
    return;
  }
  state[i] = 1;
  A[i] = ((u64)dslot[i] << 32) | (u64)dm[i];
  B[i] = (u64)(u32)g_dev.tok[off[r] + s];
  cand[i] = s;
  gtab_insert(tk, tv, mask, gkey(A[i], B[i], salt), (u32)i);
}

__global__ void k_group_resolve(i64 n, int round, i32* state, const u64* A, const u64* B, const i64* cand,
                                i64* leader, i64* o, i64* L, const u64* tk, const u32* tv, u64 mask,
                                unsigned int* active, unsigned int* collide) {
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || state[i] != 1) return;
  u32 m = gtab_find(tk, tv, mask, gkey(A[i], B[i], round));  // round includes the attempt's salt
  if (m == kNil || A[m] != A[i] || B[m] != B[i]) {
    atomicAdd(collide, 1u);
    state[i] = 0;
    L[i] = -1;
    return;
  }
  if ((i64)m == i) {
    state[i] = 0;
    L[i] = cand[i];
  } else {
    leader[i] = m;
    o[i] = cand[i] + 1;
    atomicAdd(active, 1u);
  }
}

__global__ void __launch_bounds__(kMatchWarpsPerBlock * 32)
    k_group_round(i64 n, i64 base, int round, const i64* off, const i64* len, i32* state, u64* A, u64* B,
                  i64* cand, const i64* leader, const i64* o, i64* L, u64* tk, u32* tv, u64 mask,
                  unsigned long long* bytes) {
  const i64 i = (i64)blockIdx.x * kMatchWarpsPerBlock + (threadIdx.x >> 5);
  if (i >= n || state[i] != 1) return;
  const i64 r = base + i, l = leader[i], rl = base + l;
  const i64 oi = o[i], ni = len[r], nl = len[rl];
  const i64 lim = min_(ni, nl) - oi;
  const i64 a = oi + warp_lcp(g_dev.tok + off[r] + oi, g_dev.tok + off[rl] + oi, lim);
  if (lane0()) {
    atomicAdd(bytes, (unsigned long long)(8 * (a - oi + 1)));
    if (a >= ni) {
      state[i] = 0;
      L[i] = a;
    } else {
      A[i] = ((u64)l << 32) | (u64)a;
      B[i] = (u64)(u32)g_dev.tok[off[r] + a];
      cand[i] = a;
      gtab_insert(tk, tv, mask, gkey(A[i], B[i], round), (u32)i);  // round includes the attempt's salt
    }
  }
}

__global__ void k_ct_reindex(const CtEntry* ct, u64 cap, char* rec, u32 rs) {
  const u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap) return;
  const CtEntry e = ct[j];
  if (e.key == kEmptyKey || e.key == kTombKey) return;
  ((NodeRec*)(rec + (u64)e.val * rs))->ctpos = (u32)j;
}

__global__ void k_arena_index(i64 n, i64 base_tok, const i64* offsets, i64* off, i64* len, i64 first) {
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  off[first + i] = base_tok + offsets[i] - offsets[0];
  len[first + i] = offsets[i + 1] - offsets[i];
}
#endif

// ---- sharded replay: state delta + match summaries ----------
// The replicated state is a fixed list of regions (node pool, child table,
// LRU pages, windows, ...).  Rank 0 keeps a shadow copy of every region as
// the replicas last received it; after each committed batch a diff pass
// emits the 64-byte chunks that differ ({region<<48 | chunk} + payload), the
// replicas scatter them (k_delta_apply) and rank 0 applies the same list to
// its shadow.  Every allocation is zero-filled and every relayout (growth,
// rehash) is a deterministic function of the state, so after the apply each
// replica's regions equal rank 0's byte for byte.
constexpr int kMaxRegions = 16;
constexpr u32 kChunkWords = 16;  // 64 bytes
struct RegionTab {
  u32* cur[kMaxRegions];
  const u32* sh[kMaxRegions];
  u64 words[kMaxRegions];       // allocated words (apply bound)
  u64 chunk0[kMaxRegions + 1];  // prefix sum of live chunks (diff)
  u64 live_words[kMaxRegions];
  int n;
};

E2_HDX int region_of(const RegionTab& t, u64 c) {
  int r = 0;
  while (r + 1 < t.n && c >= t.chunk0[r + 1]) ++r;
  return r;
}

#if E2_DEVICE_BUILD
// One thread per 16-byte quad, four quads per chunk (lanes 4k..4k+3).
__global__ void __launch_bounds__(256) k_delta_diff(RegionTab t, u64 quads, u64* idx, uint4* pay, u64 cap,
                                                    unsigned long long* count) {
  for (u64 q0 = (u64)blockIdx.x * blockDim.x; q0 < quads; q0 += (u64)gridDim.x * blockDim.x) {
    const u64 q = q0 + threadIdx.x;
    const bool in = q < quads;
    const u64 c = q >> 2;
    const u32 part = (u32)(q & 3);
    bool diff = false;
    uint4 v = make_uint4(0, 0, 0, 0);
    int r = 0;
    u64 cc = 0;
    if (in) {
      r = region_of(t, c);
      cc = c - t.chunk0[r];
      const u64 w = cc * kChunkWords + part * 4;
      const u64 lw = t.live_words[r];
      if (w + 4 <= lw) {
        v = *(const uint4*)(t.cur[r] + w);
        const uint4 o = *(const uint4*)(t.sh[r] + w);
        diff = v.x != o.x || v.y != o.y || v.z != o.z || v.w != o.w;
      } else if (w < lw) {
        u32 vv[4] = {0, 0, 0, 0};
        for (u64 k = 0; k < 4 && w + k < lw; ++k) {
          vv[k] = t.cur[r][w + k];
          diff |= vv[k] != t.sh[r][w + k];
        }
        v = make_uint4(vv[0], vv[1], vv[2], vv[3]);
      }
    }
    // any quad of the chunk differs -> the whole chunk goes
    const unsigned lane_id = threadIdx.x & 31;
    const unsigned grp = 0xfu << (lane_id & ~3u);
    const unsigned any = __ballot_sync(0xffffffffu, diff) & grp;
    const bool lead = in && part == 0 && any != 0;
    const unsigned leads = __ballot_sync(0xffffffffu, lead);
    unsigned long long base = 0;
    if (lane_id == 0 && leads) base = atomicAdd(count, (unsigned long long)__popc(leads));
    base = __shfl_sync(0xffffffffu, base, 0);
    const u64 slot = base + (u64)__popc(leads & ((1u << (lane_id & ~3u)) - 1u));
    if (any && in && slot < cap) {
      if (part == 0) idx[slot] = ((u64)r << 48) | cc;
      pay[slot * 4 + part] = v;
    }
  }
}

__global__ void __launch_bounds__(256) k_delta_apply(RegionTab t, u64 n, const u64* idx, const uint4* pay) {
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < n * 4; q += (u64)gridDim.x * blockDim.x) {
    const u64 j = q >> 2;
    const u32 part = (u32)(q & 3);
    const u64 e = idx[j];
    const int r = (int)(e >> 48);
    const u64 w = (e & ((1ull << 48) - 1)) * kChunkWords + part * 4;
    const u64 words = t.words[r];
    const uint4 v = pay[q];
    if (w + 4 <= words) {
      *(uint4*)(t.cur[r] + w) = v;
    } else {
      const u32 vv[4] = {v.x, v.y, v.z, v.w};
      for (u64 k = 0; k < 4 && w + k < words; ++k) t.cur[r][w + k] = vv[k];
    }
  }
}

// Order-independent digest of a region's live words (tests: replica == rank 0).
__global__ void k_digest(const u32* p, u64 words, unsigned long long* out) {
  u64 acc = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (u64)gridDim.x * blockDim.x)
    acc += mix64((i << 32) ^ (u64)p[i]);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

// Match summaries: K1's per-request results as rows [S, dslot, dm, hints].
__global__ void k_shard_pack(i64 lo, i64 cnt, const i64* S, const u32* dslot, const u32* dm, const u32* path,
                             int hstride, char* out, u64 row_bytes, const unsigned int* deepest) {
  const i64 i = (i64)blockIdx.x;
  if (i == 0 && threadIdx.x == 0) {
    ((u64*)out)[0] = *deepest;
    ((u64*)out)[1] = (u64)cnt;
  }
  if (i >= cnt) return;
  char* row = out + 16 + (u64)i * row_bytes;
  const i64 w = lo + i;
  if (threadIdx.x == 0) {
    *(i64*)row = S[w];
    ((u32*)row)[2] = dslot[w];
    ((u32*)row)[3] = dm[w];
  }
  const u32* src = path + (u64)w * hstride;
  u32* dst = (u32*)(row + 16);
  for (int k = threadIdx.x; k < hstride; k += blockDim.x) {
    const u32 v = src[k];
    dst[k] = v;
    if (v == kNil) break;  // rows are kNil-terminated
  }
}

__global__ void k_shard_unpack(int world, i64 per, i64 nb, const char* in, u64 row_bytes, u64 slice_bytes, i64* S,
                               u32* dslot, u32* dm, u32* path, int hstride, unsigned int* deepest) {
  const i64 i = (i64)blockIdx.x;  // batch row
  if (i >= nb) return;
  const i64 k = i / per, j = i - k * per;
  const char* sl = in + (u64)k * slice_bytes;
  if (j == 0 && threadIdx.x == 0) atomicMax(deepest, (unsigned int)((const u64*)sl)[0]);
  const char* row = sl + 16 + (u64)j * row_bytes;
  if (threadIdx.x == 0) {
    S[i] = *(const i64*)row;
    dslot[i] = ((const u32*)row)[2];
    dm[i] = ((const u32*)row)[3];
  }
  const u32* src = (const u32*)(row + 16);
  u32* dst = path + (u64)i * hstride;
  for (int q = threadIdx.x; q < hstride; q += blockDim.x) {
    const u32 v = src[q];
    dst[q] = v;
    if (v == kNil) break;
  }
}
#endif

}  // namespace

// last error of calls without a handle (e2_create, e2_generate)
thread_local std::string g_err;
void e2_set_global_error(const char* m) { g_err = m; }

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
// A batched replay in progress (e2_replay, or the sharded replay's steps).
struct ReplaySession {
  bool active = false;
  bool device_ptrs = false;
  bool stopped = false;
  i64 n = 0, B = 0, next_b0 = 0, cur_b = 0, done = 0;
  i64 cb0 = 0, cnb = 0;  // the current batch
  i64 carried = 0;       // streamed replay: requests of the previous chunk at the front of the arrays
  // prune ticks (driver prune_interval_ms): (combined request index it
  // precedes, tick time); batches are cut at these indices
  std::vector<std::pair<i64, double>> ticks;
  size_t tick_pos = 0;
  SerialArgs a;
  e2_decision* out = nullptr;  // caller's buffers
  e2_cost* costs = nullptr;
  double* ratios = nullptr;
  e2_decision* d_dec = nullptr;  // device-side buffers the kernels write
  e2_cost* d_cost = nullptr;
  double* d_rat = nullptr;
  std::string fail;
  int fail_code = 0;
  int saved_stream_valid = 0;
  void* saved_stream = nullptr;
};

// The delta a sharded replay's rank 0 sends after each batch.
struct DeltaHdr {
  u64 magic;
  i64 n_chunks;
  i64 done;
  i32 fail_code;
  i32 want_hstride;
  u32 n_regions;
  u32 pad;
  u64 region_words[kMaxRegions];
  char msg[256];
  Hot hot;
};
constexpr u64 kDeltaMagic = 0x4532444c54413031ull;  // "E2DLTA01"
constexpr size_t kDeltaHdrBytes = (sizeof(DeltaHdr) + 63) / 64 * 64;

struct ShardState {
  bool on = false;
  int rank = 0, world = 1;
  // rank 0: shadow copy of each region as the replicas hold it
  std::vector<u32*> sh;
  std::vector<u64> sh_words;
  std::vector<const void*> sh_src;  // region pointer the shadow was taken from
  // rank 0: the last delta (chunk list + payload), library-owned
  u64* dl_idx = nullptr;
  uint4* dl_pay = nullptr;
  u64 dl_cap = 0;
  unsigned long long* dl_count = nullptr;
  DeltaHdr hdr;
  i64 row_bytes = 0;
};

struct e2_handle {
  Dev d;
  Hot hot;
  int G = 0;
  e2_sched_cfg cfg;
  e2_time_model model;
  e2_policy pol;
  Stream stream = 0;
  Stream own_stream_handle = 0;
  bool own_stream = false;
  // token arena
  i32* tok = nullptr;
  i64 tok_len = 0, tok_cap = 0;
  // per-request arena index for replays / api
  i64* r_off = nullptr;
  i64* r_len = nullptr;
  i64 r_cap = 0;
  // batch work arrays
  i64 bcap = 0;
  i64 *b_S = nullptr, *b_L = nullptr, *b_cand = nullptr, *b_leader = nullptr, *b_o = nullptr;
  u32 *b_dslot = nullptr, *b_dm = nullptr, *b_path = nullptr;
  i32* b_state = nullptr;
  u64 *b_A = nullptr, *b_B = nullptr;
  u64* g_tk = nullptr;
  u32* g_tv = nullptr;
  u64 g_mask = 0;
  int n_sm = 148;
  Hot dev_hot;  // the hot state last pushed to / pulled from the device
  bool dev_hot_valid = false;
  // pinned host staging for the per-call API: [Hot][ApiOut][off, len][tokens]
  char* pin = nullptr;
  size_t pin_cap = 0;
  bool no_pipe = false;      // E2_NO_PIPE=1: single-warp replays (dev comparisons)
  bool no_prefetch = false;  // E2_NO_PREFETCH=1: no prefetch warp (dev comparisons)
  bool no_top = false;       // E2_NO_TOP=1: K1 without the staged top (dev comparisons)
  unsigned int* d_cnt = nullptr;       // [0] active, [1] collisions, [2] deepest K1 path beyond the hint stride
  int hstride = kPathHint;             // K1 path hints per request (grown when paths get deeper)
  int want_hstride = kPathHint;
  unsigned long long* d_bytes = nullptr;  // [0] match bytes, [1] group bytes
  ApiOut* d_api = nullptr;
  ApiOut api;
  // resident staging for host-buffer replays
  i64 st_cap = 0, st_cost_cap = 0, st_rat_cap = 0;
  i64 *st_ids = nullptr, *st_out = nullptr, *st_offs = nullptr;
  double* st_arr = nullptr;
  e2_decision* st_dec = nullptr;
  e2_cost* st_cost = nullptr;
  double* st_rat = nullptr;
  // autoscale queue stats (global_scheduler.hpp:157-158): host-side, fed by
  // note_admitted; prefix root id -> bucket -> (sum, count)
  std::map<u64, std::map<i64, std::pair<double, i64>>> queue_stats;
  u32 nsets = 0;          // node-cache sets of the serial kernel
  size_t serial_smem = 0;  // its dynamic shared memory
  i64 req_cap = 0;         // d.req_tail capacity
  char* top_img = nullptr;  // K1's staged top image (device)
  i64 top_rows = 0;         // valid rows of b_path from the last K1 batch
  ReplaySession rs;
  ShardState sh;
  // streamed replays (e2_replay_set_continue): the next replay continues the
  // driver state of the previous one; the last finish_lag requests' ids,
  // arrivals and output lengths are carried so their note_finished calls
  // land in the next chunk exactly where a single replay would make them
  bool cont = false;
  double next_tick = 0;  // streamed replays: the next prune tick (driver prune_interval_ms)
  i64 prev_total = 0;   // requests replayed since the last reset
  i64 carry_n = 0;
  i64 *carry_ids = nullptr, *carry_out = nullptr;
  double* carry_arr = nullptr;
  i64 carry_cap = 0;
  i64 *cb_ids = nullptr, *cb_out = nullptr;  // combined [carry | chunk] arrays
  double* cb_arr = nullptr;
  i64 cb_cap = 0;
  // per-call session (k_session): a resident warp fed through pinned,
  // device-mapped command/result blocks
  bool sess_on = false;
  bool no_session = false;  // E2_NO_SESSION=1: every per-call op is its own launch
  Stream sess_stream = 0;
  void* sess_cmd = nullptr;  // SessCmd + tokens (pinned, mapped)
  void* sess_res = nullptr;  // SessRes (pinned, mapped)
  i64 sess_tok_cap = 0;
  unsigned long long sess_next = 1;  // the next command number
  u64 sess_idle_ns = 2000000;
  std::vector<i32> sess_last;  // tokens of the last committed op sent through the session
  i64 sess_last_off = 0;
  bool sess_last_ok = false;
  i64 sess_ops = 0, sess_starts = 0, sess_relaunch = 0, sess_stops = 0;
  i64 sess_why[5] = {0, 0, 0, 0, 0};
  // reserve_* dry run: report (dry_hit) instead of growing
  bool dry = false, dry_hit = false;
  // profiling
  bool prof = false;
  e2_profile acc;
#if E2_DEVICE_BUILD
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  std::vector<cudaEvent_t> ev_pool;
#endif
  std::string err;
};

namespace {

#if E2_DEVICE_BUILD
cudaEvent_t ev_get(e2_handle* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}
struct Timed {
  e2_handle* h;
  int k;
  cudaEvent_t a = nullptr, b = nullptr;
  Timed(e2_handle* hh, int kk) : h(hh), k(kk) {
    if (h->prof) {
      a = ev_get(h);
      b = ev_get(h);
      CK(cudaEventRecord(a, h->stream));
    }
  }
  ~Timed() {
    if (h->prof) {
      cudaEventRecord(b, h->stream);
      h->ev.push_back({k, {a, b}});
    }
  }
};
void prof_flush(e2_handle* h) {
  if (h->ev.empty()) return;
  ssync(h->stream);
  for (auto& e : h->ev) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e.second.first, e.second.second);
    h->acc.ms[e.first] += ms;
    h->ev_pool.push_back(e.second.first);
    h->ev_pool.push_back(e.second.second);
  }
  h->ev.clear();
}
#else
struct Timed {
  Timed(e2_handle*, int) {}
};
void prof_flush(e2_handle*) {}
#endif

// The kernels read the handle's pointers/config from constant memory.
void upload_dev(e2_handle* h) {
#if E2_DEVICE_BUILD
  // skipped when the constant bank already holds this descriptor (calls are
  // serialised across handles, and each call completes before returning)
  static Dev last;
  static bool last_valid = false;
  if (last_valid && memcmp(&last, &h->d, sizeof(Dev)) == 0) return;
  CK(cudaMemcpyToSymbolAsync(g_dev, &h->d, sizeof(Dev), 0, cudaMemcpyHostToDevice, h->stream));
  last = h->d;
  last_valid = true;
#else
  g_dev_h = h->d;
#endif
}

// The host mirror of the hot state is pushed only when it differs from the
// last state known to be on the device (a per-call API op would otherwise
// upload ~7 KB per call for nothing).
void push_hot(e2_handle* h) {
  if (h->dev_hot_valid && memcmp(&h->hot, &h->dev_hot, sizeof(Hot)) == 0) return;
  h2d(h->d.hot_g, &h->hot, sizeof(Hot), h->stream);
  h->dev_hot = h->hot;
  h->dev_hot_valid = true;
}
bool session_active(const e2_handle* h);
void pull_hot(e2_handle* h) {
  if (session_active(h)) return;  // h->hot is the session's last published state
  d2h(&h->hot, h->d.hot_g, sizeof(Hot), h->stream);
  ssync(h->stream);
  h->dev_hot = h->hot;
  h->dev_hot_valid = true;
}

void zero_ptrs(Dev& d) {
  Cfg c = d.cfg;
  memset(&d, 0, sizeof(d));
  d.cfg = c;
}

// ---- capacity management ---------------------------------------------------
void host_rehash_ct(e2_handle* h, u64 new_cap) {
  Dev& d = h->d;
  const u64 old_cap = d.ct ? d.ct_mask + 1 : 0;
  std::vector<CtEntry> old(old_cap);
  if (old_cap) {
    d2h(old.data(), d.ct, old_cap * sizeof(CtEntry), h->stream);
    ssync(h->stream);
  }
  CtEntry empty;
  empty.key = kEmptyKey;
  empty.val = 0;
  empty.pad = 0;
  std::vector<CtEntry> nt(new_cap, empty);
  const u64 mask = new_cap - 1;
  for (u64 i = 0; i < old_cap; ++i) {
    const u64 k = old[i].key;
    if (k == kEmptyKey || k == kTombKey) continue;
    u64 j = mix64(k) & mask;
    while (nt[j].key != kEmptyKey) j = (j + 1) & mask;
    nt[j] = old[i];
  }
  dfree(d.ct);
  d.ct = talloc<CtEntry>(new_cap);
  h2d(d.ct, nt.data(), new_cap * sizeof(CtEntry), h->stream);
  // every node's record holds the position of its own entry (ctpos)
#if E2_DEVICE_BUILD
  k_ct_reindex<<<(unsigned)((new_cap + 255) / 256), 256, 0, h->stream>>>(d.ct, new_cap, d.rec, d.rs);
  CK(cudaGetLastError());
#else
  for (u64 j = 0; j < new_cap; ++j) {
    const u64 k = nt[j].key;
    if (k == kEmptyKey || k == kTombKey) continue;
    ((NodeRec*)(d.rec + (u64)nt[j].val * d.rs))->ctpos = (u32)j;
  }
#endif
  ssync(h->stream);
  d.ct_mask = mask;
}

void reserve_nodes(e2_handle* h, u64 need) {
  Dev& d = h->d;
  if (need <= d.node_cap && d.rec) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  const int G = h->G;
  u64 cap = std::max<u64>(need, (u64)d.node_cap * 2);
  cap = std::max<u64>(cap, 1024);
  if (cap > 0xfffffff0ull) throw Fail(E2_ERR_ARG, "node capacity exceeds 32-bit slots");
  const u64 keep = h->hot.slots_used;
  grow(d.rec, keep * d.rs, cap * d.rs, h->stream);
  d.node_cap = (u32)cap;
  // child table at load <= 1/2
  const u64 ct = pow2_at_least(2 * cap);
  if (!d.ct || ct > d.ct_mask + 1) host_rehash_ct(h, ct);
  // LRU pages: each page holds >= 1 key; keys <= cached nodes
  const u64 pages = cap / 2 + 1024 * (u64)G;
  if (pages > d.page_cap || !d.pg_la) {
    const u64 kp = h->hot.pages_used;
    grow(d.pg_la, kp * kPage, pages * kPage, h->stream);
    grow(d.pg_id, kp * kPage, pages * kPage, h->stream);
    grow(d.pg_slot, kp * kPage, pages * kPage, h->stream);
    grow(d.free_pages, h->hot.free_top, pages, h->stream);
    d.page_cap = (u32)pages;
  }
  // directory ring per instance
  const u64 dcap = pow2_at_least(std::max<u64>(cap / 8 + 1024, 1024));
  if (dcap > d.dcap) {
    DirEntry* nd = talloc<DirEntry>(dcap * G);
    if (d.dir) {
      std::vector<DirEntry> od(d.dcap * (u64)G), pd(dcap * G);
      d2h(od.data(), d.dir, od.size() * sizeof(DirEntry), h->stream);
      ssync(h->stream);
      for (int g = 0; g < G; ++g) {
        for (u32 k = 0; k < h->hot.dir_n[g]; ++k)
          pd[(u64)g * dcap + k] = od[(u64)g * d.dcap + ((h->hot.dir_head[g] + k) & (d.dcap - 1))];
        h->hot.dir_head[g] = 0;
      }
      h2d(nd, pd.data(), pd.size() * sizeof(DirEntry), h->stream);
      ssync(h->stream);
      dfree(d.dir);
    }
    d.dir = nd;
    d.dcap = (u32)dcap;
    push_hot(h);
  }
  // plan scratch
  if (!d.scr_slot) {
    d.scap = 1u << 16;
    d.vcap = 1u << 16;
    d.scr_slot = talloc<u32>((u64)d.scap * G);
    d.scr_la = talloc<u64>((u64)d.scap * G);
    d.scr_id = talloc<u64>((u64)d.scap * G);
    d.scr_val = talloc<i64>((u64)d.scap * G + 1);
    d.vic_slot = talloc<u32>(d.vcap);
    d.vic_tok = talloc<i64>(d.vcap);
  }
}

// relayout a monotone-index ring (per instance) into a larger capacity
template <typename T>
void ring_regrow(e2_handle* h, T*& arr, u64 oldcap, u64 newcap, const u64* heads, const u64* tails) {
  const int G = h->G;
  T* na = talloc<T>(newcap * G);
  if (arr && oldcap) {
    std::vector<T> o(oldcap * G), n(newcap * G);
    d2h(o.data(), arr, o.size() * sizeof(T), h->stream);
    ssync(h->stream);
    for (int g = 0; g < G; ++g)
      for (u64 i = heads[g]; i < tails[g]; ++i) n[(u64)g * newcap + (i & (newcap - 1))] = o[(u64)g * oldcap + (i & (oldcap - 1))];
    h2d(na, n.data(), n.size() * sizeof(T), h->stream);
    ssync(h->stream);
  }
  dfree(arr);
  arr = na;
}

void reserve_window(e2_handle* h, u64 entries) {
  Dev& d = h->d;
  const u64 cap = pow2_at_least(std::max<u64>(entries, 1024));
  if (cap <= d.wcap) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  // scheduled entries stay until their hit stamps are undone (ws_done)
  ring_regrow(h, d.win, d.wcap, cap, h->hot.ws_done, h->hot.ws_tail);
  ring_regrow(h, d.comp, d.wcap, cap, h->hot.wc_head, h->hot.wc_tail);
  d.wcap = cap;
}

// Path log rings: grown (up to a bound) when an instance's live log passes
// half the ring; entries that do not fit are simply not logged (their hit
// stamps are undone by the parent-chain walk instead).
constexpr u64 kPlogMin = 1ull << 16, kPlogMax = 1ull << 21;
void reserve_plog(e2_handle* h) {
  Dev& d = h->d;
  if (!d.plog && h->dry) {
    h->dry_hit = true;
    return;
  }
  if (!d.plog) {
    d.pcap = kPlogMin;
    d.plog = talloc<u32>(d.pcap * (u64)h->G);
    return;
  }
  u64 live = 0;
  for (int g = 0; g < h->G; ++g) live = std::max<u64>(live, h->hot.pl_tail[g] - h->hot.pl_head[g]);
  if (live * 2 <= d.pcap || d.pcap >= kPlogMax) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  const u64 cap = std::min<u64>(d.pcap * 4, kPlogMax);
  ring_regrow(h, d.plog, d.pcap, cap, h->hot.pl_head, h->hot.pl_tail);
  d.pcap = cap;
}

void reserve_fifo(e2_handle* h, u64 entries) {
  Dev& d = h->d;
  u64 cap = pow2_at_least(std::max<u64>(entries, 64));
  if (cap <= d.fcap) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  ring_regrow(h, d.fifo_req, d.fcap, cap, h->hot.fifo_head, h->hot.fifo_tail);
  ring_regrow(h, d.fifo_tail, d.fcap, cap, h->hot.fifo_head, h->hot.fifo_tail);
  d.fcap = cap;
}

void reserve_inflight(e2_handle* h, u64 live) {
  Dev& d = h->d;
  const u64 cap = pow2_at_least(std::max<u64>(4 * live + 64, 1024));
  if (d.inf && cap <= d.inf_mask + 1) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  const u64 oc = d.inf ? d.inf_mask + 1 : 0;
  std::vector<InfRec> old(oc);
  if (oc) {
    d2h(old.data(), d.inf, oc * sizeof(InfRec), h->stream);
    ssync(h->stream);
  }
  InfRec empty;
  memset(&empty, 0, sizeof(empty));
  empty.key = kNoInflight;
  std::vector<InfRec> nt(cap, empty);
  const u64 mask = cap - 1;
  for (u64 i = 0; i < oc; ++i) {
    if (old[i].key == kNoInflight) continue;
    u64 j = mix64((u64)old[i].key) & mask;
    while (nt[j].key != kNoInflight) j = (j + 1) & mask;
    nt[j] = old[i];
  }
  dfree(d.inf);
  d.inf = talloc<InfRec>(cap);
  h2d(d.inf, nt.data(), cap * sizeof(InfRec), h->stream);
  ssync(h->stream);
  d.inf_mask = mask;
}

void reserve_tokens(e2_handle* h, i64 need) {
  if (need + 128 <= h->tok_cap) return;
  if (h->dry) {
    h->dry_hit = true;
    return;
  }
  i64 cap = std::max<i64>(need + 128, h->tok_cap * 2);
  cap = std::max<i64>(cap, 1 << 16);
  grow(h->tok, (size_t)h->tok_len, (size_t)cap, h->stream);
  h->tok_cap = cap;
  h->d.tok = h->tok;
}

void reserve_requests(e2_handle* h, i64 need) {
  if (need <= h->r_cap) return;
  i64 cap = std::max<i64>(need, h->r_cap * 2);
  cap = std::max<i64>(cap, 1024);
  grow(h->r_off, 0, cap, h->stream);
  grow(h->r_len, 0, cap, h->stream);
  h->r_cap = cap;
}

void reserve_batch(e2_handle* h, i64 B) {
  if (h->dry) {
    if ((h->want_hstride > h->hstride && h->bcap > 0) || B > h->bcap) h->dry_hit = true;
    return;
  }
  if (h->want_hstride > h->hstride && h->bcap > 0) {
    // paths got deeper than the hint stride in an earlier batch
    dfree(h->b_path);
    h->hstride = h->want_hstride;
    h->b_path = talloc<u32>(h->bcap * h->hstride);
  }
  if (B <= h->bcap) return;
  i64 cap = std::max<i64>(B, 256);
  dfree(h->b_S);
  dfree(h->b_L);
  dfree(h->b_cand);
  dfree(h->b_leader);
  dfree(h->b_o);
  dfree(h->b_dslot);
  dfree(h->b_dm);
  dfree(h->b_path);
  dfree(h->b_state);
  dfree(h->b_A);
  dfree(h->b_B);
  dfree(h->g_tk);
  dfree(h->g_tv);
  h->b_S = talloc<i64>(cap);
  h->b_L = talloc<i64>(cap);
  h->b_cand = talloc<i64>(cap);
  h->b_leader = talloc<i64>(cap);
  h->b_o = talloc<i64>(cap);
  h->b_dslot = talloc<u32>(cap);
  h->b_dm = talloc<u32>(cap);
  h->b_path = talloc<u32>(cap * h->hstride);
  h->b_state = talloc<i32>(cap);
  h->b_A = talloc<u64>(cap);
  h->b_B = talloc<u64>(cap);
  u64 t = pow2_at_least(2 * (u64)cap);
  h->g_tk = talloc<u64>(t);
  h->g_tv = talloc<u32>(t);
  h->g_mask = t - 1;
  h->bcap = cap;
}

void check_hot_error(e2_handle* h) {
  if (h->hot.err == 0) return;
  static const char* why[] = {"",
                              "prompt exceeds every GPU's KV capacity",
                              "global_scheduler: cached spans are not root-contiguous on any GPU",
                              "prefix_tree: insert of empty sequence",
                              "prefix_tree: cached_child_count underflow",
                              "device node pool exhausted",
                              "device child table full",
                              "device LRU page pool exhausted",
                              "device LRU directory exhausted",
                              "device load window ring exhausted",
                              "device inflight map exhausted",
                              "device plan scratch exhausted",
                              "internal: walk did not find a matched child",
                              "prefix_tree: split boundary outside edge",
                              "device FIFO ring exhausted"};
  int code = h->hot.err;
  int w = h->hot.why;
  std::string msg = (w >= 0 && w < (int)(sizeof(why) / sizeof(why[0]))) ? why[w] : "device error";
  h->hot.err = 0;
  h->hot.why = 0;
  push_hot(h);
  ssync(h->stream);
  throw Fail(code, msg);
}

// Ensure capacities for `req` more requests with `toks` more tokens.
void reserve_for(e2_handle* h, i64 req, i64 toks) {
  reserve_tokens(h, h->tok_len + toks);
  reserve_nodes(h, (u64)h->hot.slots_used + 5 * (u64)req + 64);
  u64 maxw = 0, maxf = 0;
  for (int g = 0; g < h->G; ++g) {
    maxw = std::max<u64>(maxw, h->hot.ws_tail[g] - h->hot.ws_done[g]);
    maxw = std::max<u64>(maxw, h->hot.wc_tail[g] - h->hot.wc_head[g]);
    maxf = std::max<u64>(maxf, h->hot.fifo_tail[g] - h->hot.fifo_head[g]);
  }
  reserve_window(h, maxw + (u64)req + 1);
  reserve_plog(h);
  reserve_fifo(h, maxf + (u64)req + 1);
  reserve_inflight(h, (u64)h->hot.inflight_n + (u64)req + 1);
}

// ---- launches ---------------------------------------------------------------
void launch_serial(e2_handle* h, const SerialArgs& a) {
  {
    Timed t(h, a.kind == 0 ? E2_K_COMMIT : E2_K_OTHER);
#if E2_DEVICE_BUILD
    h->acc.launches[a.kind == 0 ? E2_K_COMMIT : E2_K_OTHER]++;
    upload_dev(h);
    // replays pipeline evictions on a second warp (the shared-memory node
    // cache variant is single-writer only)
#if defined(E2_SMEM_NODECACHE)
    const unsigned threads = 32;
#else
    const unsigned threads = (a.kind == 0 && !h->no_pipe) ? 128 : 32;  // warps: decide, evict, prefetch, books
    SerialArgs ka = a;
    ka.no_prefetch = h->no_prefetch ? 1 : 0;
#endif
    k_serial<<<1, threads, h->serial_smem, h->stream>>>(ka, h->nsets);
    CK(cudaGetLastError());
#else
    Scr s;
    memset(&s, 0, sizeof(s));
    const u32 ne = h->nsets * kWays;
    std::vector<u32> tag(ne, kNil), tick(ne, 0), dirty(ne, 0);
    std::vector<u64> data((size_t)ne * h->d.rs / 8);
    NCache nc;
    nc.nsets = h->nsets;
    nc.clock = 0;
    nc.victim = 0;
    nc.tag = tag.data();
    nc.tick = tick.data();
    nc.dirty = dirty.data();
    nc.data = (char*)data.data();
    g_dev_h = h->d;
    g_hot_h = h->d.hot_g;
    g_nc_h = nc;
    serial_body(&s, a);
#endif
  }
}

// A K1 path reached `levels` >= the hint stride: grow it for later batches.
void note_depth(e2_handle* h, u64 levels) {
  if (levels < (u64)h->hstride) return;
  int want = h->hstride;
  while ((u64)want <= levels && want < kMaxHint) want *= 2;
  h->want_hstride = std::max(h->want_hstride, want);
}

// K1 over requests [base+lo, base+lo+cnt) of the arena index; results land
// in the batch arrays at [lo, lo+cnt).  Returns the deepest path seen when it
// reached the hint stride (0 otherwise) via note_depth on the device path.
void k1_slice(e2_handle* h, i64 base, i64 lo, i64 cnt) {
  if (cnt <= 0) return;
  [[maybe_unused]] Dev& d = h->d;  // the host emulation's match reads the arena through it
#if E2_DEVICE_BUILD
  const i64 blocks = (cnt + kMatchWarpsPerBlock * kTile - 1) / (kMatchWarpsPerBlock * kTile);
  const unsigned grid = (unsigned)std::min<i64>(blocks, (i64)h->n_sm * kMatchBlocksPerSM);
  upload_dev(h);
  if (!h->top_img) h->top_img = (char*)dalloc(kTopBytes);
  if (!h->no_top) {
    // the staged top, from the root children the previous batch walked through
    // (its path rows, still in b_path: rebuilt before this launch overwrites them)
    Timed tt(h, E2_K_OTHER);
    h->acc.launches[E2_K_OTHER]++;
    k_top_build<<<1, 1024, 0, h->stream>>>(h->b_path, h->hstride, std::min<i64>(h->top_rows, h->bcap), h->top_img);
    CK(cudaGetLastError());
  }
  h->acc.launches[E2_K_MATCH]++;
  dset(h->d_cnt + 2, 0, 8, h->stream);  // [2] deepest path, [3] work counter
  {
    Timed t(h, E2_K_MATCH);  // the kernel alone (roofline denominator)
    k_match<<<grid, kMatchWarpsPerBlock * 32, 0, h->stream>>>(cnt, base + lo, h->r_off, h->r_len, h->b_S + lo,
                                                             h->b_dslot + lo, h->b_dm + lo,
                                                             h->b_path + lo * h->hstride, h->hstride, h->d_bytes,
                                                             h->d_cnt + 2, h->d_cnt + 3,
                                                             h->no_top ? nullptr : h->top_img);
    CK(cudaGetLastError());
  }
  h->top_rows = lo + cnt;
#else
  h->d_cnt[2] = 0;
  for (i64 w = lo; w < lo + cnt; ++w) {
    const i64 r = base + w;
    g_dev_h = h->d;
    MatchRes m = match_one(d.tok + h->r_off[r], h->r_len[r], h->b_path + w * h->hstride, h->hstride);
    h->b_S[w] = m.S;
    h->b_dslot[w] = m.div_slot;
    h->b_dm[w] = m.div_m;
    h->d_bytes[0] += (unsigned long long)m.bytes;
    if (m.levels >= h->hstride) h->d_cnt[2] = std::max<unsigned int>(h->d_cnt[2], (unsigned int)m.levels);
  }
#endif
  h->acc.match_requests += cnt;
}

// Leader rounds over the batch [0, n) (K1 results in b_S/b_dslot/b_dm):
// produces b_L and b_leader.  `deepest`: K1's deepest path beyond the hint
// stride (device: already in d_cnt[2]).
void group_rounds(e2_handle* h, i64 base, i64 n) {
  [[maybe_unused]] Dev& d = h->d;
  if (n == 1) {
    // single sequence: no intra-batch dependency
#if !E2_DEVICE_BUILD
    note_depth(h, h->d_cnt[2]);
#endif
    d2d(h->b_L, h->b_S, 8, h->stream);
    dset(h->b_leader, 0xff, 8, h->stream);  // -1: no in-batch leader
#if E2_DEVICE_BUILD
    unsigned int c2 = 0;
    d2h(&c2, h->d_cnt + 2, 4, h->stream);
    ssync(h->stream);
    note_depth(h, c2);
#endif
    return;
  }
#if E2_DEVICE_BUILD
  Timed t(h, E2_K_GROUP);
  const u64 tsz = h->g_mask + 1;
  const unsigned tg = (unsigned)((n + 255) / 256);
  // A 64-bit key collision between two different (divergence point, next
  // token) pairs is detected by k_group_resolve; the grouping then restarts
  // with a fresh salt (a new hash family), so a collision costs one retry.
  for (int attempt = 0;; ++attempt) {
    if (attempt == 8) throw Fail(E2_ERR_ARG, "intra-batch grouping: repeated hash collisions");
    const int salt = attempt * 4096;
    dset(h->g_tk, 0, tsz * 8, h->stream);
    dset(h->g_tv, 0xff, tsz * 4, h->stream);
    h->acc.launches[E2_K_GROUP]++;
    k_group_init<<<tg, 256, 0, h->stream>>>(n, base, h->r_off, h->r_len, h->b_S, h->b_dslot, h->b_dm, h->b_state,
                                            h->b_A, h->b_B, h->b_cand, h->b_L, h->g_tk, h->g_tv, h->g_mask,
                                            h->b_leader, salt);
    CK(cudaGetLastError());
    bool collided = false;
    for (int round = 0;; ++round) {
      dset(h->d_cnt, 0, 8, h->stream);
      h->acc.launches[E2_K_GROUP]++;
      k_group_resolve<<<tg, 256, 0, h->stream>>>(n, round + salt, h->b_state, h->b_A, h->b_B, h->b_cand,
                                                 h->b_leader, h->b_o, h->b_L, h->g_tk, h->g_tv, h->g_mask, h->d_cnt,
                                                 h->d_cnt + 1);
      CK(cudaGetLastError());
      unsigned int cnt[3];
      d2h(cnt, h->d_cnt, 12, h->stream);
      ssync(h->stream);
      note_depth(h, cnt[2]);
      if (cnt[1]) {
        collided = true;
        h->acc.group_retries++;
        break;
      }
      if (cnt[0] == 0) break;
      dset(h->g_tk, 0, tsz * 8, h->stream);
      dset(h->g_tv, 0xff, tsz * 4, h->stream);
      unsigned grid = (unsigned)((n + kMatchWarpsPerBlock - 1) / kMatchWarpsPerBlock);
      h->acc.launches[E2_K_GROUP]++;
      k_group_round<<<grid, kMatchWarpsPerBlock * 32, 0, h->stream>>>(
          n, base, round + 1 + salt, h->r_off, h->r_len, h->b_state, h->b_A, h->b_B, h->b_cand, h->b_leader,
          h->b_o, h->b_L, h->g_tk, h->g_tv, h->g_mask, h->d_bytes + 1);
      CK(cudaGetLastError());
    }
    if (!collided) break;
  }
#else
  note_depth(h, h->d_cnt[2]);
  // host emulation: the same recursion with std::map grouping
  const i64* S = h->b_S;
  std::vector<i32> st(n);
  std::vector<u64> A(n), B(n);
  std::vector<i64> cand(n), leader(n, -1), o(n);
  i64* L = h->b_L;
  for (i64 i = 0; i < n; ++i) {
    const i64 r = base + i;
    if (S[i] >= h->r_len[r]) {
      st[i] = 0;
      L[i] = S[i];
      continue;
    }
    st[i] = 1;
    A[i] = ((u64)h->b_dslot[i] << 32) | h->b_dm[i];
    B[i] = (u64)(u32)d.tok[h->r_off[r] + S[i]];
    cand[i] = S[i];
  }
  for (int round = 0;; ++round) {
    std::map<std::pair<u64, u64>, i64> first;
    for (i64 i = 0; i < n; ++i)
      if (st[i] == 1) first.emplace(std::make_pair(A[i], B[i]), i);
    i64 active = 0;
    for (i64 i = 0; i < n; ++i) {
      if (st[i] != 1) continue;
      i64 m = first[std::make_pair(A[i], B[i])];
      if (m == i) {
        st[i] = 0;
        L[i] = cand[i];
      } else {
        leader[i] = m;
        o[i] = cand[i] + 1;
        active++;
      }
    }
    if (!active) break;
    for (i64 i = 0; i < n; ++i) {
      if (st[i] != 1) continue;
      const i64 r = base + i, rl = base + leader[i];
      const i64 lim = std::min(h->r_len[r], h->r_len[rl]) - o[i];
      const i64 a = o[i] + warp_lcp(d.tok + h->r_off[r] + o[i], d.tok + h->r_off[rl] + o[i], lim);
      if (a >= h->r_len[r]) {
        st[i] = 0;
        L[i] = a;
      } else {
        A[i] = ((u64)leader[i] << 32) | (u64)a;
        B[i] = (u64)(u32)d.tok[h->r_off[r] + a];
        cand[i] = a;
      }
    }
  }
  for (i64 i = 0; i < n; ++i) h->b_leader[i] = leader[i];
#endif
}

// K1 + leader rounds for requests [base, base+n) of the arena index.
// Produces h->b_L[0..n).
void launch_match(e2_handle* h, i64 base, i64 n) {
  if (n == 0) return;
  reserve_batch(h, n);
  k1_slice(h, base, 0, n);
  group_rounds(h, base, n);
}

// Per-call API staging (pinned host memory).
constexpr size_t kPinHead = (sizeof(Hot) + sizeof(ApiOut) + 63) / 64 * 64;

// Pinned staging for the per-call API (async copies; reused after the call's
// synchronisation).
char* pin_reserve(e2_handle* h, size_t bytes) {
  const size_t need = kPinHead + 16 + bytes;
  if (need > h->pin_cap) {
    const size_t cap = std::max<size_t>(need, 2 * h->pin_cap + (1 << 16));
#if E2_DEVICE_BUILD
    if (h->pin) {
      ssync(h->stream);  // no async copy may still read the old buffer
      cudaFreeHost(h->pin);
    }
    CK(cudaMallocHost((void**)&h->pin, cap));
#else
    free(h->pin);
    h->pin = (char*)malloc(cap);
#endif
    h->pin_cap = cap;
  }
  return h->pin;
}

// Append tokens only (per-call API: the serial kernel gets offset/length as
// arguments).
void append_host_tokens(e2_handle* h, const i32* seq, i64 len) {
  reserve_tokens(h, h->tok_len + len);
  char* p = pin_reserve(h, (size_t)len * 4);
  i32* t = (i32*)(p + kPinHead + 16);
  memcpy(t, seq, (size_t)len * 4);
  h2d(h->tok + h->tok_len, t, (size_t)len * 4, h->stream);
  h->tok_len += len;
}


// ---- per-call session (host side of k_session) -----------------------------
e2_handle* g_sess_owner = nullptr;  // at most one session: g_dev is shared by every handle
bool session_active(const e2_handle* h) { return h->sess_on; }

#if E2_DEVICE_BUILD
SessCmd* sess_cmd(e2_handle* h) { return (SessCmd*)h->sess_cmd; }
SessRes* sess_res(e2_handle* h) { return (SessRes*)h->sess_res; }

// Wait until k_session left (stop command, idle timeout or error) and take
// the state it wrote back to HBM as the device's.
void session_stop(e2_handle* h) {
  if (h) h->sess_last_ok = false;
  if (!h || !h->sess_on) return;
  h->sess_stops++;
  SessCmd* c = sess_cmd(h);
  c->stop = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  c->seq = h->sess_next++;
  const cudaError_t e = cudaStreamSynchronize(h->sess_stream);
  c->stop = 0;
  h->sess_on = false;
  if (g_sess_owner == h) g_sess_owner = nullptr;
  if (e != cudaSuccess) throw Fail(E2_ERR_CUDA, std::string("session: ") + cudaGetErrorString(e));
  h->dev_hot = h->hot;  // the kernel's last published hot state, now in hot_g
  h->dev_hot_valid = true;
}

void session_launch(e2_handle* h) {
  k_session<<<1, 32, h->serial_smem, h->sess_stream>>>(sess_cmd(h), sess_res(h), h->sess_next, h->b_path, h->hstride,
                                                      h->nsets, h->sess_idle_ns);
  CK(cudaGetLastError());
  h->sess_starts++;
}

void session_start(e2_handle* h) {
  if (g_sess_owner && g_sess_owner != h) session_stop(g_sess_owner);
  if (!h->sess_stream) CK(cudaStreamCreateWithFlags(&h->sess_stream, cudaStreamNonBlocking));
  push_hot(h);
  upload_dev(h);
  ssync(h->stream);  // every earlier copy and launch of h is complete
  memcpy((void*)&sess_res(h)->hot, &h->hot, sizeof(Hot));  // the warp publishes changed words only
  session_launch(h);
  h->sess_on = true;
  g_sess_owner = h;
}

void session_buffers(e2_handle* h, i64 ntok) {
  if (h->sess_cmd && ntok <= h->sess_tok_cap) return;
  session_stop(h);
  if (h->sess_cmd) cudaFreeHost(h->sess_cmd);
  h->sess_cmd = nullptr;
  const i64 cap = std::max<i64>(ntok, std::max<i64>(2 * h->sess_tok_cap, 1 << 14));
  CK(cudaHostAlloc(&h->sess_cmd, kSessTok + (size_t)cap * 4 + kSessFirst + 64, cudaHostAllocMapped));
  memset(h->sess_cmd, 0, kSessTok);
  h->sess_tok_cap = cap;
  if (!h->sess_res) {
    CK(cudaHostAlloc(&h->sess_res, sizeof(SessRes), cudaHostAllocMapped));
    memset(h->sess_res, 0, sizeof(SessRes));
  }
  // command numbers restart with the new block (the old one is gone)
  h->sess_next = 1;
}

// Would reserve_for / reserve_batch grow anything for this op?
bool session_fits(e2_handle* h, i64 len, bool need_match) {
  h->dry = true;
  h->dry_hit = false;
  reserve_for(h, 1, len);
  if (need_match) reserve_batch(h, 1);
  h->dry = false;
  return !h->dry_hit;
}

bool session_kind(i32 k) {
  switch (k) {
    case OP_SCHEDULE:
    case OP_DECIDE:
    case OP_PREFILL:
    case OP_EVICT:
    case OP_FINISHED:
    case OP_LOAD_COST:
    case OP_GPU_LOAD:
    case OP_MATCH:
    case OP_WINDOW:
    case OP_INFLIGHT_GET:
      return true;
    default:
      return false;
  }
}

// Run one per-call op through the session.  False: not taken (the caller
// uses the launch path; any running session is stopped first).
bool session_op(e2_handle* h, OpDesc op, const i32* seq, i64 len, bool need_match, bool transient) {
  int why = 0;
  if (h->no_session) why = 1;
  else if (!session_kind(op.kind)) why = 2;
  else if (!h->dev_hot_valid || memcmp(&h->hot, &h->dev_hot, sizeof(Hot)) != 0) why = 3;
  else if (!session_fits(h, seq ? len : 0, need_match)) why = 4;
  if (why) {
    h->sess_why[why]++;
    session_stop(h);
    return false;
  }
  session_buffers(h, seq ? len : 0);
  if (!h->sess_on) session_start(h);
  SessCmd* c = sess_cmd(h);
  SessRes* r = sess_res(h);
  // the same prompt as the last committed op (schedule, then its
  // note_prefill_cached): its tokens are already in the arena
  const bool reuse = seq && h->sess_last_ok && (i64)h->sess_last.size() == len &&
                     memcmp(h->sess_last.data(), seq, (size_t)len * 4) == 0;
  if (seq) {
    if (!reuse) memcpy((char*)c + kSessTok, seq, (size_t)len * 4);
    op.off = reuse ? h->sess_last_off : h->tok_len;
    op.len = len;
    if (need_match) op.L = kMatchInline;
  }
  c->op = op;
  c->ntok = (seq && !reuse) ? len : 0;
  c->need_match = (seq && need_match) ? 1 : 0;
  c->stop = 0;
  const unsigned long long want = h->sess_next;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  c->seq = want;
  for (u64 spin = 1; r->seq != want; ++spin) {
    if ((spin & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(h->sess_stream);
      if (q == cudaErrorNotReady) continue;
      if (q != cudaSuccess) {
        h->sess_on = false;
        if (g_sess_owner == h) g_sess_owner = nullptr;
        throw Fail(E2_ERR_CUDA, std::string("session: ") + cudaGetErrorString(q));
      }
      if (r->seq == want) break;
      // the warp left on its idle timeout before it saw this command: its
      // hot state is in HBM (h->dev_hot); a fresh warp picks the command up
      h->sess_relaunch++;
      session_launch(h);
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  h->sess_next = want + 1;
  h->sess_ops++;
  if (seq && !reuse) {
    if (!transient) {
      h->sess_last.assign(seq, seq + len);
      h->sess_last_off = h->tok_len;
      h->sess_last_ok = true;
    }
    h->tok_len += len;
  }
  memcpy(&h->hot, (const void*)&r->hot, sizeof(Hot));
  memcpy(&h->api, (const void*)&r->api, sizeof(ApiOut));
  h->dev_hot = h->hot;
  h->dev_hot_valid = true;
  if (h->hot.err) {
    session_stop(h);
    check_hot_error(h);
  }
  return true;
}

void session_free(e2_handle* h) {
  try {
    session_stop(h);
  } catch (...) {
  }
  if (h->sess_res && getenv("E2_SESSION_DEBUG")) {
    const SessRes* r = sess_res(h);
    const double n = std::max<double>(1.0, (double)r->pad[3]);
    fprintf(stderr,
            "session: %lld ops, %lld launches (%lld relaunches), %lld stops, not taken %lld/%lld/%lld/%lld; per op us: "
            "in %.2f op %.2f out %.2f\n",
            (long long)h->sess_ops, (long long)h->sess_starts, (long long)h->sess_relaunch, (long long)h->sess_stops,
            (long long)h->sess_why[1], (long long)h->sess_why[2], (long long)h->sess_why[3], (long long)h->sess_why[4],
            r->pad[0] / n / 1e3, r->pad[1] / n / 1e3, r->pad[2] / n / 1e3);
  }
  if (h->sess_cmd) cudaFreeHost(h->sess_cmd);
  if (h->sess_res) cudaFreeHost(h->sess_res);
  if (h->sess_stream) cudaStreamDestroy(h->sess_stream);
  h->sess_cmd = h->sess_res = nullptr;
  h->sess_stream = 0;
}
#else
void session_stop(e2_handle*) {}
bool session_op(e2_handle*, OpDesc, const i32*, i64, bool, bool) { return false; }
void session_free(e2_handle*) {}
#endif

// One API op on one sequence (or none): append, match, run.
// `transient`: the op stores no reference to the sequence (decide, match,
// note_eviction: splits only cut existing edges), so its arena bytes are
// handed back afterwards and read-only calls do not grow device memory.
void run_api(e2_handle* h, OpDesc op, const i32* seq, i64 len, bool need_match, bool transient = false) {
  const i64 tok_mark = h->tok_len;
  struct Rollback {
    e2_handle* h;
    i64 mark;
    bool on;
    ~Rollback() {
      if (on) h->tok_len = mark;
    }
  } rb{h, tok_mark, transient};
  if (session_op(h, op, seq, len, need_match, transient)) return;
  reserve_for(h, 1, len);
  if (seq) {
    append_host_tokens(h, seq, len);
    op.off = h->tok_len - len;
    op.len = len;
    if (need_match) {
      reserve_batch(h, 1);
      op.L = kMatchInline;  // the serial kernel matches the sequence itself
    }
  }
  SerialArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = 1;
  a.op = op;
  a.out = h->d_api;
  a.hint = need_match ? h->b_path : nullptr;
  a.L = nullptr;
  a.hstride = h->hstride;
  push_hot(h);
  launch_serial(h, a);
  // one synchronisation for the mirrored hot state and the op's result
  char* p = pin_reserve(h, 0);
  d2h(p, h->d.hot_g, sizeof(Hot), h->stream);
  d2h(p + sizeof(Hot), h->d_api, sizeof(ApiOut), h->stream);
  ssync(h->stream);
  memcpy(&h->hot, p, sizeof(Hot));
  memcpy(&h->api, p + sizeof(Hot), sizeof(ApiOut));
  h->dev_hot = h->hot;
  h->dev_hot_valid = true;
  check_hot_error(h);
}

std::recursive_mutex g_lock;  // g_dev (constant memory) is shared by every handle

// guard: every entry point.  Entry points other than the per-call ops
// (guard_api) first end the running session, so their launches, copies and
// reads of the HBM hot state see the session's final state.
template <typename F>
int guard(e2_handle* h, F&& f, bool api = false) {
  std::lock_guard<std::recursive_mutex> lk(g_lock);
  try {
    if (g_sess_owner && (!api || g_sess_owner != h)) session_stop(g_sess_owner);
    f();
    return E2_OK;
  } catch (const Fail& e) {
    if (h) h->err = e.what();
    else g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (h) h->err = e.what();
    else g_err = e.what();
    return E2_ERR_ARG;
  }
}

// INT64_MIN marks an empty inflight slot (e2_state.cuh kNoInflight); the
// reference's std::map accepts it, this implementation rejects it loudly.
bool bad_id(e2_handle* h, int64_t id) {
  if (id == kNoInflight) {
    h->err = "request id INT64_MIN is reserved";
    return true;
  }
  return false;
}

bool bad_gpu(e2_handle* h, int32_t g) {
  if (g < 0 || g >= h->G) {
    h->err = "gpu id out of range";
    return true;
  }
  return false;
}

void copy_decision(e2_handle* h, e2_decision* out, e2_cost* costs, double* ratios) {
  if (out) *out = h->api.dec;
  if (costs)
    for (int i = 0; i < h->api.dec.n_costs; ++i) costs[i] = h->api.costs[i];
  if (ratios && h->api.dec.has_ratios)
    for (int g = 0; g < h->G; ++g) ratios[g] = h->api.ratios[g];
}

// ---- autoscale (global_scheduler.cpp:236-338), host-orchestrated --------------
// Out of the hot path: it only fires after note_admitted fills the
// queue statistics, which the trace driver never does.
struct HostTree {
  std::vector<NodeRec> hdr;
  std::vector<u64> cmask, lamask;
  std::vector<double> la;
  std::vector<i32> hits;
  std::vector<std::vector<u32>> kids;  // sorted by first token
  std::vector<i32> tok;
};

void pull_tree(e2_handle* h, HostTree& t) {
  const u64 n = h->hot.slots_used;
  const int G = h->G;
  t.hdr.resize(n);
  t.cmask.resize(n);
  t.lamask.resize(n);
  t.la.resize(n * G);
  t.hits.resize(n * G);
  std::vector<char> raw(n * h->d.rs);
  d2h(raw.data(), h->d.rec, raw.size(), h->stream);
  ssync(h->stream);
  for (u64 s = 0; s < n; ++s) {
    NodeRec* r = (NodeRec*)(raw.data() + s * h->d.rs);
    t.hdr[s] = *r;
    t.cmask[s] = r->cmask;
    t.lamask[s] = r->lamask;
    for (int g = 0; g < G; ++g) {
      t.la[s * G + g] = rla(r)[g];
      t.hits[s * G + g] = rhits(r, G)[g];
    }
  }
  t.tok.resize(h->tok_len);
  d2h(t.tok.data(), h->tok, h->tok_len * 4, h->stream);
  ssync(h->stream);
  t.kids.assign(n, {});
  for (u64 s = 1; s < n; ++s) {
    if (t.hdr[s].edge_len == 0) continue;
    t.kids[t.hdr[s].parent].push_back((u32)s);
  }
  for (auto& k : t.kids)
    std::sort(k.begin(), k.end(), [&](u32 a, u32 b) { return t.hdr[a].first_tok < t.hdr[b].first_tok; });
}

double host_load(e2_handle* h, int g, double now) {
  OpDesc op;
  memset(&op, 0, sizeof(op));
  op.kind = OP_GPU_LOAD;
  op.gpu = g;
  op.now = now;
  run_api(h, op, nullptr, 0, false);
  return h->api.v;
}

void run_simple(e2_handle* h, i32 kind, int gpu, i64 x, double now) {
  OpDesc op;
  memset(&op, 0, sizeof(op));
  op.kind = kind;
  op.gpu = gpu;
  op.x = x;
  op.now = now;
  run_api(h, op, nullptr, 0, false);
}

double host_prefill_time(const e2_time_model& m, i64 missed) {
  if (missed <= 0) return 0.0;
  volatile double a = m.prefill_per_token_ms * (double)missed;
  volatile double b = m.prefill_base_ms + a;
  return b;
}

// The subtree ops collect their nodes into vic_slot: size it from the host copy.
u64 subtree_size(const HostTree& t, u32 n) {
  u64 c = 0;
  std::vector<u32> st{n};
  while (!st.empty()) {
    const u32 x = st.back();
    st.pop_back();
    ++c;
    for (u32 y : t.kids[x]) st.push_back(y);
  }
  return c;
}
void reserve_victims(e2_handle* h, u64 need) {
  Dev& d = h->d;
  if (need <= d.vcap) return;
  const u64 cap = pow2_at_least(need);
  if (cap > 0xffffffffull) throw Fail(E2_ERR_ARG, "victim scratch exceeds 32-bit indices");
  dfree(d.vic_slot);
  dfree(d.vic_tok);
  d.vic_slot = talloc<u32>(cap);
  d.vic_tok = talloc<i64>(cap);
  d.vcap = (u32)cap;
}

void replicate_prefix(e2_handle* h, u32 root_child, int target, double now) {
  run_simple(h, OP_MARK_NODE, target, root_child, now);
  run_simple(h, OP_EXPIRE_ALL, 0, 0, now);  // windowed hits for all instances
  HostTree t;
  pull_tree(h, t);
  const int G = h->G;
  struct Kid {
    u32 node;
    double load;
  };
  std::vector<Kid> kids;
  for (u32 ch : t.kids[root_child]) {
    i64 toks = 0;
    std::vector<u32> st{ch};
    while (!st.empty()) {
      u32 x = st.back();
      st.pop_back();
      toks += t.hdr[x].edge_len;
      for (u32 y : t.kids[x]) st.push_back(y);
    }
    i64 hits = 0;
    for (int g = 0; g < G; ++g) hits += t.hits[(u64)ch * G + g];
    volatile double ld = (double)hits * host_prefill_time(h->model, toks);
    kids.push_back({ch, ld});
  }
  std::sort(kids.begin(), kids.end(), [&](const Kid& a, const Kid& b) {
    if (a.load != b.load) return a.load > b.load;
    return t.hdr[a.node].id < t.hdr[b.node].id;
  });
  double stay = 0, move = 0;
  std::vector<u32> moving;
  for (auto& k : kids) {
    if (move < stay) {
      moving.push_back(k.node);
      move += k.load;
    } else {
      stay += k.load;
    }
  }
  for (u32 n : moving) {
    u64 owners = 0;
    std::vector<u32> st{n};
    while (!st.empty()) {
      u32 x = st.back();
      st.pop_back();
      owners |= t.cmask[x];
      for (u32 y : t.kids[x]) st.push_back(y);
    }
    reserve_victims(h, subtree_size(t, n));
    run_simple(h, OP_MARK_SUBTREE, target, n, now);
    for (int g = 0; g < G; ++g)
      if (((owners >> g) & 1ull) && g != target) run_simple(h, OP_UNCACHE_SUBTREE, g, n, now);
  }
}

void check_autoscale(e2_handle* h, double now) {
  if (h->queue_stats.empty()) return;
  const double H = h->cfg.history_window_ms;
  const i64 cur = (i64)std::floor(now / H);
  for (auto it = h->queue_stats.begin(); it != h->queue_stats.end();) {
    auto& buckets = it->second;
    while (!buckets.empty() && buckets.begin()->first < cur - 1) buckets.erase(buckets.begin());
    if (buckets.empty()) {
      it = h->queue_stats.erase(it);
      continue;
    }
    bool fired = false;
    auto pi = buckets.find(cur - 1);
    auto ci = buckets.find(cur);
    if (pi != buckets.end() && ci != buckets.end() && pi->second.second > 0 && ci->second.second > 0) {
      const double pm = pi->second.first / (double)pi->second.second;
      const double cm = ci->second.first / (double)ci->second.second;
      if (pm > 0 && cm >= 2.0 * pm) {
        session_stop(h);  // host-orchestrated: a tree pull, subtree ops on the launch path
        HostTree t;
        pull_tree(h, t);
        u32 rc = kNil;
        for (u32 ch : t.kids[kRoot])
          if (t.hdr[ch].id == it->first) rc = ch;
        int src = -1;
        if (rc != kNil) {
          for (int s = 0; s < h->G; ++s)
            if (h->hot.redirect[s] >= 0 && ((t.cmask[rc] >> s) & 1ull)) {
              src = s;
              break;
            }
        }
        if (src >= 0) {
          int target = -1;
          double tl = 0;
          for (int g = 0; g < h->G; ++g) {
            if ((t.cmask[rc] >> g) & 1ull) continue;
            double l = host_load(h, g, now);
            if (target < 0 || l < tl) {
              target = g;
              tl = l;
            }
          }
          if (target >= 0) {
            replicate_prefix(h, rc, target, now);
            h->hot.stats[kStAutoscale]++;
            push_hot(h);
            fired = true;
          }
        }
      }
    }
    if (fired)
      it = h->queue_stats.erase(it);
    else
      ++it;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* e2_backend(void) {
#if E2_DEVICE_BUILD
  return "b200";
#else
  return "hostsim";
#endif
}

int e2_create(int32_t n_gpus, const e2_sched_cfg* cfg, const e2_time_model* model, const e2_policy* policy,
              e2_handle** out) {
  *out = nullptr;
  // ConfigError checks — global_scheduler.cpp:8-15, 27-37
  if (n_gpus < 1) {
    g_err = "cluster needs at least one GPU";
    return E2_ERR_CONFIG;
  }
  if (!(cfg->history_window_ms > 0)) {
    g_err = "history_window_ms must be > 0";
    return E2_ERR_CONFIG;
  }
  if (!(cfg->th_bal > 1.0)) {
    g_err = "th_bal must be > 1";
    return E2_ERR_CONFIG;
  }
  if (!(cfg->imbal_ratio > 0.0 && cfg->imbal_ratio <= 1.0)) {
    g_err = "imbal_ratio must be in (0,1]";
    return E2_ERR_CONFIG;
  }
  if (cfg->priority_groups < 1) {
    g_err = "priority_groups must be >= 1";
    return E2_ERR_CONFIG;
  }
  if (cfg->kv_capacity_tokens <= 0) {
    g_err = "kv_capacity_tokens must be > 0";
    return E2_ERR_CONFIG;
  }
  if (cfg->default_output_len < 0) {
    g_err = "default_output_len must be >= 0";
    return E2_ERR_CONFIG;
  }
  if (n_gpus > E2_MAX_GPUS) {
    g_err = "this implementation supports at most 64 instances";
    return E2_ERR_ARG;
  }
  e2_handle* h = new e2_handle();
  memset(&h->d, 0, sizeof(h->d));  // every device pointer null until allocated (teardown on failure)
  int rc = guard(nullptr, [&] {
    h->G = n_gpus;
    h->cfg = *cfg;
    h->model = *model;
    h->pol = *policy;
    memset(&h->hot, 0, sizeof(h->hot));
    memset(&h->acc, 0, sizeof(h->acc));
    for (int g = 0; g < kMaxG; ++g) h->hot.redirect[g] = -1;
    h->hot.next_id = 1;  // root holds id 0 (prefix_tree.cpp:9-12)
    h->hot.slots_used = 1;
    Cfg c;
    memset(&c, 0, sizeof(c));
    c.G = n_gpus;
    c.gtop = 1;
    while (c.gtop < std::min(n_gpus, 32)) c.gtop *= 2;
    c.mode = policy->mode == E2_MODE_ROUND_ROBIN ? 1 : 0;
    c.rebalance = policy->rebalance;
    c.autoscale = policy->autoscale;
    c.pd_balance = policy->pd_balance;
    c.H = cfg->history_window_ms;
    c.th_bal = cfg->th_bal;
    c.imbal = cfg->imbal_ratio;
    c.cap = cfg->kv_capacity_tokens;
    c.default_out = cfg->default_output_len;
    c.c0 = model->prefill_base_ms;
    c.c1 = model->prefill_per_token_ms;
    c.c2 = model->decode_per_token_ms;
    c.c3 = model->iteration_base_ms;
    zero_ptrs(h->d);
    h->d.cfg = c;
    h->d.rs = rec_stride(n_gpus);
    for (int g = 0; g < kMaxG; ++g) h->hot.ws_head_t[g] = h->hot.wc_head_t[g] = 1.0 / 0.0;
    {
      // node cache: as many 4-way sets as fit in ~150 KB of shared memory
      u32 ne = 1;
#if defined(E2_SMEM_NODECACHE)
      while ((u64)(ne * 2) * (h->d.rs + 12) <= 150u * 1024 && ne * 2 <= 1024) ne *= 2;
#else
      ne = kWays;  // no node cache: the tag arrays stay as a stub
#endif
      h->nsets = std::max<u32>(ne / kWays, 1);
      const u32 e = h->nsets * kWays;
      h->serial_smem = kScrBytes + ((3 * e * 4 + 15) / 16) * 16 + (size_t)e * h->d.rs;
    }
#if E2_DEVICE_BUILD
    CK(cudaFuncSetAttribute(k_serial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->serial_smem));
    CK(cudaFuncSetAttribute(k_session, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->serial_smem));
#if !defined(E2_NO_L1_PREF)
    // the serial kernel is one block per SM: the smallest shared-memory
    // configuration that fits it leaves the rest to L1 (A/B: C4 +4.5 %,
    // C2 +2.3 %, C5 +3.8 % together with the 512-level path scratch)
    CK(cudaFuncSetAttribute(k_serial, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_session, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
#endif
#endif
#if E2_DEVICE_BUILD
    {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, dev));
      const char* np = getenv("E2_NO_PIPE");
      h->no_pipe = np && np[0] == '1';
      const char* npf = getenv("E2_NO_PREFETCH");
      h->no_prefetch = npf && npf[0] == '1';
      const char* ntp = getenv("E2_NO_TOP");
      h->no_top = ntp && ntp[0] == '1';
      const char* nse = getenv("E2_NO_SESSION");
      h->no_session = nse && nse[0] == '1';
      const char* sid = getenv("E2_SESSION_IDLE_US");
      if (sid) h->sess_idle_ns = (u64)std::max(0.0, atof(sid) * 1000.0);
    }
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream_handle = h->stream;
    h->own_stream = true;
#endif
    h->d.hot_g = talloc<Hot>(1);
    h->d_api = talloc<ApiOut>(1);
    h->d_cnt = talloc<unsigned int>(4);
    h->d.xp_slot = talloc<u32>(kXPath + 1);
    h->d.xp_m = talloc<u32>(kXPath + 1);
    h->d.xp_cm = talloc<u64>(kXPath + 1);
    h->d.xp_la0 = talloc<u64>(kXPath + 1);
    h->d.xp_flag = talloc<u32>(kXPath + 1);
    h->d_bytes = talloc<unsigned long long>(2);
    reserve_nodes(h, 1024);
    reserve_window(h, 1024);
    reserve_plog(h);
    reserve_fifo(h, 64);
    reserve_inflight(h, 64);
    reserve_tokens(h, 1 << 16);
    reserve_requests(h, 1024);
    // root node: slot 0, id 0
    NodeRec root;
    memset(&root, 0, sizeof(root));
    root.parent = kNil;
    h2d(h->d.rec, &root, sizeof(root), h->stream);
    push_hot(h);
    ssync(h->stream);
  });
  if (rc != E2_OK) {
    if (g_err.empty()) g_err = h->err;
    e2_destroy(h);  // frees what was allocated before the failure, and the stream
    return rc;
  }
  *out = h;
  return E2_OK;
}

namespace {
void shadow_free(e2_handle* h);  // (sharded replay, below)
}

void e2_destroy(e2_handle* h) {
  if (!h) return;
  {
    std::lock_guard<std::recursive_mutex> lk(g_lock);
    session_free(h);
  }
  shadow_free(h);
  Dev& d = h->d;
  void* ptrs[] = {d.rec, d.ct, d.win, d.comp, d.plog, d.dir, d.pg_la, d.pg_id, d.pg_slot, d.free_pages, d.inf, d.fifo_req,
                  d.fifo_tail, d.req_tail, d.scr_slot, d.scr_val, d.scr_la, d.scr_id, d.vic_slot, d.vic_tok, d.hot_g,
                  d.xp_slot, d.xp_m, d.xp_cm, d.xp_la0, d.xp_flag,
                  h->tok, h->r_off, h->r_len, h->b_S, h->b_L, h->b_cand, h->b_leader, h->b_o, h->b_dslot, h->b_dm,
                  h->b_path, h->b_state, h->b_A, h->b_B, h->g_tk, h->g_tv, h->d_cnt, h->d_bytes, h->d_api,
                  h->st_ids, h->st_out, h->st_offs, h->st_arr, h->st_dec, h->st_cost, h->st_rat,
                  h->carry_ids, h->carry_out, h->carry_arr, h->cb_ids, h->cb_out, h->cb_arr, h->top_img};
  for (void* p : ptrs) dfree(p);
#if E2_DEVICE_BUILD
  for (auto& e : h->ev) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  if (h->own_stream) cudaStreamDestroy(h->own_stream_handle);
  if (h->pin) cudaFreeHost(h->pin);
#else
  free(h->pin);
#endif
  delete h;
}

const char* e2_last_error(const e2_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }

int e2_reset(e2_handle* h) {
  return guard(h, [&] {
    Dev& d = h->d;
    const u64 used = h->hot.slots_used;
    dset(d.rec, 0, used * d.rs, h->stream);
    {
      CtEntry e;
      e.key = kEmptyKey;
      e.val = 0;
      e.pad = 0;
      std::vector<CtEntry> empty_ct(d.ct_mask + 1, e);
      h2d(d.ct, empty_ct.data(), empty_ct.size() * sizeof(CtEntry), h->stream);
      InfRec z;
      memset(&z, 0, sizeof(z));
      z.key = kNoInflight;
      std::vector<InfRec> empty_inf(d.inf_mask + 1, z);
      h2d(d.inf, empty_inf.data(), empty_inf.size() * sizeof(InfRec), h->stream);
      ssync(h->stream);
    }
    memset(&h->hot, 0, sizeof(h->hot));
    for (int g = 0; g < kMaxG; ++g) {
      h->hot.redirect[g] = -1;
      h->hot.ws_head_t[g] = h->hot.wc_head_t[g] = 1.0 / 0.0;
    }
    h->hot.next_id = 1;
    h->hot.slots_used = 1;
    NodeRec root;
    memset(&root, 0, sizeof(root));
    root.parent = kNil;
    h2d(d.rec, &root, sizeof(root), h->stream);
    push_hot(h);
    ssync(h->stream);
    h->tok_len = 0;
    h->queue_stats.clear();
    h->prev_total = 0;
    h->carry_n = 0;
    h->next_tick = 0;
  });
}

int e2_replay_set_continue(e2_handle* h, int32_t on) {
  return guard(h, [&] { h->cont = on != 0; });
}

int e2_set_stream(e2_handle* h, void* stream) {
  return guard(h, [&] {
#if E2_DEVICE_BUILD
    ssync(h->stream);
    h->stream = stream ? (Stream)stream : h->own_stream_handle;
#else
    (void)stream;
#endif
  });
}

int e2_schedule(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int64_t request_id, double arrival_ms,
                double now, e2_decision* out, e2_cost* costs, double* ratios) {
  if (bad_id(h, request_id)) return E2_ERR_ARG;
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_SCHEDULE;
    op.id = request_id;
    op.arr = arrival_ms;
    op.now = now;
    static const i32 dummy = 0;
    run_api(h, op, prompt_len ? prompt : &dummy, prompt_len, true);
    copy_decision(h, out, costs, ratios);
    if (h->pol.mode == E2_MODE_PREFIX_AWARE && h->pol.autoscale) check_autoscale(h, now);
  }, true);
}

int e2_decide(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int64_t request_id, double now,
              e2_decision* out, e2_cost* costs, double* ratios) {
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_DECIDE;
    op.id = request_id;
    op.now = now;
    static const i32 dummy = 0;
    run_api(h, op, prompt_len ? prompt : &dummy, prompt_len, true, true);
    copy_decision(h, out, costs, ratios);
  }, true);
}

int e2_note_admitted(e2_handle* h, int64_t request_id, double now) {
  if (bad_id(h, request_id)) return E2_ERR_ARG;
  return guard(h, [&] {
    if (h->pol.mode != E2_MODE_PREFIX_AWARE) return;
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_INFLIGHT_GET;
    op.id = request_id;
    run_api(h, op, nullptr, 0, false);
    if (!h->api.i0) return;
    const i64 bucket = (i64)std::floor(now / h->cfg.history_window_ms);
    auto& cell = h->queue_stats[h->api.u0][bucket];
    cell.first += now - h->api.v;
    cell.second += 1;
  }, true);
}

int e2_note_prefill_cached(e2_handle* h, const int32_t* prompt, int64_t prompt_len, int32_t gpu, double now) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    if (h->pol.mode != E2_MODE_PREFIX_AWARE || prompt_len == 0) return;
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_PREFILL;
    op.gpu = gpu;
    op.now = now;
    run_api(h, op, prompt, prompt_len, true);
  }, true);
}

int e2_note_eviction(e2_handle* h, const int32_t* seq, int64_t seq_len, int64_t tail_len, int32_t gpu, double now) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    if (h->pol.mode != E2_MODE_PREFIX_AWARE || seq_len == 0 || tail_len <= 0) return;
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_EVICT;
    op.gpu = gpu;
    op.x = tail_len;
    op.now = now;
    run_api(h, op, seq, seq_len, true, true);
  }, true);
}

int e2_note_finished(e2_handle* h, int64_t request_id, double now, int64_t output_len) {
  if (bad_id(h, request_id)) return E2_ERR_ARG;
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_FINISHED;
    op.id = request_id;
    op.now = now;
    op.x = output_len;
    run_api(h, op, nullptr, 0, false);
  }, true);
}

int e2_decode_ratio(e2_handle* h, int32_t gpu, double* out) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    pull_hot(h);
    const i64 ip = h->hot.inflight_prompt[gpu];
    *out = ip <= 0 ? 0.0 : (double)h->hot.inflight_cached[gpu] / (double)ip;
  }, true);
}

int e2_gpu_load_ms(e2_handle* h, int32_t gpu, double now, double* out) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] { *out = host_load(h, gpu, now); }, true);
}

int e2_prune_dead_nodes(e2_handle* h, double now, int64_t* removed) {
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_PRUNE_DEAD;
    op.now = now;
    run_api(h, op, nullptr, 0, false);
    *removed = h->api.i0;
  });
}

int e2_cached_tokens(e2_handle* h, int32_t gpu, int64_t* out) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    pull_hot(h);
    *out = h->hot.cached_tokens[gpu];
  }, true);
}

int e2_node_count(e2_handle* h, int64_t* out) {
  return guard(h, [&] {
    pull_hot(h);
    *out = h->hot.node_count;
  }, true);
}

int e2_redirects(e2_handle* h, int32_t* out) {
  return guard(h, [&] {
    pull_hot(h);
    for (int g = 0; g < h->G; ++g) out[g] = h->hot.redirect[g];
  }, true);
}

int e2_get_stats(e2_handle* h, e2_stats* out) {
  return guard(h, [&] {
    pull_hot(h);
    out->exploit = h->hot.stats[kStExploit];
    out->explore = h->hot.stats[kStExplore];
    out->decode_pressure = h->hot.stats[kStPressure];
    out->round_robin = h->hot.stats[kStRoundRobin];
    out->redirected = h->hot.stats[kStRedirected];
    out->rebalance_installs = h->hot.stats[kStInstalls];
    out->autoscale_events = h->hot.stats[kStAutoscale];
    out->tree_reads = h->hot.stats[kStTreeReads];
  }, true);
}

int e2_load_cost(e2_handle* h, int32_t gpu, int64_t missed_tokens, double now, e2_cost* out) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_LOAD_COST;
    op.gpu = gpu;
    op.x = missed_tokens;
    op.now = now;
    run_api(h, op, nullptr, 0, false);
    *out = h->api.costs[0];
  }, true);
}

int e2_match(e2_handle* h, const int32_t* seq, int64_t len, int64_t* matched_len, int64_t* cached_len,
             int64_t* per_gpu) {
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_MATCH;
    static const i32 dummy = 0;
    run_api(h, op, len ? seq : &dummy, len, true, true);
    if (matched_len) *matched_len = h->api.i0;
    if (cached_len) *cached_len = h->api.i1;
    if (per_gpu)
      for (int g = 0; g < h->G; ++g) per_gpu[g] = h->api.ext[g];
  }, true);
}

int e2_window_sizes(e2_handle* h, int32_t gpu, double now, int64_t* n_scheduled, int64_t* n_completed,
                    int64_t* inflight_cached, int64_t* inflight_prompt) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_WINDOW;
    op.gpu = gpu;
    op.now = now;
    run_api(h, op, nullptr, 0, false);
    if (n_scheduled) *n_scheduled = h->api.i0;
    if (n_completed) *n_completed = h->api.i1;
    if (inflight_cached) *inflight_cached = h->api.i2;
    if (inflight_prompt) *inflight_prompt = h->api.i3;
  }, true);
}

// ---- export / dump (host-side; off the hot path) ---------------------------
namespace {
void expire_all(e2_handle* h, double now) { run_simple(h, OP_EXPIRE_ALL, 0, 0, now); }

// Ring positions [head, tail) of instance g's window ring (T = WinEnt or
// CompEnt), oldest first.
extern "C++" template <typename T>
std::vector<T> pull_ring(e2_handle* h, const T* ring, int g, u64 head, u64 tail) {
  std::vector<T> out(tail - head);
  const u64 cap = h->d.wcap;
  for (u64 i = head; i < tail;) {
    const u64 at = i & (cap - 1);
    const u64 run = std::min<u64>(tail - i, cap - at);
    d2h(out.data() + (i - head), ring + (u64)g * cap + at, run * sizeof(T), h->stream);
    i += run;
  }
  ssync(h->stream);
  return out;
}

void dfs_order(const HostTree& t, std::vector<std::pair<u32, int>>& order) {
  std::vector<std::pair<u32, int>> st{{kRoot, 0}};
  while (!st.empty()) {
    auto [x, dep] = st.back();
    st.pop_back();
    order.push_back({x, dep});
    const auto& k = t.kids[x];
    for (size_t i = k.size(); i-- > 0;) st.push_back({k[i], dep + 1});
  }
}
}  // namespace

int e2_export_size(e2_handle* h, int64_t* n_nodes, int64_t* n_tokens) {
  return guard(h, [&] {
    HostTree t;
    pull_tree(h, t);
    std::vector<std::pair<u32, int>> order;
    dfs_order(t, order);
    i64 nt = 0;
    for (auto& [x, dep] : order) nt += t.hdr[x].edge_len;
    *n_nodes = (i64)order.size();
    *n_tokens = nt;
  });
}

int e2_export(e2_handle* h, double now, e2_node* nodes, int32_t* tokens, double* last_access, int64_t* hits) {
  return guard(h, [&] {
    expire_all(h, now);
    HostTree t;
    pull_tree(h, t);
    std::vector<std::pair<u32, int>> order;
    dfs_order(t, order);
    const int G = h->G;
    i64 off = 0;
    for (size_t i = 0; i < order.size(); ++i) {
      const u32 x = order[i].first;
      const NodeRec& hd = t.hdr[x];
      if (nodes) {
        nodes[i].id = hd.id;
        nodes[i].parent_id = x == kRoot ? hd.id : t.hdr[hd.parent].id;
        nodes[i].edge_off = off;
        nodes[i].edge_len = hd.edge_len;
        nodes[i].caching_mask = t.cmask[x];
        nodes[i].last_access_mask = t.lamask[x];
        nodes[i].pin_count = 0;
      }
      if (tokens && hd.edge_len) memcpy(tokens + off, t.tok.data() + hd.edge_off, (size_t)hd.edge_len * 4);
      off += hd.edge_len;
      for (int g = 0; g < G; ++g) {
        if (last_access) last_access[i * G + g] = ((t.lamask[x] >> g) & 1ull) ? t.la[(u64)x * G + g] : 0.0;
        if (hits) hits[i * G + g] = t.hits[(u64)x * G + g];
      }
    }
  });
}

// snapshot(now)'s windows (global_scheduler.cpp:384-389): after pruning at
// now, the scheduled and completed entries, oldest first.
int e2_window_entries(e2_handle* h, int32_t gpu, double now, double* sched_t, int64_t* sched_missed,
                      int64_t* sched_est, double* comp_t, int64_t* comp_out) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  return guard(h, [&] {
    OpDesc op;
    memset(&op, 0, sizeof(op));
    op.kind = OP_WINDOW;  // prunes gpu's window at now
    op.gpu = gpu;
    op.now = now;
    run_api(h, op, nullptr, 0, false);
    const auto ws = pull_ring(h, h->d.win, gpu, h->hot.ws_head[gpu], h->hot.ws_tail[gpu]);
    for (size_t i = 0; i < ws.size(); ++i) {
      if (sched_t) sched_t[i] = ws[i].t;
      if (sched_missed) sched_missed[i] = ws[i].missed;
      if (sched_est) sched_est[i] = ws[i].est;
    }
    const auto wc = pull_ring(h, h->d.comp, gpu, h->hot.wc_head[gpu], h->hot.wc_tail[gpu]);
    for (size_t i = 0; i < wc.size(); ++i) {
      if (comp_t) comp_t[i] = wc[i].t;
      if (comp_out) comp_out[i] = wc[i].out;
    }
  });
}

// NodeSnapshot::hits (prefix_tree.cpp:436-448), in-window stamps only.  The
// counter identity (DESIGN §3 fact 3) says node n's hits on g are the
// in-window scheduled entries of g whose prompt passes through n; that
// prompt's path is the parent chain of the entry's tail slot (splits insert
// above it, the slot keeps the suffix).  So each entry's time is stamped on
// its chain, entries in window order; the per-node counts must equal the
// device's counters (checked).
int e2_export_hit_stamps(e2_handle* h, double now, double* stamps, int64_t cap, int64_t* n_stamps) {
  return guard(h, [&] {
    expire_all(h, now);
    HostTree t;
    pull_tree(h, t);
    const int G = h->G;
    const u64 n = t.hdr.size();
    std::vector<std::vector<double>> st(n * (u64)G);
    for (int g = 0; g < G; ++g) {
      const auto ws = pull_ring(h, h->d.win, g, h->hot.ws_head[g], h->hot.ws_tail[g]);
      for (const WinEnt& e : ws)
        for (u32 x = e.slot; x != kRoot && x != kNil && x < n; x = t.hdr[x].parent) st[(u64)x * G + g].push_back(e.t);
    }
    std::vector<std::pair<u32, int>> order;
    dfs_order(t, order);
    i64 k = 0;
    for (auto& [x, dep] : order)
      for (int g = 0; g < G; ++g) {
        const auto& v = st[(u64)x * G + g];
        if ((i64)v.size() != (i64)t.hits[(u64)x * G + g])
          throw Fail(E2_ERR_SIM, "hit stamps disagree with the hit counters");
        for (double s : v) {
          if (stamps && k < cap) stamps[k] = s;
          k++;
        }
      }
    if (n_stamps) *n_stamps = k;
    if (stamps && k > cap) throw Fail(E2_ERR_ARG, "stamps buffer too small");
  });
}

int e2_debug_dump(e2_handle* h, double now, char* buf, size_t cap, size_t* needed) {
  return guard(h, [&] {
    expire_all(h, now);
    HostTree t;
    pull_tree(h, t);
    std::vector<std::pair<u32, int>> order;
    dfs_order(t, order);
    std::string s;
    const int G = h->G;
    char tmp[64];
    for (auto& [x, dep] : order) {
      for (int i = 0; i < dep; ++i) s += "  ";
      snprintf(tmp, sizeof(tmp), "d%d len=%u gpus=[", dep, t.hdr[x].edge_len);
      s += tmp;
      bool first = true;
      for (int g = 0; g < G; ++g)
        if ((t.cmask[x] >> g) & 1ull) {
          if (!first) s += ",";
          s += std::to_string(g);
          first = false;
        }
      s += "] hits=[";
      first = true;
      for (int g = 0; g < G; ++g) {
        i32 c = t.hits[(u64)x * G + g];
        if (c == 0) continue;
        if (!first) s += ",";
        s += std::to_string(g) + ":" + std::to_string(c);
        first = false;
      }
      s += "]\n";
    }
    if (needed) *needed = s.size();
    if (buf && cap > 0) {
      size_t k = std::min(cap - 1, s.size());
      memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
  });
}

// ---- batched replay ---------------------------------------------------------
// One replay is begin / (next, match, commit)* / end.  e2_replay runs the
// steps back to back; the sharded replay (e2_shard_*) runs the same steps
// with K1 split across ranks and rank 0's state shipped as a delta.
namespace {
void replay_begin(e2_handle* h, const int32_t* tokens, const int64_t* offsets, const int64_t* ids,
                  const double* arrivals, const int64_t* output_lens, int64_t n, const e2_driver_cfg* drv,
                  e2_decision* out, e2_cost* costs, double* ratios, bool device_ptrs) {
  if (!h->queue_stats.empty() && h->pol.autoscale && h->pol.mode == E2_MODE_PREFIX_AWARE)
    throw Fail(E2_ERR_ARG, "replay with pending autoscale queue statistics is not supported");
  ReplaySession& S = h->rs;
  S = ReplaySession();
  S.n = n;
  S.device_ptrs = device_ptrs;
  S.out = out;
  S.costs = costs;
  S.ratios = ratios;
  if (n <= 0) {
    S.active = true;
    return;
  }
  const int G = h->G;
  i64 off0 = 0, offn = 0;
  if (device_ptrs) {
    d2h(&off0, offsets, 8, h->stream);
    d2h(&offn, offsets + n, 8, h->stream);
    ssync(h->stream);
  } else {
    off0 = offsets[0];
    offn = offsets[n];
    for (i64 i = 0; i < n; ++i)
      if (ids[i] == kNoInflight) throw Fail(E2_ERR_ARG, "request id INT64_MIN is reserved");
  }
  const i64 ntok = offn - off0;
  // streamed continuation: the previous chunk's last finish_lag requests
  // go in front (their note_finished calls fall in this chunk)
  const bool cont = h->cont && h->prev_total > 0;
  if (cont && drv->eviction == E2_EVICT_FIFO_TAIL)
    throw Fail(E2_ERR_ARG, "streamed replays support the mirror-LRU and no-eviction drivers only");
  const i64 C = cont ? std::min<i64>(h->carry_n, std::max<i64>(drv->finish_lag, 0)) : 0;
  S.carried = C;
  reserve_for(h, n, ntok);
  reserve_requests(h, C + n);
  // token arena: append the trace
  const i64 base_tok = h->tok_len;
  const i64 pad = (4 - (base_tok & 3)) & 3;  // 16-byte align the trace start
  reserve_tokens(h, base_tok + pad + ntok);
  const i64 tstart = base_tok + pad;
  if (device_ptrs)
    d2d(h->tok + tstart, tokens + off0, (size_t)ntok * 4, h->stream);
  else
    h2d(h->tok + tstart, tokens + off0, (size_t)ntok * 4, h->stream);
  h->tok_len = tstart + ntok;
  // per-request arrays resident on the device
  i64 *d_ids = nullptr, *d_out = nullptr, *d_offs = nullptr;
  double* d_arr = nullptr;
  if (device_ptrs) {
    d_ids = (i64*)ids;
    d_arr = (double*)arrivals;
    d_out = (i64*)output_lens;
    d_offs = (i64*)offsets;
    S.d_dec = out;
    S.d_cost = costs;
    S.d_rat = ratios;
  } else {
    if (n > h->st_cap) {
      for (void* p : {(void*)h->st_ids, (void*)h->st_out, (void*)h->st_offs, (void*)h->st_arr, (void*)h->st_dec}) dfree(p);
      h->st_ids = talloc<i64>(n);
      h->st_arr = talloc<double>(n);
      h->st_out = talloc<i64>(n);
      h->st_offs = talloc<i64>(n + 1);
      h->st_dec = talloc<e2_decision>(n);
      h->st_cap = n;
    }
    if (costs && n * (G + 1) > h->st_cost_cap) {
      dfree(h->st_cost);
      h->st_cost = talloc<e2_cost>((size_t)n * (G + 1));
      h->st_cost_cap = n * (G + 1);
    }
    if (ratios && n * G > h->st_rat_cap) {
      dfree(h->st_rat);
      h->st_rat = talloc<double>((size_t)n * G);
      h->st_rat_cap = n * G;
    }
    d_ids = h->st_ids;
    d_arr = h->st_arr;
    d_out = h->st_out;
    d_offs = h->st_offs;
    S.d_dec = h->st_dec;
    S.d_cost = costs ? h->st_cost : nullptr;
    S.d_rat = ratios ? h->st_rat : nullptr;
    h2d(d_ids, ids, n * 8, h->stream);
    h2d(d_arr, arrivals, n * 8, h->stream);
    h2d(d_out, output_lens, n * 8, h->stream);
    h2d(d_offs, offsets, (n + 1) * 8, h->stream);
  }
#if E2_DEVICE_BUILD
  {
    Timed t(h, E2_K_OTHER);
    h->acc.launches[E2_K_OTHER]++;
    k_arena_index<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(n, tstart, d_offs, h->r_off, h->r_len, C);
    CK(cudaGetLastError());
  }
#else
  for (i64 i = 0; i < n; ++i) {
    h->r_off[C + i] = tstart + d_offs[i] - d_offs[0];
    h->r_len[C + i] = d_offs[i + 1] - d_offs[i];
  }
#endif
  if (h->cont) {
    // combined [carry | chunk] ids, arrivals and output lengths
    const i64 need = C + n;
    if (need > h->cb_cap) {
      dfree(h->cb_ids);
      dfree(h->cb_arr);
      dfree(h->cb_out);
      h->cb_cap = need + need / 4;
      h->cb_ids = talloc<i64>(h->cb_cap);
      h->cb_arr = talloc<double>(h->cb_cap);
      h->cb_out = talloc<i64>(h->cb_cap);
    }
    if (C) {
      d2d(h->cb_ids, h->carry_ids, C * 8, h->stream);
      d2d(h->cb_arr, h->carry_arr, C * 8, h->stream);
      d2d(h->cb_out, h->carry_out, C * 8, h->stream);
      dset(h->r_off, 0, C * 8, h->stream);  // carried requests are never replayed again
      dset(h->r_len, 0, C * 8, h->stream);
    }
    d2d(h->cb_ids + C, d_ids, n * 8, h->stream);
    d2d(h->cb_arr + C, d_arr, n * 8, h->stream);
    d2d(h->cb_out + C, d_out, n * 8, h->stream);
    d_ids = h->cb_ids;
    d_arr = h->cb_arr;
    d_out = h->cb_out;
  }
  // prune ticks: the simulator's cadence on the driver clock
  if (drv->prune_interval_ms > 0) {
    std::vector<double> arr_h((size_t)n);
    if (device_ptrs) {
      d2h(arr_h.data(), arrivals, (size_t)n * 8, h->stream);
      ssync(h->stream);
    } else {
      memcpy(arr_h.data(), arrivals, (size_t)n * 8);
    }
    double now = cont ? h->hot.drv_now : 0.0;
    double t = cont ? h->next_tick : drv->prune_interval_ms;
    for (i64 i = 0; i < n; ++i) {
      now = std::max(now, arr_h[(size_t)i]);
      while (t <= now) {
        S.ticks.push_back({C + i, t});
        t += drv->prune_interval_ms;
      }
    }
    h->next_tick = t;
  }
  // driver state (a streamed continuation keeps the driver clock)
  if (!cont) {
    h->hot.drv_now = 0;
    for (int g = 0; g < G; ++g) h->hot.fifo_head[g] = h->hot.fifo_tail[g] = 0;
  }
  push_hot(h);
  S.B = drv->batch > 0 ? drv->batch : 16384;
  reserve_batch(h, std::min<i64>(S.B, n));
  if (C + n > h->req_cap) {
    dfree(h->d.req_tail);
    h->d.req_tail = talloc<u32>(C + n);
    h->req_cap = C + n;
  }
  SerialArgs& a = S.a;
  memset(&a, 0, sizeof(a));
  a.kind = 0;
  a.eviction = drv->eviction;
  a.prefill = drv->prefill_cached;
  a.off = h->r_off;
  a.len = h->r_len;
  a.ids = d_ids;
  a.arr = d_arr;
  a.outl = d_out;
  a.L = h->b_L;
  a.S = h->b_S;
  a.lead = h->b_leader;
  a.hint = h->b_path;
  // the kernels index every per-request array by the combined index C + i
  a.dec = S.d_dec ? S.d_dec - C : nullptr;
  a.costs = S.d_cost ? S.d_cost - C * (G + 1) : nullptr;
  a.ratios = S.d_rat ? S.d_rat - C * G : nullptr;
  a.trunk = drv->trunk_len;
  a.hw = drv->high_water;
  a.lag = drv->finish_lag;
  // Batch sizes ramp up geometrically from kFirstBatch: a batch is matched
  // against the tree at its start, so early batches (a cold tree) would
  // leave most requests without K1 path hints.
  S.cur_b = std::min<i64>(S.B, n <= 4 * kFirstBatch ? kShortFirstBatch : kFirstBatch);
  S.next_b0 = C;
  S.n = C + n;  // batches run over the combined index range [C, C + n)
  S.done = C;
  S.active = true;
}

// The next batch [cb0, cb0+cnb); false when the replay is complete or stopped.
bool replay_next(e2_handle* h) {
  ReplaySession& S = h->rs;
  if (!S.active) throw Fail(E2_ERR_ARG, "no replay in progress");
  if (S.stopped || S.next_b0 >= S.n) {
    S.cnb = 0;
    return false;
  }
  // prune ticks due before this batch's first request (prune_dead_nodes at
  // the tick time; a batch never spans a tick, so K1 matches the pruned tree)
  while (S.tick_pos < S.ticks.size() && S.ticks[S.tick_pos].first <= S.next_b0) {
    run_simple(h, OP_PRUNE_DEAD, 0, 0, S.ticks[S.tick_pos].second);
    S.tick_pos++;
  }
  S.cb0 = S.next_b0;
  S.cnb = std::min<i64>(S.cur_b, S.n - S.next_b0);
  if (S.tick_pos < S.ticks.size()) S.cnb = std::min<i64>(S.cnb, S.ticks[S.tick_pos].first - S.next_b0);
  S.next_b0 += S.cnb;
  S.cur_b = std::min<i64>(S.B, S.cur_b * 2);
  reserve_batch(h, S.cnb);
  return true;
}

// The serial decide/commit pass over the current batch (K1 + leader rounds done).
void replay_commit(e2_handle* h) {
  ReplaySession& S = h->rs;
  SerialArgs& a = S.a;
  a.L = h->b_L;
  a.S = h->b_S;
  a.lead = h->b_leader;
  a.hint = h->b_path;  // the hint stride may have grown
  a.hstride = h->hstride;
  a.base = S.cb0;
  a.n = S.cnb;
  launch_serial(h, a);
  pull_hot(h);
  S.done = S.cb0 + h->hot.done;
  if (h->hot.err) {
    try {
      check_hot_error(h);
    } catch (const Fail& e) {
      S.fail = e.what();
      S.fail_code = e.code;
    }
    S.stopped = true;
  }
}

void replay_after_batch(e2_handle* h) {
  if (!h->rs.stopped) reserve_plog(h);
}

void replay_end(e2_handle* h, int64_t* n_done) {
  ReplaySession& S = h->rs;
  if (!S.active) throw Fail(E2_ERR_ARG, "no replay in progress");
  S.active = false;
  prof_flush(h);
  const i64 C = S.carried;
  const i64 done = S.done - C;  // requests of this call decided
  if (h->cont && S.n > 0) {
    // keep the last finish_lag requests of [carry | chunk] for the next chunk
    const i64 upto = S.done;  // combined index one past the last decided request
    const i64 keep = std::min<i64>(upto, std::max<i64>(S.a.lag, 0));
    if (keep > h->carry_cap) {
      dfree(h->carry_ids);
      dfree(h->carry_arr);
      dfree(h->carry_out);
      h->carry_cap = keep + 16;
      h->carry_ids = talloc<i64>(h->carry_cap);
      h->carry_arr = talloc<double>(h->carry_cap);
      h->carry_out = talloc<i64>(h->carry_cap);
    }
    if (keep) {
      d2d(h->carry_ids, S.a.ids + (upto - keep), keep * 8, h->stream);
      d2d(h->carry_arr, S.a.arr + (upto - keep), keep * 8, h->stream);
      d2d(h->carry_out, S.a.outl + (upto - keep), keep * 8, h->stream);
      ssync(h->stream);
    }
    h->carry_n = keep;
  }
  h->prev_total = h->cont ? h->prev_total + std::max<i64>(done, 0) : 0;
  if (!S.device_ptrs && done > 0) {
    const int G = h->G;
    d2h(S.out, S.d_dec, (size_t)done * sizeof(e2_decision), h->stream);
    if (S.costs) d2h(S.costs, S.d_cost, (size_t)done * (G + 1) * sizeof(e2_cost), h->stream);
    if (S.ratios) d2h(S.ratios, S.d_rat, (size_t)done * G * 8, h->stream);
    ssync(h->stream);
  }
  if (n_done) *n_done = done;
  if (S.fail_code) throw Fail(S.fail_code, S.fail + " (request index " + std::to_string(done) + ")");
}

int replay_impl(e2_handle* h, const int32_t* tokens, const int64_t* offsets, const int64_t* ids,
                const double* arrivals, const int64_t* output_lens, int64_t n, const e2_driver_cfg* drv,
                e2_decision* out, e2_cost* costs, double* ratios, int64_t* n_done, bool device_ptrs) {
  if (n_done) *n_done = 0;
  return guard(h, [&] {
    if (n <= 0) return;
    replay_begin(h, tokens, offsets, ids, arrivals, output_lens, n, drv, out, costs, ratios, device_ptrs);
    try {
      while (replay_next(h)) {
        launch_match(h, h->rs.cb0, h->rs.cnb);
        replay_commit(h);
        replay_after_batch(h);
      }
    } catch (...) {
      h->rs.active = false;
      throw;
    }
    replay_end(h, n_done);
  });
}

// ---- sharded replay: regions, delta export/apply ---------------------------
RegionTab state_regions(e2_handle* h) {
  Dev& d = h->d;
  const u64 G = (u64)h->G;
  RegionTab t;
  memset(&t, 0, sizeof(t));
  auto add = [&](void* p, u64 bytes) {
    t.cur[t.n] = (u32*)p;
    t.words[t.n] = p ? bytes / 4 : 0;
    t.live_words[t.n] = t.words[t.n];
    t.n++;
  };
  add(d.rec, (u64)d.node_cap * d.rs);
  add(d.ct, (d.ct_mask + 1) * sizeof(CtEntry));
  add(d.win, d.wcap * G * sizeof(WinEnt));
  add(d.comp, d.wcap * G * sizeof(CompEnt));
  add(d.plog, d.pcap * G * 4);
  add(d.dir, (u64)d.dcap * G * sizeof(DirEntry));
  add(d.pg_la, (u64)d.page_cap * kPage * 8);
  add(d.pg_id, (u64)d.page_cap * kPage * 8);
  add(d.pg_slot, (u64)d.page_cap * kPage * 4);
  add(d.free_pages, (u64)d.page_cap * 4);
  add(d.inf, (d.inf_mask + 1) * sizeof(InfRec));
  add(d.fifo_req, d.fcap * G * 8);
  add(d.fifo_tail, d.fcap * G * 8);
  add(d.req_tail, (u64)h->req_cap * 4);
  // only the used part of the node pool can have changed
  t.live_words[0] = std::min<u64>(t.words[0], (u64)h->hot.slots_used * d.rs / 4);
  return t;
}

// (Re)take rank 0's shadow of every region whose allocation changed since
// the last snapshot (all of them on the first call).
void shadow_sync(e2_handle* h) {
  ShardState& sh = h->sh;
  RegionTab t = state_regions(h);
  if ((int)sh.sh.size() != t.n) {
    sh.sh.assign(t.n, nullptr);
    sh.sh_words.assign(t.n, 0);
    sh.sh_src.assign(t.n, nullptr);
  }
  for (int r = 0; r < t.n; ++r) {
    if (sh.sh_src[r] == t.cur[r] && sh.sh_words[r] == t.words[r]) continue;
    dfree(sh.sh[r]);
    sh.sh[r] = talloc<u32>(std::max<u64>(t.words[r], 1));
    if (t.words[r]) d2d(sh.sh[r], t.cur[r], t.words[r] * 4, h->stream);
    sh.sh_words[r] = t.words[r];
    sh.sh_src[r] = t.cur[r];
  }
  ssync(h->stream);
}

void shadow_free(e2_handle* h) {
  ShardState& sh = h->sh;
  for (u32* p : sh.sh) dfree(p);
  sh.sh.clear();
  sh.sh_words.clear();
  sh.sh_src.clear();
  dfree(sh.dl_idx);
  dfree(sh.dl_pay);
  dfree(sh.dl_count);
  sh.dl_idx = nullptr;
  sh.dl_pay = nullptr;
  sh.dl_count = nullptr;
  sh.dl_cap = 0;
}

// Apply n chunks (idx/payload) to the regions of `t` (cur pointers).
void delta_apply(e2_handle* h, const RegionTab& t, u64 n, const u64* idx, const uint4* pay) {
  if (!n) return;
#if E2_DEVICE_BUILD
  const u64 q = n * 4;
  const unsigned grid = (unsigned)std::min<u64>((q + 255) / 256, (u64)h->n_sm * 8);
  k_delta_apply<<<grid, 256, 0, h->stream>>>(t, n, idx, pay);
  CK(cudaGetLastError());
#else
  (void)h;
  for (u64 j = 0; j < n; ++j) {
    const int r = (int)(idx[j] >> 48);
    const u64 w0 = (idx[j] & ((1ull << 48) - 1)) * kChunkWords;
    const u32* src = (const u32*)&pay[j * 4];
    for (u64 k = 0; k < kChunkWords && w0 + k < t.words[r]; ++k) t.cur[r][w0 + k] = src[k];
  }
#endif
}

// Rank 0, after a committed batch: diff the regions against the shadow into
// dl_idx/dl_pay, fill the header, apply the chunks to the shadow.
void delta_export(e2_handle* h) {
  ShardState& sh = h->sh;
  RegionTab t = state_regions(h);
  if ((int)sh.sh.size() != t.n) throw Fail(E2_ERR_ARG, "shard: shadow not initialised");
  u64 total = 0;
  for (int r = 0; r < t.n; ++r) {
    if (sh.sh_src[r] != t.cur[r] || sh.sh_words[r] != t.words[r])
      throw Fail(E2_ERR_ARG, "shard: a region moved inside a batch");
    t.sh[r] = sh.sh[r];
    t.chunk0[r] = total;
    total += (t.live_words[r] + kChunkWords - 1) / kChunkWords;
  }
  t.chunk0[t.n] = total;
  u64 n = 0;
#if E2_DEVICE_BUILD
  if (!sh.dl_count) sh.dl_count = talloc<unsigned long long>(1);
  for (int pass = 0; pass < 2; ++pass) {
    if (!sh.dl_idx) {
      sh.dl_cap = std::max<u64>(sh.dl_cap, 1 << 16);
      sh.dl_idx = talloc<u64>(sh.dl_cap);
      sh.dl_pay = talloc<uint4>(sh.dl_cap * 4);
    }
    dset(sh.dl_count, 0, 8, h->stream);
    const u64 quads = total * 4;
    if (quads) {
      const unsigned grid = (unsigned)std::min<u64>((quads + 255) / 256, (u64)h->n_sm * 8);
      k_delta_diff<<<grid, 256, 0, h->stream>>>(t, quads, sh.dl_idx, sh.dl_pay, sh.dl_cap, sh.dl_count);
      CK(cudaGetLastError());
    }
    unsigned long long c = 0;
    d2h(&c, sh.dl_count, 8, h->stream);
    ssync(h->stream);
    n = c;
    if (n <= sh.dl_cap) break;
    dfree(sh.dl_idx);
    dfree(sh.dl_pay);
    sh.dl_idx = nullptr;
    sh.dl_cap = n + n / 4;
  }
#else
  std::vector<u64> idx;
  std::vector<uint4> pay;
  for (int r = 0; r < t.n; ++r) {
    const u64 lw = t.live_words[r];
    for (u64 c = 0; c * kChunkWords < lw; ++c) {
      const u64 w0 = c * kChunkWords;
      bool diff = false;
      for (u64 k = 0; k < kChunkWords && w0 + k < lw; ++k) diff |= t.cur[r][w0 + k] != t.sh[r][w0 + k];
      if (!diff) continue;
      idx.push_back(((u64)r << 48) | c);
      u32 v[kChunkWords] = {0};
      for (u64 k = 0; k < kChunkWords && w0 + k < lw; ++k) v[k] = t.cur[r][w0 + k];
      for (int q = 0; q < 4; ++q) pay.push_back(uint4{v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]});
    }
  }
  n = idx.size();
  if (n > sh.dl_cap) {
    dfree(sh.dl_idx);
    dfree(sh.dl_pay);
    sh.dl_cap = n + n / 4 + 16;
    sh.dl_idx = talloc<u64>(sh.dl_cap);
    sh.dl_pay = talloc<uint4>(sh.dl_cap * 4);
  }
  if (n) {
    memcpy(sh.dl_idx, idx.data(), n * 8);
    memcpy(sh.dl_pay, pay.data(), n * 64);
  }
#endif
  // the replicas will hold exactly this: bring the shadow along
  RegionTab ts = t;
  for (int r = 0; r < t.n; ++r) ts.cur[r] = sh.sh[r];
  delta_apply(h, ts, n, sh.dl_idx, sh.dl_pay);
  DeltaHdr& hd = sh.hdr;
  memset(&hd, 0, sizeof(hd));
  hd.magic = kDeltaMagic;
  hd.n_chunks = (i64)n;
  hd.done = h->rs.done;
  hd.fail_code = h->rs.fail_code;
  hd.want_hstride = h->want_hstride;
  hd.n_regions = (u32)t.n;
  for (int r = 0; r < t.n; ++r) hd.region_words[r] = t.words[r];
  snprintf(hd.msg, sizeof(hd.msg), "%s", h->rs.fail.c_str());
  hd.hot = h->hot;
  h->acc.delta_chunks += (i64)n;
  h->acc.delta_bytes += (i64)(kDeltaHdrBytes + n * 8 + n * 64);
  ssync(h->stream);
}

u64 delta_bytes_of(u64 n) { return kDeltaHdrBytes + (n * 8 + 63) / 64 * 64 + n * 64; }

void shard_check(e2_handle* h, bool rank0) {
  if (!h->sh.on || !h->rs.active) throw Fail(E2_ERR_ARG, "no sharded replay in progress");
  if (rank0 && h->sh.rank != 0) throw Fail(E2_ERR_ARG, "this step runs on rank 0 only");
  if (!rank0 && h->sh.rank == 0) throw Fail(E2_ERR_ARG, "this step runs on the replicas only");
}
}  // namespace

int e2_replay(e2_handle* h, const int32_t* tokens, const int64_t* offsets, const int64_t* ids, const double* arrivals,
              const int64_t* output_lens, int64_t n, const e2_driver_cfg* drv, e2_decision* out, e2_cost* costs,
              double* ratios, int64_t* n_done) {
  return replay_impl(h, tokens, offsets, ids, arrivals, output_lens, n, drv, out, costs, ratios, n_done, false);
}

int e2_replay_device(e2_handle* h, const int32_t* d_tokens, const int64_t* d_offsets, const int64_t* d_ids,
                     const double* d_arrivals, const int64_t* d_output_lens, int64_t n, const e2_driver_cfg* drv,
                     e2_decision* d_out, e2_cost* d_costs, double* d_ratios, void* stream, int64_t* n_done) {
#if E2_DEVICE_BUILD
  Stream saved = h->stream;
  if (stream) h->stream = (Stream)stream;
  int rc = replay_impl(h, d_tokens, d_offsets, d_ids, d_arrivals, d_output_lens, n, drv, d_out, d_costs, d_ratios,
                       n_done, true);
  h->stream = saved;
  return rc;
#else
  (void)stream;
  return replay_impl(h, d_tokens, d_offsets, d_ids, d_arrivals, d_output_lens, n, drv, d_out, d_costs, d_ratios,
                     n_done, true);
#endif
}

// ---- sharded replay ------------------------------------------
int e2_shard_begin(e2_handle* h, const int32_t* d_tokens, const int64_t* d_offsets, const int64_t* d_ids,
                   const double* d_arrivals, const int64_t* d_output_lens, int64_t n, const e2_driver_cfg* drv,
                   e2_decision* d_out, e2_cost* d_costs, double* d_ratios, int32_t rank, int32_t world) {
  return guard(h, [&] {
    if (world < 1 || rank < 0 || rank >= world) throw Fail(E2_ERR_ARG, "shard: bad rank/world");
    if (n <= 0) throw Fail(E2_ERR_ARG, "shard: empty trace");
    if (h->cont) throw Fail(E2_ERR_ARG, "shard: streamed continuation is not supported");
    if (drv->prune_interval_ms > 0) throw Fail(E2_ERR_ARG, "shard: prune ticks inside a sharded replay are not supported");
    h->sh.on = true;
    h->sh.rank = rank;
    h->sh.world = world;
    replay_begin(h, d_tokens, d_offsets, d_ids, d_arrivals, d_output_lens, n, drv, rank == 0 ? d_out : nullptr,
                 rank == 0 ? d_costs : nullptr, rank == 0 ? d_ratios : nullptr, true);
    if (rank == 0) shadow_sync(h);
  });
}

int e2_shard_next(e2_handle* h, int64_t* b0, int64_t* nb, int64_t* row_bytes) {
  return guard(h, [&] {
    if (!h->sh.on) throw Fail(E2_ERR_ARG, "no sharded replay in progress");
    const bool more = replay_next(h);
    *b0 = h->rs.cb0;
    *nb = more ? h->rs.cnb : 0;
    h->sh.row_bytes = 16 + 4 * (i64)h->hstride;
    *row_bytes = h->sh.row_bytes;
  });
}

int e2_shard_match(e2_handle* h, int64_t lo, int64_t cnt, void* d_slice) {
  return guard(h, [&] {
    if (!h->sh.on || !h->rs.active) throw Fail(E2_ERR_ARG, "no sharded replay in progress");
    if (lo < 0 || cnt < 0 || lo + cnt > h->rs.cnb) throw Fail(E2_ERR_ARG, "shard: slice outside the batch");
    const u64 rb = (u64)h->sh.row_bytes;
#if E2_DEVICE_BUILD
    if (cnt > 0) {
      k1_slice(h, h->rs.cb0, lo, cnt);
    } else {
      dset(h->d_cnt + 2, 0, 4, h->stream);
    }
    k_shard_pack<<<(unsigned)std::max<i64>(cnt, 1), 128, 0, h->stream>>>(lo, cnt, h->b_S, h->b_dslot, h->b_dm,
                                                                         h->b_path, h->hstride, (char*)d_slice, rb,
                                                                         h->d_cnt + 2);
    CK(cudaGetLastError());
    ssync(h->stream);
#else
    h->d_cnt[2] = 0;
    k1_slice(h, h->rs.cb0, lo, cnt);
    char* out = (char*)d_slice;
    ((u64*)out)[0] = h->d_cnt[2];
    ((u64*)out)[1] = (u64)cnt;
    for (i64 i = 0; i < cnt; ++i) {
      char* row = out + 16 + (u64)i * rb;
      const i64 w = lo + i;
      *(i64*)row = h->b_S[w];
      ((u32*)row)[2] = h->b_dslot[w];
      ((u32*)row)[3] = h->b_dm[w];
      memcpy(row + 16, h->b_path + (u64)w * h->hstride, (size_t)h->hstride * 4);
    }
#endif
  });
}

int e2_shard_commit(e2_handle* h, const void* d_gathered, int64_t per, int64_t* delta_bytes) {
  return guard(h, [&] {
    shard_check(h, true);
    const i64 nb = h->rs.cnb;
    const int world = h->sh.world;
    if (per * world < nb) throw Fail(E2_ERR_ARG, "shard: slices do not cover the batch");
    const u64 rb = (u64)h->sh.row_bytes, slice = 16 + (u64)per * rb;
#if E2_DEVICE_BUILD
    dset(h->d_cnt + 2, 0, 4, h->stream);
    if (nb > 0)
      k_shard_unpack<<<(unsigned)nb, 128, 0, h->stream>>>(world, per, nb, (const char*)d_gathered, rb, slice, h->b_S,
                                                         h->b_dslot, h->b_dm, h->b_path, h->hstride, h->d_cnt + 2);
    CK(cudaGetLastError());
#else
    h->d_cnt[2] = 0;
    for (i64 i = 0; i < nb; ++i) {
      const i64 k = i / per, j = i - k * per;
      const char* sl = (const char*)d_gathered + (u64)k * slice;
      if (j == 0) h->d_cnt[2] = std::max<unsigned int>(h->d_cnt[2], (unsigned int)((const u64*)sl)[0]);
      const char* row = sl + 16 + (u64)j * rb;
      h->b_S[i] = *(const i64*)row;
      h->b_dslot[i] = ((const u32*)row)[2];
      h->b_dm[i] = ((const u32*)row)[3];
      memcpy(h->b_path + (u64)i * h->hstride, row + 16, (size_t)h->hstride * 4);
    }
#endif
    group_rounds(h, h->rs.cb0, nb);
    replay_commit(h);
    delta_export(h);
    replay_after_batch(h);
    shadow_sync(h);  // regions a growth moved are re-taken whole (the replicas regrow identically)
    *delta_bytes = (int64_t)delta_bytes_of((u64)h->sh.hdr.n_chunks);
  });
}

int e2_shard_delta_copy(e2_handle* h, void* d_dst) {
  return guard(h, [&] {
    shard_check(h, true);
    const u64 n = (u64)h->sh.hdr.n_chunks;
    char* dst = (char*)d_dst;
    h2d(dst, &h->sh.hdr, sizeof(DeltaHdr), h->stream);
    if (n) {
      d2d(dst + kDeltaHdrBytes, h->sh.dl_idx, n * 8, h->stream);
      d2d(dst + kDeltaHdrBytes + (n * 8 + 63) / 64 * 64, h->sh.dl_pay, n * 64, h->stream);
    }
    ssync(h->stream);
  });
}

int e2_shard_apply(e2_handle* h, const void* d_delta, int64_t bytes) {
  return guard(h, [&] {
    shard_check(h, false);
    if (bytes < (int64_t)kDeltaHdrBytes) throw Fail(E2_ERR_ARG, "shard: delta too short");
    DeltaHdr hd;
    d2h(&hd, d_delta, sizeof(DeltaHdr), h->stream);
    ssync(h->stream);
    if (hd.magic != kDeltaMagic) throw Fail(E2_ERR_ARG, "shard: not a delta");
    const u64 n = (u64)hd.n_chunks;
    if ((u64)bytes != delta_bytes_of(n)) throw Fail(E2_ERR_ARG, "shard: delta size mismatch");
    RegionTab t = state_regions(h);
    if ((int)hd.n_regions != t.n) throw Fail(E2_ERR_ARG, "shard: region count mismatch");
    for (int r = 0; r < t.n; ++r)
      if (hd.region_words[r] != t.words[r]) throw Fail(E2_ERR_ARG, "shard: replica capacity diverged");
    const char* src = (const char*)d_delta;
    delta_apply(h, t, n, (const u64*)(src + kDeltaHdrBytes),
                (const uint4*)(src + kDeltaHdrBytes + (n * 8 + 63) / 64 * 64));
    h->hot = hd.hot;
    h->dev_hot_valid = false;
    push_hot(h);
    h->want_hstride = std::max(h->want_hstride, (int)hd.want_hstride);
    h->rs.done = hd.done;
    if (hd.fail_code) {
      h->rs.fail_code = hd.fail_code;
      h->rs.fail = hd.msg;
      h->rs.stopped = true;
    }
    ssync(h->stream);
    replay_after_batch(h);
  });
}

int e2_state_digest(e2_handle* h, uint64_t* out, int32_t cap, int32_t* n_out) {
  return guard(h, [&] {
    RegionTab t = state_regions(h);
    if (cap < t.n + 1) throw Fail(E2_ERR_ARG, "digest: output too small");
    for (int r = 0; r < t.n; ++r) {
      // the node pool's live part; every other region whole
      const u64 words = t.live_words[r];
#if E2_DEVICE_BUILD
      unsigned long long* d = talloc<unsigned long long>(1);
      if (words) {
        k_digest<<<(unsigned)std::min<u64>((words + 255) / 256, (u64)h->n_sm * 8), 256, 0, h->stream>>>(t.cur[r], words, d);
        CK(cudaGetLastError());
      }
      unsigned long long v = 0;
      d2h(&v, d, 8, h->stream);
      ssync(h->stream);
      dfree(d);
      out[r] = v;
#else
      u64 acc = 0;
      for (u64 i = 0; i < words; ++i) acc += mix64((i << 32) ^ (u64)t.cur[r][i]);
      out[r] = acc;
#endif
    }
    Hot hot = h->hot;
    memset(hot.phase_cycles, 0, sizeof(hot.phase_cycles));
    hot.phase_last = hot.phase_last1 = 0;
    u64 acc = 0;
    const u64* w = (const u64*)&hot;
    for (size_t i = 0; i < sizeof(Hot) / 8; ++i) acc += mix64(((u64)i << 40) ^ w[i]);
    out[t.n] = acc;
    *n_out = t.n + 1;
  });
}

int e2_shard_end(e2_handle* h, int64_t* n_done) {
  if (n_done) *n_done = 0;
  return guard(h, [&] {
    if (!h->sh.on) throw Fail(E2_ERR_ARG, "no sharded replay in progress");
    h->sh.on = false;
    shadow_free(h);
    replay_end(h, n_done);
  });
}

int e2_profile_get(e2_handle* h, e2_profile* out) {
  return guard(h, [&] {
    prof_flush(h);
    unsigned long long b[2] = {0, 0};
    d2h(b, h->d_bytes, 16, h->stream);
    ssync(h->stream);
    *out = h->acc;
    out->match_bytes = (i64)b[0];
  });
}

int e2_profile_reset(e2_handle* h, int32_t enable_timing) {
  return guard(h, [&] {
    prof_flush(h);
    memset(&h->acc, 0, sizeof(h->acc));
    h->prof = enable_timing != 0;
    dset(h->d_bytes, 0, 16, h->stream);
    ssync(h->stream);
  });
}

}  // extern "C"

#ifdef E2_PHASES
// dev-only: per-phase cycle totals of the serial replay (E2_PHASES builds)
extern "C" int e2_debug_phases(e2_handle* h, uint64_t* out) {
  return guard(h, [&] {
    pull_hot(h);
    for (int i = 0; i < 48; ++i) out[i] = h->hot.phase_cycles[i];
  });
}
#endif
