// e2_common.cuh — SIMT-generic primitives shared by every kernel.
//
// Device build (nvcc, sm_100a): code runs as one 32-lane warp; scalar control
// logic is executed redundantly by all lanes (uniform values), single writes
// go through lane 0 followed by __syncwarp, and the warp-cooperative pieces
// (child-table probes, LRU page edits, per-instance cost lanes) use
// ballot/shuffle.
//
// Host emulation build (E2_HOSTSIM, g++; TEST-ONLY, never linked into the
// product library): the same source with a warp width of 1, so the CPU test
// suite can exercise the engine's control logic without a GPU.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__) && !defined(E2_HOSTSIM)
#define E2_DEVICE_BUILD 1
#define E2_HD __device__ __forceinline__
#define E2_HDX __host__ __device__ __forceinline__
#define E2_D __device__ __forceinline__
// Every engine function is inlined into the serial kernel: measured on C2,
// device calls (ABI register save/restore, no optimisation across the call)
// cost ~35% of the per-request time (99.6k vs 73.1k decisions/s with only
// decide inlined).  -DE2_NOINLINE keeps the call structure (profiling).
#if defined(E2_NOINLINE)
#define E2_DNI __device__ __noinline__
#else
#define E2_DNI __device__ __forceinline__
#endif
#else
#define E2_DEVICE_BUILD 0
#define E2_HD inline
#define E2_HDX inline
#define E2_D inline
#define E2_DNI
#endif

// E2_WARP: the warp-cooperative code paths (32 lanes).  Scalar builds use a
// width of 1: the host emulation, and the single-thread device engine
// (E2_SCALAR, e2_serial.cu).
#if E2_DEVICE_BUILD && !defined(E2_SCALAR)
#define E2_WARP 1
#else
#define E2_WARP 0
#endif

namespace e2 {

typedef int64_t i64;
typedef uint64_t u64;
typedef int32_t i32;
typedef uint32_t u32;

constexpr u32 kNil = 0xffffffffu;
constexpr u32 kRoot = 0;
constexpr int kMaxG = 64;

#if E2_WARP
constexpr int kWidth = 32;
E2_D int lane() { return (int)(threadIdx.x & 31); }
E2_D void wsync() { __syncwarp(); }
E2_D u32 ballot(bool p) { return __ballot_sync(0xffffffffu, p); }
E2_D bool any(bool p) { return __any_sync(0xffffffffu, p); }
template <typename T>
E2_D T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <typename T>
E2_D T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
E2_D T shfl_down1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
E2_D int ffs32(u32 m) { return __ffs((int)m) - 1; }
E2_D int popc32(u32 m) { return __popc(m); }
E2_D int popc64(u64 m) { return __popcll(m); }
E2_D int ffs64(u64 m) { return __ffsll((long long)m) - 1; }
// Exact IEEE double ops with explicit rounding so nvcc never contracts a*b+c
// into an FMA: the reference's bits are computed unfused (SURVEY 7 hard part 4).
E2_D double dmul(double a, double b) { return __dmul_rn(a, b); }
E2_D double dadd(double a, double b) { return __dadd_rn(a, b); }
E2_D double dsub(double a, double b) { return __dsub_rn(a, b); }
E2_D double ddiv(double a, double b) { return __ddiv_rn(a, b); }
E2_D double i2d(i64 v) { return __ll2double_rn((long long)v); }
#elif E2_DEVICE_BUILD
// single-thread device engine: lane 0 of a width-1 "warp"
constexpr int kWidth = 1;
E2_D int lane() { return 0; }
E2_D void wsync() {}
E2_D u32 ballot(bool p) { return p ? 1u : 0u; }
E2_D bool any(bool p) { return p; }
template <typename T>
E2_D T shfl(T v, int) { return v; }
template <typename T>
E2_D T shfl_up1(T v) { return v; }
template <typename T>
E2_D T shfl_down1(T v) { return v; }
E2_D int ffs32(u32 m) { return __ffs((int)m) - 1; }
E2_D int popc32(u32 m) { return __popc(m); }
E2_D int popc64(u64 m) { return __popcll(m); }
E2_D int ffs64(u64 m) { return __ffsll((long long)m) - 1; }
E2_D double dmul(double a, double b) { return __dmul_rn(a, b); }
E2_D double dadd(double a, double b) { return __dadd_rn(a, b); }
E2_D double dsub(double a, double b) { return __dsub_rn(a, b); }
E2_D double ddiv(double a, double b) { return __ddiv_rn(a, b); }
E2_D double i2d(i64 v) { return __ll2double_rn((long long)v); }
#else
constexpr int kWidth = 1;
inline int lane() { return 0; }
inline void wsync() {}
inline u32 ballot(bool p) { return p ? 1u : 0u; }
inline bool any(bool p) { return p; }
template <typename T>
inline T shfl(T v, int) { return v; }
template <typename T>
inline T shfl_up1(T v) { return v; }
template <typename T>
inline T shfl_down1(T v) { return v; }
inline int ffs32(u32 m) { return m ? __builtin_ctz(m) : -1; }
inline int popc32(u32 m) { return __builtin_popcount(m); }
inline int popc64(u64 m) { return __builtin_popcountll(m); }
inline int ffs64(u64 m) { return m ? __builtin_ctzll(m) : -1; }
inline double dmul(double a, double b) {
  volatile double r = a * b;
  return r;
}
inline double dadd(double a, double b) {
  volatile double r = a + b;
  return r;
}
inline double dsub(double a, double b) {
  volatile double r = a - b;
  return r;
}
inline double ddiv(double a, double b) {
  volatile double r = a / b;
  return r;
}
inline double i2d(i64 v) { return (double)v; }
#endif

E2_HD bool lane0() { return lane() == 0; }

// Block-scope memory fence (hand-off flags between the replay's warps)
#if E2_DEVICE_BUILD
E2_D void fence_block() { __threadfence_block(); }
#else
inline void fence_block() {}
#endif

// L1 prefetch of a global address (no-op in the host emulation)
#if E2_DEVICE_BUILD
E2_D void pf(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
#else
inline void pf(const void*) {}
#endif
#if E2_DEVICE_BUILD
E2_D bool thread0() { return threadIdx.x == 0; }  // lane 0 of warp 0
#else
inline bool thread0() { return true; }
#endif

// Warp vote over positions [0, n) (n <= 32): bit j = f(j).  On the device
// lane j evaluates f(j); the host emulation loops, so both builds probe the
// same 32-wide windows.
template <typename F>
E2_D u32 vote(int n, F&& f) {
#if E2_WARP
  const int l = lane();
  return ballot(l < n && f(l));
#else
  u32 m = 0;
  for (int j = 0; j < n; ++j)
    if (f(j)) m |= 1u << j;
  return m;
#endif
}

template <typename T>
E2_HDX T min_(T a, T b) { return a < b ? a : b; }
template <typename T>
E2_HDX T max_(T a, T b) { return a > b ? a : b; }

// Bit pattern of a non-negative double is monotone as an unsigned integer;
// last_access values are always >= +0 (prefix_tree.cpp:21-24, 48-49).
E2_HDX u64 dbits(double d) {
  u64 u;
  memcpy(&u, &d, 8);
  return u;
}
E2_HDX double bitsd(u64 u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}

E2_HDX u64 mix64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

}  // namespace e2
