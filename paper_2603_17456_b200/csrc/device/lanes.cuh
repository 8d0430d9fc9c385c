// Lane-group abstraction for the warp-per-instance engine.
//
// The engine is written once as warp-synchronous code: scalar control flow is
// executed uniformly by every lane of the group (all lanes hold identical
// register copies of scalar state), data-parallel loops stride over lanes, and
// every store to shared instance state in a scalar section goes through
// G::put (one writer, fenced by __syncwarp on both sides).
//
//   WarpLanes   -- the product: one 32-lane warp on sm_100a owns one instance.
//   SerialLanes -- a 1-lane host build of the SAME engine source, used only by
//                  the CPU test tier to debug engine logic without a GPU. It is
//                  never linked into the product library.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define MF_FN __device__ __forceinline__
#define MF_NOINLINE __device__ __noinline__
#else
#define MF_FN inline
#define MF_NOINLINE
#endif

// unroll factor of the lane-strided hot loops: 1 measured fastest (icache-bound;
// A/B of 1/2/4 on the bench workload, profiles/r01_ab_engine_builds.txt)
#ifndef MF_UNROLL_N
#define MF_UNROLL_N 1
#endif
#define MF_PRAGMA_(x) _Pragma(#x)
#define MF_PRAGMA(x) MF_PRAGMA_(x)
#if defined(__CUDACC__)
#define MF_UNROLL MF_PRAGMA(unroll MF_UNROLL_N)
#else
#define MF_UNROLL
#endif

namespace mfb {

#if defined(__CUDACC__)
struct WarpLanes {
  static constexpr int N = 32;
  MF_FN int lane() const { return threadIdx.x & 31; }
  MF_FN bool leader() const { return (threadIdx.x & 31) == 0; }
  MF_FN void sync() const { __syncwarp(); }
  template <class T>
  MF_FN void put(T* p, T v) const {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *p = v;
    __syncwarp();
  }
  MF_FN int shfl_xor(int v, int m) const { return __shfl_xor_sync(0xffffffffu, v, m); }
  MF_FN unsigned shfl_xor(unsigned v, int m) const { return __shfl_xor_sync(0xffffffffu, v, m); }
  MF_FN double shfl_xor(double v, int m) const { return __shfl_xor_sync(0xffffffffu, v, m); }
  MF_FN unsigned long long shfl_xor(unsigned long long v, int m) const {
    return __shfl_xor_sync(0xffffffffu, v, m);
  }
  MF_FN long long shfl_xor(long long v, int m) const { return __shfl_xor_sync(0xffffffffu, v, m); }
  MF_FN int shfl(int v, int src) const { return __shfl_sync(0xffffffffu, v, src); }
  MF_FN double shfl(double v, int src) const { return __shfl_sync(0xffffffffu, v, src); }
  MF_FN unsigned long long shfl(unsigned long long v, int src) const {
    return __shfl_sync(0xffffffffu, v, src);
  }
  MF_FN int shfl_up(int v, int d) const { return __shfl_up_sync(0xffffffffu, v, d); }
  MF_FN unsigned ballot(bool p) const { return __ballot_sync(0xffffffffu, p); }
  MF_FN bool any(bool p) const { return __any_sync(0xffffffffu, p); }
  MF_FN unsigned match_any(int v) const { return __match_any_sync(0xffffffffu, v); }
  MF_FN unsigned lanemask_lt() const { return (1u << (threadIdx.x & 31)) - 1u; }
  MF_FN int sum(int v) const { return __reduce_add_sync(0xffffffffu, (unsigned)v); }
  MF_FN int atomic_add(int* p, int v) const { return atomicAdd(p, v); }
  MF_FN unsigned atomic_or(unsigned* p, unsigned v) const { return atomicOr(p, v); }
  // set a byte flag to 1, returning its previous value (32-bit CAS on the word)
  MF_FN int atomic_exch_u8(uint8_t* p) const {
    unsigned* w = reinterpret_cast<unsigned*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
    const unsigned sh = (unsigned)(reinterpret_cast<uintptr_t>(p) & 3) * 8u;
    const unsigned old = atomicOr(w, 1u << sh);
    return (old >> sh) & 0xffu;
  }
  // Warp minimum of a NON-NEGATIVE, non-NaN double (+0 <= x <= +inf). Such
  // values order like their IEEE bit patterns read as unsigned integers, so two
  // 32-bit redux.sync steps (high word, then low word among the lanes holding
  // the minimal high word) replace a 5-step shuffle/compare butterfly. The
  // result is the same IEEE value (bit pattern) on every lane.
  MF_FN double min_nonneg(double v) const {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  }
  MF_FN unsigned long long min_u64(unsigned long long v) const {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
  }
  // Lexicographic warp argmin of (t, k) for t >= 0 or t == -0 (no NaN; -0 and
  // +0 compare equal as with `<`/`==`): the lowest lane holding the minimal
  // (t, k) wins; returns that lane's (t, k, payload) on every lane.
  MF_FN void argmin_tk(double* t, unsigned long long* k, int* payload) const {
    const double tc = *t + 0.0;  // -0 -> +0 (round-to-nearest)
    const unsigned long long tb = (unsigned long long)__double_as_longlong(tc);
    const unsigned long long tm = min_u64(tb);
    const unsigned long long km = min_u64(tb == tm ? *k : ~0ull);
    const unsigned win = __ballot_sync(0xffffffffu, tb == tm && *k == km);
    const int src = __ffs(win) - 1;
    *t = __shfl_sync(0xffffffffu, *t, src);
    *k = km;
    *payload = __shfl_sync(0xffffffffu, *payload, src);
  }
  // exclusive prefix sum of v over lanes; *total receives the warp sum
  MF_FN int excl_scan(int v, int* total) const {
    int x = v;
    const int l = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, d);
      if (l >= d) x += y;
    }
    *total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  }
};
#endif

struct SerialLanes {
  static constexpr int N = 1;
  inline int lane() const { return 0; }
  inline bool leader() const { return true; }
  inline void sync() const {}
  template <class T>
  inline void put(T* p, T v) const { *p = v; }
  template <class T>
  inline T shfl_xor(T v, int) const { return v; }
  template <class T>
  inline T shfl(T v, int) const { return v; }
  inline int shfl_up(int v, int) const { return v; }
  inline unsigned ballot(bool p) const { return p ? 1u : 0u; }
  inline bool any(bool p) const { return p; }
  inline unsigned match_any(int) const { return 1u; }
  inline unsigned lanemask_lt() const { return 0u; }
  inline int sum(int v) const { return v; }
  inline int atomic_add(int* p, int v) const {
    int o = *p;
    *p = o + v;
    return o;
  }
  inline unsigned atomic_or(unsigned* p, unsigned v) const {
    unsigned o = *p;
    *p = o | v;
    return o;
  }
  inline int atomic_exch_u8(uint8_t* p) const {
    int o = *p;
    *p = 1;
    return o;
  }
  inline int excl_scan(int v, int* total) const {
    *total = v;
    return 0;
  }
  inline double min_nonneg(double v) const { return v; }
  inline unsigned long long min_u64(unsigned long long v) const { return v; }
  inline void argmin_tk(double*, unsigned long long*, int*) const {}
};

}  // namespace mfb
