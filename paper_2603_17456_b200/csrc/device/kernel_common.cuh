// Per-warp shared-memory plan and instance staging shared by the two kernels
// (engine_kernel.cu: one warp per instance; engine_gang.cu: lock-step gangs).
// Each kernel lives in its own translation unit so that its copy of the
// engine is register-allocated for its own occupancy (a gang of 32 warps per
// SM: 64 registers; the one-warp kernel of sparse launches: up to 128).
#pragma once
#include <cuda_runtime.h>

#include "../host/instance.hpp"
#include "engine.cuh"

namespace mfb {

// Per-warp shared-memory plan of one launch: the descriptor copy, then the
// hot arrays of an instance whenever its capacities fit (active-flow state +
// route cache + per-step rates, the event pool, per-link residual / count).
struct SmemPlan {
  int ES;  // event pool entries
  int NL;  // link -> slot map entries (0: map stays in global memory)
  int TS;  // slots
  int bytes;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

constexpr int kFrzWords = 32;  // on-chip member frozen bits: active sets up to 1024 flows

// Per-warp shared memory: the descriptor copy, the event pool, the link ->
// slot map and the per-slot filling state. The active-flow arrays stay in
// global memory (L1/L2): measured sweep instances reach 250-900 active flows,
// and keeping shared memory small lets ~19 warps share an SM.
__host__ inline SmemPlan make_plan(int nlinks) {
  SmemPlan p{};
  p.ES = mfh::kSmemEvents;
  p.NL = 0;
  p.TS = mfh::kSmemSlots;
  int b = align16(sizeof(Inst));
  b += align16(p.ES * 8) * 2 + align16(p.ES * 4) * 3;
  b += align16(p.TS * 8) + 3 * align16(p.TS * 4) + 2 * align16(p.TS * 2);
  b += align16(kFrzWords * 4);
  p.bytes = align16(b);
  return p;
}

static __device__ __forceinline__ int sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return (int)r;
}

// Copies instance `src`'s descriptor into this warp's shared-memory region
// `base` and stages the event pool and the per-slot filling state there when
// the instance's capacities fit the plan. Returns whether the slot state is on
// chip (the filling rounds are specialised on it).
static __device__ __noinline__ bool stage_instance(const Inst* __restrict__ src, unsigned char* base,
                                            const SmemPlan& plan) {
  const int lane = threadIdx.x & 31;
  Inst* d = reinterpret_cast<Inst*>(base);
  {  // descriptor copy (8-byte words across the warp)
    const unsigned long long* s8 = reinterpret_cast<const unsigned long long*>(src);
    unsigned long long* d8 = reinterpret_cast<unsigned long long*>(d);
    for (int w = lane; w < (int)(sizeof(Inst) / 8); w += 32) d8[w] = s8[w];
  }
  __syncwarp();
  bool slots_on_chip = false;
  if (lane == 0) {
    unsigned char* q = base + align16(sizeof(Inst));
    auto take = [&](int bytes) {
      unsigned char* r = q;
      q += align16(bytes);
      return r;
    };
    if (d->E_cap <= plan.ES) {
      double* et = reinterpret_cast<double*>(take(plan.ES * 8));
      unsigned long long* es = reinterpret_cast<unsigned long long*>(take(plan.ES * 8));
      int* ek = reinterpret_cast<int*>(take(plan.ES * 4));
      int* ea = reinterpret_cast<int*>(take(plan.ES * 4));
      int* eb = reinterpret_cast<int*>(take(plan.ES * 4));
      d->e_t_home = d->e_t;  // the engine moves entries between chip and home
      d->e_seq_home = d->e_seq;
      d->e_kind_home = d->e_kind;
      d->e_a_home = d->e_a;
      d->e_b_home = d->e_b;
      d->e_t = et;
      d->e_seq = es;
      d->e_kind = ek;
      d->e_a = ea;
      d->e_b = eb;
    } else {
      q += 2 * align16(plan.ES * 8) + 3 * align16(plan.ES * 4);
    }
    if (plan.TS > 0 && d->TS_cap > 0 && d->A_cap <= 32 * kFrzWords) {
      // per-step slot state on chip; the slot bookkeeping stays in HBM
      // (its capacity bound must not change across suspend / resume)
      d->sl_res = reinterpret_cast<double*>(take(plan.TS * 8));
      d->sl_cnt = reinterpret_cast<int*>(take(plan.TS * 4));
      d->sl_mb = reinterpret_cast<int*>(take(plan.TS * 4));
      d->sl_end = reinterpret_cast<int*>(take(plan.TS * 4));
      d->sl_tl = reinterpret_cast<unsigned short*>(take(plan.TS * 2));
      d->sl_sat = reinterpret_cast<unsigned short*>(take(plan.TS * 2));
      d->c_frz = reinterpret_cast<unsigned*>(take(kFrzWords * 4));
      slots_on_chip = true;
    }
  }
  slots_on_chip = __shfl_sync(0xffffffffu, slots_on_chip, 0);
  __syncwarp();
  return slots_on_chip;
}

// The SM's home claim group (see the kernels below).
static __device__ __forceinline__ int home_group(const int* __restrict__ goff, int n, int groups, int nsm,
                                          long long slice_ns) {
  int home = 0;
  const int* __restrict__ gmap = slice_ns > 0 ? goff : goff + groups + 1;
  const long long pos = (long long)sm_id() * n / nsm;
  while (home + 1 < groups && gmap[home + 1] <= pos) ++home;
  return home;
}

// next instance for this warp (-1: none left), home group first
static __device__ __forceinline__ int claim(const int* __restrict__ order, const int* __restrict__ goff,
                                     int groups, int home, int* __restrict__ next) {
  int i = -1;
  if ((threadIdx.x & 31) == 0) {
    for (int k = 0; k < groups && i < 0; ++k) {
      const int gi = (home + k) % groups;
      const int c = atomicAdd(&next[gi], 1);
      if (goff[gi] + c < goff[gi + 1]) i = order[goff[gi] + c];
    }
  }
  return __shfl_sync(0xffffffffu, i, 0);
}

// host side of the gang kernel (engine_gang.cu)
void gang_kernel_init();
int gang_kernel_blocks_per_sm(bool ext, int threads, int bytes);
void gang_kernel_launch(bool ext, int grid, int threads, int bytes, cudaStream_t stream, const Inst* insts,
                        const int* order, int n, int groups, int nsm, int* next, SmemPlan plan,
                        long long budget, long long slice_ns, int* remaining);

}  // namespace mfb
