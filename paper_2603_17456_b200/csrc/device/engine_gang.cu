// sm_100a lock-step gang kernel (see kernel_common.cuh for why it has its own
// translation unit).
#include <cuda_runtime.h>

#include "kernel_common.cuh"

namespace mfb {

// Gang variant: a block of W warps, each owning its own instance (and its own
// slice of shared memory), advances all W instances ONE EVENT at a time in
// lock step, with a block barrier between popping the event, its handler, its
// policy classes, its filling and its completion events. The engine is
// instruction-fetch bound (ncu: 50-68 % of warp stalls "no instruction", ~40k
// SASS instructions, warps of one SM in different phases); in lock step the W
// warps of a block run through the same code at about the same time (A/B,
// profiles/r02_gang_ab.txt:
// one barrier per event +13-15 %, the phase barriers another +3 %, two
// events per barrier -17 %, two 16-warp gangs per SM +5 % over one of 32).
template <bool kAalo>
__global__ void __launch_bounds__(1024, 1)
    mfsim_gang_kernel(const Inst* __restrict__ insts, const int* __restrict__ order, int n,
                      int groups, int nsm, int* __restrict__ next, SmemPlan plan,
                      long long budget, long long slice_ns, int* __restrict__ remaining) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long t0;
  const int nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char* mine = smem + (threadIdx.x >> 5) * plan.bytes;
  Inst* d = reinterpret_cast<Inst*>(mine);
  unsigned long long deadline = 0;
  if (slice_ns > 0) {
    if (threadIdx.x == 0) t0 = now_ns();
    __syncthreads();
    deadline = t0 + (unsigned long long)slice_ns;
  }
  const int* __restrict__ goff = order + n;
  const int home = home_group(goff, n, groups, nsm, slice_ns);
  Engine<WarpLanes, kAalo> eng(*d, false);
  int state = 0;  // 0: claim next, 1: running an instance, 2: no work left
  // first claims by block: the gang's warps take consecutive instances of the
  // claim order (similar per-event cost, so less waiting at the barrier)
  __shared__ int base0;
  if (threadIdx.x == 0) base0 = atomicAdd(&next[home], nw);
  __syncthreads();
  int first = -1;
  if (goff[home] + base0 + (int)(threadIdx.x >> 5) < goff[home + 1])
    first = order[goff[home] + base0 + (threadIdx.x >> 5)];
#if defined(MF_GANG_PROF)
  // lock-step efficiency: busy cycles of this warp's events vs the whole loop
  __shared__ unsigned long long busy_sum, iters;
  if (threadIdx.x == 0) busy_sum = iters = 0;
  __syncthreads();
  const long long loop0 = clock64();
  long long busy = 0, n_it = 0;
#endif
  for (;;) {
    if (state == 0) {
      const int i = first >= 0 ? first : claim(order, goff, groups, home, next);
      first = -1;
      if (i < 0) {
        state = 2;
      } else {
        eng.chip = stage_instance(insts + i, mine, plan);
        if (eng.begin(budget)) state = 1;
      }
    }
    if (state == 1) {
#if defined(MF_GANG_PROF)
      const long long b0 = clock64();
#endif
      const int r = eng.step_head(deadline);
#if defined(MF_GANG_PROF)
      busy += clock64() - b0;
      ++n_it;
#endif
      if (r != 0) {
        const bool done = eng.end(r == 1);
        if (done && lane == 0) atomicSub(remaining, 1);
        __syncwarp();
        state = 0;
      }
    }
    // barriers between popping the event, its handler, the policy classes,
    // the filling and the completion events: the gang's warps run each
    // phase's code together
    __syncthreads();
#if defined(MF_GANG_PROF)
    long long b1 = clock64();
#endif
    if (state == 1) {
      if (eng.step_dispatch() != 0) {
        const bool done = eng.end(true);
        if (done && lane == 0) atomicSub(remaining, 1);
        __syncwarp();
        state = 0;
      }
    }
#if defined(MF_GANG_PROF)
    busy += clock64() - b1;
#endif
    __syncthreads();
#if defined(MF_GANG_PROF)
    b1 = clock64();
#endif
    if (state == 1) eng.settle_decide();
#if defined(MF_GANG_PROF)
    busy += clock64() - b1;
#endif
    __syncthreads();
#if defined(MF_GANG_PROF)
    b1 = clock64();
#endif
    if (state == 1) eng.settle_allocate();
#if defined(MF_GANG_PROF)
    busy += clock64() - b1;
#endif
    __syncthreads();
    if (state == 1) {
      eng.settle_finish();
      if (eng.s.err) {
        const bool done = eng.end(true);
        if (done && lane == 0) atomicSub(remaining, 1);
        __syncwarp();
        state = 0;
      }
    }
    if (!__syncthreads_or(state != 2)) break;
  }
#if defined(MF_GANG_PROF)
  if (lane == 0) {
    atomicAdd(&busy_sum, (unsigned long long)busy);
    atomicAdd(&iters, (unsigned long long)n_it);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    printf("gangprof block %d sm %d: loop %lld cycles, warps %d, busy share %.3f, events %llu\n", blockIdx.x,
           sm_id(), clock64() - loop0, blockDim.x >> 5,
           (double)busy_sum / ((double)(clock64() - loop0) * (blockDim.x >> 5)), iters);
#endif
}

void gang_kernel_init() {
  for (auto k : {mfsim_gang_kernel<false>, mfsim_gang_kernel<true>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

int gang_kernel_blocks_per_sm(bool ext, int threads, int bytes) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ext ? mfsim_gang_kernel<true> : mfsim_gang_kernel<false>,
                                                threads, bytes);
  return per_sm;
}

void gang_kernel_launch(bool ext, int grid, int threads, int bytes, cudaStream_t stream, const Inst* insts,
                        const int* order, int n, int groups, int nsm, int* next, SmemPlan plan,
                        long long budget, long long slice_ns, int* remaining) {
  auto kern = ext ? mfsim_gang_kernel<true> : mfsim_gang_kernel<false>;
  kern<<<grid, threads, bytes, stream>>>(insts, order, n, groups, nsm, next, plan, budget, slice_ns, remaining);
}

}  // namespace mfb
