// sm_100a lock-step gang kernel (see kernel_common.cuh for why it has its own
// translation unit).
#include <cuda_runtime.h>

#include "kernel_common.cuh"

namespace mfb {

// Gang variant: a block of W warps, each owning its own instance (and its own
// slice of shared memory), advances all W instances ONE EVENT at a time in
// lock step (one block barrier per event). The engine is instruction-fetch
// bound (ncu: 50-68 % of warp stalls "no instruction", ~40k SASS instructions,
// warps of one SM in different phases); in lock step the W warps of a block
// run through the same code at about the same time.
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
      const int r = eng.step(deadline);
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

// Re-sorts every claim group by its instances' CURRENT active-flow count,
// descending, before a time-sliced gang launch: the 32 warps of a gang then
// take instances of similar per-event cost at this point of their runs (the
// static claim order only knows the offered load). A suspended instance's
// count is in its scalar-state blob; fresh and finished instances count 0.
// One block; keys (group, -active, position) bitonic-sorted in shared memory.
__global__ void __launch_bounds__(1024)
    mfsim_order_kernel(const Inst* __restrict__ insts, const int* __restrict__ in, int* __restrict__ out,
                       int n, int groups, int n2) {
  extern __shared__ __align__(16) unsigned long long key[];
  const int* __restrict__ goff = in + n;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    unsigned long long k = ~0ull;
    if (i < n) {
      const int id = in[i];
      int g = 0;
      while (g + 1 < groups && goff[g + 1] <= i) ++g;
      int a = 0;
      if (*insts[id].phase == 1) a = reinterpret_cast<const Sc*>(insts[id].sc_blob)->n_active;
      a = a < 0 ? 0 : (a > 0xFFFFF ? 0xFFFFF : a);
      k = ((unsigned long long)g << 52) | ((unsigned long long)(0xFFFFF - a) << 32) | (unsigned)i;
    }
    key[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = key[i], b = key[ixj];
          if (((i & k) == 0) == (a > b)) {
            key[i] = b;
            key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = in[(int)(key[i] & 0xffffffffu)];
  for (int i = threadIdx.x; i < 2 * (groups + 1); i += blockDim.x) out[n + i] = in[n + i];
}

bool order_kernel_launch(cudaStream_t stream, const Inst* insts, const int* in, int* out, int n, int groups) {
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  const int bytes = n2 * 8;
  if (bytes > 200 * 1024) return false;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(mfsim_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    init = true;
  }
  mfsim_order_kernel<<<1, 1024, bytes, stream>>>(insts, in, out, n, groups, n2);
  return true;
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
