// sm_100a entry point and CUDA backend.
//
// mfsim_engine_kernel is a persistent grid: each warp repeatedly claims the
// next unclaimed simulation instance (atomic work counter, so long-running
// instances -- Karuna, overload -- do not stall a static partition) and runs
// that instance's entire event loop on the device (engine.cuh). Grid =
// blocks_per_sm x 148 SMs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

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

__device__ __forceinline__ int sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return (int)r;
}

// Copies instance `src`'s descriptor into this warp's shared-memory region
// `base` and stages the event pool and the per-slot filling state there when
// the instance's capacities fit the plan. Returns whether the slot state is on
// chip (the filling rounds are specialised on it).
__device__ __noinline__ bool stage_instance(const Inst* __restrict__ src, unsigned char* base,
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
__device__ __forceinline__ int home_group(const int* __restrict__ goff, int n, int groups, int nsm,
                                          long long slice_ns) {
  int home = 0;
  const int* __restrict__ gmap = slice_ns > 0 ? goff : goff + groups + 1;
  const long long pos = (long long)sm_id() * n / nsm;
  while (home + 1 < groups && gmap[home + 1] <= pos) ++home;
  return home;
}

// next instance for this warp (-1: none left), home group first
__device__ __forceinline__ int claim(const int* __restrict__ order, const int* __restrict__ goff,
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

// order[0, n): instance ids in claim groups (one per policy), estimated work
// descending within a group; order[n + g] = offset of group g. A warp claims
// from its SM's home group first, then from the others. SMs are mapped onto
// the groups in proportion to their sizes for time-sliced launches (every
// warp busy for the slice) and in proportion to their estimated work,
// order[n + groups + 1 + g], for launches that run to completion (the
// makespan is the most loaded SM's).
template <bool kAalo>
__global__ void __launch_bounds__(32)
    mfsim_engine_kernel(const Inst* __restrict__ insts, const int* __restrict__ order, int n,
                        int groups, int nsm, int* __restrict__ next, SmemPlan plan,
                        long long budget, long long slice_ns, int* __restrict__ remaining) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  Inst* d = reinterpret_cast<Inst*>(smem);
  // time-sliced launches: every warp works until the same device-clock deadline
  unsigned long long deadline = 0;
  if (slice_ns > 0) {
    __shared__ unsigned long long t0;
    if (lane == 0) t0 = now_ns();
    __syncwarp();
    deadline = t0 + (unsigned long long)slice_ns;
  }
  const int* __restrict__ goff = order + n;
  const int home = home_group(goff, n, groups, nsm, slice_ns);
  for (;;) {
    const int i = claim(order, goff, groups, home, next);
    if (i < 0) return;
    const bool slots_on_chip = stage_instance(insts + i, smem, plan);
    Engine<WarpLanes, kAalo> eng(*d, slots_on_chip);
    const bool done = eng.run(budget, deadline);
    if (done && lane == 0) atomicSub(remaining, 1);
    __syncwarp();
  }
}

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

}  // namespace mfb

namespace mfh {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

class CudaBackend final : public Backend {
 public:
  explicit CudaBackend(int device) : device_(device) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&own_, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_ = own_;
    ck(cudaEventCreate(&e0_), "cudaEventCreate");
    ck(cudaEventCreate(&e1_), "cudaEventCreate");
    ck(cudaMalloc(&counter_, (1 + kMaxGroups) * sizeof(int)), "cudaMalloc counter");
    ck(cudaMallocHost(&remain_host_, sizeof(int)), "cudaMallocHost");
    ck(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device), "attr");
    for (auto k : {mfb::mfsim_engine_kernel<false>, mfb::mfsim_engine_kernel<true>})
      ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024),
         "smem attr");
    for (auto k : {mfb::mfsim_gang_kernel<false>, mfb::mfsim_gang_kernel<true>})
      ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024),
         "smem attr");
    // warps per lock-step gang: 32 (one gang per SM) measured +13 % over the
    // one-warp kernel on the bench workload (profiles/r02_gang_ab.txt)
    if (const char* g = getenv("MFSIM_GANG")) gang_ = atoi(g);
    if (gang_ < 1) gang_ = 1;
    if (gang_ > 32) gang_ = 32;
    if (const char* g = getenv("MFSIM_GANG_MIN")) gang_min_ = atoi(g);  // tests: force small batches
    // deep per-warp call chains (noinline handlers) need more than the default
    ck(cudaDeviceSetLimit(cudaLimitStackSize, 4096), "stack limit");
  }
  ~CudaBackend() override {
    cudaFree(counter_);
    cudaFreeHost(remain_host_);
    cudaEventDestroy(e0_);
    cudaEventDestroy(e1_);
    cudaStreamDestroy(own_);
  }
  const char* name() const override { return "cuda-sm100a"; }
  void* dev_alloc(size_t n) override {
    void* p = nullptr;
    ck(cudaMalloc(&p, n), "cudaMalloc");
    return p;
  }
  void dev_free(void* p) override { cudaFree(p); }
  void* host_alloc(size_t n) override {
    void* p = nullptr;
    ck(cudaMallocHost(&p, n), "cudaMallocHost");
    return p;
  }
  void host_free(void* p) override { cudaFreeHost(p); }
  void h2d(void* d, const void* h, size_t n) override {
    if (n) ck(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, stream_), "H2D");
  }
  void d2h(void* h, const void* d, size_t n) override {
    if (n) ck(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, stream_), "D2H");
  }
  void launch(const mfb::Inst* d, const int* order, int n, const LaunchHint& hint,
              long long budget, long long slice_ns, int active) override {
    const mfb::SmemPlan plan = mfb::make_plan(hint.nlinks);
    // lock step pays off only when every SM holds a full gang: a batch of a
    // few (large) instances keeps one warp per instance, spread over the SMs
    if (active <= 0 || active > n) active = n;
    if (gang_ > 1) {
      // one gang block per SM of as many warps as the running instances fill
      // (up to MFSIM_GANG); thinner than kMinGang warps the one-warp kernel is used
      const bool forced = gang_min_ >= 0 && active >= gang_min_;
      const int w = forced ? gang_ : std::min(gang_, active / sms_);
      if (forced || w >= kMinGang) {
        launch_gang(d, order, n, hint, budget, slice_ns, plan, w);
        return;
      }
    }
    int per_sm = 0;
    // the lean kernel unless the batch holds Aalo instances (extension code compiled out)
    auto kern = hint.aalo ? mfb::mfsim_engine_kernel<true> : mfb::mfsim_engine_kernel<false>;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32,
                                                     plan.bytes),
       "occupancy");
    if (per_sm < 1) per_sm = 1;
    // one wave of one-warp blocks lands round-robin over the SMs: with `active`
    // instances left, ceil(active / SMs) warps per SM keep them on distinct SMs
    const int want = (active + sms_ - 1) / sms_;
    if (want < per_sm) per_sm = want > 0 ? want : 1;
    int grid = sms_ * per_sm;
    ck(cudaMemsetAsync(counter_ + 1, 0, sizeof(int) * kMaxGroups, stream_), "memset");
    ck(cudaEventRecord(e0_, stream_), "event");
    last_kernel_ = "mfsim_engine_kernel";
    kern<<<grid, 32, plan.bytes, stream_>>>(
        d, order, n, hint.groups, sms_, counter_ + 1, plan, budget, slice_ns, counter_);
    ck(cudaGetLastError(), "launch");
    ck(cudaEventRecord(e1_, stream_), "event");
    ++launches_;
    timed_ = true;
    last_grid_ = grid;
  }
  void launch_gang(const mfb::Inst* d, const int* order, int n, const LaunchHint& hint,
                   long long budget, long long slice_ns, const mfb::SmemPlan& plan, int w) {
    auto kern = hint.aalo ? mfb::mfsim_gang_kernel<true> : mfb::mfsim_gang_kernel<false>;
    const int threads = 32 * w;
    const int bytes = plan.bytes * w;
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, bytes), "occupancy");
    if (per_sm < 1) throw DeviceError("gang block does not fit an SM");
    int grid = sms_;  // one gang per SM: its warps share the SM's instruction cache
    const int need = (n + w - 1) / w;
    if (need < grid) grid = need > 0 ? need : 1;
    ck(cudaMemsetAsync(counter_ + 1, 0, sizeof(int) * kMaxGroups, stream_), "memset");
    ck(cudaEventRecord(e0_, stream_), "event");
    last_kernel_ = "mfsim_gang_kernel";
    kern<<<grid, threads, bytes, stream_>>>(d, order, n, hint.groups, sms_, counter_ + 1, plan,
                                             budget, slice_ns, counter_);
    ck(cudaGetLastError(), "launch");
    ck(cudaEventRecord(e1_, stream_), "event");
    ++launches_;
    timed_ = true;
    last_grid_ = grid;
  }
  // instances not yet finished (a fresh batch sets it to n)
  void set_remaining(int n) override {
    *remain_host_ = n;
    ck(cudaMemcpyAsync(counter_, remain_host_, sizeof(int), cudaMemcpyHostToDevice, stream_),
       "remaining");
    ck(cudaStreamSynchronize(stream_), "remaining");
  }
  int remaining() override {
    ck(cudaMemcpyAsync(remain_host_, counter_, sizeof(int), cudaMemcpyDeviceToHost, stream_),
       "remaining");
    ck(cudaStreamSynchronize(stream_), "remaining");
    return *remain_host_;
  }
  void sync() override {
    ck(cudaStreamSynchronize(stream_), "kernel");
    if (timed_) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, e0_, e1_) == cudaSuccess) last_ms_ = ms;
      timed_ = false;
    }
  }
  // any caller stream, including 0 (the legacy default stream)
  void set_stream(void* s) override { stream_ = static_cast<cudaStream_t>(s); }
  double last_kernel_ms() const override { return last_ms_; }
  int kernel_launches() const override { return launches_; }
  const char* last_kernel() const override { return last_kernel_; }

 private:
  int device_;
  cudaStream_t own_ = nullptr, stream_ = nullptr;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
  int* counter_ = nullptr;
  int* remain_host_ = nullptr;
  int sms_ = 148;
  int gang_ = 32;  // warps per block in lock step (MFSIM_GANG; 1 = one-warp kernel)
  static constexpr int kMinGang = 16;  // thinnest gang worth its barrier
  const char* last_kernel_ = "";
  int gang_min_ = -1;  // fewest instances for a gang launch (-1: a full gang per SM)
  int last_grid_ = 0;
  int launches_ = 0;
  bool timed_ = false;
  double last_ms_ = 0.0;
};

}  // namespace

std::unique_ptr<Backend> make_backend(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw DeviceError("no CUDA device visible: the B200 engine has no CPU fallback");
  if (device < 0 || device >= n) throw DeviceError("CUDA device index out of range");
  return std::make_unique<CudaBackend>(device);
}

}  // namespace mfh
