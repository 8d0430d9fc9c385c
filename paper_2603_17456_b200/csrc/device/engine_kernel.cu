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
#include "kernel_common.cuh"

namespace mfb {

// order[0, n): instance ids in claim groups (one per policy), estimated work
// descending within a group; order[n + g] = offset of group g. A warp claims
// from its SM's home group first, then from the others. SMs are mapped onto
// the groups in proportion to their sizes for time-sliced launches (every
// warp busy for the slice) and in proportion to their estimated work,
// order[n + groups + 1 + g], for launches that run to completion (the
// makespan is the most loaded SM's).
template <bool kAalo>
__global__ void __maxnreg__(128)
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
    mfb::gang_kernel_init();
    ck(cudaGetLastError(), "gang smem attr");
    // warps per lock-step gang: 32 (one gang per SM) measured +13 % over the
    // one-warp kernel on the bench workload (profiles/r02_gang_ab.txt)
    if (const char* g = getenv("MFSIM_GANG")) gang_ = atoi(g);
    if (gang_ < 1) gang_ = 1;
    if (gang_ > 32) gang_ = 32;
    if (const char* g = getenv("MFSIM_GANG_MIN")) gang_min_ = atoi(g);  // tests: force small batches
    if (const char* g = getenv("MFSIM_GANG_MINW")) min_gang_ = std::max(2, atoi(g));
    if (const char* g = getenv("MFSIM_GANG_BLOCKS")) gang_blocks_ = std::max(1, atoi(g));
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
      // Gang blocks per SM and warps per gang from the running instances: two
      // gangs of up to 16 warps per SM (a slow warp then holds up half of the
      // SM), else one gang of up to 32, else the one-warp kernel (A/B,
      // profiles/r02_gang_ab.txt: 2x16 +5 % over 1x32 at 4736 instances,
      // 2x9 +8 % over 1x18 at 2800, 1x13 +13 % over one warp each at 2000)
      if (gang_min_ >= 0 && active >= gang_min_) {  // tests: a gang even for small batches
        launch_gang(d, order, n, hint, budget, slice_ns, plan, gang_, 1);
        return;
      }
      for (int b = gang_blocks_; b >= 1; --b) {
        const int w = std::min(std::min(gang_, 32 / b), active / (sms_ * b));
        if (w >= (b > 1 ? min_gang_split_ : min_gang_)) {
          launch_gang(d, order, n, hint, budget, slice_ns, plan, w, b);
          return;
        }
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
                   long long budget, long long slice_ns, const mfb::SmemPlan& plan, int w, int blocks) {
    const int threads = 32 * w;
    const int bytes = plan.bytes * w;
    const int per_sm = mfb::gang_kernel_blocks_per_sm(hint.aalo, threads, bytes);
    if (per_sm < 1) throw DeviceError("gang block does not fit an SM");
    int grid = sms_ * std::min(blocks, per_sm);  // gangs per SM: a gang's warps share the SM's instruction cache
    const int need = (n + w - 1) / w;
    if (need < grid) grid = need > 0 ? need : 1;
    ck(cudaMemsetAsync(counter_ + 1, 0, sizeof(int) * kMaxGroups, stream_), "memset");
    ck(cudaEventRecord(e0_, stream_), "event");
    const int* ord = order;
    last_kernel_ = "mfsim_gang_kernel";
    mfb::gang_kernel_launch(hint.aalo, grid, threads, bytes, stream_, d, ord, n, hint.groups, sms_, counter_ + 1,
                            plan, budget, slice_ns, counter_);
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
  int gang_blocks_ = 2;  // most gang blocks per SM (MFSIM_GANG_BLOCKS)
  int min_gang_split_ = 8;  // thinnest gang when an SM holds two
  int min_gang_ = 12;  // thinnest gang worth its barrier (MFSIM_GANG_MINW; A/B: 13 warps +13 %, 9 warps +1 %)
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
