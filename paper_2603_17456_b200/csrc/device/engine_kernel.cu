// sm_100a entry point and CUDA backend.
//
// mfsim_engine_kernel is a persistent grid: each warp repeatedly claims the
// next unclaimed simulation instance (atomic work counter, so long-running
// instances -- Karuna, overload -- do not stall a static partition) and runs
// that instance's entire event loop on the device (engine.cuh). Grid =
// blocks_per_sm x 148 SMs.
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../host/instance.hpp"
#include "engine.cuh"

namespace mfb {

constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    mfsim_engine_kernel(const Inst* __restrict__ insts, int n, int* __restrict__ next) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int i = 0;
    if (lane == 0) i = atomicAdd(next, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n) return;
    Engine<WarpLanes> eng(insts[i]);
    eng.run();
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
    ck(cudaMalloc(&counter_, sizeof(int)), "cudaMalloc counter");
    int sms = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mfb::mfsim_engine_kernel,
                                                     32 * mfb::kWarpsPerBlock, 0),
       "occupancy");
    if (per_sm < 1) per_sm = 1;
    grid_ = sms * per_sm;
    // deep per-warp call chains (noinline handlers) need more than the default
    ck(cudaDeviceSetLimit(cudaLimitStackSize, 16384), "stack limit");
  }
  ~CudaBackend() override {
    cudaFree(counter_);
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
  void launch(const mfb::Inst* d, int n) override {
    ck(cudaMemsetAsync(counter_, 0, sizeof(int), stream_), "memset");
    int grid = grid_;
    const int warps_needed = (n + mfb::kWarpsPerBlock - 1) / mfb::kWarpsPerBlock;
    if (warps_needed < grid) grid = warps_needed > 0 ? warps_needed : 1;
    ck(cudaEventRecord(e0_, stream_), "event");
    mfb::mfsim_engine_kernel<<<grid, 32 * mfb::kWarpsPerBlock, 0, stream_>>>(d, n, counter_);
    ck(cudaGetLastError(), "launch");
    ck(cudaEventRecord(e1_, stream_), "event");
    ++launches_;
    timed_ = true;
  }
  void sync() override {
    ck(cudaStreamSynchronize(stream_), "kernel");
    if (timed_) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, e0_, e1_) == cudaSuccess) last_ms_ = ms;
      timed_ = false;
    }
  }
  void set_stream(void* s) override { stream_ = s ? static_cast<cudaStream_t>(s) : own_; }
  double last_kernel_ms() const override { return last_ms_; }
  int kernel_launches() const override { return launches_; }

 private:
  int device_;
  cudaStream_t own_ = nullptr, stream_ = nullptr;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
  int* counter_ = nullptr;
  int grid_ = 148;
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
