// TEST-ONLY serial host build of the device engine.
//
// Compiles engine.cuh with the 1-lane SerialLanes group so the CPU test tier
// can exercise the exact engine logic (event order, class construction,
// filling, RMLQ, Algorithm 1) against the oracle without a GPU. It is linked
// into build/libmfsim_emu.so only; the product library libmfsim_b200.so links
// the CUDA backend (engine_kernel.cu) and has no CPU path.
#include <cstdlib>
#include <cstring>

#include "../host/instance.hpp"
#include "engine.cuh"

namespace mfh {

namespace {

class EmuBackend final : public Backend {
 public:
  const char* name() const override { return "host-emulation(test-only)"; }
  void* dev_alloc(size_t n) override { return std::calloc(1, n); }
  void dev_free(void* p) override { std::free(p); }
  void* host_alloc(size_t n) override { return std::calloc(1, n); }
  void host_free(void* p) override { std::free(p); }
  void h2d(void* d, const void* h, size_t n) override {
    if (n) std::memcpy(d, h, n);
  }
  void d2h(void* h, const void* d, size_t n) override {
    if (n) std::memcpy(h, d, n);
  }
  void launch(const mfb::Inst* d, const int*, int n, const LaunchHint&, long long budget,
              long long) override {
    for (int i = 0; i < n; ++i) {
      mfb::Inst local = d[i];
      mfb::Engine<mfb::SerialLanes> eng(local);
      if (eng.run(budget)) --remaining_;
    }
    ++launches_;
  }
  void set_remaining(int n) override { remaining_ = n; }
  int remaining() override { return remaining_; }
  void sync() override {}
  void set_stream(void*) override {}
  double last_kernel_ms() const override { return 0.0; }
  int kernel_launches() const override { return launches_; }

 private:
  int launches_ = 0;
  int remaining_ = 0;
};

}  // namespace

std::unique_ptr<Backend> make_backend(int) { return std::make_unique<EmuBackend>(); }

}  // namespace mfh
