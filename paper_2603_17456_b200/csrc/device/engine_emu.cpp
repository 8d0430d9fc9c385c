// TEST-ONLY serial host build of the device engine.
//
// Compiles engine.cuh with the 1-lane SerialLanes group so the CPU test tier
// can exercise the exact engine logic (event order, class construction,
// filling, RMLQ, Algorithm 1) against the oracle without a GPU. It is linked
// into build/libmfsim_emu.so only; the product library libmfsim_b200.so links
// the CUDA backend (engine_kernel.cu) and has no CPU path.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

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
              long long, int) override {
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
  const char* last_kernel() const override { return "host-emulation"; }

 private:
  int launches_ = 0;
  int remaining_ = 0;
};

}  // namespace

std::unique_ptr<Backend> make_backend(int) { return std::make_unique<EmuBackend>(); }

}  // namespace mfh

// TEST-ONLY: one allocate_rates call (allocator.cpp:28-126) through the
// engine's filling code on a star fabric (host h: up link 2h, down link
// 2h+1), the counterpart of oracle/ref_harness.cpp ref_allocate_star.
// caps[i] = NaN: flow i uncapped. variant 0: per-link filling
// (allocate_generic), 1: link-slot filling (allocate_slots).
extern "C" int mfsim_emu_allocate_star(int hosts, double cap, int n, const int* src, const int* dst,
                                       const int* cls_of, int ncls, const double* caps, int variant,
                                       double* rates_out) {
  using namespace mfb;
  const int nl = 2 * hosts, rm = 2;
  if (n <= 0 || ncls <= 0 || hosts <= 0) return 1;
  std::vector<double> capv(nl, cap), lres(nl, cap), srate(n), scap(n, MF_INF), slres(nl);
  std::vector<int> lcnt(nl, 0), ord, cls(ncls + 1, 0), ul(n), afid(n), hk(n), hidx(n);
  std::vector<int> slcnt(nl, 0), slmb(nl), slend(nl);
  std::vector<unsigned short> arl(n * rm), asl(n * rm), stl(nl), sllink(nl), sltl(nl), slsat(nl),
      cmem(n * rm);
  std::vector<uint8_t> arn(n, (uint8_t)rm);
  std::vector<unsigned> frz((n + 31) / 32 + 1);
  std::vector<unsigned long long> xhi(n), xlo(n);
  bool has_caps = false;
  for (int i = 0; i < n; ++i) {
    if (src[i] == dst[i] || cls_of[i] < 0 || cls_of[i] >= ncls) return 1;
    afid[i] = i;
    arl[i * rm] = asl[i * rm] = (unsigned short)(2 * src[i]);
    arl[i * rm + 1] = asl[i * rm + 1] = (unsigned short)(2 * dst[i] + 1);
    if (caps && !std::isnan(caps[i])) {
      scap[i] = caps[i];
      has_caps = true;
    }
  }
  for (int c = 0; c < ncls; ++c) {  // classes[c] in flow-id order (ref_allocate_star)
    cls[c] = (int)ord.size();
    for (int i = 0; i < n; ++i)
      if (cls_of[i] == c) ord.push_back(i);
  }
  cls[ncls] = n;
  for (int j = 0; j < nl; ++j) sllink[j] = (unsigned short)j;
  Inst I{};
  I.p.policy = POL_FS;
  I.rmax = rm;
  I.nlinks = nl;
  I.cap = capv.data();
  I.a_fid = afid.data();
  I.a_rl = arl.data();
  I.a_rn = arn.data();
  I.l_res = lres.data();
  I.l_cnt = lcnt.data();
  I.s_rate = srate.data();
  I.s_cap = scap.data();
  I.s_ord = ord.data();
  I.s_cls = cls.data();
  I.s_ul = ul.data();
  I.s_tl = stl.data();
  I.h_keys = hk.data();
  I.f_hidx = hidx.data();
  I.x_hi = xhi.data();
  I.x_lo = xlo.data();
  I.TS_cap = variant == 1 ? nl : 0;
  I.a_sl = asl.data();
  I.sl_link = sllink.data();
  I.sl_res = slres.data();
  I.sl_cnt = slcnt.data();
  I.sl_mb = slmb.data();
  I.sl_end = slend.data();
  I.sl_tl = sltl.data();
  I.sl_sat = slsat.data();
  I.c_mem = cmem.data();
  I.c_frz = frz.data();
  Engine<SerialLanes> eng(I);
  std::memset(&eng.s, 0, sizeof(eng.s));
  eng.s.n_active = n;
  eng.s.sl_hw = nl;
  eng.s.sat_max = 1e-12 * cap;
  if (variant == 1)
    eng.allocate_slots<false>(ncls, has_caps);
  else
    eng.allocate_generic(ncls, has_caps);
  if (eng.s.err) return 5;
  for (int i = 0; i < n; ++i) rates_out[i] = srate[i];
  return 0;
}
