// Instance construction and execution on the host side of the C ABI.
//
// A simulation instance is everything Engine::run (engine.cpp:595-657) needs:
// the fabric's link capacities and routes, the request list with derived
// deadlines, and the policy block. Workload-mode instances are built from a
// Config exactly as run_simulation does (sim_api.cpp:8-35); manual instances
// (engine.hpp:124-133) come from a line-oriented spec. Instances are packed
// into one device arena and executed by a Backend (CUDA for the product).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../device/layout.h"
#include "config.hpp"
#include "scheduler.hpp"
#include "topology.hpp"
#include "workload.hpp"

namespace mfh {

// First-attempt capacities; they match the per-warp shared-memory plan of the
// kernel, so instances that stay within them run with their hot state on chip.
// An instance that outgrows one is re-run with a larger, global-memory bound.
constexpr int kDefaultActive = 1024;  // first-attempt active-set capacity
constexpr int kSmemEvents = 64;       // event pool staged on chip
constexpr int kSmemLinks = 1024;      // link -> slot map staged on chip
#ifndef MF_SMEM_SLOTS
#define MF_SMEM_SLOTS 96
#endif
// per-slot filling state staged on chip: 96 slots let 32 warps per SM stay
// resident (the 64-register limit) and cost nothing per warp against 128 or
// 256 (A/B, profiles/r01_ab_engine_builds.txt calls 9 and 11)
constexpr int kSmemSlots = MF_SMEM_SLOTS;

struct LaunchHint {
  int rmax = 1;    // longest route of any instance
  int nlinks = 1;  // most links of any instance
  int groups = 1;  // claim groups (one per policy): order[n .. n+groups] holds their offsets
  bool aalo = false;  // some instance runs an extension policy (aalo / varys: the kernel variant with their code)
};
constexpr int kMaxGroups = 8;

// Device execution backend: the product build links the CUDA backend only.
class Backend {
 public:
  virtual ~Backend() = default;
  virtual const char* name() const = 0;
  virtual void* dev_alloc(size_t bytes) = 0;
  virtual void dev_free(void* p) = 0;
  virtual void* host_alloc(size_t bytes) = 0;  // pinned staging
  virtual void host_free(void* p) = 0;
  virtual void h2d(void* dst, const void* src, size_t n) = 0;  // stream-ordered
  virtual void d2h(void* dst, const void* src, size_t n) = 0;
  // order: device array, a permutation of [0, n) giving the claim order, in
  // hint.groups contiguous groups whose offsets follow at order[n..n+groups];
  // budget: events per instance in this launch (<= 0: run to completion)
  // active: instances not finished yet (the host's last count; sizes the grid so
  // that a few remaining instances land on distinct SMs)
  virtual void launch(const mfb::Inst* d_insts, const int* order, int n, const LaunchHint& hint,
                      long long budget, long long slice_ns, int active) = 0;
  virtual void set_remaining(int n) = 0;
  virtual int remaining() = 0;
  virtual void sync() = 0;
  virtual void set_stream(void* stream) = 0;
  virtual double last_kernel_ms() const = 0;
  virtual int kernel_launches() const = 0;
  virtual const char* last_kernel() const = 0;
};
std::unique_ptr<Backend> make_backend(int device);

// Fabric-derived tables shared by all instances on the same topology/layout.
struct TopoImage {
  std::vector<double> cap;
  RouteTable routes;
  std::vector<int> rt_reuse, rt_p2d, rt_coll;
  int lr_cap = 1;  // max distinct links one request's load touches
  int hosts = 0;   // hosts of the fabric
};
std::shared_ptr<TopoImage> build_topo_image(const Fabric& f, const Layout& lay);

struct ManualImage;  // manual-mode state image (manual_spec.cpp)

struct InstanceInput {
  mfb::InstParams p{};
  std::shared_ptr<TopoImage> topo;
  std::vector<HostRequest> reqs;
  std::shared_ptr<ManualImage> manual;  // null = workload mode
  std::string policy;
  long seed = 0;
  double rate = 0.0;
  double slo_mult = 3.0;
  bool deadlines_ready = false;
  int a_cap = 0;  // active-set capacity (0 = default)
  int e_boost = 0;
};

struct InstanceOutput {
  long long out[mfb::OUT_N] = {};
  std::vector<double> ttft;  // -1 = unfinished
  std::vector<uint8_t> pruned;
  std::vector<double> stall;
  std::vector<int> rbatch;
  std::vector<double> c_rel, c_done, c_stall;  // detail >= 1
  std::vector<double> f_fin;                   // detail >= 2
  std::vector<uint8_t> f_band, f_level;
  std::vector<double> b_done;
};

// Workload-mode instance from config keys (policy, fabric, layout, workload).
// Deadlines are NOT derived here; see derive_deadlines.
InstanceInput workload_instance(const Config& cfg);

// derive_slos (workload.cpp:177-217) for many instances at once: one isolated
// single-request FS run per distinct (tokens, reuse bits, unit, source) key,
// all executed in a single device launch.
void derive_deadlines(Backend& be, const std::vector<InstanceInput*>& insts);

InstanceInput manual_instance(const std::string& spec);

// request inputs regardless of mode (manual images keep their own arrays)
double request_arrival(const InstanceInput& in, int r);
double request_deadline(const InstanceInput& in, int r);

// A packed, device-resident set of instances.
class Batch {
 public:
  Batch(Backend& be, std::vector<InstanceInput> inputs);
  ~Batch();
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;

  void upload();          // H2D of all inputs (stream-ordered) + reset()
  void upload_inputs();   // H2D of the inputs only (state untouched)
  void reset();           // every instance back to its initial state (fresh run)
  // device event loops (stream-ordered): at most `budget` events per instance
  // and, with slice_ns > 0, until that much device time has passed
  void launch(long long budget = 0, long long slice_ns = 0);
  int remaining();        // instances not finished yet (synchronises)
  void download(int detail);  // D2H; detail 0 requests, 1 +coflows, 2 +flows/batches
  // upload + launch + download, re-running instances that hit a capacity
  // bound with doubled capacities
  void run(int detail);

  int size() const { return static_cast<int>(inputs_.size()); }
  const InstanceInput& input(int i) const { return inputs_[i]; }
  const InstanceOutput& output(int i) const;  // per-request columns parsed on first read
  size_t input_bytes() const { return in_bytes_; }
  size_t output_bytes(int detail) const;
  size_t device_bytes() const { return in_bytes_ + st_bytes_ + out_bytes_; }

 private:
  void pack();
  void release();
  Backend& be_;
  std::vector<InstanceInput> inputs_;
  mutable std::vector<InstanceOutput> outputs_;
  mutable std::vector<char> parsed_;  // per-request columns copied out of out_host_
  std::vector<mfb::Inst> desc_;
  char* in_host_ = nullptr;
  char* out_host_ = nullptr;
  char* in_dev_ = nullptr;
  char* st_dev_ = nullptr;
  char* out_dev_ = nullptr;
  mfb::Inst* desc_dev_ = nullptr;
  int* order_dev_ = nullptr;
  int* phase_dev_ = nullptr;
  int remaining_ = 0;  // instances not finished at the last remaining() / reset()
  std::vector<int> order_;
  LaunchHint hint_;
  size_t in_bytes_ = 0, st_bytes_ = 0, out_bytes_ = 0;
  struct OutView {
    size_t out, ttft, pruned, stall, rbatch;
  };
  std::vector<OutView> oview_;
};

// errors: translate a device status into the reference's exception classes
void raise_status(long long status, long long check);
const char* check_name(int chk);

}  // namespace mfh
