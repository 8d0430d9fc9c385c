// Host configuration layer: the reference's `section.key = value` format
// (config.hpp:12-40, config.cpp:28-110) and the typed parameter groups read
// from it (engine.cpp:8-47, workload.cpp:30-48, rmlq.cpp:8-27,
// policy_factory.cpp:27-43, topology.cpp:147-165). Same keys, same defaults,
// same validation, same error classes (types.hpp:30-45).
#pragma once
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace mfh {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct WorkloadError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SimError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InternalError : std::logic_error {
  using std::logic_error::logic_error;
};
// CUDA / device failures (no reference counterpart; reported as INTERNAL)
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Config {
 public:
  static Config parse(const std::string& text);
  static Config load(const std::string& path);

  void set(const std::string& key, const std::string& value) { kv_[key] = value; }
  bool has(const std::string& key) const { return kv_.count(key) != 0; }
  std::optional<std::string> raw(const std::string& key) const;

  std::string str(const std::string& key, const std::string& dflt) const;
  double num(const std::string& key, double dflt) const;
  long integer(const std::string& key, long dflt) const;
  bool flag(const std::string& key, bool dflt) const;
  double need_num(const std::string& key) const;

  const std::map<std::string, std::string>& entries() const { return kv_; }

 private:
  double to_double(const std::string& key, const std::string& v) const;
  std::map<std::string, std::string> kv_;
};

// ---- parameter groups

struct CostModel {  // engine.hpp:19-28
  int layers = 4;
  double alpha = 1e-3;
  double beta = 1e-6;
  double kv = 1000;
  double coll = 250;
  double layer_cost(double tokens) const { return alpha + beta * tokens; }
  static CostModel from(const Config& c);
};

struct Layout {  // engine.hpp:31-43
  int units = 1;
  int hosts_per_unit = 2;
  int decode_hosts = 1;
  int host(int unit, int k) const { return unit * hosts_per_unit + k; }
  int lead(int unit) const { return host(unit, 0); }
  int decode(int unit) const { return units * hosts_per_unit + (unit % decode_hosts); }
  int total_hosts() const { return units * hosts_per_unit + decode_hosts; }
  static Layout from(const Config& c);
};

struct RunParams {  // engine.hpp:45-52
  std::optional<double> horizon;
  double horizon_slack = 300.0;
  double tick = 1e-3;
  long max_batch_tokens = 8192;
  long livelock = 1000000;
  static RunParams from(const Config& c);
};

struct WorkloadSpec {  // workload.hpp:31-44
  double rate = 1.0;
  long count = 100;
  double prompt_mean = 2000.0;
  double prompt_sigma = 0.0;
  double reuse_mean = 0.5;
  double reuse_skew = 1.0;
  uint64_t seed = 1;
  std::string trace;
  double slo_mult = 3.0;
  static WorkloadSpec from(const Config& c);
};

struct RmlqParams {  // rmlq.hpp:18-27
  int K = 8;
  double E = 4.0;
  double U = 0.5;
  std::vector<double> thresholds;
  static RmlqParams make(int K, double E, double U);
  static RmlqParams from(const Config& c);
};

struct InterParams {  // rmlq.hpp:56-59
  bool pruning = true;
  double drop_frac = 0.05;
  static InterParams from(const Config& c);
};

}  // namespace mfh
