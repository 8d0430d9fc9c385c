// Request synthesis on the host. The inputs must be bit-identical to the
// reference's (workload.cpp:11-175): same splitmix64 stream, same glibc libm
// transcendentals (log1p, log, sqrt, cos, exp, pow, llround), same operation
// order, compiled without FP contraction.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "config.hpp"

namespace mfh {

struct HostRequest {
  double arrival = 0.0;
  long tokens = 0;
  double reuse = 0.0;
  int unit = 0;
  int source = -1;
  int layers = 0;
  double deadline = 0.0;  // absolute; +inf until derive_slos
};

struct SplitMix {  // workload.hpp:14-29
  uint64_t state;
  explicit SplitMix(uint64_t seed) : state(seed) {}
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
  double exponential(double rate);
  double lognormal(double mean, double sigma);
};

std::vector<HostRequest> synthesize(const WorkloadSpec& spec, const Layout& layout,
                                    const CostModel& cost, long max_batch_tokens);

// arrival_s,prompt_tokens,reuse_fraction,source_unit (workload.cpp:132-175)
std::vector<HostRequest> read_trace(const std::string& path, const Layout& layout,
                                    const CostModel& cost);

}  // namespace mfh
