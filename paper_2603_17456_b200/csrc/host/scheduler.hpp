// Scheduler-policy interface on the host, mirroring the reference plugin ABI
// (scheduler.hpp:15-66, policy_factory.cpp:7-43): the same five policy names,
// the same factory keys (mfs.K/E/U, inter.enable_pruning,
// inter.drop_budget_frac) and the same hook set. What changed is where the
// hooks execute: decide() / on_flow_released / on_layer_boundary /
// on_promotion_tick / on_batch_event run inside the device event loop
// (csrc/device/engine.cuh); a host Scheduler object describes its policy to the
// device through configure().
#pragma once
#include <memory>
#include <string>

#include "../device/layout.h"
#include "config.hpp"

namespace mfh {

enum class PolicyKind { FairShare, SJF, EDF, Karuna, MFS, Aalo, Varys };

// fs|sjf|edf|karuna|mfs, plus the extensions aalo and varys (no reference counterpart)
PolicyKind parse_policy(const std::string& name);
const char* policy_name(PolicyKind k);

class Scheduler {
 public:
  virtual ~Scheduler() = default;
  virtual const char* name() const = 0;
  virtual PolicyKind kind() const = 0;
  virtual bool wants_promotion_ticks() const { return false; }
  // Fill the device-side policy block of an instance.
  virtual void configure(mfb::InstParams& p) const;
};

class FairShareScheduler : public Scheduler {  // baselines.cpp:46-51
 public:
  const char* name() const override { return "fs"; }
  PolicyKind kind() const override { return PolicyKind::FairShare; }
};

class SjfScheduler : public Scheduler {  // baselines.cpp:23-57
 public:
  const char* name() const override { return "sjf"; }
  PolicyKind kind() const override { return PolicyKind::SJF; }
};

class EdfScheduler : public Scheduler {  // baselines.cpp:59-90
 public:
  const char* name() const override { return "edf"; }
  PolicyKind kind() const override { return PolicyKind::EDF; }
};

class KarunaScheduler : public Scheduler {  // baselines.cpp:92-135
 public:
  const char* name() const override { return "karuna"; }
  PolicyKind kind() const override { return PolicyKind::Karuna; }
};

class MfsScheduler : public Scheduler {  // rmlq.hpp:61-101
 public:
  MfsScheduler(RmlqParams rmlq, InterParams inter) : rmlq_(std::move(rmlq)), inter_(inter) {}
  const char* name() const override { return "mfs"; }
  PolicyKind kind() const override { return PolicyKind::MFS; }
  bool wants_promotion_ticks() const override { return true; }
  void configure(mfb::InstParams& p) const override;
  const RmlqParams& rmlq() const { return rmlq_; }

 private:
  RmlqParams rmlq_;
  InterParams inter_;
};

// Extension (BASELINE configs[1] "Varys/Aalo-style
// coflow"): Aalo's D-CLAS. Coflow = (batch, target layer, stage); queue from
// attained service against thresholds Q0 * E^i (aalo.Q0, aalo.E, aalo.K);
// one priority class per coflow, FIFO (batch-major) within a queue. The
// reference has no such policy: its oracle is oracle/mfsim_oracle.c (policy 5).
class AaloScheduler : public Scheduler {
 public:
  AaloScheduler(int K, double E, double Q0) : K_(K), E_(E), Q0_(Q0) {}
  const char* name() const override { return "aalo"; }
  PolicyKind kind() const override { return PolicyKind::Aalo; }
  void configure(mfb::InstParams& p) const override;
  static std::unique_ptr<AaloScheduler> from(const Config& cfg);

 private:
  int K_;
  double E_, Q0_;
};

// Extension: Varys-style SEBF + MADD (clairvoyant coflow scheduling). Coflows
// as in Aalo; one class per coflow ordered by its effective bottleneck
// Gamma = max over links of (remaining bytes over the link) / capacity; every
// member capped at remaining / Gamma (MADD). Oracle: mfsim_oracle.c policy 6.
class VarysScheduler : public Scheduler {
 public:
  const char* name() const override { return "varys"; }
  PolicyKind kind() const override { return PolicyKind::Varys; }
};

std::unique_ptr<Scheduler> make_scheduler(PolicyKind kind, const Config& cfg);

}  // namespace mfh
