// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// Full-precision trace harness around the UNMODIFIED reference simulator
// (/root/reference/proj/src/core, compiled in place by oracle/Makefile into
// oracle/_ref/libmfsim_ref.so). It exposes a small C ABI so the Python tests
// and bench.py's cpu_baseline leg can run the reference on the same inputs as
// the B200 engine and compare bit patterns, which the reference itself only
// prints at %.9g (metrics.cpp:77-81).
//
//   * ref_run_config : mirrors run_simulation (sim_api.cpp:8-35) but keeps the
//                      RunResult (engine.hpp:107-113) and counts decide() calls
//                      with a forwarding scheduler (pattern of
//                      test_engine.cpp:295-315).
//   * ref_run_manual : builds a manual instance (engine.hpp:124-133) from the
//                      text spec shared with the B200 host (see
//                      paper_2603_17456_b200/csrc/host/manual_spec.cpp).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "core/baselines.hpp"
#include "core/engine.hpp"
#include "core/metrics.hpp"
#include "core/rmlq.hpp"
#include "core/scheduler.hpp"
#include "core/sim_api.hpp"
#include "core/workload.hpp"

using namespace mfsim;

namespace {

struct CountingSched : Scheduler {
  Scheduler& inner;
  long decides = 0;
  explicit CountingSched(Scheduler& s) : inner(s) {}
  const char* name() const override { return inner.name(); }
  PolicyDecision decide(const SchedView& v) override {
    ++decides;
    return inner.decide(v);
  }
  void on_flow_released(Flow& f, const SchedView& v) override { inner.on_flow_released(f, v); }
  void on_layer_boundary(BatchId b, const SchedView& v) override { inner.on_layer_boundary(b, v); }
  bool on_promotion_tick(BatchId b, const SchedView& v) override {
    return inner.on_promotion_tick(b, v);
  }
  void on_batch_event(const SchedView& v) override { inner.on_batch_event(v); }
  bool wants_promotion_ticks() const override { return inner.wants_promotion_ticks(); }
  long pruned_count() const override { return inner.pruned_count(); }
  std::vector<RequestId> take_newly_pruned() override { return inner.take_newly_pruned(); }
};

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

char* dupstr(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

struct ref_result {
  long events;
  long steps;
  long pruned_count;
  int n_req;
  int n_flows;
  int n_coflows;
  int n_batches;
  double t_run_s;    // Engine::run wall time
  double t_setup_s;  // workload generation + derive_slos
  double* req_arrival;
  double* req_deadline;
  double* req_done;  // NaN when unfinished
  unsigned char* req_pruned;
  double* req_stall;
  int* req_batch;
  double* flow_finish;  // -1 (kNoTime) when unfinished
  int* flow_band;       // final priority band / level
  int* flow_level;
  double* cof_release;
  double* cof_done;
  double* cof_stall;
  double* pipe_done;  // per batch
  char* summary_json;
  char* requests_csv;
  int err;            // 0 ok, else mfsim.h error code
  char errmsg[512];
};

void ref_free(ref_result* r) {
  if (!r) return;
  std::free(r->req_arrival);
  std::free(r->req_deadline);
  std::free(r->req_done);
  std::free(r->req_pruned);
  std::free(r->req_stall);
  std::free(r->req_batch);
  std::free(r->flow_finish);
  std::free(r->flow_band);
  std::free(r->flow_level);
  std::free(r->cof_release);
  std::free(r->cof_done);
  std::free(r->cof_stall);
  std::free(r->pipe_done);
  std::free(r->summary_json);
  std::free(r->requests_csv);
  std::free(r);
}

}  // extern "C"

namespace {

void fill(ref_result* out, const Engine& eng, const RunResult& res, long steps,
          const std::string& policy, long seed, double rate) {
  out->events = res.events;
  out->steps = steps;
  out->pruned_count = res.pruned_count;
  out->n_req = static_cast<int>(res.requests.size());
  out->n_flows = static_cast<int>(res.flow_finish.size());
  out->n_coflows = static_cast<int>(res.coflows.size());
  out->n_batches = static_cast<int>(eng.batches().size());
  std::vector<double> arr, dl, done, stall, pdone;
  std::vector<unsigned char> pr;
  std::vector<int> rb;
  for (const RequestRow& r : res.requests) {
    arr.push_back(r.arrival);
    dl.push_back(r.deadline);
    done.push_back(r.done ? *r.done : std::nan(""));
    pr.push_back(r.pruned ? 1 : 0);
    stall.push_back(r.stall);
  }
  for (const Request& r : eng.requests()) rb.push_back(r.batch);
  std::vector<int> band, level;
  for (const Flow& f : eng.flows()) {
    band.push_back(static_cast<int>(f.priority.band));
    level.push_back(f.priority.level);
  }
  std::vector<double> cr, cd, cs;
  for (const CoflowRow& c : res.coflows) {
    cr.push_back(c.release);
    cd.push_back(c.done);
    cs.push_back(c.stall);
  }
  for (const BatchPipeline& p : eng.pipelines()) pdone.push_back(p.done_t);
  out->req_arrival = dup(arr);
  out->req_deadline = dup(dl);
  out->req_done = dup(done);
  out->req_pruned = dup(pr);
  out->req_stall = dup(stall);
  out->req_batch = dup(rb);
  out->flow_finish = dup(res.flow_finish);
  out->flow_band = dup(band);
  out->flow_level = dup(level);
  out->cof_release = dup(cr);
  out->cof_done = dup(cd);
  out->cof_stall = dup(cs);
  out->pipe_done = dup(pdone);
  MetricsReport m = build_metrics(res);
  out->summary_json = dupstr(summary_json(m, policy, seed, rate));
  out->requests_csv = dupstr(requests_csv(m));
}

template <typename Fn>
int guarded(ref_result* out, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    out->err = 2;
    std::snprintf(out->errmsg, sizeof out->errmsg, "%s", e.what());
  } catch (const WorkloadError& e) {
    out->err = 3;
    std::snprintf(out->errmsg, sizeof out->errmsg, "%s", e.what());
  } catch (const IoError& e) {
    out->err = 4;
    std::snprintf(out->errmsg, sizeof out->errmsg, "%s", e.what());
  } catch (const SimError& e) {
    out->err = 5;
    std::snprintf(out->errmsg, sizeof out->errmsg, "%s", e.what());
  } catch (const std::exception& e) {
    out->err = 6;
    std::snprintf(out->errmsg, sizeof out->errmsg, "%s", e.what());
  }
  return out->err;
}

using Clock = std::chrono::steady_clock;

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep)) out.push_back(cur);
  return out;
}

double num(const std::string& s) {
  if (s == "-") return kNoTime;
  return std::strtod(s.c_str(), nullptr);
}

}  // namespace

extern "C" {

// Run one simulation from `key = value` config text (sim_api.cpp:8-35).
int ref_run_config(const char* config_text, ref_result** out_p) {
  auto* out = static_cast<ref_result*>(std::calloc(1, sizeof(ref_result)));
  *out_p = out;
  return guarded(out, [&] {
    Config cfg = Config::from_string(config_text);
    auto t0 = Clock::now();
    PolicyKind kind = parse_policy(cfg.get_string("policy", "fs"));
    Topology topo = build_topology(cfg);
    ClusterLayout layout = ClusterLayout::from_config(cfg);
    CostModel cost = CostModel::from_config(cfg);
    EngineParams params = EngineParams::from_config(cfg);
    WorkloadSpec spec = WorkloadSpec::from_config(cfg);
    std::vector<Request> requests;
    if (!spec.trace_path.empty())
      requests = load_trace(spec.trace_path, layout, cost);
    else
      requests = generate_workload(spec, layout, cost, params.max_batch_tokens);
    derive_slos(requests, spec.slo_multiplier, topo, layout, cost, params);
    auto sched = make_scheduler(kind, cfg);
    CountingSched counting(*sched);
    Engine engine(topo, counting, params);
    engine.load_workload(std::move(requests), layout, cost);
    auto t1 = Clock::now();
    RunResult res = engine.run();
    auto t2 = Clock::now();
    out->t_setup_s = std::chrono::duration<double>(t1 - t0).count();
    out->t_run_s = std::chrono::duration<double>(t2 - t1).count();
    fill(out, engine, res, counting.decides, policy_name(kind), static_cast<long>(spec.seed),
         spec.rate_rps);
  });
}

// Deadlines only (workload generation + derive_slos), for input parity.
int ref_derive_deadlines(const char* config_text, ref_result** out_p) {
  auto* out = static_cast<ref_result*>(std::calloc(1, sizeof(ref_result)));
  *out_p = out;
  return guarded(out, [&] {
    Config cfg = Config::from_string(config_text);
    Topology topo = build_topology(cfg);
    ClusterLayout layout = ClusterLayout::from_config(cfg);
    CostModel cost = CostModel::from_config(cfg);
    EngineParams params = EngineParams::from_config(cfg);
    WorkloadSpec spec = WorkloadSpec::from_config(cfg);
    std::vector<Request> requests;
    if (!spec.trace_path.empty())
      requests = load_trace(spec.trace_path, layout, cost);
    else
      requests = generate_workload(spec, layout, cost, params.max_batch_tokens);
    derive_slos(requests, spec.slo_multiplier, topo, layout, cost, params);
    std::vector<double> arr, dl;
    for (const Request& r : requests) {
      arr.push_back(r.arrival);
      dl.push_back(r.deadline);
    }
    out->n_req = static_cast<int>(requests.size());
    out->req_arrival = dup(arr);
    out->req_deadline = dup(dl);
  });
}

// Manual instance from the line-oriented spec (see manual_spec.cpp):
//   policy <name> | set <key> <value> | param <field> <value>
//   node <role> | link <from> <to> <cap> | duplex <a> <b> <cap>
//   request <arrival> <deadline> [prompt_tokens]
//   batch <admit_at> <members,..|-> <costs,..|->
//   flow <batch> <request> <stage> <src> <dst> <size> <target> <release|-> <deadline|->
int ref_run_manual(const char* spec_text, ref_result** out_p) {
  auto* out = static_cast<ref_result*>(std::calloc(1, sizeof(ref_result)));
  *out_p = out;
  return guarded(out, [&] {
    std::istringstream in(spec_text);
    std::string line;
    Config cfg;
    std::string policy = "fs";
    EngineParams params;
    Topology topo;
    struct Op {
      std::vector<std::string> tok;
    };
    std::vector<Op> ops;
    bool routes = false;
    while (std::getline(in, line)) {
      if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
      std::istringstream ls(line);
      std::vector<std::string> tok;
      std::string t;
      while (ls >> t) tok.push_back(t);
      if (tok.empty()) continue;
      const std::string& k = tok[0];
      if (k == "policy") {
        policy = tok.at(1);
      } else if (k == "set") {
        cfg.set(tok.at(1), tok.at(2));
      } else if (k == "param") {
        const std::string& f = tok.at(1);
        double v = std::strtod(tok.at(2).c_str(), nullptr);
        if (f == "promotion_tick") params.promotion_tick = v;
        else if (f == "horizon") params.horizon = v;
        else if (f == "horizon_slack") params.horizon_slack = v;
        else if (f == "max_batch_tokens") params.max_batch_tokens = static_cast<long>(v);
        else if (f == "livelock_events") params.livelock_events = static_cast<long>(v);
        else throw ConfigError("unknown param " + f);
      } else if (k == "node") {
        std::string role = tok.size() > 1 ? tok[1] : "prefill";
        NodeRole r = role == "decode" ? NodeRole::DecodeGPU
                     : role == "switch" ? NodeRole::Switch : NodeRole::PrefillGPU;
        topo.add_node(r, "n");
      } else if (k == "link") {
        topo.add_link(std::stoi(tok.at(1)), std::stoi(tok.at(2)), num(tok.at(3)));
      } else if (k == "duplex") {
        topo.add_duplex(std::stoi(tok.at(1)), std::stoi(tok.at(2)), num(tok.at(3)));
      } else {
        ops.push_back({tok});
      }
    }
    topo.build_routes();
    routes = true;
    (void)routes;
    PolicyKind kind = parse_policy(policy);
    auto sched = make_scheduler(kind, cfg);
    CountingSched counting(*sched);
    Engine eng(topo, counting, params);
    for (const Op& op : ops) {
      const auto& tok = op.tok;
      if (tok[0] == "request") {
        Request r;
        r.arrival = num(tok.at(1));
        r.deadline = std::strtod(tok.at(2).c_str(), nullptr);
        if (tok.size() > 3) r.prompt_tokens = std::stol(tok[3]);
        eng.add_request(r);
      } else if (tok[0] == "batch") {
        std::vector<RequestId> members;
        std::vector<double> costs;
        if (tok.at(2) != "-")
          for (auto& s : split(tok[2], ',')) members.push_back(std::stoi(s));
        if (tok.at(3) != "-")
          for (auto& s : split(tok[3], ',')) costs.push_back(std::strtod(s.c_str(), nullptr));
        eng.add_manual_batch(members, costs, num(tok.at(1)));
      } else if (tok[0] == "flow") {
        Stage st = tok.at(3) == "reuse" ? Stage::Reuse
                   : tok[3] == "collective" ? Stage::Collective : Stage::P2D;
        std::optional<SimTime> rel, dl;
        if (tok.at(8) != "-") rel = std::strtod(tok[8].c_str(), nullptr);
        if (tok.at(9) != "-") dl = std::strtod(tok[9].c_str(), nullptr);
        eng.add_manual_flow(std::stoi(tok.at(1)), std::stoi(tok.at(2)), st, std::stoi(tok.at(4)),
                            std::stoi(tok.at(5)), std::strtod(tok.at(6).c_str(), nullptr),
                            std::stoi(tok.at(7)), rel, dl);
      } else {
        throw ConfigError("unknown manual spec op " + tok[0]);
      }
    }
    auto t1 = Clock::now();
    RunResult res = eng.run();
    out->t_run_s = std::chrono::duration<double>(Clock::now() - t1).count();
    fill(out, eng, res, counting.decides, policy_name(kind), 0, 0.0);
  });
}

// Raw allocator entry point for the K3 parity cases (allocator.cpp:28-126):
// a star of `hosts` hosts with capacity `cap`; flows given as src/dst pairs;
// classes as a flat list with class ids; optional caps (NaN = uncapped).
int ref_allocate_star(int hosts, double cap, int nflows, const int* src, const int* dst,
                      const int* cls_of, int ncls, const double* caps, double* rates_out) {
  try {
    Topology topo = build_star(hosts, cap);
    std::vector<Flow> flows(nflows);
    for (int i = 0; i < nflows; ++i) {
      flows[i].id = i;
      flows[i].src = src[i];
      flows[i].dst = dst[i];
      flows[i].size = flows[i].remaining = 1.0;
      flows[i].state = FlowState::Active;
    }
    PriorityClasses classes(ncls);
    for (int i = 0; i < nflows; ++i) classes[cls_of[i]].push_back(i);
    RateCaps rc;
    bool has = false;
    if (caps)
      for (int i = 0; i < nflows; ++i)
        if (!std::isnan(caps[i])) {
          rc[i] = caps[i];
          has = true;
        }
    auto a = allocate_rates(flows, topo, classes, has ? &rc : nullptr, 0.0);
    for (int i = 0; i < nflows; ++i) rates_out[i] = a.rate(i);
    return 0;
  } catch (...) {
    return 6;
  }
}

}  // extern "C"
