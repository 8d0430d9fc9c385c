#include "instance.hpp"

#include <mutex>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>
#include <tuple>

namespace mfh {

using namespace mfb;

namespace {

constexpr double kInfD = std::numeric_limits<double>::infinity();
constexpr double kNoTime = -1.0;

int pow2(long n) {
  long p = 1;
  while (p < n) p <<= 1;
  return static_cast<int>(p);
}

// libstdc++ bucket count reached by n single insertions (see engine.cuh)
int hash_buckets(int n) {
  static const int at[] = {0,     13,     29,     59,     127,    257,    541,
                           1109,  2357,   5087,   10273,  20753,  42043,  85229,
                           172933, 351061, 712697, 1447153, 2938679};
  static const int bk[] = {13,    29,     59,     127,    257,    541,     1109,
                           2357,  5087,   10273,  20753,  42043,  85229,   172933,
                           351061, 712697, 1447153, 2938679, 5967347};
  int b = 13;
  for (int i = 0; i < 19; ++i)
    if (n > at[i]) b = bk[i];
  return b;
}

}  // namespace

// ---------------------------------------------------------------- manual mode

struct ManualImage {
  std::vector<double> r_arrival, r_deadline;
  std::vector<long long> r_tokens;
  std::vector<int> r_batch, r_open;
  // batches
  std::vector<std::vector<int>> members;
  std::vector<std::vector<double>> costs;
  std::vector<double> admit_at;
  std::vector<int> b_ffirst, b_fcount;
  // flows
  struct F {
    int req, batch, stage, route, tl, coflow = -1;
    double size, relat, dl;
    bool scripted;
  };
  std::vector<F> flows;
  // per (batch, layer)
  std::vector<std::vector<std::vector<int>>> reuse, p2d;  // [b][layer][...]
  std::vector<std::vector<int>> coll;                     // [b][layer] coflow or -1
  struct C {
    int batch, layer;
    std::vector<int> members;
  };
  std::vector<C> coflows;
  double last_admit = 0.0;
};

namespace {

std::vector<std::string> split_csv(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, ',')) out.push_back(cur);
  return out;
}

double parse_d(const std::string& s) { return std::strtod(s.c_str(), nullptr); }

}  // namespace

// Line-oriented manual instance spec (shared with oracle/ref_harness.cpp):
//   policy <name> | set <key> <value> | param <field> <value>
//   node <prefill|decode|switch> | link <from> <to> <cap> | duplex <a> <b> <cap>
//   request <arrival> <deadline> [prompt_tokens]
//   batch <admit_at> <members,..|-> <costs,..|->
//   flow <batch> <request> <reuse|collective|p2d> <src> <dst> <size> <target>
//        <release_at|-> <deadline|->
// Operations are applied in file order, like the engine's add_* calls
// (engine.cpp:114-220), so flow / batch / coflow ids and push seqs match.
InstanceInput manual_instance(const std::string& spec) {
  auto img = std::make_shared<ManualImage>();
  Config cfg;
  std::string policy = "fs";
  RunParams rp;
  Fabric fab;
  std::vector<std::vector<std::string>> ops;
  std::istringstream text(spec);
  std::string line;
  while (std::getline(text, line)) {
    const size_t h = line.find('#');
    if (h != std::string::npos) line.resize(h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    for (std::string t; ls >> t;) tok.push_back(t);
    if (tok.empty()) continue;
    const std::string& k = tok[0];
    auto need = [&](size_t n) {
      if (tok.size() < n) throw ConfigError("manual spec: too few fields in '" + line + "'");
    };
    if (k == "policy") {
      need(2);
      policy = tok[1];
    } else if (k == "set") {
      need(3);
      cfg.set(tok[1], tok[2]);
    } else if (k == "param") {
      need(3);
      const double v = parse_d(tok[2]);
      if (tok[1] == "promotion_tick") rp.tick = v;
      else if (tok[1] == "horizon") rp.horizon = v;
      else if (tok[1] == "horizon_slack") rp.horizon_slack = v;
      else if (tok[1] == "max_batch_tokens") rp.max_batch_tokens = static_cast<long>(v);
      else if (tok[1] == "livelock_events") rp.livelock = static_cast<long>(v);
      else throw ConfigError("manual spec: unknown param " + tok[1]);
    } else if (k == "node") {
      const std::string role = tok.size() > 1 ? tok[1] : "prefill";
      fab.add_node(role == "decode" ? NodeRole::Decode
                   : role == "switch" ? NodeRole::Switch : NodeRole::Prefill);
    } else if (k == "link") {
      need(4);
      fab.add_link(std::stoi(tok[1]), std::stoi(tok[2]), parse_d(tok[3]));
    } else if (k == "duplex") {
      need(4);
      fab.add_duplex(std::stoi(tok[1]), std::stoi(tok[2]), parse_d(tok[3]));
    } else {
      ops.push_back(tok);
    }
  }
  auto sched = make_scheduler(parse_policy(policy), cfg);

  auto topo = std::make_shared<TopoImage>();
  for (const Link& l : fab.links()) topo->cap.push_back(l.capacity);
  ManualImage& m = *img;
  int n_flows = 0;
  for (const auto& tok : ops) {
    if (tok[0] == "request") {
      if (tok.size() < 3) throw ConfigError("manual spec: request needs arrival and deadline");
      m.r_arrival.push_back(tok[1] == "-" ? -1.0 : parse_d(tok[1]));
      m.r_deadline.push_back(parse_d(tok[2]));
      m.r_tokens.push_back(tok.size() > 3 ? std::stoll(tok[3]) : 0);
      m.r_batch.push_back(-1);
      m.r_open.push_back(0);
    } else if (tok[0] == "batch") {
      if (tok.size() < 4) throw ConfigError("manual spec: batch needs admit, members, costs");
      std::vector<int> mem;
      std::vector<double> cost;
      if (tok[2] != "-")
        for (auto& s : split_csv(tok[2])) mem.push_back(std::stoi(s));
      if (tok[3] != "-")
        for (auto& s : split_csv(tok[3])) cost.push_back(parse_d(s));
      const int b = static_cast<int>(m.members.size());
      for (int r : mem) {
        if (r < 0 || r >= static_cast<int>(m.r_batch.size()))
          throw ConfigError("manual spec: batch member out of range");
        m.r_batch[r] = b;
      }
      const double at = tok[1] == "-" ? -1.0 : parse_d(tok[1]);
      m.members.push_back(mem);
      m.costs.push_back(cost);
      m.admit_at.push_back(at);
      m.last_admit = std::max(m.last_admit, at);
      m.b_ffirst.push_back(n_flows);
      m.b_fcount.push_back(0);
      const size_t L = cost.size();
      m.reuse.emplace_back(L);
      m.p2d.emplace_back(L);
      m.coll.emplace_back(L, -1);
    } else if (tok[0] == "flow") {
      if (tok.size() < 10) throw ConfigError("manual spec: flow needs 9 fields");
      ManualImage::F f{};
      f.batch = std::stoi(tok[1]);
      f.req = std::stoi(tok[2]);
      f.stage = tok[3] == "reuse" ? ST_REUSE : tok[3] == "collective" ? ST_COLL : ST_P2D;
      const int src = std::stoi(tok[4]), dst = std::stoi(tok[5]);
      f.size = parse_d(tok[6]);
      f.tl = std::stoi(tok[7]);
      f.scripted = tok[8] != "-";
      f.relat = f.scripted ? parse_d(tok[8]) : 0.0;
      f.dl = tok[9] != "-" ? parse_d(tok[9]) : std::nan("");
      if (f.batch < 0 || f.batch >= static_cast<int>(m.members.size()))
        throw ConfigError("manual spec: flow batch out of range");
      // flows_by_batch must be contiguous for the device batch ranges
      if (m.b_fcount[f.batch] > 0 && m.b_ffirst[f.batch] + m.b_fcount[f.batch] != n_flows)
        throw ConfigError("manual spec: a batch's flows must be added contiguously");
      if (m.b_fcount[f.batch] == 0) m.b_ffirst[f.batch] = n_flows;
      if (f.req >= 0) {
        const auto& mem = m.members[f.batch];
        if (std::find(mem.begin(), mem.end(), f.req) == mem.end())
          throw ConfigError("manual spec: a flow's request must belong to its batch");
        m.r_open[f.req] += 1;
      }
      try {
        f.route = topo->routes.add(fab, src, dst);
      } catch (const SimError&) {
        f.route = -1;  // unreachable: raised when the flow is released
      }
      const int fid = n_flows++;
      m.b_fcount[f.batch] += 1;
      const int idx = f.tl - 1;
      const int L = static_cast<int>(m.costs[f.batch].size());
      if (idx >= 0 && idx < L) {
        if (f.stage == ST_REUSE) m.reuse[f.batch][idx].push_back(fid);
        else if (f.stage == ST_P2D) m.p2d[f.batch][idx].push_back(fid);
        else {
          int& c = m.coll[f.batch][idx];
          if (c < 0) {
            c = static_cast<int>(m.coflows.size());
            m.coflows.push_back({f.batch, f.tl, {}});
          }
          m.coflows[c].members.push_back(fid);
          f.coflow = c;
        }
      }
      m.flows.push_back(f);
    } else {
      throw ConfigError("manual spec: unknown op '" + tok[0] + "'");
    }
  }
  if (topo->routes.count() == 0) topo->routes.add(fab, 0, 0);  // keep CSR non-empty
  topo->lr_cap = std::max<int>(1, static_cast<int>(fab.links().size()));

  InstanceInput in;
  sched->configure(in.p);
  in.policy = sched->name();
  in.p.tick = rp.tick;
  in.p.horizon = rp.horizon ? *rp.horizon : m.last_admit + rp.horizon_slack;
  in.p.livelock = rp.livelock;
  in.p.max_batch_tokens = rp.max_batch_tokens;
  in.p.workload_mode = 0;
  in.topo = topo;
  in.manual = img;
  in.deadlines_ready = true;
  return in;
}

double request_arrival(const InstanceInput& in, int r) {
  return in.manual ? in.manual->r_arrival[r] : in.reqs[r].arrival;
}
double request_deadline(const InstanceInput& in, int r) {
  return in.manual ? in.manual->r_deadline[r] : in.reqs[r].deadline;
}

// ------------------------------------------------------------- workload mode

std::shared_ptr<TopoImage> build_topo_image(const Fabric& f, const Layout& lay) {
  auto t = std::make_shared<TopoImage>();
  for (const Link& l : f.links()) t->cap.push_back(l.capacity);
  const int U = lay.units, H = lay.hosts_per_unit;
  t->rt_reuse.assign(static_cast<size_t>(U) * U, -1);
  t->rt_p2d.assign(U, -1);
  t->rt_coll.assign(static_cast<size_t>(U) * H * H, -1);
  for (int u = 0; u < U; ++u) t->rt_p2d[u] = t->routes.add(f, lay.lead(u), lay.decode(u));
  for (int u = 0; u < U; ++u)
    for (int i = 0; i < H; ++i)
      for (int j = 0; j < H; ++j)
        if (i != j) t->rt_coll[(u * H + i) * H + j] = t->routes.add(f, lay.host(u, i), lay.host(u, j));
  for (int s = 0; s < U; ++s)
    for (int d = 0; d < U; ++d)
      if (s != d) t->rt_reuse[s * U + d] = t->routes.add(f, lay.lead(s), lay.lead(d));
  // per-request distinct-link bound: own reuse + p2d routes + the unit's collectives
  int lr = 1;
  for (int u = 0; u < U; ++u) {
    std::vector<int> ls;
    auto add_route = [&](int rid) {
      if (rid < 0) return;
      for (int k = t->routes.off[rid]; k < t->routes.off[rid + 1]; ++k)
        ls.push_back(t->routes.links[k]);
    };
    add_route(t->rt_p2d[u]);
    for (int i = 0; i < H; ++i)
      for (int j = 0; j < H; ++j)
        if (i != j) add_route(t->rt_coll[(u * H + i) * H + j]);
    std::sort(ls.begin(), ls.end());
    ls.erase(std::unique(ls.begin(), ls.end()), ls.end());
    lr = std::max(lr, static_cast<int>(ls.size()) + t->routes.rmax);
  }
  t->lr_cap = lr;
  return t;
}

// Topology images are immutable once built; the instances of a sweep share
// one per distinct (fabric, layout) key text instead of rebuilding the fabric
// and its routes. A miss validates in the reference order (fabric, layout).
std::shared_ptr<TopoImage> shared_topo_image(const Config& cfg) {
  std::string key;
  for (const char* k : {"topology.kind", "topology.hosts", "topology.nics_per_host",
                        "topology.link_bytes_per_s", "topology.link_gbps",
                        "topology.oversubscription", "cluster.prefill_units",
                        "cluster.hosts_per_unit", "cluster.decode_hosts"})
    key += (cfg.has(k) ? "=" + cfg.str(k, "") : std::string("-")) + '\x1f';
  static std::mutex mu;
  static std::map<std::string, std::weak_ptr<TopoImage>> cache;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end())
      if (auto t = it->second.lock()) return t;
  }
  const Fabric fab = Fabric::from(cfg);
  const Layout lay = Layout::from(cfg);
  auto t = build_topo_image(fab, lay);
  t->hosts = fab.hosts();
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = t;
  return t;
}

InstanceInput workload_instance(const Config& cfg) {
  InstanceInput in;
  const PolicyKind kind = parse_policy(cfg.str("policy", "fs"));
  in.topo = shared_topo_image(cfg);
  const Layout lay = Layout::from(cfg);
  const CostModel cost = CostModel::from(cfg);
  const RunParams rp = RunParams::from(cfg);
  const WorkloadSpec spec = WorkloadSpec::from(cfg);
  if (spec.trace.empty())
    in.reqs = synthesize(spec, lay, cost, rp.max_batch_tokens);
  else
    in.reqs = read_trace(spec.trace, lay, cost);
  auto sched = make_scheduler(kind, cfg);
  sched->configure(in.p);
  if (lay.total_hosts() > in.topo->hosts)
    throw ConfigError("config key 'cluster.prefill_units': layout needs " +
                      std::to_string(lay.total_hosts()) + " hosts, topology has " +
                      std::to_string(in.topo->hosts));
  double last = 0.0;
  for (HostRequest& r : in.reqs) {
    if (r.tokens > rp.max_batch_tokens)
      throw WorkloadError("request: prompt of " + std::to_string(r.tokens) +
                          " tokens exceeds the batch token cap");
    if (r.unit < 0 || r.unit >= lay.units) throw WorkloadError("request: prefill unit out of range");
    if (r.layers <= 0) r.layers = cost.layers;
    if (r.layers > cost.layers) throw WorkloadError("request: more layers than the model");
    const double reuse_bytes = r.reuse * static_cast<double>(r.tokens) * cost.kv;
    if (reuse_bytes > 0.0 && (r.source < 0 || r.source >= lay.units || r.source == r.unit))
      throw WorkloadError("request: reuse_fraction > 0 needs a reuse_source");
    last = std::max(last, r.arrival);
  }
  in.policy = sched->name();
  in.seed = static_cast<long>(spec.seed);
  in.rate = spec.rate;
  in.slo_mult = spec.slo_mult;
  in.p.tick = rp.tick;
  in.p.horizon = rp.horizon ? *rp.horizon : last + rp.horizon_slack;
  in.p.livelock = rp.livelock;
  in.p.max_batch_tokens = rp.max_batch_tokens;
  in.p.layers = cost.layers;
  in.p.alpha = cost.alpha;
  in.p.beta = cost.beta;
  in.p.kv = cost.kv;
  in.p.coll = cost.coll;
  in.p.units = lay.units;
  in.p.hpu = lay.hosts_per_unit;
  in.p.decode_hosts = lay.decode_hosts;
  in.p.workload_mode = 1;
  return in;
}

void derive_deadlines(Backend& be, const std::vector<InstanceInput*>& insts) {
  // One isolated run per distinct key (workload.cpp:199-217). The run depends
  // only on the fabric, the engine/cost parameters and the key, so identical
  // probes of different instances (seeds, loads, SLO scales, policies of one
  // sweep) are simulated once.
  std::vector<InstanceInput> probes;
  std::vector<std::vector<int>> probe_of(insts.size());
  std::map<std::tuple<const void*, std::string, long, long, int, int>, int> cache;
  for (size_t i = 0; i < insts.size(); ++i) {
    InstanceInput& in = *insts[i];
    InstParams fsp = in.p;
    FairShareScheduler fs;
    fs.configure(fsp);
    fsp.horizon = 0.0 + 1e9;  // horizon reset, slack 1e9 (workload.cpp:189-191)
    // key of the probe parameters, field by field (struct padding is not data)
    static_assert(sizeof(InstParams) == 368, "new InstParams field: add it to the probe key");
    std::string pkey;
    auto put = [&pkey](auto v) { pkey.append(reinterpret_cast<const char*>(&v), sizeof(v)); };
    put(fsp.policy), put(fsp.K);
    for (double t : fsp.thr) put(t);
    put(fsp.tick), put(fsp.horizon), put(fsp.livelock), put(fsp.max_batch_tokens), put(fsp.layers);
    put(fsp.alpha), put(fsp.beta), put(fsp.kv), put(fsp.coll), put(fsp.units), put(fsp.hpu);
    put(fsp.decode_hosts), put(fsp.prune_enable), put(fsp.drop_frac), put(fsp.workload_mode);
    probe_of[i].resize(in.reqs.size());
    // Within an instance the reference caches on the reuse fraction rounded to
    // 1e-9 (workload.cpp:203-205): a request reuses the isolated TTFT of the
    // FIRST request of its (tokens, llround(frac * 1e9), unit, source) bucket.
    std::map<std::tuple<long, long, int, int>, int> bucket;
    for (size_t r = 0; r < in.reqs.size(); ++r) {
      const HostRequest& q = in.reqs[r];
      const auto bk = std::make_tuple(static_cast<long>(q.tokens),
                                      static_cast<long>(std::llround(q.reuse * 1e9)), q.unit, q.source);
      if (auto b = bucket.find(bk); b != bucket.end()) {
        probe_of[i][r] = b->second;
        continue;
      }
      // the bucket's first request: its probe is shared across instances by
      // the exact reuse bits (the run depends on the exact fraction)
      long bits;
      std::memcpy(&bits, &q.reuse, sizeof(bits));
      auto key = std::make_tuple(static_cast<const void*>(in.topo.get()), pkey, q.tokens, bits, q.unit,
                                 q.source);
      auto it = cache.find(key);
      if (it != cache.end()) {
        probe_of[i][r] = it->second;
        bucket.emplace(bk, it->second);
        continue;
      }
      InstanceInput p;
      p.p = fsp;
      p.topo = in.topo;
      HostRequest pr = q;
      pr.arrival = 0.0;
      pr.deadline = kInfD;
      p.reqs.push_back(pr);
      p.policy = "fs";
      const int id = static_cast<int>(probes.size());
      probes.push_back(std::move(p));
      cache.emplace(key, id);
      bucket.emplace(bk, id);
      probe_of[i][r] = id;
    }
  }
  if (probes.empty()) return;
  // memory-bounded chunks of probes (each a tiny single-request instance)
  std::vector<double> low(probes.size(), -1.0);
  const size_t chunk = 32768;
  for (size_t b0 = 0; b0 < probes.size(); b0 += chunk) {
    const size_t b1 = std::min(probes.size(), b0 + chunk);
    std::vector<InstanceInput> part(std::make_move_iterator(probes.begin() + b0),
                                    std::make_move_iterator(probes.begin() + b1));
    Batch batch(be, std::move(part));
    batch.run(0);
    for (size_t k = b0; k < b1; ++k) {
      const InstanceOutput& o = batch.output(static_cast<int>(k - b0));
      if (o.ttft.size() != 1 || o.ttft[0] == -1.0)
        throw InternalError("isolated oracle run did not finish");
      low[k] = o.ttft[0];
    }
  }
  for (size_t i = 0; i < insts.size(); ++i) {
    InstanceInput& in = *insts[i];
    for (size_t r = 0; r < in.reqs.size(); ++r) {
      HostRequest& q = in.reqs[r];
      q.deadline = q.arrival + in.slo_mult * low[probe_of[i][r]];
    }
    in.deadlines_ready = true;
  }
}

// -------------------------------------------------------------- packing

namespace {

struct Region {
  size_t off = 0;
  char* dev = nullptr;
  char* host = nullptr;
  size_t take(size_t bytes) {
    off = (off + 63) & ~size_t(63);
    size_t o = off;
    off += bytes ? bytes : 8;
    return o;
  }
};

struct Carver {
  Region in, st, out;
  bool real = false;
  template <class T>
  T* I(size_t n, const T* src = nullptr, size_t ncopy = 0) {  // uploaded input
    size_t o = in.take(sizeof(T) * n);
    if (real && src && ncopy) std::memcpy(in.host + o, src, sizeof(T) * ncopy);
    return real ? reinterpret_cast<T*>(in.dev + o) : nullptr;
  }
  template <class T>
  T* Ih(size_t n, T** host_view) {  // uploaded input filled in place
    size_t o = in.take(sizeof(T) * n);
    *host_view = real ? reinterpret_cast<T*>(in.host + o) : nullptr;
    return real ? reinterpret_cast<T*>(in.dev + o) : nullptr;
  }
  template <class T>
  T* S(size_t n) {  // device-only state
    size_t o = st.take(sizeof(T) * n);
    return real ? reinterpret_cast<T*>(st.dev + o) : nullptr;
  }
  template <class T>
  T* O(size_t n, size_t* off) {  // level-0 output (one D2H for the batch)
    size_t o = out.take(sizeof(T) * n);
    *off = o;
    return real ? reinterpret_cast<T*>(out.dev + o) : nullptr;
  }
};

template <class T>
T* host_of(const Carver& c, T* dev) {
  return reinterpret_cast<T*>(c.in.host + (reinterpret_cast<char*>(dev) - c.in.dev));
}

void carve_topo(Carver& c, TopoImage& t, Inst& d) {
  d.cap = c.I<double>(t.cap.size(), t.cap.data(), t.cap.size());
  d.route_off = c.I<int>(t.routes.off.size(), t.routes.off.data(), t.routes.off.size());
  d.route_links = c.I<int>(t.routes.links.size(), t.routes.links.data(), t.routes.links.size());
  d.rt_reuse = c.I<int>(t.rt_reuse.size(), t.rt_reuse.data(), t.rt_reuse.size());
  d.rt_p2d = c.I<int>(t.rt_p2d.size(), t.rt_p2d.data(), t.rt_p2d.size());
  d.rt_coll = c.I<int>(t.rt_coll.size(), t.rt_coll.data(), t.rt_coll.size());
}

void carve_instance(Carver& c, const InstanceInput& in, Inst& d, const Inst& topo_ptrs,
                    size_t* o_out, size_t* o_ttft, size_t* o_pruned, size_t* o_stall,
                    size_t* o_rbatch) {
  const TopoImage& t = *in.topo;
  const ManualImage* m = in.manual.get();
  std::memset(&d, 0, sizeof(Inst));
  d.p = in.p;
  d.cap = topo_ptrs.cap;
  d.route_off = topo_ptrs.route_off;
  d.route_links = topo_ptrs.route_links;
  d.rt_reuse = topo_ptrs.rt_reuse;
  d.rt_p2d = topo_ptrs.rt_p2d;
  d.rt_coll = topo_ptrs.rt_coll;
  d.nlinks = static_cast<int>(t.cap.size());
  d.rmax = std::max(1, t.routes.rmax);

  // ---- capacities
  long n_req, F, B, C, PL, RP, PP, CM, E, A, MP;
  const int units = in.p.units;
  if (!m) {
    n_req = static_cast<long>(in.reqs.size());
    const long L = in.p.layers;
    const long per = static_cast<long>(in.p.hpu) * (in.p.hpu - 1);
    F = 0;
    for (const HostRequest& r : in.reqs) {
      const double tokens = static_cast<double>(r.tokens);
      const double reuse_bytes = r.reuse * tokens * in.p.kv;
      const double p2d_bytes = tokens * in.p.kv;
      F += static_cast<long>(r.layers) * ((reuse_bytes > 0.0) + (p2d_bytes > 0.0));
    }
    const bool coll = in.p.coll > 0.0 && in.p.hpu > 1;
    B = std::max(1L, n_req);
    if (coll) F += B * L * per;
    C = coll ? B * L : 1;
    PL = B * L;
    RP = PP = n_req * L;
    CM = coll ? B * L * per : 1;
    E = in.e_boost > 0 ? 2 * n_req + 4L * units + 64 + in.e_boost : kSmemEvents;
    MP = n_req;
  } else {
    n_req = static_cast<long>(m->r_arrival.size());
    F = static_cast<long>(m->flows.size());
    B = static_cast<long>(m->members.size());
    C = static_cast<long>(m->coflows.size());
    PL = 0;
    RP = PP = CM = MP = 0;
    for (size_t b = 0; b < m->members.size(); ++b) {
      PL += static_cast<long>(m->costs[b].size());
      MP += static_cast<long>(m->members[b].size());
      for (auto& v : m->reuse[b]) RP += static_cast<long>(v.size());
      for (auto& v : m->p2d[b]) PP += static_cast<long>(v.size());
    }
    for (auto& cf : m->coflows) CM += static_cast<long>(cf.members.size());
    E = B * 3 + F + 64 + in.e_boost;
  }
  // first-attempt active-set bound: the on-chip plan's 1024, or MFSIM_ACTIVE_CAP
  // for runs known to be large (an overflow re-runs the batch from the start)
  long a_first = kDefaultActive;
  if (const char* e = std::getenv("MFSIM_ACTIVE_CAP")) a_first = std::max(1L, std::atol(e));
  A = in.a_cap > 0 ? in.a_cap : std::min<long>(std::max<long>(F, 1), a_first);

  A = std::max<long>(A, 1);
  const long X = A * d.rmax;
  const int LR = t.lr_cap;
  d.n_req = static_cast<int>(n_req);
  d.n_arr = m ? 0 : static_cast<int>(n_req);
  d.F_cap = static_cast<int>(std::max(F, 1L));
  d.B_cap = static_cast<int>(std::max(B, 1L));
  d.C_cap = static_cast<int>(std::max(C, 1L));
  d.E_cap = static_cast<int>(E);
  d.A_cap = static_cast<int>(A);
  d.PL_cap = static_cast<int>(std::max(PL, 1L));
  d.RP_cap = static_cast<int>(std::max(RP, 1L));
  d.PP_cap = static_cast<int>(std::max(PP, 1L));
  d.CM_cap = static_cast<int>(std::max(CM, 1L));
  d.MP_cap = static_cast<int>(std::max(MP, 1L));
  d.LR_cap = LR;
  d.X_cap = static_cast<int>(X);
  d.host_init = m ? 1 : 0;
  const size_t nr = static_cast<size_t>(std::max(n_req, 1L));

  // ---- request inputs
  if (!m) {
    std::vector<double> arr(n_req), dl(n_req), reuse(n_req);
    std::vector<long long> tok(n_req);
    std::vector<int> unit(n_req), src(n_req), lay(n_req), order(n_req);
    for (long i = 0; i < n_req; ++i) {
      const HostRequest& r = in.reqs[i];
      arr[i] = r.arrival;
      dl[i] = r.deadline;
      reuse[i] = r.reuse;
      tok[i] = r.tokens;
      unit[i] = r.unit;
      src[i] = r.source;
      lay[i] = r.layers;
    }
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      if (arr[a] != arr[b]) return arr[a] < arr[b];
      return a < b;
    });
    // per-unit FIFO lists in arrival-processing order
    std::vector<int> qoff(units + 1, 0), mp(n_req);
    for (long i = 0; i < n_req; ++i) ++qoff[unit[i] + 1];
    for (int u = 0; u < units; ++u) qoff[u + 1] += qoff[u];
    std::vector<int> fill(qoff.begin(), qoff.end() - 1);
    for (long k = 0; k < n_req; ++k) {
      const int r = order[k];
      mp[fill[unit[r]]++] = r;
    }
    d.r_arrival = c.I<double>(nr, arr.data(), n_req);
    d.r_deadline = c.I<double>(nr, dl.data(), n_req);
    d.r_tokens = c.I<long long>(nr, tok.data(), n_req);
    d.r_reuse = c.I<double>(nr, reuse.data(), n_req);
    d.r_unit = c.I<int>(nr, unit.data(), n_req);
    d.r_src = c.I<int>(nr, src.data(), n_req);
    d.r_layers = c.I<int>(nr, lay.data(), n_req);
    d.arr_order = c.I<int>(nr, order.data(), n_req);
    d.q_off = c.I<int>(units + 1, qoff.data(), units + 1);
    d.m_pool = c.I<int>(nr, mp.data(), n_req);
  } else {
    std::vector<double> zeros(n_req, 0.0);
    std::vector<int> units0(n_req, 0), srcm(n_req, -1), lay0(n_req, 0);
    d.r_arrival = c.I<double>(nr, m->r_arrival.data(), n_req);
    d.r_deadline = c.I<double>(nr, m->r_deadline.data(), n_req);
    d.r_tokens = c.I<long long>(nr, m->r_tokens.data(), n_req);
    d.r_reuse = c.I<double>(nr, zeros.data(), n_req);
    d.r_unit = c.I<int>(nr, units0.data(), n_req);
    d.r_src = c.I<int>(nr, srcm.data(), n_req);
    d.r_layers = c.I<int>(nr, lay0.data(), n_req);
    d.arr_order = c.I<int>(1);
    d.q_off = c.I<int>(1);
    std::vector<int> mp;
    for (auto& mem : m->members) mp.insert(mp.end(), mem.begin(), mem.end());
    d.m_pool = c.I<int>(std::max<size_t>(mp.size(), 1), mp.data(), mp.size());
  }

  // ---- state: host-initialised in manual mode, device-initialised otherwise
  auto state = [&](auto* tag, size_t n) {
    using T = std::remove_pointer_t<decltype(tag)>;
    return m ? c.I<T>(n) : c.S<T>(n);
  };
  const size_t nF = d.F_cap, nB = d.B_cap, nC = d.C_cap, nA = d.A_cap, nPL = d.PL_cap;
  d.r_batch = state((int*)nullptr, nr);
  d.r_pruned = state((uint8_t*)nullptr, nr);
  d.r_ttft = c.O<double>(nr, o_ttft);
  d.r_open = state((int*)nullptr, nr);
  d.r_lastfin = state((double*)nullptr, nr);
  d.r_rank = state((int*)nullptr, nr);
  d.u_busy = c.S<uint8_t>(std::max(units, 1));
  d.q_head = c.S<int>(std::max(units, 1));
  d.q_tail = c.S<int>(std::max(units, 1));
  d.f_size = state((double*)nullptr, nF);
  d.f_rel = state((double*)nullptr, nF);
  d.f_fin = state((double*)nullptr, nF);
  d.f_dl = state((double*)nullptr, nF);
  d.f_relat = state((double*)nullptr, m ? nF : 1);
  d.f_req = state((int*)nullptr, nF);
  d.f_batch = state((int*)nullptr, nF);
  d.f_cof = state((int*)nullptr, nF);
  d.f_route = state((int*)nullptr, nF);
  d.f_apos = state((int*)nullptr, nF);
  d.f_rank = state((int*)nullptr, nF);
  d.f_tl = state((int*)nullptr, nF);
  d.f_hidx = c.S<int>(nF);
  d.f_stage = state((uint8_t*)nullptr, nF);
  d.f_state = state((uint8_t*)nullptr, nF);
  d.f_band = state((uint8_t*)nullptr, nF);
  d.f_level = state((uint8_t*)nullptr, nF);
  d.f_scripted = state((uint8_t*)nullptr, nF);
  d.a_fid = c.S<int>(nA);
  d.a_rem = c.S<double>(nA);
  d.a_rate = c.S<double>(nA);
  d.a_evt = c.S<double>(nA);
  d.a_evseq = c.S<unsigned long long>(nA);
  d.a_rl = c.S<unsigned short>(nA * d.rmax);
  d.a_rn = c.S<uint8_t>(nA);
  d.b_unit = state((int*)nullptr, nB);
  d.b_layers = state((int*)nullptr, nB);
  d.b_lbase = state((int*)nullptr, nB);
  d.b_admit = state((double*)nullptr, nB);
  d.b_done = state((double*)nullptr, nB);
  d.b_departed = state((uint8_t*)nullptr, nB);
  d.b_admitted = state((uint8_t*)nullptr, nB);
  d.b_open = state((int*)nullptr, nB);
  d.b_rank = state((int*)nullptr, nB);
  d.b_ffirst = state((int*)nullptr, nB);
  d.b_fcount = state((int*)nullptr, nB);
  d.b_moff = state((int*)nullptr, nB);
  d.b_mcnt = state((int*)nullptr, nB);
  d.pl_cost = state((double*)nullptr, nPL);
  d.pl_started = state((uint8_t*)nullptr, nPL);
  d.pl_done = state((uint8_t*)nullptr, nPL);
  d.pl_start = state((double*)nullptr, nPL);
  d.pl_end = state((double*)nullptr, nPL);
  d.pl_coll = state((int*)nullptr, nPL);
  d.pl_roff = state((int*)nullptr, nPL);
  d.pl_rcnt = state((int*)nullptr, nPL);
  d.pl_poff = state((int*)nullptr, nPL);
  d.pl_pcnt = state((int*)nullptr, nPL);
  const size_t nAT = d.p.policy == mfb::POL_AALO ? 3 * nPL : 1;
  d.pl_att = state((double*)nullptr, nAT);
  d.pl_asum = c.S<double>(nAT);
  d.rpool = state((int*)nullptr, d.RP_cap);
  d.ppool = state((int*)nullptr, d.PP_cap);
  d.c_batch = state((int*)nullptr, nC);
  d.c_layer = state((int*)nullptr, nC);
  d.c_open = state((int*)nullptr, nC);
  d.c_rel = state((double*)nullptr, nC);
  d.c_done = state((double*)nullptr, nC);
  d.c_moff = state((int*)nullptr, nC);
  d.c_mcnt = state((int*)nullptr, nC);
  d.cpool = state((int*)nullptr, d.CM_cap);
  d.e_t = state((double*)nullptr, d.E_cap);
  d.e_seq = state((unsigned long long*)nullptr, d.E_cap);
  d.e_kind = state((int*)nullptr, d.E_cap);
  d.e_a = state((int*)nullptr, d.E_cap);
  d.e_b = state((int*)nullptr, d.E_cap);
  const size_t nl = std::max(d.nlinks, 1);
  d.l_res = c.S<double>(nl);
  d.l_cnt = c.S<int>(nl);
  d.l_off = c.S<int>(nl);
  d.l_x = c.S<double>(nl);
  d.l_y = c.S<double>(nl);
  const size_t pA = static_cast<size_t>(pow2(static_cast<long>(nA)));
  d.s_rate = c.S<double>(nA);
  d.s_cap = c.S<double>(nA);
  d.s_ord = c.S<int>(2 * pA);
  d.s_cls = c.S<int>(nA + 1);
  d.s_ul = c.S<int>(nA);
  // slot filling state: host-sized for the global fallback (the kernel stages
  // the per-slot arrays in shared memory when they fit its plan)
  // slots: at most the per-warp shared-memory plan (kSmemSlots), so the
  // bound is the same in HBM and on chip and survives suspend / resume
  const size_t nts = std::min<size_t>({nl, nA * d.rmax, static_cast<size_t>(kSmemSlots)});
  d.TS_cap = (std::getenv("MFSIM_FORCE_GLOBAL") || nA * d.rmax > 65535) ? 0 : static_cast<int>(nts);
  if (const char* cap = std::getenv("MFSIM_SLOT_CAP"))  // test knob: per-step slot overflow
    d.TS_cap = std::min(d.TS_cap, std::atoi(cap));
  d.l2s = c.S<unsigned short>(nl);
  d.a_sl = c.S<unsigned short>(nA * d.rmax);
  d.sl_link = c.S<unsigned short>(nts);
  d.sl_ref = c.S<unsigned short>(nts);
  d.sl_free = c.S<unsigned short>(nts);
  d.sl_res = c.S<double>(nts);
  d.sl_cnt = c.S<int>(nts);
  d.sl_mb = c.S<int>(nts);
  d.sl_end = c.S<int>(nts);
  d.sl_tl = c.S<unsigned short>(nts);
  d.sl_sat = c.S<unsigned short>(nts);
  d.c_mem = c.S<unsigned short>(nA * d.rmax);
  d.c_frz = c.S<unsigned>((nA + 31) / 32);
  d.s_tl = c.S<unsigned short>(nl);
  d.srt = c.S<int>(nA);
  d.srt_add = c.S<int>(nA);
  d.s_k0 = c.S<unsigned long long>(nA);
  d.s_k1 = c.S<unsigned long long>(nA);
  d.s_k2 = c.S<unsigned long long>(nA);
  d.s_k3 = c.S<unsigned long long>(nA);
  d.h_keys = c.S<int>(nA);
  d.h_next = c.S<int>(nA);
  d.h_bkt = c.S<int>(hash_buckets(static_cast<int>(nA)));
  d.h_rank = c.S<int>(nA);
  const size_t pX = static_cast<size_t>(pow2(X));
  d.x_hi = c.S<unsigned long long>(pX);
  d.x_lo = c.S<unsigned long long>(pX);
  d.x_val = c.S<double>(pX);
  d.x_pre = c.S<double>(pX);
  d.x_seg = c.S<int>(pX);
  d.y_key = c.S<unsigned long long>(pX);
  d.y_val = c.S<double>(pX);
  d.x_aux = c.S<int>(pX);
  d.y_aux = c.S<int>(pX);
  const size_t pB = static_cast<size_t>(pow2(static_cast<long>(nB)));
  d.g_batches = c.S<int>(nB);
  d.g_req = c.S<int>(nr);
  d.g_rbat = c.S<int>(nr);
  d.g_loff = c.S<int>(nr);
  d.g_lcnt = c.S<int>(nr);
  d.g_link = c.S<int>(nr * LR);
  d.g_load = c.S<double>(nr * LR);
  d.g_rpos = c.S<int>(nr);
  d.g_inpool = c.S<uint8_t>(nr);
  d.g_tmp = c.S<double>(nr);
  d.g_pruned = c.S<int>(nr);
  d.g_slot_b = c.S<int>(nB);
  d.g_slot_off = c.S<int>(nB);
  d.g_slot_cnt = c.S<int>(nB);
  d.g_tok = c.S<double>(nB);
  d.g_red = c.S<double>(nB);
  d.g_dlo = c.S<double>(nB);
  d.g_sig = c.S<int>(pB);
  d.g_sk0 = c.S<unsigned long long>(nB);
  d.g_sk1 = c.S<unsigned long long>(nB);
  d.g_sk2 = c.S<unsigned long long>(nB);
  d.c_stall = c.S<double>(nC);
  d.b_stall = c.S<double>(nB);
  d.r_stall = c.O<double>(nr, o_stall);
  d.out = c.O<long long>(OUT_N, o_out);
  d.sc_blob = c.S<unsigned char>(kScBlob);
  d.o_pruned = c.O<uint8_t>(nr, o_pruned);
  d.o_rbatch = c.O<int>(nr, o_rbatch);

  // ---- manual-mode state image
  d.seq0 = m ? static_cast<long long>(m->members.size()) : static_cast<long long>(n_req);
  d.n_ev0 = m ? static_cast<int>(m->members.size()) : 0;
  d.n_flows0 = m ? static_cast<int>(m->flows.size()) : 0;
  d.n_batches0 = m ? static_cast<int>(m->members.size()) : 0;
  d.n_coflows0 = m ? static_cast<int>(m->coflows.size()) : 0;
  if (m && c.real) {
    for (long r = 0; r < n_req; ++r) {
      host_of(c, d.r_batch)[r] = m->r_batch[r];
      host_of(c, d.r_pruned)[r] = 0;
      host_of(c, d.r_open)[r] = m->r_open[r];
      host_of(c, d.r_lastfin)[r] = kNoTime;
      host_of(c, d.r_rank)[r] = -1;
    }
    int pl = 0, moff = 0, rp = 0, pp = 0, cm = 0;
    for (size_t b = 0; b < m->members.size(); ++b) {
      const int L = static_cast<int>(m->costs[b].size());
      host_of(c, d.b_unit)[b] = 0;
      host_of(c, d.b_layers)[b] = L;
      host_of(c, d.b_lbase)[b] = pl;
      host_of(c, d.b_admit)[b] = m->admit_at[b];
      host_of(c, d.b_done)[b] = kNoTime;
      host_of(c, d.b_departed)[b] = 0;
      host_of(c, d.b_admitted)[b] = 0;
      host_of(c, d.b_open)[b] = m->b_fcount[b];
      host_of(c, d.b_rank)[b] = -1;
      host_of(c, d.b_ffirst)[b] = m->b_ffirst[b];
      host_of(c, d.b_fcount)[b] = m->b_fcount[b];
      host_of(c, d.b_moff)[b] = moff;
      host_of(c, d.b_mcnt)[b] = static_cast<int>(m->members[b].size());
      moff += static_cast<int>(m->members[b].size());
      for (int l = 0; l < L; ++l, ++pl) {
        host_of(c, d.pl_cost)[pl] = m->costs[b][l];
        host_of(c, d.pl_started)[pl] = 0;
        host_of(c, d.pl_done)[pl] = 0;
        host_of(c, d.pl_start)[pl] = kNoTime;
        host_of(c, d.pl_end)[pl] = kNoTime;
        host_of(c, d.pl_coll)[pl] = m->coll[b][l];
        host_of(c, d.pl_roff)[pl] = rp;
        host_of(c, d.pl_rcnt)[pl] = static_cast<int>(m->reuse[b][l].size());
        for (int f : m->reuse[b][l]) host_of(c, d.rpool)[rp++] = f;
        host_of(c, d.pl_poff)[pl] = pp;
        host_of(c, d.pl_pcnt)[pl] = static_cast<int>(m->p2d[b][l].size());
        for (int f : m->p2d[b][l]) host_of(c, d.ppool)[pp++] = f;
        if (d.p.policy == mfb::POL_AALO)
          for (int k = 0; k < 3; ++k) host_of(c, d.pl_att)[3 * pl + k] = 0.0;
      }
      // initial BatchAdmit event, pushed by add_manual_batch (engine.cpp:178)
      host_of(c, d.e_t)[b] = m->admit_at[b];
      host_of(c, d.e_seq)[b] = b;
      host_of(c, d.e_kind)[b] = EV_ADMIT;
      host_of(c, d.e_a)[b] = static_cast<int>(b);
      host_of(c, d.e_b)[b] = -1;
    }
    for (size_t ci = 0; ci < m->coflows.size(); ++ci) {
      const auto& cf = m->coflows[ci];
      host_of(c, d.c_batch)[ci] = cf.batch;
      host_of(c, d.c_layer)[ci] = cf.layer;
      host_of(c, d.c_open)[ci] = static_cast<int>(cf.members.size());
      host_of(c, d.c_rel)[ci] = kNoTime;
      host_of(c, d.c_done)[ci] = kNoTime;
      host_of(c, d.c_moff)[ci] = cm;
      host_of(c, d.c_mcnt)[ci] = static_cast<int>(cf.members.size());
      for (int f : cf.members) host_of(c, d.cpool)[cm++] = f;
    }
    for (size_t i = 0; i < m->flows.size(); ++i) {
      const auto& f = m->flows[i];
      host_of(c, d.f_size)[i] = f.size;
      host_of(c, d.f_rel)[i] = kNoTime;
      host_of(c, d.f_fin)[i] = kNoTime;
      host_of(c, d.f_dl)[i] = f.dl;
      host_of(c, d.f_relat)[i] = f.relat;
      host_of(c, d.f_req)[i] = f.req;
      host_of(c, d.f_batch)[i] = f.batch;
      host_of(c, d.f_cof)[i] = f.coflow;
      host_of(c, d.f_route)[i] = f.route;
      host_of(c, d.f_apos)[i] = -1;
      host_of(c, d.f_rank)[i] = 0;
      host_of(c, d.f_tl)[i] = f.tl;
      host_of(c, d.f_stage)[i] = static_cast<uint8_t>(f.stage);
      host_of(c, d.f_state)[i] = FL_PENDING;
      host_of(c, d.f_band)[i] = BD_EARLY;
      host_of(c, d.f_level)[i] = 1;
      host_of(c, d.f_scripted)[i] = f.scripted ? 1 : 0;
    }
  }
}

}  // namespace

Batch::Batch(Backend& be, std::vector<InstanceInput> inputs) : be_(be), inputs_(std::move(inputs)) {
  pack();
}

Batch::~Batch() { release(); }

void Batch::release() {
  if (in_host_) be_.host_free(in_host_);
  if (out_host_) be_.host_free(out_host_);
  if (in_dev_) be_.dev_free(in_dev_);
  if (st_dev_) be_.dev_free(st_dev_);
  if (out_dev_) be_.dev_free(out_dev_);
  if (desc_dev_) be_.dev_free(desc_dev_);
  if (order_dev_) be_.dev_free(order_dev_);
  if (phase_dev_) be_.dev_free(phase_dev_);
  in_host_ = out_host_ = in_dev_ = st_dev_ = out_dev_ = nullptr;
  desc_dev_ = nullptr;
  order_dev_ = nullptr;
  phase_dev_ = nullptr;
}

void Batch::pack() {
  release();
  const int n = size();
  desc_.assign(n, Inst{});
  oview_.assign(n, OutView{});
  outputs_.assign(n, InstanceOutput{});
  // distinct topologies, carved once
  std::vector<TopoImage*> topos;
  for (auto& in : inputs_)
    if (std::find(topos.begin(), topos.end(), in.topo.get()) == topos.end())
      topos.push_back(in.topo.get());
  for (int pass = 0; pass < 2; ++pass) {
    Carver c;
    c.real = pass == 1;
    if (c.real) {
      c.in.dev = in_dev_;
      c.in.host = in_host_;
      c.st.dev = st_dev_;
      c.out.dev = out_dev_;
      c.out.host = out_host_;
    }
    std::vector<Inst> tp(topos.size());
    for (size_t t = 0; t < topos.size(); ++t) carve_topo(c, *topos[t], tp[t]);
    for (int i = 0; i < n; ++i) {
      size_t t = std::find(topos.begin(), topos.end(), inputs_[i].topo.get()) - topos.begin();
      OutView& ov = oview_[i];
      carve_instance(c, inputs_[i], desc_[i], tp[t], &ov.out, &ov.ttft, &ov.pruned, &ov.stall,
                     &ov.rbatch);
    }
    if (!c.real) {
      hint_ = LaunchHint{};
      for (const Inst& d : desc_) {
        hint_.rmax = std::max(hint_.rmax, d.rmax);
        hint_.nlinks = std::max(hint_.nlinks, d.nlinks);
        hint_.aalo = hint_.aalo || d.p.policy == mfb::POL_AALO || d.p.policy == mfb::POL_VARYS;
      }
      in_bytes_ = c.in.off;
      st_bytes_ = c.st.off;
      out_bytes_ = c.out.off;
      in_host_ = static_cast<char*>(be_.host_alloc(in_bytes_ + 64));
      out_host_ = static_cast<char*>(be_.host_alloc(out_bytes_ + 64));
      in_dev_ = static_cast<char*>(be_.dev_alloc(in_bytes_ + 64));
      st_dev_ = static_cast<char*>(be_.dev_alloc(st_bytes_ + 64));
      out_dev_ = static_cast<char*>(be_.dev_alloc(out_bytes_ + 64));
      desc_dev_ = static_cast<Inst*>(be_.dev_alloc(sizeof(Inst) * std::max(n, 1)));
      order_dev_ = static_cast<int*>(be_.dev_alloc(sizeof(int) * (n + 2 * (kMaxGroups + 1))));
      phase_dev_ = static_cast<int*>(be_.dev_alloc(sizeof(int) * std::max(n, 1)));
    }
  }
  for (int i = 0; i < n; ++i) desc_[i].phase = phase_dev_ + i;
  // claim order: estimated work descending (Karuna's capped filling and MFS's
  // promotions cost the most per event; the per-event cost grows with the
  // offered load, i.e. the active set), so the longest instances start first
  // and consecutive claims -- the 32 warps of a lock-step gang -- get
  // instances of similar per-event cost
  std::vector<double> cost(n);
  for (int i = 0; i < n; ++i) {
    const Inst& d = desc_[i];
    static const double factor[] = {1.0, 1.6, 1.1, 12.0, 2.5, 1.5, 4.0};
    const int pol = d.p.policy >= 0 && d.p.policy < 7 ? d.p.policy : 0;
    const double load = inputs_[i].rate > 0.0 ? inputs_[i].rate : 1.0;
    cost[i] = factor[pol] * (double(d.F_cap) + 2.0 * d.n_req) * (1.0 + load);
  }
  // claim groups: one per policy, so that the warps sharing an SM run the same
  // policy's code (the engine's instruction footprint exceeds the i-cache)
  order_.resize(n);
  std::iota(order_.begin(), order_.end(), 0);
  std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) {
    if (desc_[a].p.policy != desc_[b].p.policy) return desc_[a].p.policy < desc_[b].p.policy;
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    // then by seed: cells of one seed share arrivals and prompts, so their
    // per-event costs are the closest (and for deadline-free policies the
    // cells that differ only in SLO scale run the same event sequence, which
    // a gang executes in perfect lock step; A/B +33 %)
    if (inputs_[a].seed != inputs_[b].seed) return inputs_[a].seed < inputs_[b].seed;
    return inputs_[a].slo_mult > inputs_[b].slo_mult;
  });
  std::vector<int> off{0};
  for (int k = 1; k < n; ++k)
    if (desc_[order_[k]].p.policy != desc_[order_[k - 1]].p.policy) off.push_back(k);
  off.push_back(n);
  hint_.groups = static_cast<int>(off.size()) - 1;
  if (hint_.groups > kMaxGroups) throw InternalError("more claim groups than the kernel supports");
  order_.insert(order_.end(), off.begin(), off.end());
  // SM -> home group map for launches that run to completion: SMs in
  // proportion to each group's estimated WORK (its cost share, in [0, n)
  // position units), so that the long (Karuna) instances spread over many
  // SMs and the makespan is not one policy's SMs. Time-sliced launches keep
  // the count-proportional map (every warp busy for the whole slice).
  double total = 0.0;
  for (int i = 0; i < n; ++i) total += cost[i];
  std::vector<int> coff{0};
  double acc = 0.0;
  for (int g = 0; g + 1 < static_cast<int>(off.size()); ++g) {
    for (int k = off[g]; k < off[g + 1]; ++k) acc += cost[order_[k]];
    if (g + 2 < static_cast<int>(off.size()))
      coff.push_back(std::max(coff.back(), std::min(n, static_cast<int>(total > 0 ? n * (acc / total) : off[g + 1]))));
  }
  coff.push_back(n);
  order_.insert(order_.end(), coff.begin(), coff.end());
}

void Batch::upload_inputs() { be_.h2d(in_dev_, in_host_, in_bytes_); }

void Batch::upload() {
  be_.h2d(in_dev_, in_host_, in_bytes_);
  be_.h2d(desc_dev_, desc_.data(), sizeof(Inst) * desc_.size());
  be_.h2d(order_dev_, order_.data(), sizeof(int) * order_.size());
  reset();
}

void Batch::reset() {
  std::vector<int> zero(size(), 0);
  be_.h2d(phase_dev_, zero.data(), sizeof(int) * zero.size());
  be_.set_remaining(size());
  remaining_ = size();
}

void Batch::launch(long long budget, long long slice_ns) {
  be_.launch(desc_dev_, order_dev_, size(), hint_, budget, slice_ns, remaining_);
}

int Batch::remaining() { return remaining_ = be_.remaining(); }

size_t Batch::output_bytes(int detail) const {
  size_t b = out_bytes_;
  if (detail >= 1)
    for (const auto& o : outputs_) b += o.out[OUT_NCOFLOWS] * 24;
  if (detail >= 2)
    for (const auto& o : outputs_) b += o.out[OUT_NFLOWS] * 10 + o.out[OUT_NBATCHES] * 8;
  return b;
}

void Batch::download(int detail) {
  // one D2H for every level-0 output of the batch (out[], ttft, stall, flags)
  be_.d2h(out_host_, out_dev_, out_bytes_);
  be_.sync();
  // counters now; the per-request columns stay in the pinned buffer until an
  // instance's output is read (output()), so a batch-wide read costs one copy
  parsed_.assign(size(), 0);
  for (int i = 0; i < size(); ++i)
    std::memcpy(outputs_[i].out, out_host_ + oview_[i].out, sizeof(outputs_[i].out));
  if (detail >= 1) {
    for (int i = 0; i < size(); ++i) {
      const Inst& d = desc_[i];
      InstanceOutput& o = outputs_[i];
      const size_t nc = static_cast<size_t>(o.out[OUT_NCOFLOWS]);
      o.c_rel.resize(nc);
      o.c_done.resize(nc);
      o.c_stall.resize(nc);
      if (nc) {
        be_.d2h(o.c_rel.data(), d.c_rel, nc * 8);
        be_.d2h(o.c_done.data(), d.c_done, nc * 8);
        be_.d2h(o.c_stall.data(), d.c_stall, nc * 8);
      }
      if (detail >= 2) {
        const size_t nf = static_cast<size_t>(o.out[OUT_NFLOWS]);
        const size_t nb = static_cast<size_t>(o.out[OUT_NBATCHES]);
        o.f_fin.resize(nf);
        o.f_band.resize(nf);
        o.f_level.resize(nf);
        o.b_done.resize(nb);
        if (nf) {
          be_.d2h(o.f_fin.data(), d.f_fin, nf * 8);
          be_.d2h(o.f_band.data(), d.f_band, nf);
          be_.d2h(o.f_level.data(), d.f_level, nf);
        }
        if (nb) be_.d2h(o.b_done.data(), d.b_done, nb * 8);
      }
    }
    be_.sync();
  }
}

const InstanceOutput& Batch::output(int i) const {
  InstanceOutput& o = outputs_[i];
  if (i < static_cast<int>(parsed_.size()) && !parsed_[i]) {
    const OutView& ov = oview_[i];
    const int n = desc_[i].n_req;
    const double* tt = reinterpret_cast<const double*>(out_host_ + ov.ttft);
    const double* st = reinterpret_cast<const double*>(out_host_ + ov.stall);
    const uint8_t* pr = reinterpret_cast<const uint8_t*>(out_host_ + ov.pruned);
    const int* rb = reinterpret_cast<const int*>(out_host_ + ov.rbatch);
    o.ttft.assign(tt, tt + n);
    o.stall.assign(st, st + n);
    o.pruned.assign(pr, pr + n);
    o.rbatch.assign(rb, rb + n);
    parsed_[i] = 1;
  }
  return o;
}

void Batch::run(int detail) {
  // Instances that outgrow a device capacity bound (active set, event pool,
  // scratch) stop with a capacity check; their bounds are raised and the
  // whole batch is re-packed and re-run, so the resident layout always holds
  // the final capacities (a later launch() re-simulates the same batch).
  // Runs to completion as a series of time slices: each launch re-sizes its
  // grid to the instances still running, so the long tail of a batch (the
  // heaviest cells) ends up one instance per SM instead of sharing SMs with
  // the warps that claimed them at the start.
  long long slice_ns = 1000000000LL;
  if (const char* e = std::getenv("MFSIM_RUN_SLICE_MS")) slice_ns = std::atoll(e) * 1000000LL;
  for (int attempt = 0; attempt < 16; ++attempt) {
    upload();
    do launch(0, slice_ns);
    while (remaining() > 0);
    download(detail);
    bool again = false;
    for (int i = 0; i < size(); ++i) {
      const long long chk = outputs_[i].out[OUT_CHECK];
      if (outputs_[i].out[OUT_STATUS] != ERR_INTERNAL) continue;
      InstanceInput& in = inputs_[i];
      if (chk == CHK_CAP_EVENTS) {
        in.e_boost = std::max(in.e_boost * 2, 1024);
        again = true;
      } else if (chk == CHK_CAP_ACTIVE || chk == CHK_CAP_SCRATCH) {
        // x4: an overflow means a large instance, and every retry re-runs it
        const long long grown = std::max<long long>(4LL * desc_[i].A_cap, 64);
        in.a_cap = static_cast<int>(std::min<long long>(grown, std::max(desc_[i].F_cap, 1)));
        again = true;
      }
    }
    if (!again) return;
    pack();
  }
}

const char* check_name(int chk) {
  switch (chk) {
    case CHK_TIME_BACKWARDS: return "event time went backwards";
    case CHK_OVERSHOOT: return "transferred more than the flow size";
    case CHK_EARLY_FINISH: return "flow completed before its bytes were transferred";
    case CHK_FINISHED_TWICE: return "flow finished twice";
    case CHK_RELEASED_TWICE: return "flow released twice";
    case CHK_COFLOW_BARRIER: return "coflow member finished after barrier";
    case CHK_COMPUTE_STATE: return "compute completion for a layer that is not running";
    case CHK_LAYER_DEPS: return "layer computed before its dependencies";
    case CHK_NO_PROGRESS: return "allocate_rates: filling made no progress";
    case CHK_URGENT_BAND: return "urgent band is reserved for last-stage flows";
    case CHK_NEG_MLU: return "mlu_to_level: negative urgency";
    case CHK_CAP_FLOWS: return "device capacity exceeded: flows";
    case CHK_CAP_ACTIVE: return "device capacity exceeded: active flows";
    case CHK_CAP_EVENTS: return "device capacity exceeded: event pool";
    case CHK_CAP_BATCHES: return "device capacity exceeded: batches";
    case CHK_CAP_COFLOWS: return "device capacity exceeded: coflows";
    case CHK_CAP_POOL: return "device capacity exceeded: pipeline pools";
    case CHK_CAP_SCRATCH: return "device capacity exceeded: scratch";
    case CHK_LIVELOCK: return "livelock: simulated time stuck";
    case CHK_EMPTY_BATCH: return "admitting an empty batch";
    case CHK_ROUTE: return "no route between flow endpoints";
    case CHK_REUSE_SOURCE: return "reuse_fraction > 0 needs a reuse_source";
    default: return "internal check failed";
  }
}

void raise_status(long long status, long long check) {
  if (status == ERR_OK) return;
  const std::string msg = check_name(static_cast<int>(check));
  switch (status) {
    case ERR_WORKLOAD: throw WorkloadError(msg);
    case ERR_SIM: throw SimError(msg);
    default: throw InternalError(msg);
  }
}

}  // namespace mfh
