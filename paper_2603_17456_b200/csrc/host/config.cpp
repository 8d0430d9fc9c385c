#include "config.hpp"

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <fstream>
#include <sstream>

namespace mfh {

namespace {
std::string strip(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}
}  // namespace

Config Config::parse(const std::string& text) {
  Config c;
  std::istringstream in(text);
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    line = strip(line);
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos)
      throw ConfigError("config line " + std::to_string(no) + ": expected key = value, got '" +
                        line + "'");
    std::string k = strip(line.substr(0, eq));
    if (k.empty()) throw ConfigError("config line " + std::to_string(no) + ": empty key");
    c.set(k, strip(line.substr(eq + 1)));
  }
  return c;
}

Config Config::load(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open config file: " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return parse(ss.str());
}

std::optional<std::string> Config::raw(const std::string& key) const {
  auto it = kv_.find(key);
  if (it == kv_.end()) return std::nullopt;
  return it->second;
}

std::string Config::str(const std::string& key, const std::string& dflt) const {
  auto v = raw(key);
  return v ? *v : dflt;
}

double Config::to_double(const std::string& key, const std::string& v) const {
  char* end = nullptr;
  const double d = std::strtod(v.c_str(), &end);
  if (end == v.c_str() || *end != '\0')
    throw ConfigError("config key '" + key + "': not a number: '" + v + "'");
  return d;
}

double Config::num(const std::string& key, double dflt) const {
  auto v = raw(key);
  return v ? to_double(key, *v) : dflt;
}

long Config::integer(const std::string& key, long dflt) const {
  auto v = raw(key);
  if (!v) return dflt;
  const double d = to_double(key, *v);
  const long l = static_cast<long>(d);
  if (static_cast<double>(l) != d)
    throw ConfigError("config key '" + key + "': expected integer, got '" + *v + "'");
  return l;
}

bool Config::flag(const std::string& key, bool dflt) const {
  auto v = raw(key);
  if (!v) return dflt;
  std::string s = *v;
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  if (s == "true" || s == "1" || s == "yes" || s == "on") return true;
  if (s == "false" || s == "0" || s == "no" || s == "off") return false;
  throw ConfigError("config key '" + key + "': expected boolean, got '" + *v + "'");
}

double Config::need_num(const std::string& key) const {
  auto v = raw(key);
  if (!v) throw ConfigError("missing required config key '" + key + "'");
  return to_double(key, *v);
}

CostModel CostModel::from(const Config& c) {
  CostModel m;
  m.layers = static_cast<int>(c.integer("model.layers", 4));
  if (m.layers < 1) throw ConfigError("config key 'model.layers': must be >= 1");
  m.alpha = c.num("model.alpha_ms", 1.0) * 1e-3;
  m.beta = c.num("model.beta_us_per_token", 1.0) * 1e-6;
  m.kv = c.num("model.kv_bytes_per_token_layer", 1000.0);
  m.coll = c.num("model.coll_bytes_per_token_layer", 250.0);
  if (m.alpha < 0 || m.beta < 0 || m.alpha + m.beta <= 0)
    throw ConfigError("config key 'model.alpha_ms': per-layer compute must be positive");
  if (m.kv < 0) throw ConfigError("config key 'model.kv_bytes_per_token_layer': must be >= 0");
  if (m.coll < 0)
    throw ConfigError("config key 'model.coll_bytes_per_token_layer': must be >= 0");
  return m;
}

Layout Layout::from(const Config& c) {
  Layout l;
  l.units = static_cast<int>(c.integer("cluster.prefill_units", 1));
  l.hosts_per_unit = static_cast<int>(c.integer("cluster.hosts_per_unit", 2));
  l.decode_hosts = static_cast<int>(c.integer("cluster.decode_hosts", l.units));
  if (l.units < 1) throw ConfigError("config key 'cluster.prefill_units': must be >= 1");
  if (l.hosts_per_unit < 1) throw ConfigError("config key 'cluster.hosts_per_unit': must be >= 1");
  if (l.decode_hosts < 1) throw ConfigError("config key 'cluster.decode_hosts': must be >= 1");
  return l;
}

RunParams RunParams::from(const Config& c) {
  RunParams p;
  if (c.has("sim.horizon_s")) p.horizon = c.need_num("sim.horizon_s");
  p.tick = c.num("sim.promotion_tick_ms", 1.0) * 1e-3;
  if (!(p.tick > 0)) throw ConfigError("config key 'sim.promotion_tick_ms': must be positive");
  p.max_batch_tokens = c.integer("workload.max_batch_tokens", 8192);
  p.livelock = c.integer("sim.livelock_events", 1000000);
  return p;
}

WorkloadSpec WorkloadSpec::from(const Config& c) {
  WorkloadSpec w;
  w.rate = c.num("workload.rate_rps", 1.0);
  w.count = c.integer("workload.request_count", 100);
  w.prompt_mean = c.num("workload.prompt_mean_tokens", 2000.0);
  w.prompt_sigma = c.num("workload.prompt_sigma", 0.0);
  w.reuse_mean = c.num("workload.reuse_fraction_mean", 0.5);
  w.reuse_skew = c.num("workload.reuse_skew", 1.0);
  w.seed = static_cast<uint64_t>(c.integer("sim.seed", 1));
  w.trace = c.str("workload.trace", "");
  w.slo_mult = c.num("workload.slo_multiplier", 3.0);
  if (!(w.rate > 0)) throw ConfigError("config key 'workload.rate_rps': must be > 0");
  if (w.count < 0) throw ConfigError("config key 'workload.request_count': must be >= 0");
  if (w.reuse_mean < 0 || w.reuse_mean > 1)
    throw ConfigError("config key 'workload.reuse_fraction_mean': must be in [0,1]");
  if (!(w.slo_mult > 0)) throw ConfigError("config key 'workload.slo_multiplier': must be > 0");
  return w;
}

RmlqParams RmlqParams::make(int K, double E, double U) {
  if (K < 2) throw ConfigError("config key 'mfs.K': need at least 2 queues");
  if (!(E > 1.0)) throw ConfigError("config key 'mfs.E': threshold ratio must exceed 1");
  if (!(U > 0.0 && U <= 1.0)) throw ConfigError("config key 'mfs.U': scale must be in (0, 1]");
  RmlqParams r;
  r.K = K;
  r.E = E;
  r.U = U;
  double q = U;
  for (int i = 1; i < K; ++i) {  // Q_i = U / E^i by repeated division
    q /= E;
    r.thresholds.push_back(q);
  }
  return r;
}

RmlqParams RmlqParams::from(const Config& c) {
  return make(static_cast<int>(c.integer("mfs.K", 8)), c.num("mfs.E", 4.0), c.num("mfs.U", 0.5));
}

InterParams InterParams::from(const Config& c) {
  InterParams p;
  p.pruning = c.flag("inter.enable_pruning", true);
  p.drop_frac = c.num("inter.drop_budget_frac", 0.05);
  if (p.drop_frac < 0) throw ConfigError("config key 'inter.drop_budget_frac': must be >= 0");
  return p;
}

}  // namespace mfh
