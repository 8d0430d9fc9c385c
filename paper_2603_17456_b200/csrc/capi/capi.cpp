// C ABI of mfsim-b200: include/mfsim.h (the reference surface,
// proj/src/capi/mfsim_capi.cpp) and include/mfsim_dev.h (device batches).
// Exceptions never cross the boundary; each failing call records a message in
// a thread-local string and returns an mfsim.h error code.
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/mfsim.h"
#include "../../../include/mfsim_dev.h"
#include "../host/config.hpp"
#include "../host/instance.hpp"
#include "../host/metrics.hpp"

using namespace mfh;

struct mfsim_config {
  Config cfg;
  mutable std::string scratch;
};

struct mfsim_dev {
  std::unique_ptr<Backend> be;
  std::vector<InstanceInput> queued;
  std::unique_ptr<Batch> batch;
  long long h2d = 0, d2h = 0;
  double kernel_ms = 0.0;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return MFSIM_OK;
  } catch (const ConfigError& e) {
    return fail(MFSIM_ERR_CONFIG, e.what());
  } catch (const WorkloadError& e) {
    return fail(MFSIM_ERR_WORKLOAD, e.what());
  } catch (const IoError& e) {
    return fail(MFSIM_ERR_IO, e.what());
  } catch (const SimError& e) {
    return fail(MFSIM_ERR_SIM, e.what());
  } catch (const std::exception& e) {
    return fail(MFSIM_ERR_INTERNAL, e.what());
  }
}

int env_device() {
  const char* s = std::getenv("MFSIM_DEVICE");
  return s ? std::atoi(s) : 0;
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

Report report_of(const InstanceInput& in, const InstanceOutput& o) {
  const long n = static_cast<long>(o.ttft.size());
  std::vector<double> arr(n), dl(n);
  for (long r = 0; r < n; ++r) {
    arr[r] = request_arrival(in, static_cast<int>(r));
    dl[r] = request_deadline(in, static_cast<int>(r));
  }
  ReportColumns c;
  c.arrival = arr.data();
  c.deadline = dl.data();
  c.done = o.ttft.data();
  c.stall = o.stall.data();
  c.pruned = o.pruned.data();
  c.requests = n;
  c.cof_release = o.c_rel.data();
  c.cof_done = o.c_done.data();
  c.cof_stall = o.c_stall.data();
  c.coflows = static_cast<long>(o.c_done.size());
  c.pruned_count = static_cast<long>(o.out[mfb::OUT_PRUNED]);
  return summarize(c);
}

const InstanceOutput& checked(const mfsim_dev* d, int i) {
  if (!d || !d->batch || i < 0 || i >= d->batch->size())
    throw std::out_of_range("mfsim_dev: no results for that instance");
  return d->batch->output(i);
}

}  // namespace

extern "C" {

const char* mfsim_version(void) { return "0.1.0-b200"; }
const char* mfsim_last_error(void) { return g_err.c_str(); }

mfsim_config* mfsim_config_create(void) { return new mfsim_config(); }

mfsim_config* mfsim_config_load(const char* path) {
  if (!path) {
    fail(MFSIM_ERR_INVALID_ARG, "mfsim_config_load: path is NULL");
    return nullptr;
  }
  auto* h = new mfsim_config();
  if (guarded([&] { h->cfg = Config::load(path); }) != MFSIM_OK) {
    delete h;
    return nullptr;
  }
  return h;
}

int mfsim_config_set(mfsim_config* cfg, const char* key, const char* value) {
  if (!cfg || !key || !value) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_config_set: NULL argument");
  cfg->cfg.set(key, value);
  return MFSIM_OK;
}

const char* mfsim_config_get(const mfsim_config* cfg, const char* key) {
  if (!cfg || !key) return nullptr;
  auto v = cfg->cfg.raw(key);
  if (!v) return nullptr;
  cfg->scratch = *v;
  return cfg->scratch.c_str();
}

void mfsim_config_destroy(mfsim_config* cfg) { delete cfg; }

int mfsim_run(const mfsim_config* cfg, const char* out_dir, char** summary_json_out) {
  if (!cfg) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_run: config is NULL");
  return guarded([&] {
    InstanceInput in = workload_instance(cfg->cfg);
    auto be = make_backend(env_device());
    derive_deadlines(*be, {&in});
    Batch batch(*be, {in});
    batch.run(1);
    const InstanceOutput& o = batch.output(0);
    raise_status(o.out[mfb::OUT_STATUS], o.out[mfb::OUT_CHECK]);
    Report rep = report_of(batch.input(0), o);
    if (out_dir && *out_dir) write_report_files(rep, in.policy, in.seed, in.rate, out_dir);
    if (summary_json_out) *summary_json_out = dup_string(summary_json_text(rep, in.policy, in.seed, in.rate));
  });
}

void mfsim_string_free(char* s) { std::free(s); }

// ------------------------------------------------------------ device batches

int mfsim_dev_create(int device, mfsim_dev** out) {
  if (!out) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_create: out is NULL");
  *out = nullptr;
  return guarded([&] {
    auto d = std::make_unique<mfsim_dev>();
    d->be = make_backend(device);
    *out = d.release();
  });
}

void mfsim_dev_destroy(mfsim_dev* d) {
  if (!d) return;
  d->batch.reset();
  delete d;
}

int mfsim_dev_set_stream(mfsim_dev* d, void* stream) {
  if (!d) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_set_stream: NULL context");
  return guarded([&] { d->be->set_stream(stream); });
}

int mfsim_dev_add_config(mfsim_dev* d, const mfsim_config* cfg) {
  if (!d || !cfg) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_add_config: NULL argument");
  return guarded([&] { d->queued.push_back(workload_instance(cfg->cfg)); });
}

int mfsim_dev_add_manual(mfsim_dev* d, const char* spec) {
  if (!d || !spec) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_add_manual: NULL argument");
  return guarded([&] { d->queued.push_back(manual_instance(spec)); });
}

int mfsim_dev_prepare(mfsim_dev* d) {
  if (!d) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_prepare: NULL context");
  return guarded([&] {
    std::vector<InstanceInput*> need;
    for (auto& in : d->queued)
      if (!in.deadlines_ready) need.push_back(&in);
    derive_deadlines(*d->be, need);
    d->batch.reset();
    d->batch = std::make_unique<Batch>(*d->be, std::move(d->queued));
    d->queued.clear();
  });
}

int mfsim_dev_upload(mfsim_dev* d) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_upload: nothing prepared");
  return guarded([&] {
    d->batch->upload();
    d->h2d = static_cast<long long>(d->batch->input_bytes());
  });
}

int mfsim_dev_launch(mfsim_dev* d) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_launch: nothing prepared");
  return guarded([&] {
    d->batch->reset();
    d->batch->launch(0);
  });
}

int mfsim_dev_upload_inputs(mfsim_dev* d) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_upload_inputs: nothing prepared");
  return guarded([&] {
    d->batch->upload_inputs();
    d->h2d = static_cast<long long>(d->batch->input_bytes());
  });
}

int mfsim_dev_reset(mfsim_dev* d) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_reset: nothing prepared");
  return guarded([&] { d->batch->reset(); });
}

int mfsim_dev_launch_budget(mfsim_dev* d, long long budget) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_launch_budget: nothing prepared");
  return guarded([&] { d->batch->launch(budget); });
}

int mfsim_dev_launch_slice(mfsim_dev* d, long long slice_ns) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_launch_slice: nothing prepared");
  return guarded([&] { d->batch->launch(0, slice_ns); });
}

int mfsim_dev_remaining(mfsim_dev* d) {
  if (!d || !d->batch) return -1;
  int r = -1;
  guarded([&] { r = d->batch->remaining(); });
  return r;
}

int mfsim_dev_sync(mfsim_dev* d, double* kernel_ms) {
  if (!d) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_sync: NULL context");
  return guarded([&] {
    d->be->sync();
    d->kernel_ms = d->be->last_kernel_ms();
    if (kernel_ms) *kernel_ms = d->kernel_ms;
  });
}

int mfsim_dev_download(mfsim_dev* d, int detail) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_download: nothing prepared");
  return guarded([&] {
    d->batch->download(detail);
    d->d2h = static_cast<long long>(d->batch->output_bytes(detail));
  });
}

int mfsim_dev_run(mfsim_dev* d, int detail) {
  if (!d || !d->batch) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_run: nothing prepared");
  return guarded([&] {
    d->batch->run(detail);
    d->h2d = static_cast<long long>(d->batch->input_bytes());
    d->d2h = static_cast<long long>(d->batch->output_bytes(detail));
  });
}

int mfsim_dev_count(const mfsim_dev* d) { return d && d->batch ? d->batch->size() : 0; }
long long mfsim_dev_h2d_bytes(const mfsim_dev* d) { return d ? d->h2d : 0; }
long long mfsim_dev_d2h_bytes(const mfsim_dev* d) { return d ? d->d2h : 0; }
long long mfsim_dev_device_bytes(const mfsim_dev* d) {
  return d && d->batch ? static_cast<long long>(d->batch->device_bytes()) : 0;
}
int mfsim_dev_kernel_launches(const mfsim_dev* d) { return d ? d->be->kernel_launches() : 0; }
const char* mfsim_dev_last_kernel(const mfsim_dev* d) { return d ? d->be->last_kernel() : ""; }

int mfsim_dev_stats_get(const mfsim_dev* d, int i, mfsim_dev_stats* s) {
  if (!s) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_stats_get: NULL output");
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const InstanceInput& in = d->batch->input(i);
    *s = mfsim_dev_stats{};
    s->status = o.out[mfb::OUT_STATUS];
    s->check = o.out[mfb::OUT_CHECK];
    s->events = o.out[mfb::OUT_EVENTS];
    s->steps = o.out[mfb::OUT_STEPS];
    s->flows = o.out[mfb::OUT_NFLOWS];
    s->batches = o.out[mfb::OUT_NBATCHES];
    s->coflows = o.out[mfb::OUT_NCOFLOWS];
    s->pruned = o.out[mfb::OUT_PRUNED];
    s->max_active = o.out[mfb::OUT_MAXACTIVE];
    s->pushes = o.out[mfb::OUT_PUSHES];
    s->algo_bytes = o.out[mfb::OUT_ALGO_BYTES];
    s->classes = o.out[mfb::OUT_CLASSES];
    s->rounds = o.out[mfb::OUT_ROUNDS];
    s->requests = static_cast<long long>(o.ttft.size());
    for (size_t r = 0; r < o.ttft.size(); ++r) {
      if (o.ttft[r] == -1.0) continue;
      ++s->finished;
      const double a = request_arrival(in, static_cast<int>(r));
      if (o.ttft[r] - a <= request_deadline(in, static_cast<int>(r)) - a) ++s->slo_met;
    }
  });
}

int mfsim_dev_counters(const mfsim_dev* d, int i, long long* out, int cap) {
  if (!out) return -1;
  int n = -1;
  guarded([&] {
    const InstanceOutput& o = checked(d, i);
    n = cap < mfb::OUT_N ? cap : mfb::OUT_N;
    for (int k = 0; k < n; ++k) out[k] = o.out[k];
  });
  return n;
}

int mfsim_dev_requests(const mfsim_dev* d, int i, double* arrival, double* deadline, double* done,
                       unsigned char* pruned, double* stall, int* batch, long cap) {
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const InstanceInput& in = d->batch->input(i);
    const long n = static_cast<long>(o.ttft.size());
    if (cap < n) throw std::length_error("mfsim_dev_requests: buffer too small");
    for (long r = 0; r < n; ++r) {
      if (arrival) arrival[r] = request_arrival(in, static_cast<int>(r));
      if (deadline) deadline[r] = request_deadline(in, static_cast<int>(r));
      if (done) done[r] = o.ttft[r];
      if (pruned) pruned[r] = o.pruned[r];
      if (stall) stall[r] = o.stall[r];
      if (batch) batch[r] = o.rbatch[r];
    }
  });
}

int mfsim_dev_flows(const mfsim_dev* d, int i, double* finish, unsigned char* band,
                    unsigned char* level, long cap) {
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const long n = static_cast<long>(o.f_fin.size());
    if (cap < n) throw std::length_error("mfsim_dev_flows: buffer too small");
    for (long f = 0; f < n; ++f) {
      if (finish) finish[f] = o.f_fin[f];
      if (band) band[f] = o.f_band[f];
      if (level) level[f] = o.f_level[f];
    }
  });
}

int mfsim_dev_coflows(const mfsim_dev* d, int i, double* release, double* done, double* stall,
                      long cap) {
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const long n = static_cast<long>(o.c_done.size());
    if (cap < n) throw std::length_error("mfsim_dev_coflows: buffer too small");
    for (long c = 0; c < n; ++c) {
      if (release) release[c] = o.c_rel[c];
      if (done) done[c] = o.c_done[c];
      if (stall) stall[c] = o.c_stall[c];
    }
  });
}

int mfsim_dev_batches(const mfsim_dev* d, int i, double* done, long cap) {
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const long n = static_cast<long>(o.b_done.size());
    if (cap < n) throw std::length_error("mfsim_dev_batches: buffer too small");
    for (long b = 0; b < n; ++b)
      if (done) done[b] = o.b_done[b];
  });
}

int mfsim_dev_summary_json(const mfsim_dev* d, int i, char** out) {
  if (!out) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_summary_json: NULL output");
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const InstanceInput& in = d->batch->input(i);
    raise_status(o.out[mfb::OUT_STATUS], o.out[mfb::OUT_CHECK]);
    *out = dup_string(summary_json_text(report_of(in, o), in.policy, in.seed, in.rate));
  });
}

int mfsim_dev_requests_csv(const mfsim_dev* d, int i, char** out) {
  if (!out) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_requests_csv: NULL output");
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const InstanceInput& in = d->batch->input(i);
    raise_status(o.out[mfb::OUT_STATUS], o.out[mfb::OUT_CHECK]);
    *out = dup_string(requests_csv_text(report_of(in, o)));
  });
}

int mfsim_dev_write_report(const mfsim_dev* d, int i, const char* out_dir) {
  if (!out_dir) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_dev_write_report: NULL directory");
  return guarded([&] {
    const InstanceOutput& o = checked(d, i);
    const InstanceInput& in = d->batch->input(i);
    raise_status(o.out[mfb::OUT_STATUS], o.out[mfb::OUT_CHECK]);
    write_report_files(report_of(in, o), in.policy, in.seed, in.rate, out_dir);
  });
}

int mfsim_route(const mfsim_config* cfg, int src, int dst, int* links, double* capacity, int cap,
                int* n) {
  if (!cfg || !n) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_route: NULL argument");
  return guarded([&] {
    const Fabric f = Fabric::from(cfg->cfg);
    if (src < 0 || dst < 0 || src >= f.nodes() || dst >= f.nodes())
      throw ConfigError("mfsim_route: node out of range");
    const std::vector<int> r = f.route(src, dst);
    *n = static_cast<int>(r.size());
    for (int k = 0; k < static_cast<int>(r.size()) && k < cap; ++k) {
      if (links) links[k] = r[k];
      if (capacity) capacity[k] = f.links()[r[k]].capacity;
    }
  });
}

int mfsim_link_count(const mfsim_config* cfg, int* n) {
  if (!cfg || !n) return fail(MFSIM_ERR_INVALID_ARG, "mfsim_link_count: NULL argument");
  return guarded([&] { *n = static_cast<int>(Fabric::from(cfg->cfg).links().size()); });
}

}  // extern "C"
