/*
 * mfsim-b200 device batch API: many independent simulation instances
 * (seeds x load x SLO scale x policy, or manual scenarios) executed by the
 * sm_100a engine in one launch, one warp per instance.
 *
 * Conventions follow the reference C ABI (proj/include/mfsim.h): int error
 * codes from mfsim.h, thread-local mfsim_last_error(), no exceptions across
 * the boundary, caller-owned inputs copied in, caller-allocated output
 * buffers. A context owns one CUDA stream (or uses the caller's, see
 * mfsim_dev_set_stream) and is not thread-safe.
 *
 * Each entry point replaces the reference call it accelerates:
 *   mfsim_dev_add_config   <- run_simulation input stage (sim_api.cpp:8-21):
 *                             build_topology, generate_workload / load_trace
 *   mfsim_dev_prepare      <- derive_slos (workload.cpp:199-217), batched:
 *                             every isolated_ttft probe of every instance in
 *                             one device launch
 *   mfsim_dev_launch       <- Engine::run (engine.cpp:595-657) per instance
 *   mfsim_dev_requests / _flows / _coflows
 *                          <- RunResult (engine.hpp:107-113)
 *   mfsim_dev_summary_json / _requests_csv / _write_report
 *                          <- summary_json / requests_csv / write_report
 *                             (metrics.cpp:84-142)
 */
#ifndef MFSIM_DEV_H
#define MFSIM_DEV_H

#include "mfsim.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfsim_dev mfsim_dev;

typedef struct mfsim_dev_stats {
  long long status;      /* MFSIM_OK or an error code for this instance */
  long long check;       /* internal check id when status != OK */
  long long events;      /* RunResult::events (engine.cpp:611) */
  long long steps;       /* scheduling steps (decide() calls) */
  long long flows;
  long long batches;
  long long coflows;
  long long pruned;      /* RunResult::pruned_count */
  long long max_active;
  long long pushes;      /* event-queue pushes (seq counter advance) */
  long long algo_bytes;  /* kernel-side algorithmic HBM bytes */
  long long requests;
  long long finished;
  long long slo_met;
  long long classes;     /* priority classes served by the allocator */
  long long rounds;      /* progressive-filling rounds of multi-flow classes */
} mfsim_dev_stats;

/* create a context on CUDA device `device` */
int mfsim_dev_create(int device, mfsim_dev** out);
void mfsim_dev_destroy(mfsim_dev* d);
/* run on the caller's cudaStream_t (NULL = the legacy default stream) */
int mfsim_dev_set_stream(mfsim_dev* d, void* cuda_stream);

/* queue one workload-mode instance from a config (policy, fabric, workload) */
int mfsim_dev_add_config(mfsim_dev* d, const mfsim_config* cfg);
/* queue one manual instance (spec text, see docs in INTEGRATION.md) */
int mfsim_dev_add_manual(mfsim_dev* d, const char* spec);
/* derive SLO deadlines (batched isolated runs on the device) and pack the
 * queued instances into device-arena images; nothing is uploaded yet */
int mfsim_dev_prepare(mfsim_dev* d);
/* H2D of all packed inputs (stream-ordered) */
int mfsim_dev_upload(mfsim_dev* d);
/* every instance from its initial state to completion, one launch on the
 * stream; returns immediately */
int mfsim_dev_launch(mfsim_dev* d);
/* H2D of the packed inputs only (running instances are not reset) */
int mfsim_dev_upload_inputs(mfsim_dev* d);
/* back to the initial state without launching */
int mfsim_dev_reset(mfsim_dev* d);
/* advance every unfinished instance by at most `budget` events (suspended
 * instances resume exactly where they stopped); returns immediately */
int mfsim_dev_launch_budget(mfsim_dev* d, long long budget);
/* advance every unfinished instance for `slice_ns` nanoseconds of device
 * time (all warps stop at the same deadline and suspend) */
int mfsim_dev_launch_slice(mfsim_dev* d, long long slice_ns);
/* instances not finished yet (synchronises the stream) */
int mfsim_dev_remaining(mfsim_dev* d);
/* wait for the stream; *kernel_ms receives the last launch's device time */
int mfsim_dev_sync(mfsim_dev* d, double* kernel_ms);
/* D2H: detail 0 = per-request results, 1 = + coflows, 2 = + flows/batches */
int mfsim_dev_download(mfsim_dev* d, int detail);
/* upload + launch + sync + download, re-running instances that hit a device
 * capacity bound with larger bounds */
int mfsim_dev_run(mfsim_dev* d, int detail);

int mfsim_dev_count(const mfsim_dev* d);
int mfsim_dev_stats_get(const mfsim_dev* d, int i, mfsim_dev_stats* out);
/* byte counts of the last upload / download (for e2e accounting) */
long long mfsim_dev_h2d_bytes(const mfsim_dev* d);
long long mfsim_dev_d2h_bytes(const mfsim_dev* d);
long long mfsim_dev_device_bytes(const mfsim_dev* d);
int mfsim_dev_kernel_launches(const mfsim_dev* d);
/* name of the kernel of the last launch ("mfsim_gang_kernel" for full batches,
 * "mfsim_engine_kernel" otherwise); static storage */
const char* mfsim_dev_last_kernel(const mfsim_dev* d);

/* raw per-instance device counters (events, steps, ..., phase cycles in
 * profiling builds); returns the number written */
int mfsim_dev_counters(const mfsim_dev* d, int i, long long* out, int cap);

/* per-request results; done = -1 when unfinished (ttft = done - arrival) */
int mfsim_dev_requests(const mfsim_dev* d, int i, double* arrival, double* deadline,
                       double* done, unsigned char* pruned, double* stall, int* batch,
                       long cap);
/* per-flow finish time (-1 unfinished) and final priority band / level */
int mfsim_dev_flows(const mfsim_dev* d, int i, double* finish, unsigned char* band,
                    unsigned char* level, long cap);
/* per-coflow release / done / stall (-1 = never) */
int mfsim_dev_coflows(const mfsim_dev* d, int i, double* release, double* done, double* stall,
                      long cap);
/* per-batch pipeline done time (-1 = never) */
int mfsim_dev_batches(const mfsim_dev* d, int i, double* done, long cap);

/* report formats of the reference (malloc'd; free with mfsim_string_free) */
int mfsim_dev_summary_json(const mfsim_dev* d, int i, char** out);
int mfsim_dev_requests_csv(const mfsim_dev* d, int i, char** out);
int mfsim_dev_write_report(const mfsim_dev* d, int i, const char* out_dir);

/* Topology::route (topology.cpp:83-89) of the fabric a config describes:
 * link ids src -> dst into links[0..cap); *n receives the route length;
 * *capacity (optional) receives each link's capacity in bytes/s */
int mfsim_route(const mfsim_config* cfg, int src, int dst, int* links, double* capacity, int cap,
                int* n);
/* number of links of the fabric a config describes */
int mfsim_link_count(const mfsim_config* cfg, int* n);

#ifdef __cplusplus
}
#endif

#endif /* MFSIM_DEV_H */
