// Reports of one finished instance, computed from the engine's column outputs.
//
// The device engine hands back per-request columns (done time, stall, pruned
// flag) and per-coflow columns (release, done, stall); the host folds them
// into the reference's two report files without building per-row objects:
//   requests.csv  -- header request_id,arrival_s,ttft_s,deadline_s,slo_met,
//                    earliness_s,stall_s; %.9g numbers, "nan" for unfinished
//                    rows (reference: metrics.cpp:84-106)
//   summary.json  -- the reference's ordered keys (metrics.cpp:108-125),
//                    dumped by nlohmann::ordered_json with 2-space indent so
//                    the bytes match the reference's
// Semantics kept from the reference: the SLO flag is (done - arrival) <=
// (deadline - arrival) (metrics.cpp:32-40), means are sequential sums in
// request / coflow id order divided by the count, p99 is the nearest rank
// ceil(0.99 n) of the sorted values (metrics.cpp:13-19).
#pragma once
#include <optional>
#include <string>
#include <vector>

namespace mfh {

// Column inputs of one instance (all by request id / coflow id).
struct ReportColumns {
  const double* arrival = nullptr;
  const double* deadline = nullptr;
  const double* done = nullptr;   // -1 = never finished
  const double* stall = nullptr;
  const unsigned char* pruned = nullptr;
  long requests = 0;
  const double* cof_release = nullptr;  // -1 = never released
  const double* cof_done = nullptr;     // -1 = never completed
  const double* cof_stall = nullptr;
  long coflows = 0;
  long pruned_count = 0;
};

// Derived per-request columns plus the scalar statistics of summary.json.
struct Report {
  std::vector<double> arrival, ttft, budget, earliness, stall;  // ttft/earliness NaN if unfinished
  std::vector<unsigned char> met;
  std::vector<double> cct, cof_stall;  // completed coflows only
  long total = 0, finished = 0, met_count = 0, pruned = 0;
  std::optional<double> attainment, ttft_mean, ttft_p99, cct_mean, cct_p99, early_mean;
  double stall_mean = 0.0;
};

Report summarize(const ReportColumns& in);
// nearest-rank quantile (q in (0, 1]) of a non-empty sample
double quantile_nearest_rank(std::vector<double> sample, double q);
std::string requests_csv_text(const Report& r);
std::string summary_json_text(const Report& r, const std::string& policy, long seed, double rate);
void write_report_files(const Report& r, const std::string& policy, long seed, double rate,
                        const std::string& dir);

}  // namespace mfh
