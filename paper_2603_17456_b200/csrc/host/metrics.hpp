// Result reduction and report formats (metrics.cpp:13-142): per-request TTFT,
// SLO flag evaluated as (done - arrival) <= (deadline - arrival), CCT and
// stall statistics, `requests.csv` with %.9g and `summary.json` through
// nlohmann::ordered_json (the same library the reference uses), so a replay
// is byte-identical to the reference's files.
#pragma once
#include <optional>
#include <string>
#include <vector>

namespace mfh {

struct RowInput {
  double arrival, deadline, stall;
  double done;  // -1 = unfinished
  bool pruned;
};

struct Report {
  struct Row {
    int id;
    double arrival;
    bool finished;
    double ttft, deadline_rel;
    bool met;
    double earliness, stall;
    bool pruned;
  };
  std::vector<Row> rows;
  std::vector<double> cct, stalls;
  long total = 0, finished = 0, met = 0, pruned = 0;
  std::optional<double> attainment, ttft_mean, ttft_p99, cct_mean, cct_p99, early_mean;
  double stall_mean = 0.0;
};

Report reduce(const std::vector<RowInput>& rows, const std::vector<double>& c_rel,
              const std::vector<double>& c_done, const std::vector<double>& c_stall,
              long pruned_count);
double nearest_rank(std::vector<double> v, double q);
std::string csv_text(const Report& r);
std::string json_text(const Report& r, const std::string& policy, long seed, double rate);
void write_files(const Report& r, const std::string& policy, long seed, double rate,
                 const std::string& dir);

}  // namespace mfh
