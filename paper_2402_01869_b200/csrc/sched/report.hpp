// Run results: per-request outcomes, realized waste buckets and the derived
// serving metrics (normalized latency, req/s, TTFT, waste report).
// Reference: proj/include/interceptsim/metrics.hpp:15-81, metrics.cpp:30-125.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ib2 {

struct RequestOutcome {
  std::int64_t id = 0;
  std::string klass;
  double arrival = 0.0, first_token = -1.0, completion = -1.0;
  std::int64_t output_tokens = 0;
  double call_time = 0.0;
  bool incomplete = false;
};

struct IterationStat {
  std::int64_t index = 0;
  double t = 0.0;
  std::int64_t batch_tokens = 0;
  double duration = 0.0;
  std::int64_t swap_in = 0, swap_out = 0, recompute_tokens = 0;
  double stall = 0.0;
};

struct WasteTotals {
  double preserve = 0.0, recompute = 0.0, stall = 0.0;
  double total() const { return preserve + recompute + stall; }
};

struct RunReport {
  std::vector<RequestOutcome> requests;
  WasteTotals waste;
  double sim_wall = 0.0, forwarding_time = 0.0, recompute_time = 0.0, gpu_kv_capacity = 0.0;
  std::int64_t iterations = 0;
  std::vector<IterationStat> iteration_log;
};

double norm_latency_of(const RunReport& r);
double throughput_of(const RunReport& r, double horizon = -1.0);
double ttft_of(const RunReport& r);
std::int64_t completed_of(const RunReport& r);

struct WasteSummary {
  double preserve_gb_min = 0, recompute_gb_min = 0, stall_gb_min = 0, total_gb_min = 0;
  double pct_of_capacity_time = 0, recompute_fraction = 0;
};
WasteSummary waste_summary(const RunReport& r);

void write_outcomes_csv(const RunReport& r, const std::string& path);
std::string report_json(const RunReport& r);

}  // namespace ib2
