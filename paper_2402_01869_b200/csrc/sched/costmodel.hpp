// Performance model the scheduler consults: the analytic forward-time curve
// (kept as the *virtual clock* so schedules stay bit-exact with the
// reference), swap time, and block-rounded KV bytes.
// Reference: proj/include/interceptsim/cost_model.hpp:20-49.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace ib2 {

struct CostModel {
  double t0 = 0.02;
  double slope_below = 3.0e-6;
  double slope_above = 5.0e-5;
  double saturation_point = 2048;
  double swap_per_token = 6.25e-5;
  double mem_per_token = 1.0e6;
  double gpu_kv_capacity = 80.0e9;
  double cpu_kv_capacity = 320.0e9;
  int block_size = 16;
  double swap_launch_overhead = 0.002;

  // Two-segment piecewise-linear forward time (cost_model.hpp:33-37).
  double t_fwd(double b) const {
    const double lo = b < saturation_point ? b : saturation_point;
    const double hi = b > saturation_point ? b - saturation_point : 0.0;
    return t0 + slope_below * lo + slope_above * hi;
  }
  double t_swap(double n) const { return swap_per_token * n; }
  std::int64_t blocks_for(std::int64_t tokens) const { return (tokens + block_size - 1) / block_size; }
  double bytes_for(std::int64_t tokens) const {
    return static_cast<double>(blocks_for(tokens)) * block_size * mem_per_token;
  }
  std::int64_t gpu_capacity_tokens() const { return static_cast<std::int64_t>(gpu_kv_capacity / mem_per_token); }
  void validate() const;
};

struct ForwardFit {
  double t0 = 0, slope_below = 0, slope_above = 0, saturation_point = 0, sse = 0;
};

ForwardFit fit_forward_curve(const std::vector<std::pair<double, double>>& pts);
std::vector<std::pair<double, double>> read_profile_csv(const std::string& path);
std::string cost_model_json(const CostModel& m);
CostModel cost_model_parse(const std::string& text);
CostModel cost_model_read(const std::string& path);
void cost_model_write(const CostModel& m, const std::string& path);

}  // namespace ib2
