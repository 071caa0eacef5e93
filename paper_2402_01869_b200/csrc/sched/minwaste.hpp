// InferCept's min-waste interception policy: the GPU-memory-waste equations
// (paper Eq. 1-5; reference proj/src/waste.cpp:8-38), the per-iteration swap
// limit N_i and its in/out split (policy.cpp:69-95), and the waste-sorted
// greedy swap-out planner (policy.cpp:97-143).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "costmodel.hpp"

namespace ib2 {

enum class PolicyKind { VanillaDiscard, ImprovedDiscard, Preserve, NaiveSwap, InferCept };
enum class Estimator { Oracle, Profiled, Dynamic };
enum class PreserveMode { Never, Heuristic, MinWaste };

struct Policy {
  PolicyKind kind = PolicyKind::InferCept;
  bool chunked_recompute = false;
  bool budgeted_swap = false;
  PreserveMode preserve_mode = PreserveMode::Never;
  double heuristic_threshold = 1.0;
  bool requeue_at_tail = false;
  static Policy named(PolicyKind k);  // policy.cpp:10-31
};

PolicyKind policy_from_name(const std::string& s);
std::string policy_to_name(PolicyKind k);
Estimator estimator_from_name(const std::string& s);
std::string estimator_to_name(Estimator e);

// Waste components of one paused context, byte*seconds.
struct Waste {
  double preserve = 0, discard_oneshot = 0, swap_naive = 0, chunk_discard = 0;
  bool keep = true;  // true = Preserve wins (ties preserve)
  double key = 0;    // min(preserve, chunk_discard)
};
double waste_preserve(const CostModel& m, double t_int, double ctx);
double waste_discard_oneshot(const CostModel& m, double ctx, double other);
double waste_swap_naive(const CostModel& m, double ctx, double batch_ctx);
double waste_chunk_discard(const CostModel& m, double ctx, double other, double chunk);
Waste assess(const CostModel& m, double t_int, double ctx, double other, double chunk);

// N_i: tokens the link can move while the iteration's forward runs.
std::int64_t swap_limit_for(const CostModel& m, double batch_tokens);

struct SwapSplit {
  std::int64_t limit = 0, in = 0, out = 0;
};
SwapSplit split_swap_budget(std::int64_t limit, std::int64_t pending_in, std::int64_t pending_out,
                            std::int64_t free_gpu, std::int64_t free_cpu);

struct Paused {
  std::int64_t id = 0;
  std::int64_t ctx = 0;
  double t_hat = 0;
};
struct Verdict {
  std::int64_t id = 0;
  std::int64_t swap_out = 0;
  bool keep_rest = false;
  Waste w;
};
std::vector<Verdict> plan_paused(const Policy& p, const CostModel& m, const std::vector<Paused>& in, double other_ctx,
                                 double chunk, std::int64_t out_budget, std::int64_t cpu_free);

}  // namespace ib2
