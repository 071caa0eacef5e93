// run_json parsing: the reference keys (proj/src/config.cpp:88-125, including
// the undocumented "profiled_means") plus this framework's additions
// ("plan_log", "executor", "exec", "clock").  Unknown keys are ignored, as before.
#include <json.hpp>

#include "base.hpp"
#include "scheduler.hpp"

namespace ib2 {

RunConfig parse_run_json(const std::string& text) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("run JSON: ") + e.what());
  }
  RunConfig c;
  try {
    c.policy = Policy::named(policy_from_name(j.contains("policy") ? j["policy"].get<std::string>() : "infercept"));
    if (j.contains("estimator")) c.estimator = estimator_from_name(j["estimator"].get<std::string>());
    if (j.contains("max_sim_seconds")) c.max_sim_seconds = j["max_sim_seconds"].get<double>();
    if (j.contains("event_log")) c.event_log = j["event_log"].get<std::string>();
    if (j.contains("dump_ledger_every")) c.ledger_every = j["dump_ledger_every"].get<int>();
    if (j.contains("collect_iterations")) c.keep_iterations = j["collect_iterations"].get<bool>();
    if (j.contains("check_invariants")) c.invariants = j["check_invariants"].get<bool>();
    if (j.contains("chunked_recompute")) c.policy.chunked_recompute = j["chunked_recompute"].get<bool>();
    if (j.contains("budgeted_swap")) c.policy.budgeted_swap = j["budgeted_swap"].get<bool>();
    if (j.contains("preserve_mode")) {
      const std::string m = j["preserve_mode"].get<std::string>();
      if (m == "never") c.policy.preserve_mode = PreserveMode::Never;
      else if (m == "heuristic") c.policy.preserve_mode = PreserveMode::Heuristic;
      else if (m == "min-waste") c.policy.preserve_mode = PreserveMode::MinWaste;
      else throw ConfigError("run JSON: unknown preserve_mode " + m);
    }
    if (j.contains("heuristic_threshold")) c.policy.heuristic_threshold = j["heuristic_threshold"].get<double>();
    if (j.contains("profiled_means"))
      for (const auto& [kind, v] : j["profiled_means"].items()) c.profiled_means[kind] = v.get<double>();
    if (j.contains("clock")) {
      const std::string k = j["clock"].get<std::string>();
      if (k == "virtual") c.clock = Clock::Virtual;
      else if (k == "device") c.clock = Clock::Device;
      else if (k == "wall") c.clock = Clock::Wall;
      else throw ConfigError("run JSON: unknown clock " + k);
    }
    if (j.contains("plan_log")) c.plan_log = j["plan_log"].get<std::string>();
    if (j.contains("executor")) c.executor = j["executor"].get<std::string>();
    if (c.executor != "none" && c.executor != "b200") throw ConfigError("run JSON: unknown executor " + c.executor);
    if (j.contains("exec")) c.exec_json = j["exec"].dump();
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("run JSON: ") + e.what());
  }
  return c;
}

}  // namespace ib2
