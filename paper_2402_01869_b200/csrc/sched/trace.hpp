// API-augmented request traces: the synthetic workload the serving hot path
// replays.  Semantics follow proj/include/interceptsim/workload.hpp:21-97 and
// trace_io.hpp (JSONL format "intercept-trace" v1).
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace ib2 {

// One API ("interception") class of Table 1: duration / count / context
// moments plus the number of tokens the API returns.
struct ApiClass {
  std::string name;
  double duration_mean = 0.0, duration_var = 0.0;
  double count_mean = 0.0, count_var = 0.0;
  double context_mean = 0.0, context_var = 0.0;
  int return_tokens = 0;
  double weight = 1.0;
};

const std::vector<ApiClass>& table1_classes();           // workload.cpp:12-22
const ApiClass* table1_class(const std::string& name);

struct ApiCall {
  std::string kind;
  double duration = 0.0;
  int return_tokens = 0;
};

// A decode run, optionally ended by an API call (absent only on the last).
struct DecodeRun {
  int decode_tokens = 0;
  std::optional<ApiCall> call;
};

struct Request {
  std::int64_t id = 0;
  double arrival = 0.0;
  int prompt_tokens = 0;
  std::vector<DecodeRun> runs;

  int total_decode() const;
  int context_at_call(std::size_t j) const;
  double total_call_time() const;
  int call_count() const;
  std::string label() const;
};

void check_request(const Request& r);                 // ValidationError
void check_trace(const std::vector<Request>& trace);  // ids unique, sorted

struct WorkloadSpec {
  std::vector<ApiClass> classes;
  int request_count = 0;
  double arrival_rate = 0.0;
  std::uint64_t seed = 0;
  int max_seq_len = 4096;
  double final_decode_mean = 32.0;
};

std::vector<Request> synthesize(const WorkloadSpec& spec);

struct ClassSummary {
  std::string name;
  std::int64_t requests = 0, interceptions = 0;
  double duration_mean = 0, duration_var = 0, count_mean = 0, count_var = 0,
         context_mean = 0, context_var = 0;
};
std::vector<ClassSummary> summarize(const std::vector<Request>& trace);

void write_trace_jsonl(const std::vector<Request>& trace, const std::string& path);
std::vector<Request> read_trace_jsonl(const std::string& path);

WorkloadSpec parse_workload_json(const std::string& text);
std::string summaries_to_json(const std::vector<ClassSummary>& s);

}  // namespace ib2
