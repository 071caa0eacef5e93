// Trace synthesis, validation, statistics and JSONL I/O.
//
// Bit-exact with the reference generator (proj/src/workload.cpp:136-217):
// stream 0 drives unit-rate Poisson gaps, stream 1+i drives request i's body,
// so request bodies depend only on (seed, i).
#include "trace.hpp"

#include <algorithm>
#include <fstream>
#include <map>
#include <unordered_set>

#include <json.hpp>

#include "base.hpp"

namespace ib2 {
using nlohmann::json;

const std::vector<ApiClass>& table1_classes() {
  // name, duration mean/var (s), calls per request mean/var, context mean/var,
  // returned tokens.  Paper Table 1 as encoded in workload.cpp:14-19.
  static const std::vector<ApiClass> k = {
      {"Math", 9e-5, 6e-5, 3.75, 1.3, 1422.0, 738.0, 20, 1.0},
      {"QA", 0.69, 0.17, 2.52, 1.73, 1846.0, 428.0, 54, 1.0},
      {"VE", 0.09, 0.014, 28.18, 15.2, 2185.0, 115.0, 11, 1.0},
      {"Chatbot", 28.6, 15.6, 4.45, 1.96, 753.0, 703.0, 65, 1.0},
      {"Image", 20.03, 7.8, 6.91, 3.93, 1247.0, 792.0, 36, 1.0},
      {"TTS", 17.24, 7.6, 6.91, 3.93, 1251.0, 792.0, 36, 1.0},
  };
  return k;
}

const ApiClass* table1_class(const std::string& name) {
  for (const auto& c : table1_classes())
    if (c.name == name) return &c;
  return nullptr;
}

int Request::total_decode() const {
  int n = 0;
  for (const auto& r : runs) n += r.decode_tokens;
  return n;
}

int Request::context_at_call(std::size_t j) const {
  int ctx = prompt_tokens;
  for (std::size_t k = 0; k <= j && k < runs.size(); ++k) {
    ctx += runs[k].decode_tokens;
    if (k < j && runs[k].call) ctx += runs[k].call->return_tokens;
  }
  return ctx;
}

double Request::total_call_time() const {
  double t = 0.0;
  for (const auto& r : runs)
    if (r.call) t += r.call->duration;
  return t;
}

int Request::call_count() const {
  int n = 0;
  for (const auto& r : runs) n += r.call ? 1 : 0;
  return n;
}

std::string Request::label() const {
  for (const auto& r : runs)
    if (r.call) return r.call->kind;
  return "plain";
}

void check_request(const Request& r) {
  const std::string who = "request " + std::to_string(r.id);
  if (r.runs.empty()) throw ValidationError(who + ": segments empty");
  if (r.prompt_tokens < 1) throw ValidationError(who + ": prompt_tokens must be >= 1");
  if (r.arrival < 0.0) throw ValidationError(who + ": negative arrival");
  const std::size_t last = r.runs.size() - 1;
  for (std::size_t i = 0; i <= last; ++i) {
    const DecodeRun& run = r.runs[i];
    if (run.decode_tokens < 1)
      throw ValidationError(who + ": segment " + std::to_string(i) + " has decode_tokens < 1");
    if (i == last && run.call) throw ValidationError(who + ": final segment carries an interception");
    if (i != last && !run.call)
      throw ValidationError(who + ": non-final segment " + std::to_string(i) + " lacks an interception");
    if (run.call && run.call->duration < 0.0) throw ValidationError(who + ": negative interception duration");
    if (run.call && run.call->return_tokens < 0) throw ValidationError(who + ": negative return_tokens");
  }
}

void check_trace(const std::vector<Request>& trace) {
  std::unordered_set<std::int64_t> seen;
  double prev = -1.0;
  for (const auto& r : trace) {
    check_request(r);
    if (!seen.insert(r.id).second) throw ValidationError("duplicate request id " + std::to_string(r.id));
    if (r.arrival < prev) throw ValidationError("trace not sorted by arrival");
    prev = r.arrival;
  }
}

namespace {

void check_spec(const WorkloadSpec& s) {
  if (s.request_count < 1) throw ConfigError("request_count must be >= 1");
  if (!(s.arrival_rate > 0.0)) throw ConfigError("arrival_rate must be > 0");
  if (s.classes.empty()) throw ConfigError("class mixture is empty");
  if (s.max_seq_len < 4) throw ConfigError("max_seq_len too small");
  double total = 0.0;
  for (const auto& c : s.classes) {
    const std::string who = "class " + c.name;
    if (!(c.weight > 0.0)) throw ConfigError(who + ": weight must be > 0");
    if (c.duration_var < 0.0 || c.count_var < 0.0 || c.context_var < 0.0)
      throw ConfigError(who + ": variances must be >= 0");
    if (!(c.context_mean > 0.0)) throw ConfigError(who + ": context_mean must be > 0");
    if (c.count_mean > 0.0 && !(c.duration_mean > 0.0)) throw ConfigError(who + ": duration_mean must be > 0");
    if (c.return_tokens < 0) throw ConfigError(who + ": return_tokens must be >= 0");
    total += c.weight;
  }
  if (std::abs(total - 1.0) > 1e-6) throw ConfigError("class weights must sum to 1");
}

std::size_t choose_class(const std::vector<ApiClass>& cls, double u) {
  double cum = 0.0;
  for (std::size_t i = 0; i < cls.size(); ++i) {
    cum += cls[i].weight;
    if (u < cum) return i;
  }
  return cls.size() - 1;
}

int round_int(double x) { return static_cast<int>(std::llround(x)); }

// Prompt share of the first context target (workload.cpp:189, 205).
int prompt_of(int target, double frac) { return std::max(1, std::min(target - 1, round_int(target * frac))); }

}  // namespace

std::vector<Request> synthesize(const WorkloadSpec& spec) {
  check_spec(spec);
  SplitMix gaps = SplitMix::for_stream(spec.seed, 0);
  std::vector<Request> out;
  out.reserve(static_cast<std::size_t>(spec.request_count));
  double clock = 0.0;
  for (int i = 0; i < spec.request_count; ++i) {
    clock += gaps.exponential(1.0);
    SplitMix g = SplitMix::for_stream(spec.seed, 1 + static_cast<std::uint64_t>(i));
    const ApiClass& cls = spec.classes[choose_class(spec.classes, g.uniform())];

    int calls = 0;
    if (cls.count_mean > 0.0) calls = std::max(1, round_int(g.lognormal(cls.count_mean, cls.count_var)));
    std::vector<double> dur(static_cast<std::size_t>(calls));
    for (double& d : dur) d = g.lognormal(cls.duration_mean, cls.duration_var);
    std::vector<int> ctx(static_cast<std::size_t>(calls));
    for (int& c : ctx) c = round_int(g.lognormal(cls.context_mean, cls.context_var));
    std::sort(ctx.begin(), ctx.end());
    const double frac = 0.5 + 0.4 * g.uniform();
    const int tail = std::max(1, round_int(g.lognormal(spec.final_decode_mean,
                                                       spec.final_decode_mean * spec.final_decode_mean)));
    Request r;
    r.id = i;
    r.arrival = clock / spec.arrival_rate;

    // Context at call j replays to exactly ctx[j] after clamping; calls that
    // no longer fit under max_seq_len are dropped (workload.cpp:179-197).
    int resume_ctx = 0;
    const int cap = spec.max_seq_len - cls.return_tokens - 1;
    for (int j = 0; j < calls; ++j) {
      const int lo = j == 0 ? 2 : resume_ctx + 1;
      if (lo > cap) break;
      const int target = std::max(std::min(ctx[j], cap), lo);
      DecodeRun run;
      if (j == 0) {
        r.prompt_tokens = prompt_of(target, frac);
        run.decode_tokens = target - r.prompt_tokens;
      } else {
        run.decode_tokens = target - resume_ctx;
      }
      run.call = ApiCall{cls.name, dur[static_cast<std::size_t>(j)], cls.return_tokens};
      r.runs.push_back(std::move(run));
      resume_ctx = target + cls.return_tokens;
    }
    DecodeRun last;
    if (r.runs.empty()) {
      int target = round_int(g.lognormal(cls.context_mean, cls.context_var));
      target = std::min(std::max(target, 2), spec.max_seq_len);
      r.prompt_tokens = prompt_of(target, frac);
      last.decode_tokens = target - r.prompt_tokens;
    } else {
      last.decode_tokens = std::max(1, std::min(tail, spec.max_seq_len - resume_ctx));
    }
    r.runs.push_back(std::move(last));
    check_request(r);
    out.push_back(std::move(r));
  }
  return out;
}

std::vector<ClassSummary> summarize(const std::vector<Request>& trace) {
  struct Acc {
    std::int64_t n = 0;
    std::vector<double> dur, cnt, ctx;
  };
  std::map<std::string, Acc> by;  // sorted by name, as the reference's output
  for (const auto& r : trace) {
    Acc& a = by[r.label()];
    a.n += 1;
    a.cnt.push_back(static_cast<double>(r.call_count()));
    std::size_t j = 0;
    for (const auto& run : r.runs) {
      if (!run.call) continue;
      a.dur.push_back(run.call->duration);
      a.ctx.push_back(static_cast<double>(r.context_at_call(j++)));
    }
  }
  auto moments = [](const std::vector<double>& xs, double& m, double& v) {
    m = 0.0;
    v = 0.0;
    if (xs.empty()) return;
    for (double x : xs) m += x;
    m /= static_cast<double>(xs.size());
    for (double x : xs) v += (x - m) * (x - m);
    v /= static_cast<double>(xs.size());
  };
  std::vector<ClassSummary> out;
  for (auto& [name, a] : by) {
    ClassSummary s;
    s.name = name;
    s.requests = a.n;
    s.interceptions = static_cast<std::int64_t>(a.dur.size());
    moments(a.dur, s.duration_mean, s.duration_var);
    moments(a.cnt, s.count_mean, s.count_var);
    moments(a.ctx, s.context_mean, s.context_var);
    out.push_back(std::move(s));
  }
  return out;
}

void write_trace_jsonl(const std::vector<Request>& trace, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw IoError("cannot open " + path + " for writing");
  f << json{{"format", "intercept-trace"}, {"version", 1}}.dump() << '\n';
  for (const auto& r : trace) {
    json runs = json::array();
    for (const auto& run : r.runs) {
      json jr;
      jr["decode"] = run.decode_tokens;
      if (run.call)
        jr["int"] = {{"kind", run.call->kind}, {"duration", run.call->duration}, {"ret", run.call->return_tokens}};
      runs.push_back(std::move(jr));
    }
    json jq;
    jq["id"] = r.id;
    jq["arrival"] = r.arrival;
    jq["prompt_tokens"] = r.prompt_tokens;
    jq["segments"] = std::move(runs);
    f << jq.dump() << '\n';
  }
  if (!f) throw IoError("write to " + path + " failed");
}

std::vector<Request> read_trace_jsonl(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open " + path);
  std::vector<Request> out;
  std::string line;
  std::size_t no = 0;
  bool header = false;
  auto where = [&] { return path + ":" + std::to_string(no) + ": "; };
  while (std::getline(f, line)) {
    ++no;
    if (line.empty()) continue;
    json j;
    try {
      j = json::parse(line);
    } catch (const json::exception& e) {
      throw ParseError(where() + e.what());
    }
    if (!header) {
      if (!j.contains("format") || j.at("format") != "intercept-trace")
        throw ParseError(where() + "missing intercept-trace header");
      if (j.at("version").get<int>() != 1) throw ParseError(where() + "unsupported trace version");
      header = true;
      continue;
    }
    try {
      Request r;
      r.id = j.at("id").get<std::int64_t>();
      r.arrival = j.at("arrival").get<double>();
      r.prompt_tokens = j.at("prompt_tokens").get<int>();
      for (const auto& js : j.at("segments")) {
        DecodeRun run;
        run.decode_tokens = js.at("decode").get<int>();
        if (js.contains("int")) {
          const json& c = js.at("int");
          run.call = ApiCall{c.at("kind").get<std::string>(), c.at("duration").get<double>(),
                             c.at("ret").get<int>()};
        }
        r.runs.push_back(std::move(run));
      }
      out.push_back(std::move(r));
    } catch (const json::exception& e) {
      throw ParseError(where() + e.what());
    }
  }
  if (!header) throw ParseError(path + ": empty file or missing header");
  std::stable_sort(out.begin(), out.end(), [](const Request& a, const Request& b) { return a.arrival < b.arrival; });
  check_trace(out);
  return out;
}

WorkloadSpec parse_workload_json(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw ParseError(std::string("workload JSON: ") + e.what());
  }
  WorkloadSpec s;
  try {
    s.request_count = j.at("request_count").get<int>();
    s.arrival_rate = j.at("arrival_rate").get<double>();
    if (j.contains("seed")) s.seed = j["seed"].get<std::uint64_t>();
    if (j.contains("max_seq_len")) s.max_seq_len = j["max_seq_len"].get<int>();
    if (j.contains("final_decode_mean")) s.final_decode_mean = j["final_decode_mean"].get<double>();
    if (!j.contains("classes") || !j["classes"].is_array() || j["classes"].empty())
      throw ConfigError("workload JSON: classes must be a non-empty array");
    double explicit_w = 0.0;
    int implicit = 0;
    for (const auto& jc : j["classes"]) {
      const std::string name = jc.at("name").get<std::string>();
      ApiClass c;
      if (const ApiClass* base = table1_class(name)) c = *base;
      c.name = name;
      auto take = [&](const char* key, auto& field) {
        if (jc.contains(key)) field = jc[key].template get<std::decay_t<decltype(field)>>();
      };
      take("duration_mean", c.duration_mean);
      take("duration_var", c.duration_var);
      take("count_mean", c.count_mean);
      take("count_var", c.count_var);
      take("context_mean", c.context_mean);
      take("context_var", c.context_var);
      take("return_tokens", c.return_tokens);
      if (jc.contains("weight")) {
        c.weight = jc["weight"].get<double>();
        explicit_w += c.weight;
      } else {
        c.weight = -1.0;
        ++implicit;
      }
      s.classes.push_back(std::move(c));
    }
    if (implicit > 0) {
      const double rest = 1.0 - explicit_w;
      if (rest <= 0.0) throw ConfigError("workload JSON: explicit weights leave no room for the rest");
      for (auto& c : s.classes)
        if (c.weight < 0.0) c.weight = rest / implicit;
    }
  } catch (const json::exception& e) {
    throw ParseError(std::string("workload JSON: ") + e.what());
  }
  return s;
}

std::string summaries_to_json(const std::vector<ClassSummary>& stats) {
  json j = json::object();
  for (const auto& s : stats)
    j[s.name] = {{"requests", s.requests},           {"interceptions", s.interceptions},
                 {"duration_mean", s.duration_mean}, {"duration_var", s.duration_var},
                 {"count_mean", s.count_mean},       {"count_var", s.count_var},
                 {"context_mean", s.context_mean},   {"context_var", s.context_var}};
  return j.dump(2);
}

}  // namespace ib2
