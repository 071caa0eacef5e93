#include "scheduler.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <thread>

#include <json.hpp>

#include "base.hpp"

namespace ib2 {

// ---------------------------------------------------------------- PosSet --

std::int64_t PosSet::size() const {
  std::int64_t n = 0;
  for (const auto& r : r_) n += r.second - r.first;
  return n;
}

void PosSet::add(std::int64_t lo, std::int64_t hi) {
  if (hi <= lo) return;
  r_.emplace_back(lo, hi);
  std::sort(r_.begin(), r_.end());
  std::vector<std::pair<std::int64_t, std::int64_t>> m;
  for (const auto& r : r_) {
    if (!m.empty() && r.first <= m.back().second) m.back().second = std::max(m.back().second, r.second);
    else m.push_back(r);
  }
  r_.swap(m);
}

std::vector<std::pair<std::int64_t, std::int64_t>> PosSet::take_low(std::int64_t n) {
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  while (n > 0 && !r_.empty()) {
    auto& f = r_.front();
    const std::int64_t k = std::min(n, f.second - f.first);
    out.emplace_back(f.first, f.first + k);
    f.first += k;
    n -= k;
    if (f.first == f.second) r_.erase(r_.begin());
  }
  return out;
}

std::vector<std::pair<std::int64_t, std::int64_t>> PosSet::take_high(std::int64_t n) {
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  while (n > 0 && !r_.empty()) {
    auto& b = r_.back();
    const std::int64_t k = std::min(n, b.second - b.first);
    out.emplace_back(b.second - k, b.second);
    b.second -= k;
    n -= k;
    if (b.first == b.second) r_.pop_back();
  }
  std::reverse(out.begin(), out.end());
  return out;
}

std::vector<std::pair<std::int64_t, std::int64_t>> PosSet::take_all() {
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  out.swap(r_);
  return out;
}

std::vector<std::pair<std::int64_t, std::int64_t>> PosSet::take_within(std::int64_t lo, std::int64_t hi) {
  std::vector<std::pair<std::int64_t, std::int64_t>> out, keep;
  for (const auto& r : r_) {
    const std::int64_t a = std::max(lo, r.first), b = std::min(hi, r.second);
    if (a >= b) {
      keep.push_back(r);
      continue;
    }
    out.emplace_back(a, b);
    if (r.first < a) keep.emplace_back(r.first, a);
    if (b < r.second) keep.emplace_back(b, r.second);
  }
  r_.swap(keep);
  return out;
}

// ------------------------------------------------------------- Scheduler --

Scheduler::Scheduler(const std::vector<Request>& trace, const CostModel& model, const RunConfig& cfg, PlanSink* sink)
    : trace_(trace), model_(model), cfg_(cfg), sink_(sink), kv_(model) {
  model_.validate();
  check_trace(trace_);
  st_.resize(trace_.size());
  for (std::size_t i = 0; i < trace_.size(); ++i) st_[i].req = &trace_[i];

  // Profiled estimator means: explicit, then Table 1, then the trace's own
  // empirical per-kind mean (engine.cpp:28-43).
  kind_mean_ = cfg_.profiled_means;
  for (const auto& c : table1_classes()) kind_mean_.emplace(c.name, c.duration_mean);
  std::unordered_map<std::string, std::pair<double, std::int64_t>> acc;
  for (const auto& r : trace_)
    for (const auto& run : r.runs)
      if (run.call) {
        auto& a = acc[run.call->kind];
        a.first += run.call->duration;
        a.second += 1;
      }
  for (const auto& [kind, a] : acc)
    if (a.second > 0) kind_mean_.emplace(kind, a.first / static_cast<double>(a.second));

  rep_.gpu_kv_capacity = model_.gpu_kv_capacity;
  if (!cfg_.event_log.empty()) {
    events_out_ = std::make_unique<std::ofstream>(cfg_.event_log);
    if (!*events_out_) throw IoError("cannot open " + cfg_.event_log + " for writing");
  }
  if (!cfg_.plan_log.empty()) {
    plans_out_ = std::make_unique<std::ofstream>(cfg_.plan_log);
    if (!*plans_out_) throw IoError("cannot open " + cfg_.plan_log + " for writing");
  }
  if (sink_) {
    const double per_block = static_cast<double>(model_.block_size) * model_.mem_per_token;
    const auto ledger_blocks = static_cast<std::int64_t>(std::floor((model_.gpu_kv_capacity + 0.5) / per_block));
    sink_->check_capacity(ledger_blocks, cfg_.estimator == Estimator::Dynamic, model_.block_size);
  }
  if (cfg_.clock != Clock::Virtual && !(sink_ && sink_->measure_steps()))
    throw ConfigError("run JSON: a measured clock (\"device\", \"wall\") needs the b200 executor");
  wall0_ = std::chrono::steady_clock::now();
}

double Scheduler::wall_seconds() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0_).count();
}

Scheduler::~Scheduler() = default;

double Scheduler::estimate_of(const Live& s) const {
  const ApiCall& call = *s.req->runs[static_cast<std::size_t>(s.run)].call;
  if (cfg_.estimator == Estimator::Oracle) return call.duration;
  if (cfg_.estimator == Estimator::Profiled) {
    auto it = kind_mean_.find(call.kind);
    return it != kind_mean_.end() ? it->second : call.duration;
  }
  return 0.0;  // Dynamic: t_now - t_call, evaluated while paused
}

// ---- plan recording ---------------------------------------------------------

void Scheduler::record(const Live& s, int kind, std::int64_t lo, std::int64_t hi) {
  if (hi <= lo && kind != ISIM_KV_RELEASE) return;
  isim_kv_op op;
  op.request_id = s.req->id;
  op.kind = kind;
  op.phase = phase_;
  op.pos_lo = lo;
  op.pos_hi = hi;
  ops_.push_back(op);
}

void Scheduler::add_span(const Live& s, std::int64_t pos, std::int64_t count, int kind, bool sample) {
  if (count <= 0) return;
  isim_row_span sp;
  sp.request_id = s.req->id;
  sp.pos = static_cast<std::int32_t>(pos);
  sp.count = static_cast<std::int32_t>(count);
  sp.kind = kind;
  sp.sample = sample ? 1 : 0;
  spans_.push_back(sp);
}

KvStatus Scheduler::op_grow(Live& s, std::int64_t n) {
  const std::int64_t lo = s.gpu.size() + s.cpu.size() + s.gone.size();
  const KvStatus r = kv_.grow(s.req->id, n);
  if (r == KvStatus::Ok && n > 0) {
    s.gpu.add(lo, lo + n);
    record(s, ISIM_KV_GROW, lo, lo + n);
  }
  return r;
}

KvStatus Scheduler::op_recompute(Live& s, std::int64_t n) {
  const KvStatus r = kv_.recompute(s.req->id, n);
  if (r == KvStatus::Ok)
    for (const auto& [lo, hi] : s.gone.take_low(n)) {
      s.gpu.add(lo, hi);
      record(s, ISIM_KV_RECOMPUTE, lo, hi);
    }
  return r;
}

KvStatus Scheduler::op_swap_in(Live& s, std::int64_t n) {
  const KvStatus r = kv_.to_gpu(s.req->id, n);
  if (r == KvStatus::Ok) {
    swapped_total_ += n;
    for (const auto& [lo, hi] : s.cpu.take_low(n)) {
      s.gpu.add(lo, hi);
      record(s, ISIM_KV_SWAP_IN, lo, hi);
    }
  }
  return r;
}

// A preserved remainder keeps the GPU prefix, so the suffix moves out; a
// discarded remainder moves the prefix out instead.  Either way the GPU copy
// stays a position prefix and restores append in position order.
KvStatus Scheduler::op_swap_out(Live& s, std::int64_t n, bool keep_rest) {
  const KvStatus r = kv_.to_cpu(s.req->id, n);
  if (r == KvStatus::Ok && n > 0) {
    swapped_total_ += n;
    for (const auto& [lo, hi] : keep_rest ? s.gpu.take_high(n) : s.gpu.take_low(n)) {
      s.cpu.add(lo, hi);
      record(s, ISIM_KV_SWAP_OUT, lo, hi);
    }
  }
  return r;
}

void Scheduler::op_discard_all(Live& s) {
  const std::int64_t n = kv_.counts(s.req->id).gpu;
  if (kv_.drop(s.req->id, n) != KvStatus::Ok || n == 0) return;
  for (const auto& [lo, hi] : s.gpu.take_all()) {
    s.gone.add(lo, hi);
    record(s, ISIM_KV_DISCARD, lo, hi);
  }
}

void Scheduler::op_release(Live& s) {
  const std::int64_t total = s.gpu.size() + s.cpu.size() + s.gone.size();
  kv_.forget(s.req->id);
  s.gpu.take_all();
  s.cpu.take_all();
  s.gone.take_all();
  record(s, ISIM_KV_RELEASE, 0, total);
}

// ---- queue movement ---------------------------------------------------------

void Scheduler::to_waiting(std::int64_t i, double key) {
  Live& s = st_[i];
  s.queue_key = key;
  s.at = Where::Waiting;
  waiting_.insert({key, i});
}

void Scheduler::to_running(std::int64_t i) {
  Live& s = st_[i];
  s.at = Where::Running;
  running_.insert({s.req->arrival, i});
}

void Scheduler::admit() {  // engine.cpp:69-76
  while (next_ < trace_.size() && trace_[next_].arrival <= now_) {
    const auto i = static_cast<std::int64_t>(next_++);
    st_[i].fresh_pending = st_[i].req->prompt_tokens;
    to_waiting(i, st_[i].req->arrival);
  }
}

void Scheduler::resume_returned() {  // engine.cpp:78-109
  while (!resumes_.empty() && resumes_.top().first <= now_) {
    const std::int64_t i = resumes_.top().second;
    resumes_.pop();
    Live& s = st_[i];
    paused_.erase(i);
    s.fresh_pending += s.req->runs[static_cast<std::size_t>(s.run)].call->return_tokens;
    s.run += 1;
    s.decoded_in_run = 0;
    s.preserved = false;
    s.t_call = 0.0;
    s.int_end = 0.0;
    const double key = cfg_.policy.requeue_at_tail ? now_ : s.req->arrival;
    const std::int64_t on_cpu = kv_.counts(s.req->id).cpu;
    if (on_cpu > 0) {
      s.swap_in_pending = on_cpu;
      s.queue_key = key;
      s.at = Where::SwapQueue;
      swapq_.insert({s.req->arrival, i});
      swap_demand_ += on_cpu;
    } else if (s.recompute_pending > 0) {
      to_waiting(i, key);
    } else {
      to_running(i);  // preserved context resident; returned tokens chunk from the running set
    }
  }
}

double Scheduler::running_gpu_tokens() const {
  double t = 0.0;
  for (const auto& [k, i] : running_) t += static_cast<double>(kv_.counts(st_[i].req->id).gpu);
  return t;
}

double Scheduler::paused_gpu_bytes() const {
  double b = 0.0;
  for (std::int64_t i : paused_) b += model_.bytes_for(kv_.counts(st_[i].req->id).gpu);
  return b;
}

void Scheduler::flip_dynamic() {  // engine.cpp:111-129
  if (cfg_.estimator != Estimator::Dynamic || cfg_.policy.preserve_mode != PreserveMode::MinWaste) return;
  const double other = running_gpu_tokens();
  const double chunk = std::max(1.0, model_.saturation_point - static_cast<double>(running_.size()));
  for (std::int64_t i : paused_) {
    Live& s = st_[i];
    if (!s.preserved) continue;
    const std::int64_t g = kv_.counts(s.req->id).gpu;
    if (g <= 0) continue;
    if (!assess(model_, now_ - s.t_call, static_cast<double>(g), other, chunk).keep) {
      op_discard_all(s);
      s.recompute_pending += g;
      s.preserved = false;
    }
  }
}

bool Scheduler::jump_idle() {  // engine.cpp:145-163
  double next = std::numeric_limits<double>::infinity();
  if (next_ < trace_.size()) next = std::min(next, trace_[next_].arrival);
  if (!resumes_.empty()) next = std::min(next, resumes_.top().first);
  if (!std::isfinite(next)) {
    std::string who = "?";
    if (!waiting_.empty()) who = std::to_string(st_[waiting_.begin()->second].req->id);
    else if (!swapq_.empty()) who = std::to_string(st_[swapq_.begin()->second].req->id);
    throw SimError("no runnable work and no pending events; request " + who + " cannot fit in GPU KV capacity");
  }
  rep_.waste.preserve += paused_gpu_bytes() * (next - now_);
  if (cfg_.clock == Clock::Wall) {  // online serving: wait for the event
    const double wait = next - (wall_seconds() + wall_offset_);
    if (wait > 0.0) std::this_thread::sleep_for(std::chrono::duration<double>(wait));
  }
  now_ = next;
  return true;
}

void Scheduler::unlink(std::int64_t i) {
  Live& s = st_[i];
  if (s.at == Where::Running) running_.erase({s.req->arrival, i});
  else if (s.at == Where::Waiting) waiting_.erase({s.queue_key, i});
  else throw SimError("detach from unexpected state for request " + std::to_string(s.req->id));
}

void Scheduler::evict(std::int64_t i) {  // engine.cpp:179-188
  Live& v = st_[i];
  const std::int64_t g = kv_.counts(v.req->id).gpu;
  op_discard_all(v);
  v.recompute_pending += g;
  v.preserved = false;
  running_.erase({v.req->arrival, i});
  to_waiting(i, v.req->arrival);
  if (events_out_) events_.push_back("evict:" + std::to_string(v.req->id));
  // Rows already batched for the victim this iteration are dropped from the
  // device batch ("ghost decodes"); the scheduler still counts them.
  // A dropped decode row's input id is already in the history (sampled by an
  // earlier iteration); a dropped FRESH span's synthetic ids are not, so its
  // positions are remembered and re-emitted as FRESH when recomputed.
  for (const auto& sp : spans_)
    if (sp.request_id == v.req->id && sp.kind == ISIM_SPAN_FRESH) v.unwritten.add(sp.pos, sp.pos + sp.count);
  spans_.erase(std::remove_if(spans_.begin(), spans_.end(),
                              [&](const isim_row_span& sp) { return sp.request_id == v.req->id; }),
               spans_.end());
}

void Scheduler::pause_for_call(std::int64_t i, std::vector<std::int64_t>& fired) {  // engine.cpp:190-202
  Live& s = st_[i];
  unlink(i);
  s.at = Where::Paused;
  paused_.insert(i);
  s.t_call = now_;
  s.int_end = now_ + s.req->runs[static_cast<std::size_t>(s.run)].call->duration;
  s.estimate = estimate_of(s);
  s.preserved = true;
  resumes_.push({s.int_end, i});
  fired.push_back(i);
}

void Scheduler::finish_request(std::int64_t i) {  // engine.cpp:204-216
  Live& s = st_[i];
  unlink(i);
  s.at = Where::Completed;
  s.completion = now_;
  s.materialized = 0;
  s.fresh_pending = 0;
  s.recompute_pending = 0;
  recomputing_.erase(i);
  s.recompute_restored = 0;
  s.unwritten.take_all();
  op_release(s);
  done_ += 1;
}

void Scheduler::dispose(const std::vector<std::int64_t>& fired, std::int64_t decode_count, std::int64_t out_budget,
                        std::int64_t* used_out, double* naive_stall) {  // engine.cpp:218-280
  if (fired.empty() || cfg_.policy.kind == PolicyKind::Preserve) return;
  if (cfg_.policy.kind == PolicyKind::NaiveSwap) {
    for (std::int64_t i : fired) {
      Live& s = st_[i];
      const std::int64_t g = kv_.counts(s.req->id).gpu;
      if (g <= 0) continue;
      if (op_swap_out(s, g, false) == KvStatus::Ok) {
        *naive_stall += model_.t_swap(static_cast<double>(g)) + model_.swap_launch_overhead;
        *used_out += g;
      } else {
        op_discard_all(s);
        s.recompute_pending += g;
      }
      s.preserved = false;
    }
    return;
  }
  std::vector<Paused> list;
  list.reserve(fired.size());
  for (std::int64_t i : fired) list.push_back({st_[i].req->id, kv_.counts(st_[i].req->id).gpu, st_[i].estimate});
  const double other = running_gpu_tokens();
  const double chunk = std::max(1.0, model_.saturation_point - static_cast<double>(decode_count));
  std::int64_t budget = 0;
  if (cfg_.policy.budgeted_swap) {
    std::int64_t ctx = 0;
    for (const auto& p : list) ctx += p.ctx;
    budget = split_swap_budget(out_budget, 0, ctx, kv_.gpu_free_tokens(), kv_.cpu_free_tokens()).out;
  }
  const auto verdicts = plan_paused(cfg_.policy, model_, list, other, chunk, budget, kv_.cpu_free_tokens());
  for (std::size_t k = 0; k < verdicts.size(); ++k) {
    Live& s = st_[fired[k]];
    const Verdict& v = verdicts[k];
    std::int64_t take = v.swap_out;
    const std::int64_t g = kv_.counts(s.req->id).gpu;
    const bool keep = v.keep_rest && g - take > 0;
    if (take > 0 && op_swap_out(s, take, keep) != KvStatus::Ok) take = 0;
    *used_out += take;
    const std::int64_t rest = kv_.counts(s.req->id).gpu;
    if (v.keep_rest && rest > 0) {
      s.preserved = true;
    } else {
      if (rest > 0) {
        op_discard_all(s);
        s.recompute_pending += rest;
      }
      s.preserved = false;
    }
  }
}

// ---- one iteration ------------------------------------------------------------

bool Scheduler::advance() {
  admit();
  resume_returned();
  if (done_ == trace_.size()) return false;
  if (now_ >= cfg_.max_sim_seconds) return false;
  phase_ = 0;  // ops recorded before an idle jump carry over into the next plan
  flip_dynamic();

  events_.clear();
  const bool logging = events_out_ != nullptr;
  const double paused_bytes = paused_gpu_bytes();  // preserve waste this iteration
  std::int64_t used_in = 0, used_out = 0, chunk_tokens = 0, recompute_tokens = 0;
  double stall = 0.0;

  // NaiveSwap: synchronous whole-context restores ahead of everything
  // (engine.cpp:303-322).
  if (cfg_.policy.kind == PolicyKind::NaiveSwap) {
    while (!swapq_.empty()) {
      const std::int64_t i = swapq_.begin()->second;
      Live& s = st_[i];
      const std::int64_t need = s.swap_in_pending;
      if (op_swap_in(s, need) != KvStatus::Ok) break;
      stall += model_.t_swap(static_cast<double>(need)) + model_.swap_launch_overhead;
      used_in += need;
      swap_demand_ -= need;
      s.swap_in_pending = 0;
      swapq_.erase(swapq_.begin());
      if (s.recompute_pending > 0) to_waiting(i, s.queue_key);
      else to_running(i);
      if (logging) events_.push_back("swapin:" + std::to_string(s.req->id));
    }
  }

  // Decode rows: one per running request with nothing pending; an allocation
  // failure evicts the newest running context, possibly itself (326-352).
  std::vector<std::int64_t> decodes;
  {
    const std::vector<Keyed> order(running_.begin(), running_.end());
    for (const auto& [key, i] : order) {
      Live& s = st_[i];
      if (s.at != Where::Running || s.fresh_pending + s.recompute_pending > 0) continue;
      const std::int64_t pos = kv_.counts(s.req->id).total();
      bool self = false;
      while (op_grow(s, 1) != KvStatus::Ok) {
        if (running_.empty())
          throw SimError("request " + std::to_string(s.req->id) +
                         " cannot obtain a decode token slot: GPU KV capacity too small");
        const std::int64_t victim = running_.rbegin()->second;
        evict(victim);
        if (victim == i) {
          self = true;
          break;
        }
      }
      if (!self) {
        s.materialized += 1;
        decodes.push_back(i);
        add_span(s, pos, 1, ISIM_SPAN_DECODE, true);
      }
    }
  }

  std::int64_t query = static_cast<std::int64_t>(decodes.size());
  const auto sat = static_cast<std::int64_t>(model_.saturation_point);

  // API-returned tokens of resumed resident requests (357-386).
  {
    const std::vector<Keyed> order(running_.begin(), running_.end());
    for (const auto& [key, i] : order) {
      Live& s = st_[i];
      if (s.at != Where::Running || s.fresh_pending <= 0) continue;
      const std::int64_t take =
          cfg_.policy.chunked_recompute ? std::min(s.fresh_pending, sat - query) : s.fresh_pending;
      if (take <= 0) continue;
      bool blocked = false;
      while (!kv_.room_for(take, s.req->id)) {
        auto v = running_.rbegin();
        while (v != running_.rend() && v->second == i) ++v;
        if (v == running_.rend()) {
          blocked = true;
          break;
        }
        evict(v->second);
      }
      if (blocked) continue;
      const std::int64_t pos = kv_.counts(s.req->id).total();
      op_grow(s, take);
      s.fresh_pending -= take;
      s.materialized += take;
      query += take;
      chunk_tokens += take;
      add_span(s, pos, take, ISIM_SPAN_FRESH, s.fresh_pending == 0);
    }
  }

  // Waiting queue: FCFS prefill / recompute chunks with head-of-line
  // blocking; recompute first, then fresh (388-424).
  std::vector<std::int64_t> recompute_ids;
  while (!waiting_.empty() && query < sat) {
    const std::int64_t i = waiting_.begin()->second;
    Live& s = st_[i];
    const std::int64_t pending = s.recompute_pending + s.fresh_pending;
    const std::int64_t take = cfg_.policy.chunked_recompute ? std::min(pending, sat - query) : pending;
    if (take <= 0 || !kv_.room_for(take, s.req->id)) break;
    const std::int64_t rec = std::min(take, s.recompute_pending);
    const std::int64_t fresh = take - rec;
    const bool completes = pending - take == 0;
    if (rec > 0) {
      const std::int64_t before = static_cast<std::int64_t>(spans_.size());
      const auto ranges = s.gone.ranges();  // lowest discarded first
      op_recompute(s, rec);
      std::int64_t left = rec;
      for (const auto& [lo, hi] : ranges) {
        if (left <= 0) break;
        const std::int64_t k = std::min(left, hi - lo);
        std::int64_t at = lo;
        for (const auto& [a, b] : s.unwritten.take_within(lo, lo + k)) {
          add_span(s, at, a - at, ISIM_SPAN_RECOMPUTE, false);
          add_span(s, a, b - a, ISIM_SPAN_FRESH, false);
          at = b;
        }
        add_span(s, at, lo + k - at, ISIM_SPAN_RECOMPUTE, false);
        left -= k;
      }
      if (fresh == 0 && completes && static_cast<std::int64_t>(spans_.size()) > before) spans_.back().sample = 1;
      if (s.recompute_restored == 0) recomputing_.insert(i);
      s.recompute_restored += rec;
      s.recompute_pending -= rec;
      recompute_ids.push_back(i);
    }
    if (fresh > 0) {
      const std::int64_t pos = kv_.counts(s.req->id).total();
      op_grow(s, fresh);
      s.fresh_pending -= fresh;
      s.materialized += fresh;
      add_span(s, pos, fresh, ISIM_SPAN_FRESH, completes);
    }
    query += take;
    chunk_tokens += take;
    recompute_tokens += rec;
    if (s.recompute_pending + s.fresh_pending == 0) {
      waiting_.erase(waiting_.begin());
      to_running(i);  // decodes from the next iteration
    } else {
      break;  // partially processed head keeps its place
    }
  }

  // Budgeted swap-in, FCFS over the swap queue (426-455).
  const std::int64_t batch_tokens = query;
  std::int64_t limit = 0;
  if (cfg_.policy.budgeted_swap) {
    limit = swap_limit_for(model_, static_cast<double>(batch_tokens));
    if (!swapq_.empty()) {
      std::int64_t room =
          split_swap_budget(limit, swap_demand_, 0, kv_.gpu_free_tokens(), kv_.cpu_free_tokens()).in;
      while (room > 0 && !swapq_.empty()) {
        const std::int64_t i = swapq_.begin()->second;
        Live& s = st_[i];
        const std::int64_t take = std::min(room, s.swap_in_pending);
        if (op_swap_in(s, take) != KvStatus::Ok) break;
        s.swap_in_pending -= take;
        swap_demand_ -= take;
        room -= take;
        used_in += take;
        if (s.swap_in_pending == 0) {
          swapq_.erase(swapq_.begin());
          if (s.recompute_pending + s.fresh_pending > 0) to_waiting(i, s.queue_key);
          else to_running(i);
        }
      }
    }
  }

  if (decodes.empty() && chunk_tokens == 0 && used_in == 0 && !(stall > 0.0)) return jump_idle();

  // The model step.  The virtual clock keeps the reference's analytic cost so
  // schedules stay bit-exact; the executor runs the real forward for the plan.
  // Measured clocks (f2) send the phase-0 ops and rows now, wait for the
  // forward, and advance by the measured time instead.
  const double d_model = model_.t_fwd(static_cast<double>(batch_tokens));
  double d_fwd = d_model;
  if (cfg_.clock != Clock::Virtual) {
    send_forward();
    const double dev = sink_->take_step_seconds();
    if (cfg_.clock == Clock::Device) d_fwd = dev;
    else d_fwd = std::max(0.0, wall_seconds() + wall_offset_ - now_);
  }
  now_ += d_fwd + stall;

  // Token effects at the iteration boundary (463-481).
  phase_ = 1;
  std::vector<std::int64_t> fired;
  for (std::int64_t i : decodes) {
    Live& s = st_[i];
    s.output_tokens += 1;
    if (s.first_token < 0.0) s.first_token = now_;
    s.decoded_in_run += 1;
    const DecodeRun& run = s.req->runs[static_cast<std::size_t>(s.run)];
    if (s.decoded_in_run == run.decode_tokens) {
      if (run.call) {
        pause_for_call(i, fired);
        if (logging) events_.push_back("fire:" + std::to_string(s.req->id));
      } else {
        finish_request(i);
        if (logging) events_.push_back("done:" + std::to_string(s.req->id));
      }
    }
  }

  double fire_stall = 0.0;
  dispose(fired, static_cast<std::int64_t>(decodes.size()), limit - used_in, &used_out, &fire_stall);
  now_ += fire_stall;
  if (cfg_.clock == Clock::Wall) wall_offset_ += stall + fire_stall;
  const double d_total = d_fwd + stall + fire_stall;

  // Realized waste (489-526).
  rep_.waste.preserve += paused_bytes * d_total;
  for (auto it = recomputing_.begin(); it != recomputing_.end();) {
    Live& s = st_[*it];
    rep_.waste.recompute += model_.bytes_for(s.recompute_restored) * d_total;
    if (s.recompute_pending == 0) {
      s.recompute_restored = 0;
      it = recomputing_.erase(it);
    } else {
      ++it;
    }
  }
  if (recompute_tokens > 0) {
    const double added = d_model - model_.t_fwd(static_cast<double>(batch_tokens - recompute_tokens));
    double others = 0.0;
    for (const auto& [key, i] : running_)
      if (std::find(recompute_ids.begin(), recompute_ids.end(), i) == recompute_ids.end())
        others += model_.bytes_for(kv_.counts(st_[i].req->id).gpu);
    rep_.waste.recompute += added * others;
  }
  const double total_stall = stall + fire_stall;
  if (total_stall > 0.0)
    rep_.waste.stall += total_stall * std::max(0.0, kv_.gpu_bytes() - paused_gpu_bytes());

  rep_.forwarding_time += d_fwd;
  if (batch_tokens > 0)
    rep_.recompute_time += d_fwd * static_cast<double>(recompute_tokens) / static_cast<double>(batch_tokens);

  iter_ += 1;
  IterationStat rec;
  rec.index = iter_;
  rec.t = now_;
  rec.batch_tokens = batch_tokens;
  rec.duration = d_total;
  rec.swap_in = used_in;
  rec.swap_out = used_out;
  rec.recompute_tokens = recompute_tokens;
  rec.stall = total_stall;
  if (cfg_.keep_iterations) rep_.iteration_log.push_back(rec);
  if (events_out_) log_iteration(rec);
  decode_rows_ += static_cast<std::int64_t>(decodes.size());
  batch_tokens_total_ += batch_tokens;
  emit_plan(rec);
  if (cfg_.invariants) verify();
  return true;
}

void Scheduler::emit_plan(const IterationStat& rec) {
  isim_batch_plan p;
  p.iteration = rec.index;
  p.t_end = rec.t;
  p.batch_tokens = rec.batch_tokens;
  p.swap_in_tokens = rec.swap_in;
  p.swap_out_tokens = rec.swap_out;
  p.recompute_tokens = rec.recompute_tokens;
  // Measured clocks already sent the phase-0 ops and the rows (send_forward).
  const std::size_t s0 = spans_sent_ ? spans_.size() : 0;
  p.n_ops = static_cast<std::int32_t>(ops_.size() - ops_sent_);
  p.n_spans = static_cast<std::int32_t>(spans_.size() - s0);
  p.ops = ops_.data() + ops_sent_;
  p.spans = spans_.data() + s0;
  if (plans_out_) {
    nlohmann::json j;
    j["it"] = rec.index;
    j["t"] = rec.t;
    j["B"] = rec.batch_tokens;
    auto ops = nlohmann::json::array();
    for (const auto& o : ops_) ops.push_back({o.request_id, o.kind, o.phase, o.pos_lo, o.pos_hi});
    auto sp = nlohmann::json::array();
    for (const auto& s : spans_) sp.push_back({s.request_id, s.pos, s.count, s.kind, s.sample});
    j["ops"] = std::move(ops);
    j["spans"] = std::move(sp);
    (*plans_out_) << j.dump() << '\n';
  }
  if (sink_ && (!spans_sent_ || p.n_ops > 0)) sink_->consume(p);
  ops_.clear();
  spans_.clear();
  ops_sent_ = 0;
  spans_sent_ = false;
}

void Scheduler::send_forward() {
  isim_batch_plan p;
  p.iteration = iter_ + 1;
  p.t_end = now_;
  p.batch_tokens = 0;
  for (const auto& sp : spans_) p.batch_tokens += sp.count;
  p.swap_in_tokens = p.swap_out_tokens = p.recompute_tokens = 0;
  p.n_ops = static_cast<std::int32_t>(ops_.size());
  p.n_spans = static_cast<std::int32_t>(spans_.size());
  p.ops = ops_.data();
  p.spans = spans_.data();
  sink_->consume(p);
  ops_sent_ = ops_.size();
  spans_sent_ = true;
}

void Scheduler::send_ops(std::vector<isim_kv_op>& ops) {
  if (ops.empty()) return;
  isim_batch_plan p;
  p.iteration = iter_;
  p.t_end = now_;
  p.batch_tokens = p.swap_in_tokens = p.swap_out_tokens = p.recompute_tokens = 0;
  p.n_ops = static_cast<std::int32_t>(ops.size());
  p.n_spans = 0;
  p.ops = ops.data();
  p.spans = nullptr;
  sink_->consume(p);
  ops.clear();
}

std::int64_t Scheduler::fast_forward(std::int64_t n, bool* finished) {
  if (cfg_.clock != Clock::Virtual) throw ConfigError("fast_forward needs the virtual clock");
  auto live = [](const Live& s) { return s.at != Where::NotArrived && s.at != Where::Completed; };
  auto make = [](std::int64_t rid, int kind, int phase, std::int64_t lo, std::int64_t hi) {
    isim_kv_op o;
    o.request_id = rid;
    o.kind = kind;
    o.phase = phase;
    o.pos_lo = lo;
    o.pos_hi = hi;
    return o;
  };
  std::vector<isim_kv_op> ops;
  if (sink_) {
    // Ops carried over from an idle jump go first, then every request the
    // sink holds (anything with positions) is released.
    ops.assign(ops_.begin() + static_cast<std::ptrdiff_t>(ops_sent_), ops_.end());
    for (const Live& s : st_)
      if (live(s) && !(s.gpu.empty() && s.cpu.empty() && s.gone.empty()))
        ops.push_back(make(s.req->id, ISIM_KV_RELEASE, 1, 0, s.gpu.size() + s.cpu.size() + s.gone.size()));
    send_ops(ops);
  }
  ops_.clear();
  spans_.clear();
  ops_sent_ = 0;
  spans_sent_ = false;
  PlanSink* keep = sink_;
  sink_ = nullptr;
  std::int64_t done = 0;
  bool fin = false;
  try {
    while (done < n) {
      const std::int64_t before = iter_;
      if (!advance()) {
        fin = true;
        break;
      }
      done += iter_ - before;
    }
  } catch (...) {
    sink_ = keep;
    throw;
  }
  sink_ = keep;
  ops_.clear();  // carried ops are reflected in the position sets handed over below
  if (finished) *finished = fin;
  if (!sink_) return done;
  // Hand-over, host positions first while the device pool is empty (each
  // batch is grown then swapped out, so it only borrows blocks), then every
  // GPU run in one plan.
  const std::int64_t batch = 8192;
  std::int64_t in_batch = 0;
  std::vector<isim_kv_op> post;
  for (const Live& s : st_) {
    if (!live(s) || s.cpu.empty()) continue;
    for (const auto& [lo, hi] : s.cpu.ranges()) {
      ops.push_back(make(s.req->id, ISIM_KV_GROW, 0, lo, hi));
      post.push_back(make(s.req->id, ISIM_KV_SWAP_OUT, 1, lo, hi));
      in_batch += hi - lo;
    }
    if (in_batch >= batch) {
      ops.insert(ops.end(), post.begin(), post.end());
      post.clear();
      send_ops(ops);
      in_batch = 0;
    }
  }
  ops.insert(ops.end(), post.begin(), post.end());
  send_ops(ops);
  for (const Live& s : st_)
    if (live(s))
      for (const auto& [lo, hi] : s.gpu.ranges()) ops.push_back(make(s.req->id, ISIM_KV_GROW, 0, lo, hi));
  send_ops(ops);
  return done;
}

void Scheduler::verify() const {  // engine.cpp:550-565
  if (kv_.gpu_bytes() > model_.gpu_kv_capacity + 1.0) throw SimError("GPU capacity invariant violated");
  if (kv_.cpu_bytes() > model_.cpu_kv_capacity + 1.0) throw SimError("CPU capacity invariant violated");
  for (const auto& s : st_) {
    if (s.at == Where::NotArrived || s.at == Where::Completed) continue;
    const KvCounts& c = kv_.counts(s.req->id);
    const std::string id = std::to_string(s.req->id);
    if (c.gpu < 0 || c.cpu < 0 || c.discarded < 0) throw SimError("negative ledger counter for request " + id);
    if (c.total() != s.materialized) throw SimError("context conservation violated for request " + id);
    if (c.discarded != s.recompute_pending) throw SimError("recompute bookkeeping mismatch for request " + id);
    // Position model agrees with the counts (new invariant).
    if (s.gpu.size() != c.gpu || s.cpu.size() != c.cpu || s.gone.size() != c.discarded)
      throw SimError("position map mismatch for request " + id);
  }
}

void Scheduler::log_iteration(const IterationStat& rec) {  // engine.cpp:567-581
  nlohmann::json j;
  j["it"] = rec.index;
  j["t"] = rec.t;
  j["B"] = rec.batch_tokens;
  j["d"] = rec.duration;
  j["swap_in"] = rec.swap_in;
  j["swap_out"] = rec.swap_out;
  j["recompute"] = rec.recompute_tokens;
  j["stall"] = rec.stall;
  j["events"] = events_;
  if (cfg_.ledger_every > 0 && rec.index % cfg_.ledger_every == 0) j["ledger"] = nlohmann::json::parse(kv_.snapshot());
  (*events_out_) << j.dump() << '\n';
}

RunReport Scheduler::conclude() {
  rep_.sim_wall = now_;
  rep_.iterations = iter_;
  rep_.requests.clear();
  rep_.requests.reserve(st_.size());
  for (const auto& s : st_) {
    RequestOutcome o;
    o.id = s.req->id;
    o.klass = s.req->label();
    o.arrival = s.req->arrival;
    o.first_token = s.first_token;
    o.completion = s.completion;
    o.output_tokens = s.output_tokens;
    o.call_time = s.req->total_call_time();
    o.incomplete = s.at != Where::Completed;
    rep_.requests.push_back(std::move(o));
  }
  return std::move(rep_);
}

}  // namespace ib2
