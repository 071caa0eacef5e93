// Iteration-level serving scheduler (CPU, one thread per replica).
//
// Behaviour is the reference engine's, decision for decision and bit for bit
// (proj/src/engine.cpp:282-548): batch formation (decode rows, API-return
// chunks, FCFS prefill/recompute chunks, budgeted swap-in), the virtual clock
// advance by CostModel::t_fwd, token effects, min-waste interception
// dispositions and realized-waste accrual.  What is new is that every ledger
// operation carries the token POSITIONS it moves and every iteration is
// emitted as an isim_batch_plan to a PlanSink -- the B200 executor -- at the
// point the reference only charged t_fwd (engine.cpp:460).
#pragma once

#include <chrono>
#include <cstdint>
#include <fstream>
#include <memory>
#include <queue>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/infercept_b200.h"
#include "costmodel.hpp"
#include "kvaccount.hpp"
#include "minwaste.hpp"
#include "report.hpp"
#include "trace.hpp"

namespace ib2 {

// What advances the scheduler's clock each iteration.
//   Virtual: CostModel::t_fwd(B), the reference's charge (engine.cpp:460);
//            schedules are bit-exact with the reference.
//   Device:  the executor's measured device time of the iteration (the step
//            synchronises); idle periods still jump to the next event.
//   Wall:    real elapsed seconds since the run started (host + device);
//            idle periods sleep until the next arrival / API return, so
//            API calls are timed by the wall clock (online serving).
// Both measured clocks keep the model's charges for what the GPU does not
// execute (NaiveSwap stalls) and for the marginal recompute cost in the
// waste accounting.
enum class Clock { Virtual, Device, Wall };

struct RunConfig {
  Clock clock = Clock::Virtual;
  Policy policy = Policy::named(PolicyKind::InferCept);
  Estimator estimator = Estimator::Oracle;
  double max_sim_seconds = 86400.0;
  bool keep_iterations = false;
  std::string event_log;
  std::string plan_log;
  int ledger_every = 0;
  bool invariants = false;
  std::unordered_map<std::string, double> profiled_means;
  std::string executor = "none";
  std::string exec_json;  // {"model":..., "pools":..., "device":N}
};
RunConfig parse_run_json(const std::string& text);  // config.cpp:88-125 + additions

// Receives one plan per iteration, in order.
class PlanSink {
 public:
  virtual ~PlanSink() = default;
  virtual void consume(const isim_batch_plan& plan) = 0;
  // Measured clocks: enable per-consume device timing; false if unsupported.
  virtual bool measure_steps() { return false; }
  // Device seconds of the work enqueued by consume() since the previous call,
  // returned once that work has completed.
  virtual double take_step_seconds() { return -1.0; }
  // Called once before the first plan: the ledger's capacity in 16-token
  // blocks and whether the position model may hold up to two GPU runs per
  // request (Dynamic estimator).  A sink with a
  // physical block pool throws ConfigError if it cannot hold that.
  virtual void check_capacity(std::int64_t /*ledger_blocks*/, bool /*two_runs*/, int /*block_size*/) {}
};

// Sorted disjoint [lo,hi) position ranges of one request in one location.
class PosSet {
 public:
  std::int64_t size() const;
  bool empty() const { return r_.empty(); }
  void add(std::int64_t lo, std::int64_t hi);
  // Remove and return the lowest / highest n positions.
  std::vector<std::pair<std::int64_t, std::int64_t>> take_low(std::int64_t n);
  std::vector<std::pair<std::int64_t, std::int64_t>> take_high(std::int64_t n);
  std::vector<std::pair<std::int64_t, std::int64_t>> take_all();
  // Remove and return the members of [lo,hi), in position order.
  std::vector<std::pair<std::int64_t, std::int64_t>> take_within(std::int64_t lo, std::int64_t hi);
  const std::vector<std::pair<std::int64_t, std::int64_t>>& ranges() const { return r_; }

 private:
  std::vector<std::pair<std::int64_t, std::int64_t>> r_;
};

class Scheduler {
 public:
  Scheduler(const std::vector<Request>& trace, const CostModel& model, const RunConfig& cfg, PlanSink* sink);
  ~Scheduler();

  bool advance();          // one iteration, or one idle jump; false when done
  // Fast-forward: release every request the sink holds, run up to n
  // iterations without the sink (scheduler only, virtual clock), then hand
  // the sink the KV layout the ledger now describes -- each live request's
  // GPU positions grown in place and its host positions grown and swapped
  // out -- as plans without rows.  Scheduling is unchanged (the sink never
  // influences decisions); the sink's KV bytes are whatever the hand-over
  // wrote, so this serves timing (the bench), not numerics.  Returns the
  // iterations run.
  std::int64_t fast_forward(std::int64_t n, bool* finished);
  RunReport conclude();    // engine.cpp:583-601

  double now() const { return now_; }
  std::int64_t iterations() const { return iter_; }
  const KvAccount& kv() const { return kv_; }
  std::int64_t completed() const { return static_cast<std::int64_t>(done_); }
  std::int64_t decode_rows() const { return decode_rows_; }
  std::int64_t batch_tokens_total() const { return batch_tokens_total_; }
  std::int64_t swapped_tokens_total() const { return swapped_total_; }

 private:
  enum class Where { NotArrived, Waiting, Running, Paused, SwapQueue, Completed };
  using Keyed = std::pair<double, std::int64_t>;

  struct Live {
    const Request* req = nullptr;
    Where at = Where::NotArrived;
    int run = 0;
    int decoded_in_run = 0;
    std::int64_t fresh_pending = 0, recompute_pending = 0, swap_in_pending = 0, recompute_restored = 0;
    double queue_key = 0.0;
    bool preserved = false;
    double t_call = 0.0, int_end = 0.0, estimate = 0.0;
    std::int64_t materialized = 0;
    double first_token = -1.0, completion = -1.0;
    std::int64_t output_tokens = 0;
    PosSet gpu, cpu, gone;  // position model
    // Prompt / API-return positions whose FRESH rows were dropped by an
    // eviction in the same iteration: their token ids never reached the
    // device history, so their recompute is emitted as FRESH (synthetic ids).
    PosSet unwritten;
  };

  // queue / lifecycle
  void admit();
  void resume_returned();
  void flip_dynamic();
  bool jump_idle();
  void unlink(std::int64_t i);
  void evict(std::int64_t i);
  void pause_for_call(std::int64_t i, std::vector<std::int64_t>& fired);
  void finish_request(std::int64_t i);
  void dispose(const std::vector<std::int64_t>& fired, std::int64_t decode_count, std::int64_t out_budget,
               std::int64_t* used_out, double* naive_stall);
  double running_gpu_tokens() const;
  double paused_gpu_bytes() const;
  double estimate_of(const Live& s) const;
  void to_waiting(std::int64_t i, double key);
  void to_running(std::int64_t i);
  void verify() const;
  void log_iteration(const IterationStat& rec);

  // ledger operations that also move positions and record plan ops
  KvStatus op_grow(Live& s, std::int64_t n);
  KvStatus op_recompute(Live& s, std::int64_t n);
  KvStatus op_swap_in(Live& s, std::int64_t n);
  KvStatus op_swap_out(Live& s, std::int64_t n, bool keep_rest);
  void op_discard_all(Live& s);
  void op_release(Live& s);
  void record(const Live& s, int kind, std::int64_t lo, std::int64_t hi);
  void add_span(const Live& s, std::int64_t pos, std::int64_t count, int kind, bool sample);
  void emit_plan(const IterationStat& rec);
  void send_forward();        // measured clocks: phase-0 ops + rows, run now
  void send_ops(std::vector<isim_kv_op>& ops);  // a plan with ops only
  double wall_seconds() const;

  const std::vector<Request>& trace_;
  const CostModel& model_;
  RunConfig cfg_;
  PlanSink* sink_;

  std::vector<Live> st_;
  KvAccount kv_;
  std::set<Keyed> waiting_, running_, swapq_;
  std::set<std::int64_t> paused_, recomputing_;
  std::int64_t swap_demand_ = 0;
  std::priority_queue<Keyed, std::vector<Keyed>, std::greater<>> resumes_;
  std::size_t next_ = 0, done_ = 0;
  double now_ = 0.0;
  std::int64_t iter_ = 0;
  RunReport rep_;
  std::unordered_map<std::string, double> kind_mean_;
  std::unique_ptr<std::ofstream> events_out_, plans_out_;

  // per-iteration scratch
  int phase_ = 0;
  std::vector<std::string> events_;
  std::vector<isim_kv_op> ops_;
  std::vector<isim_row_span> spans_;
  std::int64_t decode_rows_ = 0, batch_tokens_total_ = 0, swapped_total_ = 0;
  std::size_t ops_sent_ = 0;  // measured clocks: ops_/spans_ already sent
  bool spans_sent_ = false;
  std::chrono::steady_clock::time_point wall0_;
  double wall_offset_ = 0.0;  // wall clock: virtual stall seconds added
};

}  // namespace ib2
