// B200 executor: turns one scheduler BatchPlan into device work.
//
// Per iteration, all on the compute stream (plans are enqueued asynchronously;
// the host never waits on the GPU outside record/sync):
//   1. plan upload: one H2D copy of rows / tiles / block deltas / swap
//      descriptors from a pinned ring;
//   2. K8 pre-phase block-table update (frees then allocs, LIFO free list);
//   3. K7 swap-in: H2D of each op's host extent into staging, scatter kernel;
//   4. forward: K9 embed -> per layer [K5 norm, K3 QKV, K4 RoPE+KV write,
//      K1 decode rows | K2 chunk tiles, K3 O (+residual), K5, K3 MLP in/out]
//      -> K5 final norm of sampling rows -> K3 LM head -> K6 argmax into the
//      token history;
//   5. K7 swap-out: gather kernel into staging, D2H into pinned host extents;
//   6. K8 post-phase frees (swap-outs, discards, releases).
// Swap copies are asynchronous cudaMemcpyAsync on a dedicated copy stream;
// staging buffers are double-buffered and ordered with events.
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <unordered_map>
#include <vector>

#include <json.hpp>

#include "executor.hpp"
#include "kernels.hpp"
#include "model.hpp"

namespace ib2 {

void set_gemm_activation_rows(std::int64_t rows);

namespace {

// First-fit allocator over the pinned host swap arena (byte offsets).
class HostArena {
 public:
  void reset(std::size_t bytes) {
    free_.clear();
    free_[0] = bytes;
    cap_ = bytes;
    used_ = 0;
  }
  static constexpr std::size_t kNone = ~std::size_t(0);
  std::size_t try_alloc(std::size_t n) {
    n = (n + 255) & ~std::size_t(255);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second >= n) {
        const std::size_t off = it->first, left = it->second - n;
        free_.erase(it);
        if (left) free_[off + n] = left;
        used_ += n;
        peak_ = std::max(peak_, used_);
        return off;
      }
    }
    return kNone;
  }
  std::string describe() const { return std::to_string(used_) + " of " + std::to_string(cap_) + " bytes in use"; }
  void release(std::size_t off, std::size_t n) {
    n = (n + 255) & ~std::size_t(255);
    used_ -= n;
    auto it = free_.emplace(off, n).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }
  std::size_t used() const { return used_; }
  std::size_t peak() const { return peak_; }

 private:
  std::map<std::size_t, std::size_t> free_;
  std::size_t cap_ = 0, used_ = 0, peak_ = 0;
};

// Positions [lo,hi) of one request living in a host extent laid out
// [L][n][2D] (n = hi0 - lo0 of the op that created it).
struct Extent {
  std::int64_t lo0, hi0;  // positions the extent was created for
  std::int64_t lo, hi;    // positions still resident on the host
  std::size_t off;        // arena offset
  std::size_t bytes;
  std::int64_t d2h_seq;   // 1-based index of the D2H batch that wrote it
  // The swap-out staging slot that held the extent's [L][n][2D] slab on the
  // way out, valid while that slot's generation is unchanged.
  int out_slot;
  std::int64_t out_gen;
  std::int64_t stage_off;
};

template <typename T>
T* dalloc(std::size_t n) {
  void* p = nullptr;
  IB2_CUDA(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

class Impl final : public B200Executor {
 public:
  Impl(const std::string& model_json, int device, const std::string& pools_json);
  ~Impl() override;

  void consume(const isim_batch_plan& plan) override;
  void sync() override;
  std::string stats_json() const override;
  std::int32_t last_tokens(std::int32_t* out, std::int32_t cap) const override;
  std::int64_t last_logits(float* out, std::int64_t cap) const override;
  std::int32_t block_table(std::int64_t request_id, std::int32_t* out, std::int32_t cap) const override;
  std::int64_t free_blocks() const override;
  void read_kv(std::int64_t request_id, std::int64_t lo, std::int64_t hi, void* out, std::int64_t cap) const override;
  void read_history(std::int64_t request_id, std::int64_t lo, std::int64_t hi, std::int32_t* out,
                    std::int64_t cap) const override;
  bool measure_steps() override {
    step_clock_ = true;
    return true;
  }
  double take_step_seconds() override;
  void check_capacity(std::int64_t ledger_blocks, bool two_runs, int block_size) override {
    if (block_size != kBlockTokens)
      throw ConfigError("executor: the cost model's block_size must be " + std::to_string(kBlockTokens));
    // Oracle / Profiled estimators keep every request's GPU positions a
    // prefix, so the device needs exactly the ledger's blocks; the Dynamic
    // estimator can leave two runs per request (at most 2 extra blocks each).
    const std::int64_t need = ledger_blocks + (two_runs ? 2LL * max_slots_ : 0);
    if (gpu_blocks_ < need)
      throw ConfigError("executor: gpu_blocks " + std::to_string(gpu_blocks_) + " < " + std::to_string(need) +
                        " (ledger capacity in blocks" + (two_runs ? " + 2 per live request for the Dynamic estimator" : "") +
                        ")");
  }

 private:
  // Measured clocks (scheduler Clock::Device / Wall): start / end events of
  // every consume() on the compute stream since the last take_step_seconds().
  bool step_clock_ = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> clk_pending_;
  std::int64_t last_iteration_ = -1;
  struct Touch {
    std::int32_t slot, lb;
    bool was_mapped;
  };
  int slot_for(std::int64_t rid);
  void apply_ops(const isim_batch_plan& p, int phase, std::vector<std::int32_t>& frees,
                 std::vector<std::int32_t>& allocs, std::vector<SwapDesc>& swaps_in, std::vector<SwapDesc>& swaps_out,
                 std::vector<std::int64_t>& released);
  void run_swaps(const std::vector<SwapDesc>& ops, const std::vector<std::int64_t>& req_of, bool swap_in);
  void forward(int n_rows, int n_drows, int n_tiles, int n_samples);
  void check_error();
  KvGeom geom() const {
    return KvGeom{pool_, gpu_blocks_, spec_.layers, spec_.heads, spec_.head_dim(), table_, max_lb_};
  }
  const f16* W(std::int64_t off) const { return off < 0 ? nullptr : weights_ + off; }

  ModelSpec spec_;
  WeightLayout wl_;
  int dev_ = 0;
  // copy_ carries D2H (swap-out), copy_in_ H2D (swap-in): PCIe is full duplex.
  cudaStream_t main_ = nullptr, copy_ = nullptr, copy_in_ = nullptr;
  // GPT-J parallel residual: the MLP branch (fc_in, fc_out) of a layer needs
  // only ln1(x), so it runs on aux_ concurrently with the attention branch;
  // its fp32 output (mlp_) is added by the O-projection epilogue, in the same
  // order as before: x = (x + attn W_o) + mlp.
  cudaStream_t aux_ = nullptr;
  bool overlap_mlp_ = true;
  std::vector<cudaEvent_t> ev_ln_, ev_mlp_;  // per layer
  float* mlp_ = nullptr;
  static constexpr int kSeqRing = 64;
  cudaEvent_t d2h_ring_[kSeqRing] = {}, h2d_ring_[kSeqRing] = {};
  std::int64_t d2h_seq_ = 0, h2d_seq_ = 0;
  struct PendingRelease {
    std::size_t off, bytes;
    std::int64_t h2d_seq;  // host memory reusable once this many H2D batches completed
  };
  std::vector<PendingRelease> pending_release_;
  void release_extent_memory(std::size_t off, std::size_t bytes) { pending_release_.push_back({off, bytes, h2d_seq_}); }
  void retire_host_memory(bool force);
  std::size_t host_alloc(std::size_t bytes);
  bool record_ = false, timing_ = false;
  bool force_row_attention_ = false;  // diagnostics: every row through K1
  bool fused_qkv_ = false;            // K4 in the QKV GEMM epilogue (opt-in)
  bool split_batch_ = false;          // decode / chunk rows as two micro-batches on two streams (opt-in)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  // diagnostics: per-iteration start events on the compute stream + the
  // iteration's composition (rows, decode rows, chunk rows, swap-in, swap-out)
  bool trace_iters_ = false;
  // per iteration: start, before forward, after forward (compute stream)
  std::vector<std::array<cudaEvent_t, 3>> iter_ev_;
  cudaEvent_t iter_mark(int which) {
    cudaEvent_t e;
    IB2_CUDA(cudaEventCreate(&e));
    IB2_CUDA(cudaEventRecord(e, main_));
    if (which == 0) iter_ev_.push_back({e, nullptr, nullptr});
    else iter_ev_.back()[which] = e;
    return e;
  }
  std::vector<std::array<std::int64_t, 5>> iter_info_;
  std::vector<std::array<double, 3>> iter_ms_;  // preamble, forward, swap-out + post phase
  // diagnostics: host/GPU timeline against a reference point taken in sync()
  cudaEvent_t trace_ref_ = nullptr;
  std::chrono::steady_clock::time_point trace_ref_host_;
  std::vector<double> iter_host_ms_;  // host time consume() started (rel. ref)
  std::vector<double> iter_lead_ms_;  // GPU start - host start of each iteration
  struct SwapTrace {
    std::int64_t iter;
    int dir;  // 0 = in (H2D), 1 = out (D2H)
    cudaEvent_t t0, t1;
    double bytes;
  };
  std::vector<SwapTrace> swap_trace_pending_;
  std::vector<std::array<double, 5>> swap_trace_;  // iter, dir, start, end (ms rel. ref), bytes
  // diagnostics: host seconds blocked per cause (plan ring, token ring, swap
  // slot reuse, host pool full) and host seconds inside consume()
  double host_block_s_[4] = {0, 0, 0, 0};
  double host_consume_s_ = 0.0;
  void sync_event(cudaEvent_t e, int cause) {
    if (!trace_iters_) {
      IB2_CUDA(cudaEventSynchronize(e));
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    IB2_CUDA(cudaEventSynchronize(e));
    host_block_s_[cause] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  f16* weights_ = nullptr;
  std::int64_t gpu_blocks_ = 0;
  int max_lb_ = 0, max_slots_ = 0, max_rows_ = 0, max_ctx_ = 0, hist_stride_ = 0, max_samples_ = 0;
  f16* pool_ = nullptr;
  std::int32_t *table_ = nullptr, *stack_ = nullptr, *top_ = nullptr, *err_ = nullptr, *hist_ = nullptr;
  float* rope_cs_ = nullptr;
  float *x_ = nullptr, *logits_ = nullptr, *part_o_ = nullptr, *part_ml_ = nullptr;
  std::int32_t* k1_counters_ = nullptr;  // K1 split arrival counters (last split merges)
  f16 *xn_ = nullptr, *qkv_ = nullptr, *attn_ = nullptr, *hid_ = nullptr, *lmrows_ = nullptr;
  std::int32_t* out_tok_ = nullptr;

  // plan upload
  // Plans in flight: the host may run this many iterations ahead of the GPU,
  // which is what lets a swap-in's H2D start long before the compute that
  // needs it.
  static constexpr int kRing = 16;
  std::size_t plan_bytes_ = 0;
  unsigned char* plan_host_[kRing] = {};      // pinned, mapped
  unsigned char* plan_host_dev_[kRing] = {};  // device view of plan_host_
  unsigned char* plan_dev_[kRing] = {};
  cudaEvent_t plan_done_[kRing] = {};
  int ring_ = 0;

  // swap
  unsigned char* host_pool_ = nullptr;
  std::size_t host_bytes_ = 0;
  HostArena arena_;
  std::unordered_map<std::int64_t, std::vector<Extent>> extents_;
  // Double-buffered swap staging.  Swap-outs: gather kernel (compute stream)
  // -> D2H on the copy stream, overlapping the next iteration.  Swap-ins: H2D
  // on the copy stream during this iteration's forward; the scatter kernel
  // runs at the start of the next iteration (the restored request cannot be
  // batched earlier: it leaves the swap queue only after this iteration).
  struct SwapBuf {
    f16* stage = nullptr;
    SwapDesc* desc_dev = nullptr;
    std::int32_t* prefix_dev = nullptr;
    SwapDesc* desc_host = nullptr;      // pinned
    std::int32_t* prefix_host = nullptr;  // pinned
    cudaEvent_t copied = nullptr;       // H2D (in) / D2H (out) finished on the copy stream
    cudaEvent_t consumed = nullptr;     // scatter (in) / gather (out) finished on the compute stream
  };
  struct PendingIn {
    int buf, n_ops, tokens;
    std::vector<std::int64_t> requests;  // whose blocks the scatter fills
  };
  static constexpr int kMaxSwapOps = 4096;
  int swap_slots_ = 3;  // staging buffers per direction
  std::vector<SwapBuf> in_, out_;
  int in_next_ = 0, out_next_ = 0;
  std::vector<std::int64_t> out_gen_;  // per swap-out slot: bumped when the slot is refilled
  // Swap-ins whose bytes are still in a swap-out staging slot (a request whose
  // API call returned before its swap-out slot was reused) are scattered from
  // that slot on the compute stream -- the same bytes, no PCIe round trip.
  struct FwdBuf {
    SwapDesc* desc_host = nullptr;  // pinned, mapped
    std::int32_t* prefix_host = nullptr;
    SwapDesc* desc_dev = nullptr;
    std::int32_t* prefix_dev = nullptr;
    cudaEvent_t done = nullptr;
  };
  static constexpr int kFwdBufs = 4;
  FwdBuf fwd_[kFwdBufs];
  int fwd_next_ = 0;
  std::int64_t swap_in_forwarded_tok_ = 0;
  std::vector<PendingIn> pending_in_;
  std::int64_t stage_tokens_ = 0;
  bool overlap_swaps_ = true;
  void flush_swap_ins();                       // all pending scatters
  void flush_swap_ins_for(const isim_batch_plan& p);  // those the plan touches
  void flush_swap_in_buffer(int buf);
  double swap_ms_ = 0.0;
  double swap_bytes_timed_ = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> swap_ev_pending_;
  std::vector<double> swap_ev_bytes_;
  cudaEvent_t new_timing_event();
  // sampled ids streamed to pinned host memory every iteration (the result
  // a serving frontend would read)
  std::int32_t* tok_host_[kRing] = {};      // pinned, mapped: the argmax kernel stores the ids here
  std::int32_t* tok_host_dev_[kRing] = {};
  cudaEvent_t tok_done_[kRing] = {};
  std::int64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
  cudaEvent_t mark_[2] = {};
 public:
  double timer(int op) override;
 private:

  // host mirrors
  std::unordered_map<std::int64_t, int> slot_of_;
  std::vector<int> free_slots_;
  std::vector<std::vector<std::uint8_t>> resid_;  // [slot][lblock] resident positions

  // record / stats
  std::vector<std::int32_t> last_tok_;
  std::vector<float> last_logits_;
  std::int64_t iters_ = 0, rows_total_ = 0, decode_rows_total_ = 0, chunk_rows_total_ = 0, swap_in_tok_ = 0,
               swap_out_tok_ = 0, samples_total_ = 0;
  double k1_bytes_timed_ = 0.0, k1_ms_ = 0.0;
  std::int64_t k1_launches_timed_ = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_free_, ev_pending_;
  std::vector<double> ev_bytes_;
  std::int64_t kernel_launches_ = 0;

  // per-iteration device views (valid during forward)
  const RowDesc* rows_dev_ = nullptr;
  const std::int32_t* drows_dev_ = nullptr;
  const TileDesc* tiles_dev_ = nullptr;
  const CombineDesc* combines_dev_ = nullptr;
  int n_combines_ = 0;
  float *chunk_ws_o_ = nullptr, *chunk_ws_ml_ = nullptr;
  const std::int32_t* samples_dev_ = nullptr;
  std::int32_t* tok_out_host_ = nullptr;
  template <typename T>
  static const void* mapped(const T* host) {
    void* d = nullptr;
    IB2_CUDA(cudaHostGetDevicePointer(&d, const_cast<T*>(host), 0));
    return d;
  }
  double k1_bytes_iter_ = 0.0;
  // Whole-step roofline (algorithmic): weights read once, KV read by K1 / K2
  // and written by K4; FLOPs of the projections, LM head and attention.  The
  // per-iteration bound is max(bytes / HBM, FLOPs / tensor peak).
  double roof_gbs_ = 6526.0, roof_tflops_ = 1662.0;
  double roof_bytes_ = 0.0, roof_flops_ = 0.0, roof_s_ = 0.0;
  int max_pos1_ = 0;
};

Impl::Impl(const std::string& model_json, int device, const std::string& pools_json) {
  spec_ = parse_model_json(model_json);
  wl_ = layout_weights(spec_);
  nlohmann::json pj = nlohmann::json::parse(pools_json.empty() ? "{}" : pools_json);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0)
    throw DeviceError("no CUDA device " + std::to_string(device) + " (B200 executor requires a GPU)");
  dev_ = device;
  IB2_CUDA(cudaSetDevice(dev_));
  cudaDeviceProp prop;
  IB2_CUDA(cudaGetDeviceProperties(&prop, dev_));
  if (prop.major != 10) throw DeviceError(std::string("executor is built for sm_100a; device is ") + prop.name);
  IB2_CUDA(cudaStreamCreateWithFlags(&main_, cudaStreamNonBlocking));
  IB2_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  IB2_CUDA(cudaStreamCreateWithFlags(&copy_in_, cudaStreamNonBlocking));
  IB2_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
  IB2_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  IB2_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  for (int i = 0; i < kSeqRing; ++i) {
    IB2_CUDA(cudaEventCreateWithFlags(&d2h_ring_[i], cudaEventDisableTiming));
    IB2_CUDA(cudaEventCreateWithFlags(&h2d_ring_[i], cudaEventDisableTiming));
  }
  record_ = pj.value("record", false);
  timing_ = pj.value("timing", false);
  force_row_attention_ = pj.value("row_attention", false);
  fused_qkv_ = pj.value("fused_qkv", getenv("IB2_FUSED_QKV") != nullptr);
  overlap_mlp_ = pj.value("overlap_mlp", getenv("IB2_NO_OVERLAP_MLP") == nullptr);
  // Off by default: measured 5.7 % slower on C4 (46.5 vs 44.0 ms per
  // iteration, profiles/r2e) -- the two chains contend for SMs (K1 fell from
  // 0.94 to 0.70 of the HBM peak) and the weights are streamed twice.
  split_batch_ = pj.value("split_batch", getenv("IB2_SPLIT_BATCH") != nullptr);
  trace_iters_ = pj.value("trace_iterations", false);

  roof_gbs_ = pj.value("roof_hbm_gbs", roof_gbs_);
  roof_tflops_ = pj.value("roof_tflops", roof_tflops_);
  max_slots_ = pj.value("max_requests", 1024);
  max_rows_ = pj.value("max_rows", 4096);
  max_ctx_ = pj.value("max_ctx", spec_.max_pos);
  max_ctx_ = (max_ctx_ + kBlockTokens - 1) / kBlockTokens * kBlockTokens;
  max_lb_ = max_ctx_ / kBlockTokens;
  hist_stride_ = max_ctx_ + 1;
  const std::int64_t M = spec_.kv_bytes_per_token();
  if (pj.contains("gpu_blocks")) {
    gpu_blocks_ = pj["gpu_blocks"].get<std::int64_t>();
  } else {
    const double cap = pj.value("gpu_kv_capacity", 1.0e9);
    const double m_cost = pj.value("mem_per_token", static_cast<double>(M));
    gpu_blocks_ = static_cast<std::int64_t>(cap / (m_cost * kBlockTokens)) + 2LL * max_slots_;
  }
  if (pj.contains("host_bytes")) {
    host_bytes_ = pj["host_bytes"].get<std::size_t>();
  } else {
    const double cpu = pj.value("cpu_kv_capacity", 4.0e9);
    const double m_cost = pj.value("mem_per_token", static_cast<double>(M));
    host_bytes_ = static_cast<std::size_t>(cpu / m_cost * static_cast<double>(M) * 1.25) + (64u << 20);
  }
  stage_tokens_ = pj.value("stage_tokens", 4096);
  swap_slots_ = std::max(2, pj.value("swap_slots", 3));
  overlap_swaps_ = pj.value("overlap_swaps", true);

  // weights
  weights_ = dalloc<f16>(wl_.total);
  for (const auto& it : wl_.items)
    launch_init_tensor(weights_ + it.off, it.count, spec_.weight_seed, it.id, it.kind, it.rows, it.cols, it.tiled,
                       main_);

  // KV pool and block tables
  const std::int64_t pool_elems = spec_.layers * gpu_blocks_ * 2LL * spec_.d_model * kBlockTokens;
  pool_ = dalloc<f16>(pool_elems);
  IB2_CUDA(cudaMemsetAsync(pool_, 0, pool_elems * sizeof(f16), main_));
  table_ = dalloc<std::int32_t>(static_cast<std::size_t>(max_slots_) * max_lb_);
  launch_fill_i32(table_, static_cast<std::int64_t>(max_slots_) * max_lb_, -1, main_);
  stack_ = dalloc<std::int32_t>(gpu_blocks_ + 16);
  launch_iota_desc(stack_, gpu_blocks_, main_);
  top_ = dalloc<std::int32_t>(1);
  err_ = dalloc<std::int32_t>(1);
  {
    const std::int32_t init[1] = {static_cast<std::int32_t>(gpu_blocks_)};
    IB2_CUDA(cudaMemcpyAsync(top_, init, 4, cudaMemcpyHostToDevice, main_));
    IB2_CUDA(cudaMemsetAsync(err_, 0, 4, main_));
  }
  hist_ = dalloc<std::int32_t>(static_cast<std::size_t>(max_slots_) * hist_stride_);
  IB2_CUDA(cudaMemsetAsync(hist_, 0, static_cast<std::size_t>(max_slots_) * hist_stride_ * 4, main_));
  resid_.assign(max_slots_, std::vector<std::uint8_t>(max_lb_, 0));
  for (int s = max_slots_ - 1; s >= 0; --s) free_slots_.push_back(s);

  // RoPE table [max_ctx][rot/2][cos,sin], computed in double on the host.
  if (spec_.rotary_dim) {
    const int half = spec_.rotary_dim / 2;
    std::vector<float> cs(static_cast<std::size_t>(max_ctx_) * spec_.rotary_dim);
    for (int p = 0; p < max_ctx_; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow(spec_.rope_theta, -2.0 * i / spec_.rotary_dim);
        const double a = static_cast<double>(p) * inv;
        cs[(static_cast<std::size_t>(p) * half + i) * 2] = static_cast<float>(std::cos(a));
        cs[(static_cast<std::size_t>(p) * half + i) * 2 + 1] = static_cast<float>(std::sin(a));
      }
    rope_cs_ = dalloc<float>(cs.size());
    IB2_CUDA(cudaMemcpy(rope_cs_, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  }

  // activations (every GEMM A operand buffer has max_rows rows)
  const std::int64_t D = spec_.d_model;
  x_ = dalloc<float>(static_cast<std::size_t>(max_rows_) * D);
  if (spec_.parallel_residual()) {
    mlp_ = dalloc<float>(static_cast<std::size_t>(max_rows_) * D);
    ev_ln_.resize(spec_.layers);
    ev_mlp_.resize(spec_.layers);
    for (int l = 0; l < spec_.layers; ++l) {
      IB2_CUDA(cudaEventCreateWithFlags(&ev_ln_[l], cudaEventDisableTiming));
      IB2_CUDA(cudaEventCreateWithFlags(&ev_mlp_[l], cudaEventDisableTiming));
    }
  }
  xn_ = dalloc<f16>(static_cast<std::size_t>(max_rows_) * D);
  qkv_ = dalloc<f16>(static_cast<std::size_t>(max_rows_) * 3 * D);
  attn_ = dalloc<f16>(static_cast<std::size_t>(max_rows_) * D);
  hid_ = dalloc<f16>(static_cast<std::size_t>(max_rows_) * spec_.ffn);
  lmrows_ = dalloc<f16>(static_cast<std::size_t>(max_rows_) * D);
  // Sampling rows and decode rows: at most one per live request.
  const std::size_t max_samples = static_cast<std::size_t>(std::min(max_rows_, max_slots_));
  max_samples_ = static_cast<int>(max_samples);
  logits_ = dalloc<float>(max_samples * spec_.vocab);
  out_tok_ = dalloc<std::int32_t>(max_rows_);
  const int max_splits = (max_ctx_ + 255) / 256;
  part_o_ = dalloc<float>(max_samples * spec_.heads * max_splits * spec_.head_dim());
  part_ml_ = dalloc<float>(max_samples * spec_.heads * max_splits * 2);
  k1_counters_ = dalloc<std::int32_t>(max_samples * spec_.heads);
  IB2_CUDA(cudaMemsetAsync(k1_counters_, 0, max_samples * spec_.heads * 4, main_));
  set_gemm_activation_rows(max_rows_);
  chunk_ws_o_ = dalloc<float>(static_cast<std::size_t>(kMaxChunkParts) * kChunkTileRows * spec_.head_dim());
  chunk_ws_ml_ = dalloc<float>(static_cast<std::size_t>(kMaxChunkParts) * kChunkTileRows * 2);

  // plan ring
  plan_bytes_ = static_cast<std::size_t>(max_rows_) * (sizeof(RowDesc) + 4 * 4) +
                static_cast<std::size_t>(kMaxChunkParts + max_rows_) * (sizeof(TileDesc) + sizeof(CombineDesc)) +
                static_cast<std::size_t>(max_slots_) * max_lb_ * 4 * 3 + 4096;
  for (int i = 0; i < kRing; ++i) {
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&plan_host_[i]), plan_bytes_ + 16, cudaHostAllocMapped));
    IB2_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&plan_host_dev_[i]), plan_host_[i], 0));
    plan_dev_[i] = dalloc<unsigned char>(plan_bytes_ + 16);
    IB2_CUDA(cudaEventCreateWithFlags(&plan_done_[i], cudaEventDisableTiming));
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&tok_host_[i]), static_cast<std::size_t>(max_rows_) * 4,
                           cudaHostAllocMapped));
    IB2_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&tok_host_dev_[i]), tok_host_[i], 0));
    IB2_CUDA(cudaEventCreateWithFlags(&tok_done_[i], cudaEventDisableTiming));
  }
  IB2_CUDA(cudaEventCreate(&mark_[0]));
  IB2_CUDA(cudaEventCreate(&mark_[1]));

  // swap path
  IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_pool_), host_bytes_, cudaHostAllocDefault));
  arena_.reset(host_bytes_);
  in_.resize(swap_slots_);
  out_.resize(swap_slots_);
  std::vector<SwapBuf*> all_bufs;
  for (auto& b : in_) all_bufs.push_back(&b);
  for (auto& b : out_) all_bufs.push_back(&b);
  for (SwapBuf* b : all_bufs) {
    b->stage = dalloc<f16>(static_cast<std::size_t>(stage_tokens_) * spec_.layers * 2 * D);
    b->desc_dev = dalloc<SwapDesc>(kMaxSwapOps + 1);
    b->prefix_dev = dalloc<std::int32_t>(kMaxSwapOps + 8);
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b->desc_host), (kMaxSwapOps + 1) * sizeof(SwapDesc),
                           cudaHostAllocMapped));
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b->prefix_host), (kMaxSwapOps + 8) * 4, cudaHostAllocMapped));
    IB2_CUDA(cudaEventCreateWithFlags(&b->copied, cudaEventDisableTiming));
    IB2_CUDA(cudaEventCreateWithFlags(&b->consumed, cudaEventDisableTiming));
  }
  out_gen_.assign(swap_slots_, 0);
  for (FwdBuf& f : fwd_) {
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&f.desc_host), (kMaxSwapOps + 1) * sizeof(SwapDesc),
                           cudaHostAllocMapped));
    IB2_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&f.prefix_host), (kMaxSwapOps + 8) * 4, cudaHostAllocMapped));
    f.desc_dev = dalloc<SwapDesc>(kMaxSwapOps + 1);
    f.prefix_dev = dalloc<std::int32_t>(kMaxSwapOps + 8);
    IB2_CUDA(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
  }
  IB2_CUDA(cudaStreamSynchronize(main_));
}

Impl::~Impl() {
  cudaDeviceSynchronize();
  for (auto& e : ev_free_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto& e : ev_pending_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (int i = 0; i < kRing; ++i) {
    cudaFreeHost(plan_host_[i]);
    cudaFree(plan_dev_[i]);
    cudaEventDestroy(plan_done_[i]);
    cudaFreeHost(tok_host_[i]);
    cudaEventDestroy(tok_done_[i]);
  }
  cudaEventDestroy(mark_[0]);
  cudaEventDestroy(mark_[1]);
  for (FwdBuf& f : fwd_) {
    cudaFreeHost(f.desc_host);
    cudaFreeHost(f.prefix_host);
    cudaFree(f.desc_dev);
    cudaFree(f.prefix_dev);
    cudaEventDestroy(f.done);
  }
  cudaFreeHost(host_pool_);
  std::vector<SwapBuf*> all_bufs;
  for (auto& b : in_) all_bufs.push_back(&b);
  for (auto& b : out_) all_bufs.push_back(&b);
  for (SwapBuf* b : all_bufs) {
    cudaFree(b->stage);
    cudaFree(b->desc_dev);
    cudaFree(b->prefix_dev);
    cudaFreeHost(b->desc_host);
    cudaFreeHost(b->prefix_host);
    cudaEventDestroy(b->copied);
    cudaEventDestroy(b->consumed);
  }
  void* ptrs[] = {weights_, pool_, table_, stack_, top_, err_, hist_, rope_cs_, x_, xn_, qkv_, attn_, hid_, lmrows_,
                  logits_, out_tok_, part_o_, part_ml_, k1_counters_, chunk_ws_o_, chunk_ws_ml_};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  cudaStreamDestroy(main_);
  cudaStreamDestroy(copy_);
  cudaStreamDestroy(copy_in_);
  cudaStreamDestroy(aux_);
  cudaEventDestroy(ev_fork_);
  cudaEventDestroy(ev_join_);
  for (cudaEvent_t e : ev_ln_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_mlp_) cudaEventDestroy(e);
  if (mlp_) cudaFree(mlp_);
  for (int i = 0; i < kSeqRing; ++i) {
    cudaEventDestroy(d2h_ring_[i]);
    cudaEventDestroy(h2d_ring_[i]);
  }
}

int Impl::slot_for(std::int64_t rid) {
  auto it = slot_of_.find(rid);
  if (it != slot_of_.end()) return it->second;
  if (free_slots_.empty()) throw DeviceError("executor: more live requests than max_requests");
  const int s = free_slots_.back();
  free_slots_.pop_back();
  slot_of_[rid] = s;
  return s;
}

// Residency bookkeeping of a phase's ops; emits the logical blocks whose
// occupancy crossed zero (in first-touch order) and the swap copy lists.
void Impl::apply_ops(const isim_batch_plan& p, int phase, std::vector<std::int32_t>& frees,
                     std::vector<std::int32_t>& allocs, std::vector<SwapDesc>& swaps_in,
                     std::vector<SwapDesc>& swaps_out, std::vector<std::int64_t>& released) {
  std::vector<Touch> touched;
  std::unordered_map<std::int64_t, std::size_t> seen;
  auto touch = [&](int slot, std::int64_t lo, std::int64_t hi, int sign) {
    if (hi > max_ctx_) throw DeviceError("executor: position beyond max_ctx");
    for (std::int64_t b = lo / kBlockTokens; b * kBlockTokens < hi; ++b) {
      const std::int64_t key = static_cast<std::int64_t>(slot) * max_lb_ + b;
      std::uint8_t& c = resid_[slot][b];
      if (!seen.count(key)) {
        seen[key] = touched.size();
        touched.push_back({slot, static_cast<std::int32_t>(b), c > 0});
      }
      const std::int64_t a = std::max(lo, b * kBlockTokens), e = std::min(hi, (b + 1) * kBlockTokens);
      const int v = static_cast<int>(c) + sign * static_cast<int>(e - a);
      if (v < 0 || v > kBlockTokens) throw DeviceError("executor: block residency out of range");
      c = static_cast<std::uint8_t>(v);
    }
  };
  for (int i = 0; i < p.n_ops; ++i) {
    const isim_kv_op& op = p.ops[i];
    if (op.phase != phase) continue;
    const int slot = slot_for(op.request_id);
    switch (op.kind) {
      case ISIM_KV_GROW:
      case ISIM_KV_RECOMPUTE:
        touch(slot, op.pos_lo, op.pos_hi, +1);
        break;
      case ISIM_KV_SWAP_IN:
        touch(slot, op.pos_lo, op.pos_hi, +1);
        swaps_in.push_back({slot, static_cast<std::int32_t>(op.pos_lo), static_cast<std::int32_t>(op.pos_hi - op.pos_lo),
                            0, 0});
        break;
      case ISIM_KV_SWAP_OUT:
        swaps_out.push_back({slot, static_cast<std::int32_t>(op.pos_lo),
                             static_cast<std::int32_t>(op.pos_hi - op.pos_lo), 0, 0});
        touch(slot, op.pos_lo, op.pos_hi, -1);
        break;
      case ISIM_KV_DISCARD:
        touch(slot, op.pos_lo, op.pos_hi, -1);
        break;
      case ISIM_KV_RELEASE:
        for (int b = 0; b < max_lb_; ++b) {
          if (!resid_[slot][b]) continue;
          const std::int64_t key = static_cast<std::int64_t>(slot) * max_lb_ + b;
          if (!seen.count(key)) {
            seen[key] = touched.size();
            touched.push_back({slot, b, true});
          }
          resid_[slot][b] = 0;
        }
        released.push_back(op.request_id);
        break;
      default:
        throw DeviceError("executor: unknown kv op kind");
    }
  }
  for (const Touch& t : touched) {
    const bool now = resid_[t.slot][t.lb] > 0;
    const std::int32_t e = t.slot * max_lb_ + t.lb;
    if (t.was_mapped && !now) frees.push_back(e);
    if (!t.was_mapped && now) allocs.push_back(e);
  }
}

void Impl::retire_host_memory(bool force) {
  if (force) {
    const auto t0 = std::chrono::steady_clock::now();
    IB2_CUDA(cudaStreamSynchronize(copy_in_));
    host_block_s_[3] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  std::size_t keep = 0;
  for (std::size_t i = 0; i < pending_release_.size(); ++i) {
    const PendingRelease& r = pending_release_[i];
    bool done = force || r.h2d_seq == 0;
    if (!done) {
      const cudaError_t q = cudaEventQuery(h2d_ring_[(r.h2d_seq - 1) % kSeqRing]);
      if (q != cudaSuccess && q != cudaErrorNotReady) IB2_CUDA(q);
      done = q == cudaSuccess;
    }
    if (done) arena_.release(r.off, r.bytes);
    else pending_release_[keep++] = r;
  }
  pending_release_.resize(keep);
}

std::size_t Impl::host_alloc(std::size_t bytes) {
  std::size_t off = arena_.try_alloc(bytes);
  if (off == HostArena::kNone) {
    retire_host_memory(true);
    off = arena_.try_alloc(bytes);
  }
  if (off == HostArena::kNone) throw DeviceError("pinned host swap pool exhausted (" + arena_.describe() + ")");
  return off;
}

// Swap-in scatters are issued lazily: the H2D of a batch overlaps later
// iterations until the restored request is touched by a plan (rows or ops),
// its staging buffer is recycled, or the executor synchronizes.
void Impl::flush_swap_in_buffer(int buf) {
  for (std::size_t i = 0; i < pending_in_.size(); ++i) {
    if (pending_in_[i].buf != buf) continue;
    const PendingIn p = pending_in_[i];
    pending_in_.erase(pending_in_.begin() + static_cast<std::ptrdiff_t>(i));
    SwapBuf& b = in_[p.buf];
    IB2_CUDA(cudaStreamWaitEvent(main_, b.copied, 0));  // descriptors + data landed (copy_in_)
    launch_swap_copy(b.desc_dev, b.prefix_dev, p.n_ops, p.tokens, geom(), b.stage, false, main_);
    ++kernel_launches_;
    IB2_CUDA(cudaEventRecord(b.consumed, main_));
    return;
  }
}

void Impl::flush_swap_ins() {
  while (!pending_in_.empty()) flush_swap_in_buffer(pending_in_.front().buf);
}

void Impl::flush_swap_ins_for(const isim_batch_plan& p) {
  if (pending_in_.empty()) return;
  std::vector<int> bufs;
  auto touched = [&](std::int64_t rid) {
    for (const PendingIn& q : pending_in_)
      if (std::find(q.requests.begin(), q.requests.end(), rid) != q.requests.end()) bufs.push_back(q.buf);
  };
  for (int i = 0; i < p.n_ops; ++i) touched(p.ops[i].request_id);
  for (int i = 0; i < p.n_spans; ++i) touched(p.spans[i].request_id);
  // Flush in issue order (a request may have batches in several buffers).
  for (std::size_t i = 0; i < pending_in_.size();) {
    if (std::find(bufs.begin(), bufs.end(), pending_in_[i].buf) != bufs.end()) flush_swap_in_buffer(pending_in_[i].buf);
    else ++i;
  }
}

void Impl::run_swaps(const std::vector<SwapDesc>& in_ops, const std::vector<std::int64_t>& req_of, bool swap_in) {
  if (in_ops.empty()) return;
  const std::int64_t D = spec_.d_model, L = spec_.layers;
  const std::size_t row_bytes = static_cast<std::size_t>(2 * D) * sizeof(f16);
  // Split ops at host-extent boundaries (swap-in) and at the staging size.
  std::vector<SwapDesc> ops;
  std::vector<std::pair<std::int64_t, std::size_t>> ext_of;  // (request, extent index)
  std::vector<std::pair<int, SwapDesc>> fwd;                 // (swap-out slot, scatter descriptor)
  std::vector<std::int64_t> fwd_reqs;
  for (std::size_t i = 0; i < in_ops.size(); ++i) {
    const SwapDesc& o = in_ops[i];
    if (!swap_in) {
      for (std::int32_t k = 0; k < o.n; k += static_cast<std::int32_t>(stage_tokens_)) {
        SwapDesc c = o;
        c.pos0 = o.pos0 + k;
        c.n = static_cast<std::int32_t>(std::min<std::int64_t>(stage_tokens_, o.n - k));
        ops.push_back(c);
        ext_of.push_back({req_of[i], 0});
      }
      continue;
    }
    auto& exts = extents_[req_of[i]];
    std::int64_t lo = o.pos0;
    const std::int64_t hi = o.pos0 + o.n;
    while (lo < hi) {
      std::size_t e = 0;
      while (e < exts.size() && !(exts[e].lo <= lo && lo < exts[e].hi)) ++e;
      if (e == exts.size()) throw DeviceError("executor: swap-in of positions not on the host");
      Extent& x = exts[e];
      if (x.out_slot >= 0 && out_gen_[x.out_slot] == x.out_gen) {
        // Still in its swap-out staging slot: forward from there.
        const std::int64_t end = std::min(hi, x.hi);
        fwd.push_back({x.out_slot,
                       SwapDesc{o.slot, static_cast<std::int32_t>(lo), static_cast<std::int32_t>(end - lo),
                                static_cast<std::int32_t>(x.hi0 - x.lo0),
                                x.stage_off + (lo - x.lo0) * 2 * D}});
        x.lo = end;
        fwd_reqs.push_back(req_of[i]);
        swap_in_forwarded_tok_ += end - lo;
        lo = end;
        continue;
      }
      const std::int64_t end = std::min({hi, x.hi, lo + stage_tokens_});
      ops.push_back({o.slot, static_cast<std::int32_t>(lo), static_cast<std::int32_t>(end - lo), 0, 0});
      ext_of.push_back({req_of[i], e});
      lo = end;
    }
  }
  if (!fwd.empty()) {
    std::stable_sort(fwd.begin(), fwd.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (std::size_t g0 = 0; g0 < fwd.size();) {
      std::size_t g1 = g0;
      while (g1 < fwd.size() && fwd[g1].first == fwd[g0].first && g1 - g0 < kMaxSwapOps) ++g1;
      FwdBuf& f = fwd_[fwd_next_];
      fwd_next_ = (fwd_next_ + 1) % kFwdBufs;
      sync_event(f.done, 2);
      f.prefix_host[0] = 0;
      const int n = static_cast<int>(g1 - g0);
      for (int k = 0; k < n; ++k) {
        f.desc_host[k] = fwd[g0 + k].second;
        f.prefix_host[k + 1] = f.prefix_host[k] + f.desc_host[k].n;
      }
      launch_copy_from_host(f.desc_dev, mapped(f.desc_host), n * sizeof(SwapDesc), main_);
      launch_copy_from_host(f.prefix_dev, mapped(f.prefix_host), (n + 1) * 4, main_);
      launch_swap_copy(f.desc_dev, f.prefix_dev, n, f.prefix_host[n], geom(), out_[fwd[g0].first].stage, false, main_);
      kernel_launches_ += 3;
      IB2_CUDA(cudaEventRecord(f.done, main_));
      g0 = g1;
    }
  }
  std::size_t first = 0;
  while (first < ops.size()) {
    std::size_t last = first;
    std::int64_t tok = 0;
    while (last < ops.size() && tok + ops[last].n <= stage_tokens_ && last - first < kMaxSwapOps) tok += ops[last++].n;
    const int n_ops = static_cast<int>(last - first);
    SwapBuf& b = swap_in ? in_[in_next_] : out_[out_next_];
    const int bi = swap_in ? in_next_ : out_next_;
    if (swap_in) in_next_ = (in_next_ + 1) % swap_slots_;
    else out_next_ = (out_next_ + 1) % swap_slots_;
    if (!swap_in) ++out_gen_[bi];  // the slot's previous slabs are about to be overwritten
    if (swap_in) flush_swap_in_buffer(bi);  // recycle: its previous batch must be scattered first
    // The pinned descriptor arrays of this buffer were last uploaded
    // swap_slots_ uses ago (swap-in: on copy_in_ before that batch's data;
    // swap-out: on the compute stream before its gather).
    sync_event(swap_in ? b.copied : b.consumed, 2);
    std::int64_t off = 0;
    b.prefix_host[0] = 0;
    for (int k = 0; k < n_ops; ++k) {
      b.desc_host[k] = ops[first + k];
      b.desc_host[k].stage_off = off;
      off += static_cast<std::int64_t>(b.desc_host[k].n) * L * 2 * D;
      b.prefix_host[k + 1] = b.prefix_host[k] + b.desc_host[k].n;
    }
    const int tokens = b.prefix_host[n_ops];
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (timing_ || trace_iters_) {
      t0 = new_timing_event();
      t1 = new_timing_event();
    }
    const double batch_bytes = static_cast<double>(tokens) * static_cast<double>(L) * static_cast<double>(row_bytes);
    if (swap_in) {
      IB2_CUDA(cudaStreamWaitEvent(copy_in_, b.consumed, 0));  // staging + descriptors free again
      IB2_CUDA(cudaMemcpyAsync(b.desc_dev, b.desc_host, n_ops * sizeof(SwapDesc), cudaMemcpyHostToDevice, copy_in_));
      IB2_CUDA(cudaMemcpyAsync(b.prefix_dev, b.prefix_host, (n_ops + 1) * 4, cudaMemcpyHostToDevice, copy_in_));
      std::int64_t need_d2h = 0;  // extents must have landed on the host
      for (int k = 0; k < n_ops; ++k)
        need_d2h = std::max(need_d2h, extents_[ext_of[first + k].first][ext_of[first + k].second].d2h_seq);
      if (need_d2h > 0) IB2_CUDA(cudaStreamWaitEvent(copy_in_, d2h_ring_[(need_d2h - 1) % kSeqRing], 0));
      if (t0) IB2_CUDA(cudaEventRecord(t0, copy_in_));
      for (int k = 0; k < n_ops; ++k) {
        const Extent& x = extents_[ext_of[first + k].first][ext_of[first + k].second];
        const std::int64_t n0 = x.hi0 - x.lo0;
        const unsigned char* src = host_pool_ + x.off + static_cast<std::size_t>(b.desc_host[k].pos0 - x.lo0) * row_bytes;
        IB2_CUDA(cudaMemcpy2DAsync(b.stage + b.desc_host[k].stage_off, static_cast<std::size_t>(b.desc_host[k].n) * row_bytes,
                                   src, static_cast<std::size_t>(n0) * row_bytes,
                                   static_cast<std::size_t>(b.desc_host[k].n) * row_bytes, L, cudaMemcpyHostToDevice,
                                   copy_in_));
        extents_[ext_of[first + k].first][ext_of[first + k].second].lo = b.desc_host[k].pos0 + b.desc_host[k].n;
      }
      IB2_CUDA(cudaEventRecord(b.copied, copy_in_));
      IB2_CUDA(cudaEventRecord(h2d_ring_[h2d_seq_ % kSeqRing], copy_in_));
      ++h2d_seq_;
      if (t1) {
        IB2_CUDA(cudaEventRecord(t1, copy_in_));
        swap_ev_pending_.push_back({t0, t1});
        swap_ev_bytes_.push_back(batch_bytes);
        if (trace_iters_ && trace_ref_) swap_trace_pending_.push_back({iters_, 0, t0, t1, batch_bytes});
      }
      std::vector<std::int64_t> reqs;
      for (int k = 0; k < n_ops; ++k)
        if (std::find(reqs.begin(), reqs.end(), ext_of[first + k].first) == reqs.end())
          reqs.push_back(ext_of[first + k].first);
      pending_in_.push_back({bi, n_ops, tokens, std::move(reqs)});
      if (!overlap_swaps_) flush_swap_ins();
    } else {
      IB2_CUDA(cudaStreamWaitEvent(main_, b.copied, 0));  // previous D2H out of this staging done
      launch_copy_from_host(b.desc_dev, mapped(b.desc_host), n_ops * sizeof(SwapDesc), main_);
      launch_copy_from_host(b.prefix_dev, mapped(b.prefix_host), (n_ops + 1) * 4, main_);
      kernel_launches_ += 2;
      launch_swap_copy(b.desc_dev, b.prefix_dev, n_ops, tokens, geom(), b.stage, true, main_);
      ++kernel_launches_;
      IB2_CUDA(cudaEventRecord(b.consumed, main_));
      IB2_CUDA(cudaStreamWaitEvent(copy_, b.consumed, 0));
      if (t0) IB2_CUDA(cudaEventRecord(t0, copy_));
      for (int k = 0; k < n_ops; ++k) {
        const std::size_t bytes = static_cast<std::size_t>(b.desc_host[k].n) * L * row_bytes;
        const std::size_t hoff = host_alloc(bytes);
        IB2_CUDA(cudaMemcpyAsync(host_pool_ + hoff, b.stage + b.desc_host[k].stage_off, bytes, cudaMemcpyDeviceToHost,
                                 copy_));
        extents_[ext_of[first + k].first].push_back({b.desc_host[k].pos0, b.desc_host[k].pos0 + b.desc_host[k].n,
                                                     b.desc_host[k].pos0, b.desc_host[k].pos0 + b.desc_host[k].n, hoff,
                                                     bytes, d2h_seq_ + 1, bi, out_gen_[bi], b.desc_host[k].stage_off});
      }
      IB2_CUDA(cudaEventRecord(b.copied, copy_));
      IB2_CUDA(cudaEventRecord(d2h_ring_[d2h_seq_ % kSeqRing], copy_));
      ++d2h_seq_;
      if (t1) {
        IB2_CUDA(cudaEventRecord(t1, copy_));
        swap_ev_pending_.push_back({t0, t1});
        swap_ev_bytes_.push_back(batch_bytes);
        if (trace_iters_ && trace_ref_) swap_trace_pending_.push_back({iters_, 1, t0, t1, batch_bytes});
      }
      if (!overlap_swaps_) IB2_CUDA(cudaStreamWaitEvent(main_, b.copied, 0));
    }
    first = last;
  }
  if (swap_in) {
    // Fully consumed extents return to the arena once the H2D copies reading
    // them have completed (the D2H stream may otherwise overwrite them).
    std::vector<std::int64_t> reqs = fwd_reqs;
    for (const auto& [rid, idx] : ext_of) {
      (void)idx;
      reqs.push_back(rid);
    }
    for (const std::int64_t rid : reqs) {
      auto& exts = extents_[rid];
      for (std::size_t e = 0; e < exts.size();) {
        if (exts[e].lo >= exts[e].hi) {
          release_extent_memory(exts[e].off, exts[e].bytes);
          exts.erase(exts.begin() + static_cast<std::ptrdiff_t>(e));
        } else {
          ++e;
        }
      }
    }
  }
}

void Impl::consume(const isim_batch_plan& p) {
  const auto consume_t0 = std::chrono::steady_clock::now();
  struct ConsumeTimer {
    const std::chrono::steady_clock::time_point t0;
    double& acc;
    ~ConsumeTimer() { acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
  } consume_timer{consume_t0, host_consume_s_};
  IB2_CUDA(cudaSetDevice(dev_));
  if (step_clock_) {
    clk_pending_.push_back({new_timing_event(), new_timing_event()});
    IB2_CUDA(cudaEventRecord(clk_pending_.back().first, main_));
  }
  retire_host_memory(false);
  if (trace_iters_) {
    iter_mark(0);
    iter_host_ms_.push_back(
        trace_ref_ ? std::chrono::duration<double, std::milli>(consume_t0 - trace_ref_host_).count() : -1.0);
  }
  const int D = spec_.d_model;

  // ---- host-side plan lowering ------------------------------------------------
  std::vector<std::int32_t> frees0, allocs0, frees1, allocs1;
  std::vector<SwapDesc> sw_in, sw_out, dummy;
  std::vector<std::int64_t> released0, released1;
  apply_ops(p, 0, frees0, allocs0, sw_in, dummy, released0);

  std::vector<RowDesc> rows;
  std::vector<std::int32_t> drows, samples;
  std::vector<TileDesc> tiles;
  // Rows of single-row spans (K1) first, then the chunk spans' rows (K2): the
  // two groups are the forward's micro-batches (split_batch_).  Sampling rows
  // stay in span order.
  std::vector<int> span_r0(p.n_spans);
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < p.n_spans; ++i) {
      const isim_row_span& sp = p.spans[i];
      const bool single = sp.count == 1 || force_row_attention_;
      if (single != (pass == 0)) continue;
      const int slot = slot_for(sp.request_id);
      const int r0 = static_cast<int>(rows.size());
      span_r0[i] = r0;
      if (sp.pos + sp.count > max_ctx_) throw DeviceError("executor: row position beyond max_ctx");
      for (int k = 0; k < sp.count; ++k)
        rows.push_back({slot, sp.pos + k, sp.kind == ISIM_SPAN_FRESH ? 1 : 0, 0, sp.request_id});
      if (single) {
        for (int k = 0; k < sp.count; ++k) drows.push_back(r0 + k);
      } else {
        for (int k = 0; k < sp.count; k += kChunkTileRows)
          tiles.push_back({r0 + k, std::min(kChunkTileRows, sp.count - k), slot, sp.pos + k, 0, 0, -1, 0});
      }
    }
  }
  for (int i = 0; i < p.n_spans; ++i)
    if (p.spans[i].sample) samples.push_back(span_r0[i] + p.spans[i].count - 1);
  const int n_rows = static_cast<int>(rows.size());
  if (n_rows > max_rows_) throw DeviceError("executor: batch exceeds max_rows");
  if (static_cast<int>(samples.size()) > max_samples_ || static_cast<int>(drows.size()) > max_samples_)
    throw DeviceError("executor: more sampling / decode rows than max_requests");
  // Split-KV for chunk tiles (one CTA per SM: K2 holds 512 TMEM columns):
  // key ranges of at most `per` keys, `per` ~ the whole (tile, head) key work
  // spread over the SMs, at least two key tiles, aligned to K2's key tile.
  std::vector<TileDesc> items;
  std::vector<CombineDesc> combines;
  {
    const int H = spec_.heads;
    const int bn = chunk_attention_key_tile(spec_.head_dim());
    std::int64_t work = 0;
    for (const TileDesc& t : tiles) work += static_cast<std::int64_t>(t.pos0 + t.nrows) * H;
    static const int min_keys = getenv("IB2_K2_MIN_KEYS") ? atoi(getenv("IB2_K2_MIN_KEYS")) : 2 * bn;
    const std::int64_t slots = 148LL * chunk_attention_ctas_per_sm(spec_.head_dim());
    std::int64_t per = std::max<std::int64_t>(min_keys, (work + slots - 1) / slots);
    per = (per + bn - 1) / bn * bn;
    int parts = 0;
    for (const TileDesc& t : tiles) {
      const int keys = t.pos0 + t.nrows;
      const int sp = static_cast<int>((keys + per - 1) / per);
      if (sp == 1 || (parts + sp) * H > kMaxChunkParts) {
        TileDesc w = t;
        w.kv_lo = 0;
        w.kv_hi = keys;
        w.part = -1;
        items.push_back(w);
        continue;
      }
      // Even split in whole key tiles.
      const int ktiles = (keys + bn - 1) / bn;
      const int step = (ktiles + sp - 1) / sp * bn;
      combines.push_back({t.row0, t.nrows, parts, 0});
      for (int lo = 0; lo < keys; lo += step) {
        TileDesc w = t;
        w.kv_lo = lo;
        w.kv_hi = std::min(keys, lo + step);
        w.part = parts++;
        items.push_back(w);
        combines.back().nparts += 1;
      }
    }
    // Longest items first (LPT): the CTAs are issued in item order, and a
    // causal prompt's last query tiles see 10-30x the keys of its first ones;
    // issued last, they set the kernel's tail (C3 recompute chunks: a 2,048-row
    // item list is 1..16 key units per item over 296 CTA slots).  Items carry
    // their rows, keys and partial slot, so the order is free.
    std::stable_sort(items.begin(), items.end(), [](const TileDesc& a, const TileDesc& b) {
      const int ka = std::min(a.kv_hi, a.pos0 + a.nrows) - a.kv_lo;
      const int kb = std::min(b.kv_hi, b.pos0 + b.nrows) - b.kv_lo;
      return ka > kb;
    });
  }

  std::vector<std::int64_t> sw_in_req;
  for (int i = 0; i < p.n_ops; ++i)
    if (p.ops[i].phase == 0 && p.ops[i].kind == ISIM_KV_SWAP_IN) sw_in_req.push_back(p.ops[i].request_id);

  // ---- upload -----------------------------------------------------------------
  const int k = ring_;
  ring_ = (ring_ + 1) % kRing;
  sync_event(plan_done_[k], 0);
  unsigned char* h = plan_host_[k];
  unsigned char* d = plan_dev_[k];
  std::size_t off = 0;
  auto put = [&](const void* src, std::size_t bytes) {
    const std::size_t at = off;
    if (at + bytes > plan_bytes_) throw DeviceError("executor: plan exceeds upload buffer");
    if (bytes) std::memcpy(h + at, src, bytes);
    off = (at + bytes + 15) & ~std::size_t(15);
    return d + at;
  };
  const RowDesc* d_rows = reinterpret_cast<const RowDesc*>(put(rows.data(), rows.size() * sizeof(RowDesc)));
  const std::int32_t* d_drows = reinterpret_cast<const std::int32_t*>(put(drows.data(), drows.size() * 4));
  const TileDesc* d_tiles = reinterpret_cast<const TileDesc*>(put(items.data(), items.size() * sizeof(TileDesc)));
  const CombineDesc* d_combines =
      reinterpret_cast<const CombineDesc*>(put(combines.data(), combines.size() * sizeof(CombineDesc)));
  const std::int32_t* d_samples = reinterpret_cast<const std::int32_t*>(put(samples.data(), samples.size() * 4));
  const std::int32_t* d_frees0 = reinterpret_cast<const std::int32_t*>(put(frees0.data(), frees0.size() * 4));
  const std::int32_t* d_allocs0 = reinterpret_cast<const std::int32_t*>(put(allocs0.data(), allocs0.size() * 4));
  launch_copy_from_host(d, plan_host_dev_[k], off, main_);
  ++kernel_launches_;
  IB2_CUDA(cudaEventRecord(plan_done_[k], main_));
  h2d_bytes_ += static_cast<std::int64_t>(off);

  // ---- pre-phase: scatters this plan depends on, block table, swap-in H2D -----
  flush_swap_ins_for(p);
  launch_block_update(table_, stack_, top_, err_, d_frees0, static_cast<int>(frees0.size()), d_allocs0,
                      static_cast<int>(allocs0.size()), main_);
  run_swaps(sw_in, sw_in_req, true);

  // ---- forward ------------------------------------------------------------------
  (void)D;
  if (trace_iters_) iter_mark(1);
  if (n_rows > 0) {
    rows_dev_ = d_rows;
    drows_dev_ = d_drows;
    tiles_dev_ = d_tiles;
    combines_dev_ = d_combines;
    n_combines_ = static_cast<int>(combines.size());
    samples_dev_ = d_samples;
    std::int64_t k1_bytes = 0;
    for (int r : drows) k1_bytes += static_cast<std::int64_t>(rows[r].pos + 1) * 2 * spec_.d_model * 2;
    k1_bytes_iter_ = static_cast<double>(k1_bytes);
    {
      const double Dd = spec_.d_model, L = spec_.layers;
      const double w_layer = Dd * (3.0 * Dd + Dd + spec_.ffn_in_width() + spec_.ffn);
      const double lm = samples.empty() ? 0.0 : Dd * spec_.vocab;
      double kv_keys = 0.0, attn = 0.0;  // keys read per layer; attention FLOPs per layer / (4 D)
      for (int r : drows) {
        kv_keys += rows[r].pos + 1;
        attn += rows[r].pos + 1;
      }
      for (int i = 0; i < p.n_spans; ++i) {
        const isim_row_span& sp = p.spans[i];
        if (sp.count == 1 || force_row_attention_) continue;
        kv_keys += sp.pos + sp.count;
        attn += static_cast<double>(sp.count) * (sp.pos + (sp.count + 1) / 2.0);
      }
      const double bytes = 2.0 * (L * w_layer + lm) + L * 2.0 * Dd * 2.0 * (kv_keys + n_rows);
      const double flops = 2.0 * n_rows * L * w_layer + 2.0 * samples.size() * lm + L * 4.0 * Dd * attn;
      roof_bytes_ += bytes;
      roof_flops_ += flops;
      roof_s_ += std::max(bytes / (roof_gbs_ * 1e9), flops / (roof_tflops_ * 1e12));
    }
    max_pos1_ = 0;
    for (int r : drows) max_pos1_ = std::max(max_pos1_, rows[r].pos + 1);
    if (!samples.empty() && !record_) sync_event(tok_done_[k], 1);  // tok_host_[k] free again
    tok_out_host_ = record_ ? nullptr : tok_host_dev_[k];
    forward(n_rows, static_cast<int>(drows.size()), static_cast<int>(items.size()), static_cast<int>(samples.size()));
    if (!samples.empty() && !record_) {
      // The argmax kernel stored the ids into tok_host_[k] (mapped) directly.
      IB2_CUDA(cudaEventRecord(tok_done_[k], main_));
      d2h_bytes_ += static_cast<std::int64_t>(samples.size()) * 4;
    }
  }

  if (trace_iters_) iter_mark(2);
  // ---- post-phase: swap-out gather + D2H, then frees -----------------------------
  std::vector<SwapDesc> dummy_in;
  apply_ops(p, 1, frees1, allocs1, dummy_in, sw_out, released1);
  if (!allocs1.empty()) throw DeviceError("executor: allocation in post phase");
  std::vector<std::int64_t> sw_out_req;
  for (int i = 0; i < p.n_ops; ++i)
    if (p.ops[i].phase == 1 && p.ops[i].kind == ISIM_KV_SWAP_OUT) sw_out_req.push_back(p.ops[i].request_id);
  run_swaps(sw_out, sw_out_req, false);
  if (!frees1.empty()) {
    const int k2 = ring_;
    ring_ = (ring_ + 1) % kRing;
    sync_event(plan_done_[k2], 0);
    std::memcpy(plan_host_[k2], frees1.data(), frees1.size() * 4);
    launch_copy_from_host(plan_dev_[k2], plan_host_dev_[k2], frees1.size() * 4, main_);
    ++kernel_launches_;
    h2d_bytes_ += static_cast<std::int64_t>(frees1.size()) * 4;
    IB2_CUDA(cudaEventRecord(plan_done_[k2], main_));
    launch_block_update(table_, stack_, top_, err_, reinterpret_cast<const std::int32_t*>(plan_dev_[k2]),
                        static_cast<int>(frees1.size()), nullptr, 0, main_);
  }
  for (std::int64_t rid : released0) (void)rid;
  for (std::int64_t rid : released1) {
    auto it = slot_of_.find(rid);
    if (it != slot_of_.end()) {
      free_slots_.push_back(it->second);
      slot_of_.erase(it);
    }
    auto ex = extents_.find(rid);
    if (ex != extents_.end()) {
      for (const Extent& x : ex->second) release_extent_memory(x.off, x.bytes);
      extents_.erase(ex);
    }
  }

  if (step_clock_) IB2_CUDA(cudaEventRecord(clk_pending_.back().second, main_));

  // ---- stats / record ------------------------------------------------------------
  // (measured clocks send one iteration as two plans: forward, then post-phase ops)
  if (p.iteration != last_iteration_) iters_ += 1;
  last_iteration_ = p.iteration;
  rows_total_ += n_rows;
  decode_rows_total_ += static_cast<std::int64_t>(drows.size());
  chunk_rows_total_ += n_rows - static_cast<std::int64_t>(drows.size());
  samples_total_ += static_cast<std::int64_t>(samples.size());
  std::int64_t it_in = 0, it_out = 0;
  for (const auto& s : sw_in) it_in += s.n;
  for (const auto& s : sw_out) it_out += s.n;
  swap_in_tok_ += it_in;
  swap_out_tok_ += it_out;
  if (trace_iters_)
    iter_info_.push_back({n_rows, static_cast<std::int64_t>(drows.size()), n_rows - static_cast<std::int64_t>(drows.size()),
                          it_in, it_out});
  if (record_) {
    flush_swap_ins();
    IB2_CUDA(cudaStreamSynchronize(copy_));
    IB2_CUDA(cudaStreamSynchronize(copy_in_));
    IB2_CUDA(cudaStreamSynchronize(main_));
    check_error();
    if (step_clock_ && p.n_spans == 0) return;  // post-phase half: keep the forward's outputs
    last_tok_.assign(p.n_spans, -1);
    std::vector<std::int32_t> toks(samples.size());
    if (!samples.empty())
      IB2_CUDA(cudaMemcpy(toks.data(), out_tok_, samples.size() * 4, cudaMemcpyDeviceToHost));
    int si = 0;
    for (int i = 0; i < p.n_spans; ++i)
      if (p.spans[i].sample) last_tok_[i] = toks[si++];
    last_logits_.resize(samples.size() * static_cast<std::size_t>(spec_.vocab));
    if (!samples.empty())
      IB2_CUDA(cudaMemcpy(last_logits_.data(), logits_, last_logits_.size() * 4, cudaMemcpyDeviceToHost));
  }
}

void Impl::forward(int n, int n_drows, int n_tiles, int n_samples) {
  const ModelSpec& m = spec_;
  const int D = m.d_model, F = m.ffn;
  const KvGeom g = geom();
  const bool rms = m.family == Family::Llama;
  // Micro-batches (split_batch_): the decode rows [0, n_drows) and the chunk
  // rows [n_drows, n) are independent (different requests), so each runs its
  // own layer chain on its own stream -- the decode chain (weight-streaming
  // GEMMs + K1: HBM bound) on aux_, the chunk chain (tensor-core GEMMs + K2)
  // on main_ -- and the GPU overlaps HBM-bound with tensor-bound work.  The
  // weights are read once per chain.
  const bool split = split_batch_ && n_drows > 0 && n_drows < n && !force_row_attention_;
  auto gemm_on = [&](cudaStream_t st, int off, const f16* a, std::int64_t w, int N, int K, Epi epi, std::int64_t bias,
                     f16* out, int ldo, float* outf, int ldf, int M, const float* addf) {
    GemmArgs ga{a, weights_ + w, M, N, K, epi, W(bias), out, ldo, outf, ldf};
    ga.addf = addf;
    ga.a_rows = max_rows_ - off;  // TMA bounds of an A operand that starts at row `off`
    ga.streamk_ok = st == main_ ? 1 : 0;
    launch_gemm(ga, st);
    ++kernel_launches_;
  };
  const bool overlap = !split && overlap_mlp_ && m.parallel_residual();
  // Interleaved (GPT-J) or no rotary: RoPE pairs are adjacent columns, so the
  // QKV GEMM epilogue can apply it and write K/V into the pool itself.
  // Opt-in (IB2_FUSED_QKV=1): measured 2.5 % slower end to end than the
  // separate K4 pass on C1 -- the epilogue's dependent row/table loads sit on
  // the QKV GEMM's critical path (one tile per CTA), costing more than K4.
  const bool fused_qkv = !split && fused_qkv_ && (m.rotary_dim == 0 || m.family == Family::GptJ) && D % 64 == 0;
  launch_embed(rows_dev_, n, hist_, hist_stride_, W(wl_.tok_emb), W(wl_.pos_emb), D, m.token_seed, m.vocab, x_, main_);
  ++kernel_launches_;
  if (split) {
    IB2_CUDA(cudaEventRecord(ev_fork_, main_));
    IB2_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
  }
  const int timed_layer = m.layers / 2;
  // One layer over rows [off, off + cnt) on stream st.  attn: 1 = K1 only
  // (decode chain), 2 = K2 only (chunk chain), 3 = both (unsplit batch).
  auto layer_rows = [&](cudaStream_t st, int off, int cnt, int attn, int l) {
    const LayerWeights& lw = wl_.layer[l];
    float* x = x_ + static_cast<std::int64_t>(off) * D;
    f16* xn = xn_ + static_cast<std::int64_t>(off) * D;
    f16* qkv = qkv_ + static_cast<std::int64_t>(off) * 3 * D;
    f16* at = attn_ + static_cast<std::int64_t>(off) * D;
    f16* hid = hid_ + static_cast<std::int64_t>(off) * F;
    const bool dec = (attn & 1) && n_drows > 0;
    launch_norm(x, D, nullptr, cnt, D, W(lw.ln1_g), W(lw.ln1_b), rms, m.norm_eps, xn, D, st);
    ++kernel_launches_;
    // The layer whose K1 is timed for the roofline keeps its MLP branch inline,
    // so K1's events measure it without concurrent kernels of this chain.
    const bool overlap_l = overlap && !(timing_ && l == timed_layer && dec);
    if (overlap_l) {  // MLP branch on aux_: fc_in(ln1(x)) -> GELU -> fc_out -> mlp_ (fp32, + bias)
      IB2_CUDA(cudaEventRecord(ev_ln_[l], st));
      IB2_CUDA(cudaStreamWaitEvent(aux_, ev_ln_[l], 0));
      gemm_on(aux_, off, xn, lw.w_in, F, D, Epi::GeluF16, lw.b_in, hid, F, nullptr, 0, cnt, nullptr);
      gemm_on(aux_, off, hid, lw.w_out, D, F, Epi::StoreF32, lw.b_out, nullptr, 0, mlp_, D, cnt, nullptr);
      IB2_CUDA(cudaEventRecord(ev_mlp_[l], aux_));
    }
    if (fused_qkv) {
      // K4 fused into the QKV epilogue: q (RoPE) -> qkv_, k (RoPE) / v -> pool.
      GemmArgs ga{xn, weights_ + lw.w_qkv, cnt, 3 * D, D, Epi::QkvRopeKv, W(lw.b_qkv), qkv, 3 * D, nullptr, 0,
                  QkvWrite{rows_dev_, g.pool, l * g.layer_stride(), g.block_stride(), g.table, g.max_lblocks,
                           m.heads, m.head_dim(), m.rotary_dim, rope_cs_}};
      launch_gemm(ga, st);
      ++kernel_launches_;
    } else {
      gemm_on(st, off, xn, lw.w_qkv, 3 * D, D, Epi::StoreF16, lw.b_qkv, qkv, 3 * D, nullptr, 0, cnt, nullptr);
      launch_rope_kv_write(qkv, rows_dev_ + off, cnt, g, l, m.rotary_dim, m.family == Family::GptJ, rope_cs_, st);
      kernel_launches_ += 2;
    }
    if (attn & 1) {
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      const bool time_k1 = timing_ && l == timed_layer && n_drows > 0;
      if (time_k1) {
        if (ev_free_.empty()) {
          cudaEvent_t a, b;
          IB2_CUDA(cudaEventCreate(&a));
          IB2_CUDA(cudaEventCreate(&b));
          ev_free_.push_back({a, b});
        }
        e0 = ev_free_.back().first;
        e1 = ev_free_.back().second;
        ev_free_.pop_back();
        IB2_CUDA(cudaEventRecord(e0, st));
      }
      launch_decode_attention(qkv_, drows_dev_, rows_dev_, n_drows, g, l, max_pos1_, part_o_, part_ml_, attn_,
                              k1_counters_, st);
      if (n_drows) ++kernel_launches_;
      if (time_k1) {
        IB2_CUDA(cudaEventRecord(e1, st));
        ev_pending_.push_back({e0, e1});
        ev_bytes_.push_back(k1_bytes_iter_ + static_cast<double>(n_drows) * 2.0 * D * 2);
      }
    }
    if (attn & 2) {
      launch_chunk_attention(qkv_, max_rows_, tiles_dev_, n_tiles, combines_dev_, n_combines_, g, l, attn_,
                             chunk_ws_o_, chunk_ws_ml_, st);
      if (n_tiles) kernel_launches_ += n_combines_ > 0 ? 2 : 1;
    }
    if (overlap_l) {
      // x = (x + attn W_o) + mlp: the MLP branch ran on aux_.
      IB2_CUDA(cudaStreamWaitEvent(st, ev_mlp_[l], 0));
      gemm_on(st, off, at, lw.w_o, D, D, Epi::ResidAdd, lw.b_o, nullptr, 0, x, D, cnt, mlp_);
    } else if (m.parallel_residual()) {
      // GPT-J: x += attn W_o + mlp(ln1(x)); both read the same xn.
      gemm_on(st, off, at, lw.w_o, D, D, Epi::ResidAdd, lw.b_o, nullptr, 0, x, D, cnt, nullptr);
      gemm_on(st, off, xn, lw.w_in, F, D, Epi::GeluF16, lw.b_in, hid, F, nullptr, 0, cnt, nullptr);
      gemm_on(st, off, hid, lw.w_out, D, F, Epi::ResidAdd, lw.b_out, nullptr, 0, x, D, cnt, nullptr);
    } else {
      gemm_on(st, off, at, lw.w_o, D, D, Epi::ResidAdd, lw.b_o, nullptr, 0, x, D, cnt, nullptr);
      launch_norm(x, D, nullptr, cnt, D, W(lw.ln2_g), W(lw.ln2_b), rms, m.norm_eps, xn, D, st);
      ++kernel_launches_;
      if (m.family == Family::Llama)
        gemm_on(st, off, xn, lw.w_in, 2 * F, D, Epi::SwiGluF16, -1, hid, F, nullptr, 0, cnt, nullptr);
      else
        gemm_on(st, off, xn, lw.w_in, F, D, Epi::GeluF16, lw.b_in, hid, F, nullptr, 0, cnt, nullptr);
      gemm_on(st, off, hid, lw.w_out, D, F, Epi::ResidAdd, lw.b_out, nullptr, 0, x, D, cnt, nullptr);
    }
  };
  for (int l = 0; l < m.layers; ++l) {
    if (split) {
      layer_rows(aux_, 0, n_drows, 1, l);
      layer_rows(main_, n_drows, n - n_drows, 2, l);
    } else {
      layer_rows(main_, 0, n, 3, l);
    }
  }
  if (split) {
    IB2_CUDA(cudaEventRecord(ev_join_, aux_));
    IB2_CUDA(cudaStreamWaitEvent(main_, ev_join_, 0));
  }
  if (n_samples > 0) {
    launch_norm(x_, D, samples_dev_, n_samples, D, W(wl_.lnf_g), W(wl_.lnf_b), rms, m.norm_eps, lmrows_, D, main_);
    gemm_on(main_, 0, lmrows_, wl_.lm_w, m.vocab, D, Epi::StoreF32, wl_.lm_b, nullptr, 0, logits_, m.vocab,
            n_samples, nullptr);
    launch_argmax(logits_, n_samples, m.vocab, samples_dev_, rows_dev_, hist_, hist_stride_, out_tok_, tok_out_host_,
                  main_);
    kernel_launches_ += 2;
  }
}

void Impl::check_error() {
  std::int32_t e = 0;
  IB2_CUDA(cudaMemcpy(&e, err_, 4, cudaMemcpyDeviceToHost));
  if (e) throw DeviceError("executor: block-table update error " + std::to_string(e));
}

void Impl::sync() {
  IB2_CUDA(cudaSetDevice(dev_));
  flush_swap_ins();
  IB2_CUDA(cudaStreamSynchronize(main_));
  IB2_CUDA(cudaStreamSynchronize(copy_));
  IB2_CUDA(cudaStreamSynchronize(copy_in_));
  check_error();
  retire_host_memory(true);  // every copy reading a released extent has completed
  for (std::size_t i = 0; i < ev_pending_.size(); ++i) {
    float ms = 0.f;
    IB2_CUDA(cudaEventElapsedTime(&ms, ev_pending_[i].first, ev_pending_[i].second));
    k1_ms_ += ms;
    k1_bytes_timed_ += ev_bytes_[i];
    ++k1_launches_timed_;
    ev_free_.push_back(ev_pending_[i]);
  }
  ev_pending_.clear();
  ev_bytes_.clear();
  for (const SwapTrace& t : swap_trace_pending_) {
    float a = 0.f, b = 0.f;
    IB2_CUDA(cudaEventElapsedTime(&a, trace_ref_, t.t0));
    IB2_CUDA(cudaEventElapsedTime(&b, trace_ref_, t.t1));
    swap_trace_.push_back({static_cast<double>(t.iter), static_cast<double>(t.dir), a, b, t.bytes});
  }
  swap_trace_pending_.clear();
  for (std::size_t i = 0; i < swap_ev_pending_.size(); ++i) {
    float ms = 0.f;
    IB2_CUDA(cudaEventElapsedTime(&ms, swap_ev_pending_[i].first, swap_ev_pending_[i].second));
    swap_ms_ += ms;
    swap_bytes_timed_ += swap_ev_bytes_[i];
    ev_free_.push_back(swap_ev_pending_[i]);
  }
  swap_ev_pending_.clear();
  swap_ev_bytes_.clear();
  if (trace_iters_ && iter_ev_.size() > 1) {
    for (std::size_t i = 0; i + 1 < iter_ev_.size(); ++i) {
      float pre = 0.f, fwd = 0.f, post = 0.f;
      IB2_CUDA(cudaEventElapsedTime(&pre, iter_ev_[i][0], iter_ev_[i][1]));
      IB2_CUDA(cudaEventElapsedTime(&fwd, iter_ev_[i][1], iter_ev_[i][2]));
      IB2_CUDA(cudaEventElapsedTime(&post, iter_ev_[i][2], iter_ev_[i + 1][0]));
      iter_ms_.push_back({pre, fwd, post});
      const std::size_t gi = iter_ms_.size() - 1;  // global iteration index
      double lead = -1e9;
      if (trace_ref_ && gi < iter_host_ms_.size() && iter_host_ms_[gi] >= 0) {
        float g = 0.f;
        if (cudaEventElapsedTime(&g, trace_ref_, iter_ev_[i][0]) == cudaSuccess) lead = g - iter_host_ms_[gi];
        else (void)cudaGetLastError();
      }
      iter_lead_ms_.push_back(lead);
      for (cudaEvent_t e : iter_ev_[i]) cudaEventDestroy(e);
    }
    iter_ev_.erase(iter_ev_.begin(), iter_ev_.end() - 1);
  }
  if (trace_iters_) {  // new reference point: GPU idle now
    if (!trace_ref_) IB2_CUDA(cudaEventCreate(&trace_ref_));
    IB2_CUDA(cudaEventRecord(trace_ref_, main_));
    IB2_CUDA(cudaEventSynchronize(trace_ref_));
    trace_ref_host_ = std::chrono::steady_clock::now();
  }
}

cudaEvent_t Impl::new_timing_event() {
  // Events come in pairs from the shared free list; split a pair if needed.
  static thread_local std::vector<cudaEvent_t> spare;
  if (spare.empty()) {
    if (ev_free_.empty()) {
      cudaEvent_t a, b;
      IB2_CUDA(cudaEventCreate(&a));
      IB2_CUDA(cudaEventCreate(&b));
      ev_free_.push_back({a, b});
    }
    spare.push_back(ev_free_.back().first);
    spare.push_back(ev_free_.back().second);
    ev_free_.pop_back();
  }
  cudaEvent_t e = spare.back();
  spare.pop_back();
  return e;
}

double Impl::take_step_seconds() {
  IB2_CUDA(cudaSetDevice(dev_));
  if (clk_pending_.empty()) return 0.0;
  IB2_CUDA(cudaEventSynchronize(clk_pending_.back().second));
  double ms = 0.0;
  for (const auto& [a, b] : clk_pending_) {
    float t = 0.f;
    IB2_CUDA(cudaEventElapsedTime(&t, a, b));
    ms += t;
    ev_free_.push_back({a, b});
  }
  clk_pending_.clear();
  return ms * 1e-3;
}

double Impl::timer(int op) {
  IB2_CUDA(cudaSetDevice(dev_));
  if (op == 0 || op == 1) {
    IB2_CUDA(cudaEventRecord(mark_[op], main_));
    return 0.0;
  }
  IB2_CUDA(cudaEventSynchronize(mark_[1]));
  float ms = 0.f;
  IB2_CUDA(cudaEventElapsedTime(&ms, mark_[0], mark_[1]));
  return ms;
}

std::string Impl::stats_json() const {
  nlohmann::json j;
  j["model"] = nlohmann::json::parse(model_json(spec_));
  j["iterations"] = iters_;
  j["rows"] = rows_total_;
  j["decode_rows"] = decode_rows_total_;
  j["chunk_rows"] = chunk_rows_total_;
  j["samples"] = samples_total_;
  j["swap_in_tokens"] = swap_in_tok_;
  j["swap_out_tokens"] = swap_out_tok_;
  j["swap_in_forwarded_tokens"] = swap_in_forwarded_tok_;
  j["swap_bytes"] = static_cast<double>(swap_in_tok_ + swap_out_tok_) * static_cast<double>(spec_.kv_bytes_per_token());
  j["gpu_blocks"] = gpu_blocks_;
  j["host_pool_bytes"] = host_bytes_;
  j["host_pool_used"] = arena_.used();
  j["host_pool_peak"] = arena_.peak();
  j["kernel_launches"] = kernel_launches_;
  j["k1_timed_launches"] = k1_launches_timed_;
  j["k1_ms"] = k1_ms_;
  j["k1_bytes"] = k1_bytes_timed_;
  j["roof_bytes"] = roof_bytes_;
  j["roof_flops"] = roof_flops_;
  j["roof_s"] = roof_s_;
  j["gemm"] = gemm_uses_tcgen05() ? "tcgen05" : "simt";
  j["h2d_bytes"] = h2d_bytes_;
  j["d2h_bytes"] = d2h_bytes_;
  j["swap_ms"] = swap_ms_;
  j["swap_bytes_timed"] = swap_bytes_timed_;
  j["kv_bytes_per_token"] = spec_.kv_bytes_per_token();
  j["host_consume_s"] = host_consume_s_;
  j["host_block_s"] = {host_block_s_[0], host_block_s_[1], host_block_s_[2], host_block_s_[3]};
  if (trace_iters_) {
    j["iter_lead_ms"] = iter_lead_ms_;
    j["iter_host_ms"] = iter_host_ms_;
    j["swap_trace"] = swap_trace_;
    j["iter_ms"] = iter_ms_;
    j["iter_info"] = iter_info_;
  }
  return j.dump();
}

std::int32_t Impl::last_tokens(std::int32_t* out, std::int32_t cap) const {
  const auto n = static_cast<std::int32_t>(last_tok_.size());
  if (out) std::memcpy(out, last_tok_.data(), std::min(n, cap) * 4);
  return n;
}

std::int64_t Impl::last_logits(float* out, std::int64_t cap) const {
  const auto n = static_cast<std::int64_t>(last_logits_.size());
  if (out) std::memcpy(out, last_logits_.data(), std::min(n, cap) * 4);
  return n;
}

std::int32_t Impl::block_table(std::int64_t rid, std::int32_t* out, std::int32_t cap) const {
  auto it = slot_of_.find(rid);
  if (it == slot_of_.end()) return 0;
  IB2_CUDA(cudaStreamSynchronize(main_));
  std::vector<std::int32_t> t(max_lb_);
  IB2_CUDA(cudaMemcpy(t.data(), table_ + static_cast<std::int64_t>(it->second) * max_lb_, max_lb_ * 4,
                      cudaMemcpyDeviceToHost));
  if (out) std::memcpy(out, t.data(), std::min(max_lb_, cap) * 4);
  return max_lb_;
}

std::int64_t Impl::free_blocks() const {
  IB2_CUDA(cudaStreamSynchronize(main_));
  std::int32_t t = 0;
  IB2_CUDA(cudaMemcpy(&t, top_, 4, cudaMemcpyDeviceToHost));
  return t;
}

void Impl::read_history(std::int64_t rid, std::int64_t lo, std::int64_t hi, std::int32_t* out,
                        std::int64_t cap) const {
  auto it = slot_of_.find(rid);
  if (it == slot_of_.end()) throw DeviceError("read_history: unknown request");
  if (lo < 0 || hi < lo || hi > hist_stride_) throw DeviceError("read_history: positions out of range");
  if (cap < hi - lo) throw DeviceError("read_history: buffer too small");
  IB2_CUDA(cudaStreamSynchronize(main_));
  if (hi > lo)
    IB2_CUDA(cudaMemcpy(out, hist_ + static_cast<std::int64_t>(it->second) * hist_stride_ + lo, (hi - lo) * 4,
                        cudaMemcpyDeviceToHost));
}

void Impl::read_kv(std::int64_t rid, std::int64_t lo, std::int64_t hi, void* out, std::int64_t cap) const {
  // Bytes of positions [lo,hi) wherever they live: a pinned host extent
  // (swapped out) or the paged GPU pool.  Layout [L][pos][2][H][hd].
  auto it = slot_of_.find(rid);
  if (it == slot_of_.end()) throw DeviceError("read_kv: unknown request");
  const std::int64_t D = spec_.d_model, L = spec_.layers, H = spec_.heads, hd = spec_.head_dim();
  const std::int64_t n = hi - lo;
  if (cap < n * L * 2 * D * 2) throw DeviceError("read_kv: buffer too small");
  IB2_CUDA(cudaStreamSynchronize(copy_));
  IB2_CUDA(cudaStreamSynchronize(copy_in_));
  IB2_CUDA(cudaStreamSynchronize(main_));
  std::vector<std::int32_t> t(max_lb_);
  IB2_CUDA(cudaMemcpy(t.data(), table_ + static_cast<std::int64_t>(it->second) * max_lb_, max_lb_ * 4,
                      cudaMemcpyDeviceToHost));
  f16* dst = static_cast<f16*>(out);
  const KvGeom g = geom();
  const std::size_t row = static_cast<std::size_t>(2 * D) * 2;
  const auto ex = extents_.find(rid);
  // One D2H per (layer, block) of the GPU-resident positions.
  std::vector<f16> blk(static_cast<std::size_t>(2 * H * kBlockTokens * hd));
  std::int64_t cached_l = -1, cached_pb = -1;
  for (std::int64_t l = 0; l < L; ++l) {
    for (std::int64_t p = lo; p < hi; ++p) {
      const Extent* on_host = nullptr;
      if (ex != extents_.end())
        for (const Extent& x : ex->second)
          if (x.lo <= p && p < x.hi) on_host = &x;
      f16* d = dst + (l * n + (p - lo)) * 2 * D;
      if (on_host) {
        const std::int64_t n0 = on_host->hi0 - on_host->lo0;
        std::memcpy(d, host_pool_ + on_host->off + (static_cast<std::size_t>(l * n0 + (p - on_host->lo0))) * row, row);
        continue;
      }
      const std::int32_t pb = t[p / kBlockTokens];
      if (pb < 0) throw DeviceError("read_kv: position neither on the GPU nor on the host");
      if (l != cached_l || pb != cached_pb) {
        IB2_CUDA(cudaMemcpy(blk.data(), pool_ + l * g.layer_stride() + static_cast<std::int64_t>(pb) * g.block_stride(),
                            blk.size() * sizeof(f16), cudaMemcpyDeviceToHost));
        cached_l = l;
        cached_pb = pb;
      }
      for (int kv = 0; kv < 2; ++kv)
        for (std::int64_t h = 0; h < H; ++h)
          std::memcpy(d + kv * D + h * hd, blk.data() + ((kv * H + h) * kBlockTokens + p % kBlockTokens) * hd, hd * 2);
    }
  }
}

}  // namespace

std::unique_ptr<B200Executor> B200Executor::create(const std::string& model_json, int device,
                                                   const std::string& pools_json) {
  return std::make_unique<Impl>(model_json, device, pools_json);
}

}  // namespace ib2
