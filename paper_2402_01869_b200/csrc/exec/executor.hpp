// B200 executor: runs one scheduler BatchPlan per call on one GPU.
//
// Owns the model weights, the paged KV pool (GPU-resident block tables with a
// device free list), the pinned host swap pool, the token history and the
// CUDA streams.  Plans are enqueued asynchronously: the scheduler never waits
// on the GPU because interceptions fire on decode counts, not token values
// (reference engine.cpp:466-481), so sampled ids stay on the device.
#pragma once

#include <cstdint>
#include <memory>
#include <string>

#include "../sched/scheduler.hpp"

namespace ib2 {

class B200Executor : public PlanSink {
 public:
  static std::unique_ptr<B200Executor> create(const std::string& model_json, int device,
                                              const std::string& pools_json);
  ~B200Executor() override = default;

  void consume(const isim_batch_plan& plan) override = 0;
  virtual void sync() = 0;
  virtual std::string stats_json() const = 0;
  virtual std::int32_t last_tokens(std::int32_t* out, std::int32_t cap) const = 0;
  virtual std::int64_t last_logits(float* out, std::int64_t cap) const = 0;
  virtual std::int32_t block_table(std::int64_t request_id, std::int32_t* out, std::int32_t cap) const = 0;
  virtual std::int64_t free_blocks() const = 0;
  // op 0 / 1: record the start / stop mark on the compute stream;
  // op 2: wait for the stop mark and return the elapsed device milliseconds.
  virtual double timer(int op) = 0;
  virtual void read_kv(std::int64_t request_id, std::int64_t lo, std::int64_t hi, void* out,
                       std::int64_t cap) const = 0;
  // Token ids of positions [lo,hi) of a request's device history (synthetic
  // prompt / API-returned ids and sampled ids, as the embed kernel reads them).
  virtual void read_history(std::int64_t request_id, std::int64_t lo, std::int64_t hi, std::int32_t* out,
                            std::int64_t cap) const = 0;
};

// Kernel test hook behind isim_debug_gemm (exec/k_gemm_tc.cu).
void debug_gemm(const void* a, const void* w, int M, int N, int K, int epi, const void* bias, void* out, int ldo,
                void* outf, int ldf, int flags, void* stream);
void debug_tile_weights(const void* src, void* dst, int N, int K, void* stream);

}  // namespace ib2
