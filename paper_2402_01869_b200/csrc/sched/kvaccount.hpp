// Host-side KV accounting: per-request token counts by location (GPU KV
// cache / CPU swap space / discarded) plus block-rounded byte totals used for
// capacity decisions.  This is the scheduler's view; the device mirrors it with
// physical block tables (executor K8) whose occupancy equals these counts.
// Arithmetic follows proj/src/memory.cpp:13-88 operation for operation (the
// byte totals are doubles with a 0.5 B slack) so decisions stay bit-exact.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>

#include "costmodel.hpp"

namespace ib2 {

enum class KvStatus { Ok, NoGpuRoom, NoCpuRoom, BadArgument };

struct KvCounts {
  std::int64_t gpu = 0, cpu = 0, discarded = 0;
  std::int64_t total() const { return gpu + cpu + discarded; }
};

class KvAccount {
 public:
  explicit KvAccount(const CostModel& m) : m_(&m) {}

  KvStatus grow(std::int64_t id, std::int64_t n);           // fresh tokens computed on GPU
  KvStatus to_cpu(std::int64_t id, std::int64_t n);         // swap-out
  KvStatus to_gpu(std::int64_t id, std::int64_t n);         // swap-in
  KvStatus drop(std::int64_t id, std::int64_t n);           // discard GPU tokens
  KvStatus recompute(std::int64_t id, std::int64_t n);      // restore discarded
  void forget(std::int64_t id);                             // release
  bool room_for(std::int64_t n, std::int64_t id) const;     // fits_gpu

  const KvCounts& counts(std::int64_t id) const;
  bool tracks(std::int64_t id) const { return map_.count(id) != 0; }
  double gpu_bytes() const { return gpu_used_; }
  double cpu_bytes() const { return cpu_used_; }
  std::int64_t gpu_free_tokens() const {
    return static_cast<std::int64_t>((m_->gpu_kv_capacity - gpu_used_) / m_->mem_per_token);
  }
  std::int64_t cpu_free_tokens() const {
    return static_cast<std::int64_t>((m_->cpu_kv_capacity - cpu_used_) / m_->mem_per_token);
  }
  const std::unordered_map<std::int64_t, KvCounts>& all() const { return map_; }
  std::string snapshot() const;

 private:
  double grow_delta(std::int64_t have, std::int64_t n) const { return m_->bytes_for(have + n) - m_->bytes_for(have); }
  double shrink_delta(std::int64_t have, std::int64_t n) const { return m_->bytes_for(have) - m_->bytes_for(have - n); }
  bool gpu_fits(double delta) const { return !(gpu_used_ + delta > m_->gpu_kv_capacity + 0.5); }

  const CostModel* m_;
  std::unordered_map<std::int64_t, KvCounts> map_;
  double gpu_used_ = 0.0;
  double cpu_used_ = 0.0;
};

}  // namespace ib2
