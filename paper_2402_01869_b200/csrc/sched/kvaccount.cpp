#include "kvaccount.hpp"

#include <json.hpp>

namespace ib2 {

namespace {
const KvCounts kNone{};
}

const KvCounts& KvAccount::counts(std::int64_t id) const {
  auto it = map_.find(id);
  return it == map_.end() ? kNone : it->second;
}

KvStatus KvAccount::grow(std::int64_t id, std::int64_t n) {
  if (n < 0) return KvStatus::BadArgument;
  if (n == 0) return KvStatus::Ok;
  const double d = grow_delta(counts(id).gpu, n);
  if (!gpu_fits(d)) return KvStatus::NoGpuRoom;
  map_[id].gpu += n;
  gpu_used_ += d;
  return KvStatus::Ok;
}

KvStatus KvAccount::to_cpu(std::int64_t id, std::int64_t n) {
  auto it = map_.find(id);
  if (n < 0 || it == map_.end() || n > it->second.gpu) return KvStatus::BadArgument;
  if (n == 0) return KvStatus::Ok;
  KvCounts& c = it->second;
  const double dc = grow_delta(c.cpu, n);
  if (cpu_used_ + dc > m_->cpu_kv_capacity + 0.5) return KvStatus::NoCpuRoom;
  const double dg = shrink_delta(c.gpu, n);
  c.gpu -= n;
  c.cpu += n;
  gpu_used_ -= dg;
  cpu_used_ += dc;
  return KvStatus::Ok;
}

KvStatus KvAccount::to_gpu(std::int64_t id, std::int64_t n) {
  auto it = map_.find(id);
  if (n < 0 || it == map_.end() || n > it->second.cpu) return KvStatus::BadArgument;
  if (n == 0) return KvStatus::Ok;
  KvCounts& c = it->second;
  const double dg = grow_delta(c.gpu, n);
  if (!gpu_fits(dg)) return KvStatus::NoGpuRoom;
  const double dc = shrink_delta(c.cpu, n);
  c.cpu -= n;
  c.gpu += n;
  cpu_used_ -= dc;
  gpu_used_ += dg;
  return KvStatus::Ok;
}

KvStatus KvAccount::drop(std::int64_t id, std::int64_t n) {
  auto it = map_.find(id);
  if (n < 0 || it == map_.end() || n > it->second.gpu) return KvStatus::BadArgument;
  if (n == 0) return KvStatus::Ok;
  KvCounts& c = it->second;
  const double dg = shrink_delta(c.gpu, n);
  c.gpu -= n;
  c.discarded += n;
  gpu_used_ -= dg;
  return KvStatus::Ok;
}

KvStatus KvAccount::recompute(std::int64_t id, std::int64_t n) {
  auto it = map_.find(id);
  if (n < 0 || it == map_.end() || n > it->second.discarded) return KvStatus::BadArgument;
  if (n == 0) return KvStatus::Ok;
  KvCounts& c = it->second;
  const double dg = grow_delta(c.gpu, n);
  if (!gpu_fits(dg)) return KvStatus::NoGpuRoom;
  c.discarded -= n;
  c.gpu += n;
  gpu_used_ += dg;
  return KvStatus::Ok;
}

void KvAccount::forget(std::int64_t id) {
  auto it = map_.find(id);
  if (it == map_.end()) return;
  gpu_used_ -= m_->bytes_for(it->second.gpu);
  cpu_used_ -= m_->bytes_for(it->second.cpu);
  map_.erase(it);
}

bool KvAccount::room_for(std::int64_t n, std::int64_t id) const {
  const double d = grow_delta(counts(id).gpu, n);
  return gpu_used_ + d <= m_->gpu_kv_capacity + 0.5;
}

std::string KvAccount::snapshot() const {
  nlohmann::json j;
  j["gpu_used"] = gpu_used_;
  j["cpu_used"] = cpu_used_;
  j["gpu_capacity"] = m_->gpu_kv_capacity;
  j["cpu_capacity"] = m_->cpu_kv_capacity;
  nlohmann::json reqs = nlohmann::json::object();
  for (const auto& [id, c] : map_)
    reqs[std::to_string(id)] = {{"gpu", c.gpu}, {"cpu", c.cpu}, {"discarded", c.discarded}};
  j["requests"] = std::move(reqs);
  return j.dump();
}

}  // namespace ib2
