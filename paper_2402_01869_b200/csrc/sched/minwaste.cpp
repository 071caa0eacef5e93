#include "minwaste.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

#include "base.hpp"

namespace ib2 {

Policy Policy::named(PolicyKind k) {
  Policy p;
  p.kind = k;
  if (k == PolicyKind::VanillaDiscard) p.requeue_at_tail = true;
  if (k == PolicyKind::Preserve) p.preserve_mode = PreserveMode::MinWaste;
  if (k == PolicyKind::InferCept) {
    p.chunked_recompute = true;
    p.budgeted_swap = true;
    p.preserve_mode = PreserveMode::MinWaste;
  }
  return p;
}

namespace {
struct NamedPolicy {
  const char* name;
  PolicyKind kind;
};
constexpr NamedPolicy kPolicies[] = {{"vanilla-discard", PolicyKind::VanillaDiscard},
                                     {"improved-discard", PolicyKind::ImprovedDiscard},
                                     {"preserve", PolicyKind::Preserve},
                                     {"swap", PolicyKind::NaiveSwap},
                                     {"infercept", PolicyKind::InferCept}};
}  // namespace

PolicyKind policy_from_name(const std::string& s) {
  for (const auto& p : kPolicies)
    if (s == p.name) return p.kind;
  throw ConfigError("unknown policy: " + s);
}

std::string policy_to_name(PolicyKind k) {
  for (const auto& p : kPolicies)
    if (p.kind == k) return p.name;
  return "?";
}

Estimator estimator_from_name(const std::string& s) {
  if (s == "oracle") return Estimator::Oracle;
  if (s == "profiled") return Estimator::Profiled;
  if (s == "dynamic") return Estimator::Dynamic;
  throw ConfigError("unknown duration estimator: " + s);
}

std::string estimator_to_name(Estimator e) {
  switch (e) {
    case Estimator::Oracle: return "oracle";
    case Estimator::Profiled: return "profiled";
    case Estimator::Dynamic: return "dynamic";
  }
  return "?";
}

// Eq. 2: context held for the whole call.
double waste_preserve(const CostModel& m, double t_int, double ctx) { return t_int * ctx * m.mem_per_token; }

// Eq. 1: one-shot recompute stalls its own and everyone else's context.
double waste_discard_oneshot(const CostModel& m, double ctx, double other) {
  const double t = m.t_fwd(ctx);
  return t * ctx * m.mem_per_token + t * other * m.mem_per_token;
}

// Eq. 3: synchronous out-and-back swap stalls the batch twice.
double waste_swap_naive(const CostModel& m, double ctx, double batch_ctx) {
  return 2.0 * m.t_swap(ctx) * batch_ctx * m.mem_per_token;
}

// Eq. 4: recompute in n = ceil(C/chunk) chunks.
double waste_chunk_discard(const CostModel& m, double ctx, double other, double chunk) {
  if (ctx <= 0.0) return 0.0;
  const double n = std::ceil(ctx / chunk);
  return m.t_fwd(ctx) * ctx * m.mem_per_token / 2.0 + n * m.t_fwd(ctx / n) * other * m.mem_per_token;
}

// Eq. 5: min(preserve, chunked discard); ties preserve.
Waste assess(const CostModel& m, double t_int, double ctx, double other, double chunk) {
  Waste w;
  w.preserve = waste_preserve(m, t_int, ctx);
  w.discard_oneshot = waste_discard_oneshot(m, ctx, other);
  w.swap_naive = waste_swap_naive(m, ctx, other + ctx);
  w.chunk_discard = waste_chunk_discard(m, ctx, other, chunk);
  w.keep = w.preserve <= w.chunk_discard;
  w.key = w.keep ? w.preserve : w.chunk_discard;
  return w;
}

std::int64_t swap_limit_for(const CostModel& m, double batch_tokens) {
  return static_cast<std::int64_t>(std::floor(m.t_fwd(batch_tokens) / m.swap_per_token));
}

// Fixed point favouring swap-in: in <= out + free_gpu, out <= free_cpu + in,
// in + out <= limit.
SwapSplit split_swap_budget(std::int64_t limit, std::int64_t pending_in, std::int64_t pending_out,
                            std::int64_t free_gpu, std::int64_t free_cpu) {
  auto nonneg = [](std::int64_t v) { return std::max<std::int64_t>(0, v); };
  SwapSplit s;
  s.limit = nonneg(limit);
  pending_in = nonneg(pending_in);
  pending_out = nonneg(pending_out);
  free_gpu = nonneg(free_gpu);
  free_cpu = nonneg(free_cpu);
  auto out_cap = [&](std::int64_t in) { return std::min({pending_out, s.limit - in, free_cpu + in}); };
  std::int64_t in = std::min(pending_in, s.limit);
  for (;;) {
    const std::int64_t next = std::min(in, nonneg(out_cap(in)) + free_gpu);
    if (next == in) break;
    in = next;
  }
  s.in = in;
  s.out = nonneg(out_cap(in));
  return s;
}

std::vector<Verdict> plan_paused(const Policy& p, const CostModel& m, const std::vector<Paused>& in, double other_ctx,
                                 double chunk, std::int64_t out_budget, std::int64_t cpu_free) {
  std::vector<Verdict> v(in.size());
  for (std::size_t i = 0; i < in.size(); ++i) {
    Verdict& d = v[i];
    d.id = in[i].id;
    d.w = assess(m, in[i].t_hat, static_cast<double>(in[i].ctx), other_ctx, chunk);
    if (p.preserve_mode == PreserveMode::Never) {
      d.keep_rest = false;
      d.w.key = p.chunked_recompute ? d.w.chunk_discard : d.w.discard_oneshot;
    } else if (p.preserve_mode == PreserveMode::Heuristic) {
      d.keep_rest = in[i].t_hat < p.heuristic_threshold;
      d.w.key = d.keep_rest ? d.w.preserve : d.w.chunk_discard;
    } else {
      d.keep_rest = d.w.keep;
    }
  }
  if (!p.budgeted_swap) return v;
  // Highest waste first; then longer context; then lower id.
  std::vector<std::size_t> rank(in.size());
  std::iota(rank.begin(), rank.end(), std::size_t{0});
  std::sort(rank.begin(), rank.end(), [&](std::size_t a, std::size_t b) {
    if (v[a].w.key != v[b].w.key) return v[a].w.key > v[b].w.key;
    if (in[a].ctx != in[b].ctx) return in[a].ctx > in[b].ctx;
    return in[a].id < in[b].id;
  });
  std::int64_t left = std::min(out_budget, cpu_free);
  for (std::size_t i : rank) {
    if (left <= 0) break;
    v[i].swap_out = std::min(left, in[i].ctx);
    left -= v[i].swap_out;
  }
  return v;
}

}  // namespace ib2
