// Paged attention over the GPU-resident block tables.
//
// K1 (decode rows): flash-decoding.  Grid = (KV split, head, row); each CTA
// scores up to kSplit positions of one (row, head) with 16-byte vector loads
// of the head's contiguous [16][hd] slice of each paged block (lanes of a
// token group own 8 dims each, dot products reduced by warp shuffles), then a
// second pass accumulates P*V; the last split of a (row, head) to finish
// merges the splits.  HBM bound:
// algorithmic bytes = 2 * ctx * hd * 2 per (row, head).
//
// K2 (chunk rows) lives in k_attn_chunk.cu (tcgen05 + TMEM + TMA).
#include <cfloat>
#include <cstdlib>

#include "kernels.hpp"

namespace ib2 {

namespace {

constexpr int kSplit = 256;       // shortest positions per K1 CTA (partial buffers are sized for it)
constexpr int kDecWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void h8_to_f32(const uint4& u, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Occupancy: at head_dim 256 the unconstrained kernel takes 96 registers (5
// CTAs per SM); capping it at 80 (6 CTAs per SM, 28 B of spills) measured
// +2 % K1 bandwidth on the C1 window, a cap of 7 CTAs -4 % (profiles/r1j).
template <int HD, int SPLIT = kSplit>
__global__ void __launch_bounds__(kDecWarps * 32, HD == 256 ? 6 : 1) decode_attn_kernel(
    const f16* __restrict__ qkv, const std::int32_t* __restrict__ drow, const RowDesc* __restrict__ rows,
    const f16* __restrict__ pool, std::int64_t layer_off, std::int64_t block_stride,
    const std::int32_t* __restrict__ table, int max_lb, int H, int max_splits, float* __restrict__ part_o,
    float* __restrict__ part_ml, f16* __restrict__ out, std::int32_t* __restrict__ counters) {
  pdl_trigger();
  pdl_wait();
  constexpr int LPT = HD / 8;   // lanes per token
  constexpr int TPW = 32 / LPT; // tokens per warp step
  const int split = blockIdx.x, h = blockIdx.y, dr = blockIdx.z;
  const int r = drow[dr];
  const RowDesc d = rows[r];
  const int ctx = d.pos + 1;
  const int start = split * SPLIT;
  if (start >= ctx) return;
  const int end = min(ctx, start + SPLIT);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPT, grp = lane / LPT;
  const int D = H * HD;

  __shared__ float s_score[SPLIT];
  __shared__ float s_red[kDecWarps];
  __shared__ float s_acc[kDecWarps][HD];

  float q[8];
  {
    const uint4 u = *reinterpret_cast<const uint4*>(qkv + static_cast<std::int64_t>(r) * 3 * D + h * HD + c * 8);
    h8_to_f32(u, q);
    const float sc = rsqrtf(static_cast<float>(HD)) * kLog2e;
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] *= sc;
  }
  const std::int32_t* tab = table + static_cast<std::int64_t>(d.slot) * max_lb;
  const f16* base = pool + layer_off;
  const int lb0 = start / kBlockTokens, lb1 = (end - 1) / kBlockTokens;

  // Pass 1: scores.
  float mx = -FLT_MAX;
  for (int lb = lb0 + warp; lb <= lb1; lb += kDecWarps) {
    const f16* kblk = base + static_cast<std::int64_t>(tab[lb]) * block_stride + (static_cast<std::int64_t>(h) * kBlockTokens) * HD;
    uint4 kv[kBlockTokens / TPW];
#pragma unroll
    for (int t = 0; t < kBlockTokens / TPW; ++t)
      kv[t] = __ldg(reinterpret_cast<const uint4*>(kblk + (t * TPW + grp) * HD + c * 8));
#pragma unroll
    for (int t = 0; t < kBlockTokens / TPW; ++t) {
      float kf[8];
      h8_to_f32(kv[t], kf);
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) dot = fmaf(q[i], kf[i], dot);
#pragma unroll
      for (int o = LPT / 2; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const int p = lb * kBlockTokens + t * TPW + grp;
      if (c == 0 && p >= start && p < end) {
        s_score[p - start] = dot;
      }
      if (p >= start && p < end) mx = fmaxf(mx, dot);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  mx = s_red[0];
#pragma unroll
  for (int w = 1; w < kDecWarps; ++w) mx = fmaxf(mx, s_red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int i = threadIdx.x; i < end - start; i += blockDim.x) {
    const float e = exp2f(s_score[i] - mx);
    s_score[i] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) s_red[warp] = sum;
  __syncthreads();

  // Pass 2: P * V.
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int lb = lb0 + warp; lb <= lb1; lb += kDecWarps) {
    const f16* vblk = base + static_cast<std::int64_t>(tab[lb]) * block_stride +
                       (static_cast<std::int64_t>(H + h) * kBlockTokens) * HD;
    uint4 vv[kBlockTokens / TPW];
#pragma unroll
    for (int t = 0; t < kBlockTokens / TPW; ++t)
      vv[t] = __ldg(reinterpret_cast<const uint4*>(vblk + (t * TPW + grp) * HD + c * 8));
#pragma unroll
    for (int t = 0; t < kBlockTokens / TPW; ++t) {
      const int p = lb * kBlockTokens + t * TPW + grp;
      const float w = (p >= start && p < end) ? s_score[p - start] : 0.f;
      float vf[8];
      h8_to_f32(vv[t], vf);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(w, vf[i], acc[i]);
    }
  }
  // Reduce token groups (lanes sharing c), then warps.
#pragma unroll
  for (int o = LPT; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  if (grp == 0)
#pragma unroll
    for (int i = 0; i < 8; ++i) s_acc[warp][c * 8 + i] = acc[i];
  __syncthreads();
  const std::int64_t slot_idx = (static_cast<std::int64_t>(dr) * H + h) * max_splits + split;
  for (int i = threadIdx.x; i < HD; i += blockDim.x) {
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) o += s_acc[w][i];
    part_o[slot_idx * HD + i] = o;
  }
  if (threadIdx.x == 0) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) l += s_red[w];
    part_ml[slot_idx * 2] = mx;
    part_ml[slot_idx * 2 + 1] = l;
  }

  // The last split of this (row, head) to finish merges all splits (in split
  // order, so the result does not depend on which CTA is last) and re-arms
  // the counter: no separate combine launch, and the merge runs in K1's tail.
  __shared__ int s_last;
  const int ns = (ctx + SPLIT - 1) / SPLIT;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&counters[dr * H + h], 1);
    s_last = prev == ns - 1;
    if (s_last) counters[dr * H + h] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const std::int64_t pb = (static_cast<std::int64_t>(dr) * H + h) * max_splits;
  float M = -FLT_MAX;
  for (int sp = 0; sp < ns; ++sp) M = fmaxf(M, __ldcg(&part_ml[(pb + sp) * 2]));
  float L = 0.f;
  for (int sp = 0; sp < ns; ++sp) L += __ldcg(&part_ml[(pb + sp) * 2 + 1]) * exp2f(__ldcg(&part_ml[(pb + sp) * 2]) - M);
  const float inv = 1.f / L;
  for (int i = threadIdx.x; i < HD; i += blockDim.x) {
    float o = 0.f;
    for (int sp = 0; sp < ns; ++sp) o += __ldcg(&part_o[(pb + sp) * HD + i]) * exp2f(__ldcg(&part_ml[(pb + sp) * 2]) - M);
    out[static_cast<std::int64_t>(r) * D + h * HD + i] = __float2half_rn(o * inv);
  }
}

template <int HD>
void launch_decode_hd(const f16* qkv, const std::int32_t* drow, const RowDesc* rows, int n, const KvGeom& g,
                      int layer, int max_pos1, float* part_o, float* part_ml, f16* out,
                      std::int32_t* counters, cudaStream_t s) {
  // Positions per CTA: 512 at head dims <= 128, 256 at 256 (measured, profiles/r3i: C4 K1 0.99 vs
  // 0.93 of the copy peak and 41.2 vs 42.0 ms per iteration; C1 K1 0.74 at 256 vs 0.70 at 512).
  // IB2_K1_SPLIT = 256 / 512 / 1024 overrides (diagnostics).
  static const int split_env = getenv("IB2_K1_SPLIT") ? atoi(getenv("IB2_K1_SPLIT")) : 0;
  const int sp = (split_env == 256 || split_env == 512 || split_env == 1024) ? split_env : (HD == 256 ? 256 : 512);
  const int ms = (max_pos1 + sp - 1) / sp;
  auto go = [&](auto kernel) {
    launch_pdl(kernel, dim3(ms, g.heads, n), dim3(kDecWarps * 32), 0, s, qkv, drow, rows, g.pool,
               layer * g.layer_stride(), g.block_stride(), g.table, g.max_lblocks, g.heads, ms, part_o, part_ml, out,
               counters);
  };
  if (sp == 256) go(decode_attn_kernel<HD, 256>);
  else if (sp == 512) go(decode_attn_kernel<HD, 512>);
  else go(decode_attn_kernel<HD, 1024>);
  IB2_LAUNCH_CHECK();
}

}  // namespace

void launch_decode_attention(const f16* qkv, const std::int32_t* drow, const RowDesc* rows, int n_drows,
                             const KvGeom& g, int layer, int max_pos_plus1, float* part_o, float* part_ml,
                             f16* out, std::int32_t* counters, cudaStream_t s) {
  if (n_drows <= 0) return;
  switch (g.head_dim) {
    case 64: launch_decode_hd<64>(qkv, drow, rows, n_drows, g, layer, max_pos_plus1, part_o, part_ml, out, counters, s); break;
    case 128: launch_decode_hd<128>(qkv, drow, rows, n_drows, g, layer, max_pos_plus1, part_o, part_ml, out, counters, s); break;
    case 256: launch_decode_hd<256>(qkv, drow, rows, n_drows, g, layer, max_pos_plus1, part_o, part_ml, out, counters, s); break;
    default: throw DeviceError("unsupported head_dim");
  }
}

int decode_split_positions() { return kSplit; }

}  // namespace ib2
