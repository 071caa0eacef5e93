// Paged attention over the GPU-resident block tables.
//
// K1 (decode rows): flash-decoding.  Grid = (KV split, head, row); each CTA
// scores up to kSplit positions of one (row, head) with 16-byte vector loads
// of the head's contiguous [16][hd] slice of each paged block (lanes of a
// token group own 8 dims each, dot products reduced by warp shuffles), then a
// second pass accumulates P*V; a combine kernel merges the splits.  HBM bound:
// algorithmic bytes = 2 * ctx * hd * 2 per (row, head).
//
// K2 (chunk rows: prefill / recompute / API-returned tokens): 64-query tiles
// of one request and one head; K and V tiles of 64 positions (4 paged blocks)
// are staged in XOR-swizzled shared memory with cp.async and consumed by
// f16 tensor-core MMAs with an online softmax (causal mask by position).
// Keys are visited in the same ascending block order as K1.
#include <cfloat>

#include "kernels.hpp"

namespace ib2 {

namespace {

constexpr int kSplit = 256;       // positions per K1 CTA
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

template <int HD>
__global__ void __launch_bounds__(kDecWarps * 32) decode_attn_kernel(
    const f16* __restrict__ qkv, const std::int32_t* __restrict__ drow, const RowDesc* __restrict__ rows,
    const f16* __restrict__ pool, std::int64_t layer_off, std::int64_t block_stride,
    const std::int32_t* __restrict__ table, int max_lb, int H, int max_splits, float* __restrict__ part_o,
    float* __restrict__ part_ml) {
  pdl_trigger();
  pdl_wait();
  constexpr int LPT = HD / 8;   // lanes per token
  constexpr int TPW = 32 / LPT; // tokens per warp step
  const int split = blockIdx.x, h = blockIdx.y, dr = blockIdx.z;
  const int r = drow[dr];
  const RowDesc d = rows[r];
  const int ctx = d.pos + 1;
  const int start = split * kSplit;
  if (start >= ctx) return;
  const int end = min(ctx, start + kSplit);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPT, grp = lane / LPT;
  const int D = H * HD;

  __shared__ float s_score[kSplit];
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
}

__global__ void decode_combine_kernel(const std::int32_t* __restrict__ drow, const RowDesc* __restrict__ rows, int H,
                                      int HD, int max_splits, const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, f16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int dr = blockIdx.x, h = blockIdx.y;
  const int r = drow[dr];
  const int ns = (rows[r].pos + 1 + kSplit - 1) / kSplit;
  const std::int64_t base = (static_cast<std::int64_t>(dr) * H + h) * max_splits;
  float M = -FLT_MAX;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, part_ml[(base + s) * 2]);
  float L = 0.f;
  for (int s = 0; s < ns; ++s) L += part_ml[(base + s) * 2 + 1] * exp2f(part_ml[(base + s) * 2] - M);
  const float inv = 1.f / L;
  for (int i = threadIdx.x; i < HD; i += blockDim.x) {
    float o = 0.f;
    for (int s = 0; s < ns; ++s) o += part_o[(base + s) * HD + i] * exp2f(part_ml[(base + s) * 2] - M);
    out[static_cast<std::int64_t>(r) * H * HD + h * HD + i] = __float2half_rn(o * inv);
  }
}

// ------------------------------------------------------------------ K2 ----

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(std::uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ void ldsm_x4(std::uint32_t addr, std::uint32_t& r0, std::uint32_t& r1, std::uint32_t& r2,
                                        std::uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(std::uint32_t addr, std::uint32_t& r0, std::uint32_t& r1, std::uint32_t& r2,
                                          std::uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, std::uint32_t a0, std::uint32_t a1, std::uint32_t a2,
                                         std::uint32_t a3, std::uint32_t b0, std::uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ std::uint32_t pack_f16(float lo, float hi) {
  const __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&v);
}

// Swizzled element offset of (row, col) in a [rows][HD] f16 tile.
template <int HD>
__device__ __forceinline__ int swz(int row, int col) {
  const int chunk = (col >> 3) ^ (row & 7);
  return row * HD + chunk * 8 + (col & 7);
}

constexpr int kTileQ = 64, kTileK = 64;

template <int HD>
__global__ void __launch_bounds__(128) chunk_attn_kernel(const f16* __restrict__ qkv,
                                                         const TileDesc* __restrict__ tiles,
                                                         const f16* __restrict__ pool, std::int64_t layer_off,
                                                         std::int64_t block_stride,
                                                         const std::int32_t* __restrict__ table, int max_lb, int H,
                                                         f16* __restrict__ out, float* __restrict__ ws_o,
                                                         float* __restrict__ ws_ml) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  f16* sQ = reinterpret_cast<f16*>(smem_raw);
  f16* sK = sQ + kTileQ * HD;
  f16* sV = sK + kTileK * HD;
  const TileDesc td = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int D = H * HD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const std::int32_t* tab = table + static_cast<std::int64_t>(td.slot) * max_lb;
  const int last_pos = td.pos0 + td.nrows - 1;
  const int kv_hi = min(td.kv_hi, last_pos + 1);
  const f16* base = pool + layer_off;

  // Q tile (rows beyond nrows load zeros).
  for (int i = tid; i < kTileQ * (HD / 8); i += 128) {
    const int row = i / (HD / 8), ch = i % (HD / 8);
    const bool ok = row < td.nrows;
    const f16* src = qkv + static_cast<std::int64_t>(td.row0 + (ok ? row : 0)) * 3 * D + h * HD + ch * 8;
    cp_async16(smem_u32(sQ + swz<HD>(row, ch * 8)), src, ok);
  }

  constexpr int NT = kTileK / 8;  // score n-tiles per warp row block
  constexpr int DT = HD / 8;      // output d-tiles
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  const float sc = rsqrtf(static_cast<float>(HD)) * kLog2e;
  const int g = lane >> 2, t4 = lane & 3;
  const int qrow0 = warp * 16;
  // Query positions of this thread's two rows (clamped for padding rows).
  const int qp0 = td.pos0 + min(qrow0 + g, td.nrows - 1);
  const int qp1 = td.pos0 + min(qrow0 + g + 8, td.nrows - 1);

  const int kt_end = (kv_hi + kTileK - 1) / kTileK;
  for (int kt = td.kv_lo / kTileK; kt < kt_end; ++kt) {
    __syncthreads();  // previous tile consumed
    for (int i = tid; i < kTileK * (HD / 8); i += 128) {
      const int row = i / (HD / 8), ch = i % (HD / 8);
      const int p = kt * kTileK + row;
      const bool ok = p < kv_hi;
      std::int64_t off = 0;
      if (ok) off = static_cast<std::int64_t>(tab[p / kBlockTokens]) * block_stride + (p % kBlockTokens) * HD + ch * 8;
      const f16* ksrc = base + off + (static_cast<std::int64_t>(h) * kBlockTokens) * HD;
      const f16* vsrc = base + off + (static_cast<std::int64_t>(H + h) * kBlockTokens) * HD;
      cp_async16(smem_u32(sK + swz<HD>(row, ch * 8)), ok ? ksrc : base, ok);
      cp_async16(smem_u32(sV + swz<HD>(row, ch * 8)), ok ? vsrc : base, ok);
    }
    cp_async_wait_all();
    __syncthreads();

    // S = Q K^T for this warp's 16 rows x 64 keys.
    float s[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD; kk += 16) {
      std::uint32_t a0, a1, a2, a3;
      {
        const int row = qrow0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = kk + (lane >> 4) * 8;
        ldsm_x4(smem_u32(sQ + swz<HD>(row, col)), a0, a1, a2, a3);
      }
#pragma unroll
      for (int j = 0; j < NT; j += 2) {
        std::uint32_t b0, b1, b2, b3;
        const int key = j * 8 + (lane & 7) + (lane >> 4) * 8;
        const int col = kk + ((lane >> 3) & 1) * 8;
        ldsm_x4(smem_u32(sK + swz<HD>(key, col)), b0, b1, b2, b3);
        mma16816(s[j], a0, a1, a2, a3, b0, b1);
        mma16816(s[j + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // Causal mask + online softmax (rows g and g+8 of the warp block).
    float mx0 = m_r[0], mx1 = m_r[1];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int kp = kt * kTileK + j * 8 + 2 * t4;
      const bool in0 = kp >= td.kv_lo && kp < kv_hi, in1 = kp + 1 >= td.kv_lo && kp + 1 < kv_hi;
      s[j][0] = in0 && kp <= qp0 ? s[j][0] * sc : -FLT_MAX;
      s[j][1] = in1 && kp + 1 <= qp0 ? s[j][1] * sc : -FLT_MAX;
      s[j][2] = in0 && kp <= qp1 ? s[j][2] * sc : -FLT_MAX;
      s[j][3] = in1 && kp + 1 <= qp1 ? s[j][3] * sc : -FLT_MAX;
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int o2 = 1; o2 < 4; o2 <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o2));
    }
    // Rows with no visible key yet (split-KV) keep m = -inf: exponentiate
    // against 0 so masked scores give exactly 0.
    const float e0 = mx0 == -FLT_MAX ? 0.f : mx0, e1 = mx1 == -FLT_MAX ? 0.f : mx1;
    const float corr0 = exp2f(m_r[0] - e0), corr1 = exp2f(m_r[1] - e1);
    m_r[0] = mx0;
    m_r[1] = mx1;
    mx0 = e0;
    mx1 = e1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      // P enters the PV MMA as f16; normalize by the sum of the same rounded
      // values so numerator and denominator agree.
      s[j][0] = __half2float(__float2half_rn(exp2f(s[j][0] - mx0)));
      s[j][1] = __half2float(__float2half_rn(exp2f(s[j][1] - mx0)));
      s[j][2] = __half2float(__float2half_rn(exp2f(s[j][2] - mx1)));
      s[j][3] = __half2float(__float2half_rn(exp2f(s[j][3] - mx1)));
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l_r[0] = l_r[0] * corr0 + rs0;
    l_r[1] = l_r[1] * corr1 + rs1;
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      o[i][0] *= corr0;
      o[i][1] *= corr0;
      o[i][2] *= corr1;
      o[i][3] *= corr1;
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < kTileK / 16; ++ks) {
      const std::uint32_t a0 = pack_f16(s[2 * ks][0], s[2 * ks][1]);
      const std::uint32_t a1 = pack_f16(s[2 * ks][2], s[2 * ks][3]);
      const std::uint32_t a2 = pack_f16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      const std::uint32_t a3 = pack_f16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int i = 0; i < DT; i += 2) {
        std::uint32_t b0, b1, b2, b3;
        const int key = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = i * 8 + (lane >> 4) * 8;
        ldsm_x4_t(smem_u32(sV + swz<HD>(key, col)), b0, b1, b2, b3);
        mma16816(o[i], a0, a1, a2, a3, b0, b1);
        mma16816(o[i + 1], a0, a1, a2, a3, b2, b3);
      }
    }
  }
  // Row sums across the quad; whole items normalize and store, split items
  // leave an fp32 partial (unnormalized o, running max m, sum l).
#pragma unroll
  for (int o2 = 1; o2 < 4; o2 <<= 1) {
    l_r[0] += __shfl_xor_sync(0xffffffffu, l_r[0], o2);
    l_r[1] += __shfl_xor_sync(0xffffffffu, l_r[1], o2);
  }
  const int r0 = qrow0 + g, r1 = qrow0 + g + 8;
  if (td.part < 0) {
    const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      const int col = h * HD + i * 8 + 2 * t4;
      if (r0 < td.nrows)
        *reinterpret_cast<__half2*>(out + static_cast<std::int64_t>(td.row0 + r0) * D + col) =
            __floats2half2_rn(o[i][0] * inv0, o[i][1] * inv0);
      if (r1 < td.nrows)
        *reinterpret_cast<__half2*>(out + static_cast<std::int64_t>(td.row0 + r1) * D + col) =
            __floats2half2_rn(o[i][2] * inv1, o[i][3] * inv1);
    }
  } else {
    const std::int64_t slot = (static_cast<std::int64_t>(td.part) * H + h) * kTileQ;
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      const int col = i * 8 + 2 * t4;
      *reinterpret_cast<float2*>(ws_o + (slot + r0) * HD + col) = make_float2(o[i][0], o[i][1]);
      *reinterpret_cast<float2*>(ws_o + (slot + r1) * HD + col) = make_float2(o[i][2], o[i][3]);
    }
    if (t4 == 0) {
      ws_ml[(slot + r0) * 2] = m_r[0];
      ws_ml[(slot + r0) * 2 + 1] = l_r[0];
      ws_ml[(slot + r1) * 2] = m_r[1];
      ws_ml[(slot + r1) * 2 + 1] = l_r[1];
    }
  }
}

// Merge the split-KV partials of one q-tile and head.
__global__ void chunk_combine_kernel(const CombineDesc* __restrict__ cds, int H, int HD,
                                     const float* __restrict__ ws_o, const float* __restrict__ ws_ml,
                                     f16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const CombineDesc c = cds[blockIdx.x];
  const int h = blockIdx.y;
  const int D = H * HD;
  for (int e = threadIdx.x; e < c.nrows * HD; e += blockDim.x) {
    const int r = e / HD, d = e % HD;
    float M = -FLT_MAX;
    for (int p = 0; p < c.nparts; ++p)
      M = fmaxf(M, ws_ml[((static_cast<std::int64_t>(c.part0 + p) * H + h) * kTileQ + r) * 2]);
    float L = 0.f, O = 0.f;
    for (int p = 0; p < c.nparts; ++p) {
      const std::int64_t slot = (static_cast<std::int64_t>(c.part0 + p) * H + h) * kTileQ + r;
      const float m = ws_ml[slot * 2];
      const float w = m == -FLT_MAX ? 0.f : exp2f(m - M);
      L += ws_ml[slot * 2 + 1] * w;
      O += ws_o[slot * HD + d] * w;
    }
    out[static_cast<std::int64_t>(c.row0 + r) * D + h * HD + d] = __float2half_rn(O / L);
  }
}

template <int HD>
void launch_chunk_hd(const f16* qkv, const TileDesc* tiles, int n_tiles, const KvGeom& g, int layer, f16* out,
                     float* ws_o, float* ws_ml, cudaStream_t s) {
  const int smem = (kTileQ + 2 * kTileK) * HD * 2;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(chunk_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  dim3 grid(n_tiles, g.heads);
  launch_pdl(chunk_attn_kernel<HD>, grid, dim3(128), smem, s, qkv, tiles, g.pool, layer * g.layer_stride(),
             g.block_stride(), g.table, g.max_lblocks, g.heads, out, ws_o, ws_ml);
  IB2_LAUNCH_CHECK();
}

template <int HD>
void launch_decode_hd(const f16* qkv, const std::int32_t* drow, const RowDesc* rows, int n, const KvGeom& g,
                      int layer, int max_splits, float* part_o, float* part_ml, f16* out, cudaStream_t s) {
  dim3 grid(max_splits, g.heads, n);
  launch_pdl(decode_attn_kernel<HD>, grid, dim3(kDecWarps * 32), 0, s, qkv, drow, rows, g.pool,
             layer * g.layer_stride(), g.block_stride(), g.table, g.max_lblocks, g.heads, max_splits, part_o, part_ml);
  IB2_LAUNCH_CHECK();
  launch_pdl(decode_combine_kernel, dim3(n, g.heads), dim3(HD), 0, s, drow, rows, g.heads, HD, max_splits, part_o,
             part_ml, out);
  IB2_LAUNCH_CHECK();
}

}  // namespace

void launch_decode_attention(const f16* qkv, const std::int32_t* drow, const RowDesc* rows, int n_drows,
                             const KvGeom& g, int layer, int max_pos_plus1, float* part_o, float* part_ml,
                             f16* out, cudaStream_t s) {
  if (n_drows <= 0) return;
  const int max_splits = (max_pos_plus1 + kSplit - 1) / kSplit;
  switch (g.head_dim) {
    case 64: launch_decode_hd<64>(qkv, drow, rows, n_drows, g, layer, max_splits, part_o, part_ml, out, s); break;
    case 128: launch_decode_hd<128>(qkv, drow, rows, n_drows, g, layer, max_splits, part_o, part_ml, out, s); break;
    case 256: launch_decode_hd<256>(qkv, drow, rows, n_drows, g, layer, max_splits, part_o, part_ml, out, s); break;
    default: throw DeviceError("unsupported head_dim");
  }
}

void launch_chunk_attention(const f16* qkv, const TileDesc* tiles, int n_tiles, const CombineDesc* combines,
                            int n_combines, const KvGeom& g, int layer, f16* out, float* ws_o, float* ws_ml,
                            cudaStream_t s) {
  if (n_tiles <= 0) return;
  switch (g.head_dim) {
    case 64: launch_chunk_hd<64>(qkv, tiles, n_tiles, g, layer, out, ws_o, ws_ml, s); break;
    case 128: launch_chunk_hd<128>(qkv, tiles, n_tiles, g, layer, out, ws_o, ws_ml, s); break;
    case 256: launch_chunk_hd<256>(qkv, tiles, n_tiles, g, layer, out, ws_o, ws_ml, s); break;
    default: throw DeviceError("unsupported head_dim");
  }
  if (n_combines > 0)
    launch_pdl(chunk_combine_kernel, dim3(n_combines, g.heads), dim3(256), 0, s, combines, g.heads, g.head_dim, ws_o,
               ws_ml, out);
}

int decode_split_positions() { return kSplit; }

}  // namespace ib2
