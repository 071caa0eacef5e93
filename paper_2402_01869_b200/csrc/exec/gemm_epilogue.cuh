// Fused GEMM epilogues shared by the SIMT and tcgen05 projection GEMMs.
#pragma once

#include "common.cuh"

namespace ib2 {

// 0.5 v (1 + tanh(u)) == v * sigmoid(2u), u = sqrt(2/pi) (v + 0.044715 v^3):
// one MUFU exp and one fast divide instead of tanhf (the CTA-pair GEMM's
// MLP-in epilogue was bound by it); agrees with the tanh form to ~1e-7.
__device__ __forceinline__ float gelu_tanh(float v) {
  const float u = 0.7978845608028654f * (v + 0.044715f * v * v * v);
  return __fdividef(v, 1.0f + __expf(-2.0f * u));
}
__device__ __forceinline__ float silu(float v) { return v / (1.0f + __expf(-v)); }

// Fused K4, 16 consecutive columns n0.. (one head part, rotary pairs inside)
// of row m: x[] are the bias-added values already rounded to f16, as the
// separate RoPE pass would read them.  q -> out, k / v -> the row's paged block.
__device__ __forceinline__ void qkv_store16(const GemmArgs& a, int m, int n0, float* x) {
  const QkvWrite& w = a.qkv;
  const int D = w.H * w.hd;
  const int part = n0 >= D ? (n0 >= 2 * D ? 2 : 1) : 0;
  const int hn = n0 - part * D, h = hn / w.hd, d0 = hn - h * w.hd;
  const RowDesc r = w.rows[m];
  if (part < 2 && d0 < w.rot) {
    const float4* cs = reinterpret_cast<const float4*>(w.rope_cs + (static_cast<std::int64_t>(r.pos) * (w.rot / 2) + d0 / 2) * 2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 c = cs[i];  // (cos, sin) of pairs 2i, 2i+1
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float co = k ? c.z : c.x, si = k ? c.w : c.y;
        const float xa = x[4 * i + 2 * k], xb = x[4 * i + 2 * k + 1];
        x[4 * i + 2 * k] = __fsub_rn(__fmul_rn(xa, co), __fmul_rn(xb, si));
        x[4 * i + 2 * k + 1] = __fadd_rn(__fmul_rn(xb, co), __fmul_rn(xa, si));
      }
    }
  }
  uint4 pk[2];
  std::uint32_t* u = reinterpret_cast<std::uint32_t*>(pk);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const __half2 hv = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
    u[i] = *reinterpret_cast<const std::uint32_t*>(&hv);
  }
  f16* dst;
  if (part == 0) {
    dst = a.out + static_cast<std::int64_t>(m) * a.ldo + n0;
  } else {
    const std::int32_t pb = w.table[static_cast<std::int64_t>(r.slot) * w.max_lb + r.pos / kBlockTokens];
    dst = w.pool + w.layer_off + static_cast<std::int64_t>(pb) * w.block_stride +
          ((static_cast<std::int64_t>(part - 1) * w.H + h) * kBlockTokens + r.pos % kBlockTokens) * w.hd + d0;
  }
  reinterpret_cast<uint4*>(dst)[0] = pk[0];
  reinterpret_cast<uint4*>(dst)[1] = pk[1];
}

// Apply the epilogue to `cnt` consecutive accumulator columns n0.. of row m.
// cnt is even; SwiGLU consumes (gate, up) pairs.
template <int CNT>
__device__ __forceinline__ void epilogue_store(const GemmArgs& a, int m, int n0, const float* acc) {
  if (m >= a.M) return;
  if (a.epi == Epi::QkvRopeKv) {  // CNT consecutive columns, rotary pairs inside
    if constexpr (CNT == 16) {
      float x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        x[i] = __half2float(__float2half_rn(acc[i] + (a.bias ? __half2float(a.bias[n0 + i]) : 0.f)));
      if (n0 + 16 <= a.N) qkv_store16(a, m, n0, x);
    } else {
      __trap();  // the executor only uses the fused QKV epilogue on tcgen05 paths (K % 64 == 0)
    }
    return;
  }
  float v[CNT];
#pragma unroll
  for (int i = 0; i < CNT; ++i) v[i] = acc[i];
  if (a.bias && a.epi != Epi::SwiGluF16) {
#pragma unroll
    for (int i = 0; i < CNT; ++i)
      if (n0 + i < a.N) v[i] += __half2float(a.bias[n0 + i]);
  }
  switch (a.epi) {
    case Epi::StoreF16:
    case Epi::GeluF16: {
      f16* o = a.out + static_cast<std::int64_t>(m) * a.ldo + n0;
#pragma unroll
      for (int i = 0; i < CNT; i += 2) {
        if (n0 + i >= a.N) break;
        float x0 = v[i], x1 = v[i + 1];
        if (a.epi == Epi::GeluF16) {
          x0 = gelu_tanh(x0);
          x1 = gelu_tanh(x1);
        }
        *reinterpret_cast<__half2*>(o + i) = __floats2half2_rn(x0, x1);
      }
      break;
    }
    case Epi::ResidAdd: {
      float* o = a.outf + static_cast<std::int64_t>(m) * a.ldf + n0;
#pragma unroll
      for (int i = 0; i < CNT; ++i)
        if (n0 + i < a.N) {
          const float r = o[i] + v[i];
          o[i] = a.addf ? r + a.addf[static_cast<std::int64_t>(m) * a.ldf + n0 + i] : r;
        }
      break;
    }
    case Epi::StoreF32: {
      float* o = a.outf + static_cast<std::int64_t>(m) * a.ldf + n0;
#pragma unroll
      for (int i = 0; i < CNT; ++i)
        if (n0 + i < a.N) o[i] = v[i];
      break;
    }
    case Epi::SwiGluF16: {
      f16* o = a.out + static_cast<std::int64_t>(m) * a.ldo + n0 / 2;
#pragma unroll
      for (int i = 0; i < CNT; i += 2)
        if (n0 + i < a.N) o[i / 2] = __float2half_rn(silu(v[i]) * v[i + 1]);
      break;
    }
  }
}

}  // namespace ib2
