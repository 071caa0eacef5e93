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

// Apply the epilogue to `cnt` consecutive accumulator columns n0.. of row m.
// cnt is even; SwiGLU consumes (gate, up) pairs.
template <int CNT>
__device__ __forceinline__ void epilogue_store(const GemmArgs& a, int m, int n0, const float* acc) {
  if (m >= a.M) return;
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
        if (n0 + i < a.N) o[i] += v[i];
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
