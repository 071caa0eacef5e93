// Reference-quality SIMT GEMM (fp32 FMA) with the same fused epilogues as
// the tcgen05 kernel.  Used for shapes the tensor-core kernel does not take
// (K not a multiple of 64) and as the in-process cross-check of K3.
#include "gemm_epilogue.cuh"
#include "kernels.hpp"
#include "model.hpp"

namespace ib2 {

namespace {

constexpr int BM = 64, BN = 64, BK = 32;

__global__ void __launch_bounds__(256) simt_gemm_kernel(GemmArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sA[BK][BM + 4];
  __shared__ float sW[BK][BN + 4];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      const int r = i / BK, c = i % BK;
      const int m = m0 + r, n = n0 + r, k = k0 + c;
      sA[c][r] = (m < a.M && k < a.K) ? __half2float(a.a[static_cast<std::int64_t>(m) * a.K + k]) : 0.f;
      sW[c][r] = (n < a.N && k < a.K) ? __half2float(a.w[weight_tile_offset(n, k, a.K)]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      float av[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = sA[k][ty * 4 + i];
        wv[i] = sW[k][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) epilogue_store<4>(a, m0 + ty * 4 + i, n0 + tx * 4, acc[i]);
}

}  // namespace

void launch_gemm_simt(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  launch_pdl(simt_gemm_kernel, grid, dim3(256), 0, s, a);
  IB2_LAUNCH_CHECK();
}

}  // namespace ib2
