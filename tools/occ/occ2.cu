// Occupancy vs register count for 192-thread CTAs.
#include <cstdio>
template <int R>
__global__ void __launch_bounds__(192, 2) k(const float* in, float* out) {
  float a[R];
#pragma unroll
  for (int i = 0; i < R; ++i) a[i] = in[threadIdx.x * R + i];
#pragma unroll
  for (int it = 0; it < 4; ++it)
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = a[i] * a[(i + 1) % R] + a[(i + 7) % R];
#pragma unroll
  for (int i = 0; i < R; ++i) out[threadIdx.x * R + i] = a[i];
}
template <int R>
void probe() {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k<R>);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k<R>, 192, 0);
  int n2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n2, k<R>, 192, 100 * 1024);
  printf("R=%d regs %d: %d CTAs/SM (0 smem), %d CTAs/SM (100 KB)\n", R, fa.numRegs, n, n2);
}
int main() {
  probe<96>();
  probe<112>();
  probe<120>();
  probe<124>();
  probe<128>();
  return 0;
}
