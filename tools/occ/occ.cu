// Occupancy probe: resident CTAs per SM for a 192-thread kernel vs dynamic
// shared memory size, with and without the max-shared carve-out.
#include <cstdio>
__global__ void __launch_bounds__(192, 2) k(int* out) {
  extern __shared__ unsigned char sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (out) out[threadIdx.x] = sm[(threadIdx.x + 1) % 192];
}
int main() {
  int dev = 0, smem_sm = 0, smem_blk = 0, resv = 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  printf("smem/SM %d, max/block %d, reserved/block %d\n", smem_sm, smem_blk, resv);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_blk);
  for (int carve = 0; carve < 2; ++carve) {
    if (carve) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    for (int kb = 96; kb <= 116; kb += 2) {
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 192, kb * 1024);
      printf("carveout %d dyn %3d KB (%6d B): %d CTAs/SM %s\n", carve, kb, kb * 1024, n, e ? cudaGetErrorString(e) : "");
    }
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 192, 115456);
    printf("carveout %d dyn 115456: %d\n", carve, n);
  }
  return 0;
}
