// Actual residency of a tcgen05.alloc kernel: 2 x SMs CTAs record (smid,
// start, end); count SMs where two CTAs overlapped in time.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__global__ void __launch_bounds__(192, 2) with_tmem(long long* rec, int cols) {
  __shared__ uint32_t slot;
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&slot))), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  while (clock64() - t0 < 2000000) {}
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(cols));
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    rec[blockIdx.x * 3] = smid;
    rec[blockIdx.x * 3 + 1] = g0;
    rec[blockIdx.x * 3 + 2] = g1;
  }
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 2 * sms;
  long long* d;
  cudaMalloc(&d, n * 3 * sizeof(long long));
  cudaFuncSetAttribute(with_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int cols : {256, 512}) {
    with_tmem<<<n, 192, 100 * 1024>>>(d, cols);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(n * 3);
    cudaMemcpy(h.data(), d, n * 3 * sizeof(long long), cudaMemcpyDeviceToHost);
    int overl = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j)
        if (h[i * 3] == h[j * 3] && h[i * 3 + 1] < h[j * 3 + 2] && h[j * 3 + 1] < h[i * 3 + 2]) ++overl;
    long long t0 = h[1], t1 = h[2];
    for (int i = 0; i < n; ++i) { t0 = std::min(t0, h[i * 3 + 1]); t1 = std::max(t1, h[i * 3 + 2]); }
    printf("cols %d: %s, overlapping same-SM CTA pairs %d, makespan %.1f us\n", cols, cudaGetErrorString(e), overl,
           (t1 - t0) / 1e3);
  }
  return 0;
}
