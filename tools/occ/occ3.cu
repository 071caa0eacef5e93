// Does tcgen05.alloc in a kernel change the occupancy the runtime reports?
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(192, 2) plain(int* o) {
  extern __shared__ unsigned char sm[];
  sm[threadIdx.x] = 1;
  __syncthreads();
  if (o) o[threadIdx.x] = sm[threadIdx.x];
}
__global__ void __launch_bounds__(192, 2) with_tmem(int* o) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&slot))), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  if (o) o[threadIdx.x] = slot;
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(256));
}
int main() {
  int a = 0, b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, plain, 192, 16384);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, with_tmem, 192, 16384);
  printf("plain %d CTAs/SM, with tcgen05.alloc %d CTAs/SM\n", a, b);
  return 0;
}
