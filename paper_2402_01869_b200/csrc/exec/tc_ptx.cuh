// Inline-PTX vocabulary of the sm_100a tensor-core kernels (K2, K3):
// mbarriers, TMA tile loads, UMMA shared-memory / instruction descriptors,
// tcgen05 MMA / commit / TMEM loads and stores.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <cstdio>

namespace ib2 {
namespace tc {

__device__ __forceinline__ std::uint32_t su32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* b, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
// Bounded waits: a phase that does not complete within ~2^34 cycles (about
// 9 s) means a protocol bug; the kernel prints the barrier and traps (the
// launch fails loudly) instead of wedging the GPU.
__device__ __forceinline__ bool mbar_try(std::uint32_t addr, std::uint32_t parity) {
  std::uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cluster(std::uint32_t addr, std::uint32_t parity) {
  std::uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __noinline__ inline void mbar_timeout(std::uint32_t addr, std::uint32_t parity) {
  printf("ib2 watchdog: mbarrier smem+0x%x parity %u stuck, block (%d,%d,%d) thread %d\n", addr, parity, blockIdx.x,
         blockIdx.y, blockIdx.z, threadIdx.x);
  __trap();
}
constexpr long long kWaitLimitCycles = 1LL << 34;
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
  const std::uint32_t a = su32(b);
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(a, parity))
    if (clock64() - t0 > kWaitLimitCycles) mbar_timeout(a, parity);
}
// Acquire at cluster scope (barriers signalled from peer CTAs over DSMEM).
__device__ __forceinline__ void mbar_wait_cluster(std::uint64_t* b, std::uint32_t parity) {
  const std::uint32_t a = su32(b);
  if (mbar_try_cluster(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_cluster(a, parity))
    if (clock64() - t0 > kWaitLimitCycles) mbar_timeout(a, parity);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(map)) : "memory");
}

// UMMA shared-memory descriptor, 128-byte swizzle, descriptor version 1.
//  K-major operand: 8-row x 128 B atoms, SBO = 1024 B between row groups
//    (LBO unused); the K step inside an atom is +32 B on the start address.
//  MN-major operand: 64-element (128 B) MN runs; LBO = bytes between
//    64-element MN blocks, SBO = bytes between 8-row K groups.
__device__ __forceinline__ std::uint64_t desc_sw128(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;  // version (sm_100)
  d |= static_cast<std::uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16: f16 A/B, f32 D, M x N, operand majors.
__host__ __device__ constexpr std::uint32_t idesc_f16(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (static_cast<std::uint32_t>(a_mn_major) << 15) | (static_cast<std::uint32_t>(b_mn_major) << 16) |
         (static_cast<std::uint32_t>(N >> 3) << 17) | (static_cast<std::uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(std::uint32_t tmem_d, std::uint64_t da, std::uint64_t db, std::uint32_t idesc,
                                        std::uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// Generic-proxy shared-memory writes -> visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(std::uint32_t* slot, std::uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(slot)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc(std::uint32_t tmem, std::uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(cols));
}

// 32 lanes x 32 bit, 16 consecutive columns -> r[0..15] (no wait).
__device__ __forceinline__ void tmem_ld16_nowait(std::uint32_t taddr, std::uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(std::uint32_t taddr, const std::uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

}  // namespace tc
}  // namespace ib2
