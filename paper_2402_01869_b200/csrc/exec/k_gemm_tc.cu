// K3: projection GEMM on 5th-generation tensor cores (sm_100a).
//
//   C[M][N] = A[M][K] . W[N][K]^T   (f16 in, fp32 accumulate in TMEM)
//
// Warp-specialized, one output tile (128 x BN) per CTA:
//   warp 0      TMA producer: A and W tiles (128 B swizzle) into a STAGES-deep
//               shared-memory ring guarded by full/empty mbarriers;
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128,
//               N=BN, K=16) x4 per 64-wide K block, tcgen05.commit frees the
//               stage; the final commit signals the epilogue;
//   warp 2      TMEM allocator (BN fp32 columns);
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x16 from their TMEM lane quarter,
//               fused bias / GELU / SwiGLU / residual-add / fp32 store.
// Tensor maps cover the full buffer capacity; TMA zero-fills the K tail and
// rows past the buffer, and the epilogue masks rows >= M.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "gemm_epilogue.cuh"
#include "kernels.hpp"

namespace ib2 {

void launch_gemm_simt(const GemmArgs& a, cudaStream_t s);

namespace {

constexpr int BM = 128, BK = 64, UMMA_K = 16;

__device__ __forceinline__ std::uint32_t su32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* b, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 B (SBO), LBO unused, descriptor version 1 (sm_100).
__device__ __forceinline__ std::uint64_t smem_desc(const void* p) {
  const std::uint64_t addr = su32(p);
  std::uint64_t d = 0;
  d |= (addr & 0x3FFFFULL) >> 4;                 // start address [0,14)
  d |= static_cast<std::uint64_t>(1) << 16;      // LBO (ignored for SW128 K-major)
  d |= static_cast<std::uint64_t>(1024 >> 4) << 32;  // SBO [32,46)
  d |= static_cast<std::uint64_t>(1) << 46;      // version
  d |= static_cast<std::uint64_t>(2) << 61;      // SWIZZLE_128B
  return d;
}

template <int BN>
__host__ __device__ constexpr std::uint32_t instr_desc() {
  return (1u << 4)                                     // D = f32
         | (0u << 7)                                   // A = f16
         | (0u << 10)                                  // B = f16
         | (static_cast<std::uint32_t>(BN >> 3) << 17) // N
         | (static_cast<std::uint32_t>(BM >> 4) << 24);// M
}

template <int BN, int STAGES>
struct TcSmem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 1) * 8 + 16 + 1024;  // + alignment slack
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                                         const __grid_constant__ CUtensorMap map_w, GemmArgs args) {
  using L = TcSmem<BN, STAGES>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L::BAR_OFF);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* done = empty + STAGES;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // M-fastest rasterization: the M tiles that share a weight tile run in the
  // same wave, so the weight tile is fetched from HBM once and re-read from L2.
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nk = (args.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_w)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const std::uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the prologue above overlapped the predecessor kernel

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        unsigned char* sa = smem + s * L::STAGE_BYTES;
        unsigned char* sb = sa + L::A_BYTES;
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        tma_load_2d(sa, &map_a, &full[s], kb * BK, m0);
        // Tile-blocked weights: rows of 128-row tile t at k block kb start at
        // physical row (t * nk + kb) * 128; BN = 256 spans two tiles.
        const int wt = n0 / 128, wr = n0 % 128;
        tma_load_2d(sb, &map_w, &full[s], 0, (wt * nk + kb) * 128 + wr);
        if (BN == 256) tma_load_2d(sb + 128 * BK * 2, &map_w, &full[s], 0, ((wt + 1) * nk + kb) * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = instr_desc<BN>();
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const unsigned char* sa = smem + s * L::STAGE_BYTES;
        const std::uint64_t da = smem_desc(sa), db = smem_desc(sa + L::A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / UMMA_K; ++k) {
          const std::uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          // +32 bytes per 16-element K step inside the 128-byte swizzle atom.
          asm volatile(
              "{\n"
              ".reg .pred p;\n"
              "setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
              "}\n" ::"r"(tmem),
              "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&empty[s]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(done))
                   : "memory");
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter (warp % 4)
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int m = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      std::uint32_t r[16];
      const std::uint32_t taddr = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
      if (n0 + c < args.N) epilogue_store<16>(args, m, n0 + c, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
  }
}


// ---- small-M path: swap-AB stream-K ------------------------------------------
//
// Decode-dominated iterations have M (tokens) of 8..256 while the N x K
// weights are 17-134 MB per projection: the GEMM is a weight stream.  C^T =
// W A^T puts 128 weight rows on the UMMA M side (TMEM lanes) and the tokens on
// the UMMA N side (NT columns), so every weight byte is read exactly once.
//
// Stream-K: the tiles x k-blocks units of work are cut into gridDim.x equal
// contiguous ranges, one per CTA (one CTA per SM), so every SM streams the
// same number of weight bytes whatever N/128 is.  A range covers whole tiles
// in its middle (epilogue straight from TMEM) and partial tiles at its ends:
// those write an fp32 partial [NT][128] into the CTA's own workspace slot,
// and the last CTA to finish a tile (atomic ticket) sums the tile's partials
// in CTA order -- deterministic -- and runs the fused epilogue.  Accumulators
// alternate between two TMEM buffers so the epilogue of one segment overlaps
// the MMAs of the next; the TMA ring never drains between segments.

template <int NT, int STAGES>
struct SkSmem {
  static constexpr int A_BYTES = BM * BK * 2;  // weights tile
  static constexpr int B_BYTES = NT * BK * 2;  // tokens tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = 2 * NT < 32 ? 32 : 2 * NT;
};

__device__ __forceinline__ void epi_one(const GemmArgs& a, int m, int n, float v) {
  if (a.bias && a.epi != Epi::SwiGluF16) v += __half2float(a.bias[n]);
  switch (a.epi) {
    case Epi::StoreF16: a.out[static_cast<std::int64_t>(m) * a.ldo + n] = __float2half_rn(v); break;
    case Epi::GeluF16: a.out[static_cast<std::int64_t>(m) * a.ldo + n] = __float2half_rn(gelu_tanh(v)); break;
    case Epi::ResidAdd: a.outf[static_cast<std::int64_t>(m) * a.ldf + n] += v; break;
    case Epi::StoreF32: a.outf[static_cast<std::int64_t>(m) * a.ldf + n] = v; break;
    default: break;
  }
}

// Epilogue of weight row n (this lane) for token m; SwiGLU pairs come from
// the neighbouring lane (gate = even row, up = odd row).
__device__ __forceinline__ void epi_row(const GemmArgs& a, int n, int m, float v, int lane) {
  if (a.epi == Epi::SwiGluF16) {
    const float up = __shfl_down_sync(0xffffffffu, v, 1);
    if (!(lane & 1) && m < a.M && n < a.N)
      a.out[static_cast<std::int64_t>(m) * a.ldo + n / 2] = __float2half_rn(silu(v) * up);
    return;
  }
  if (m < a.M && n < a.N) epi_one(a, m, n, v);
}

__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, std::uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Unit range [start(c), start(c+1)) of CTA c; the CTA owning unit u.
__device__ __forceinline__ std::int64_t sk_start(int c, std::int64_t U, int G) { return c * U / G; }
__device__ __forceinline__ int sk_owner(std::int64_t u, std::int64_t U, int G) {
  return static_cast<int>(((u + 1) * G - 1) / U);
}

template <int NT, int STAGES>
__global__ void __launch_bounds__(256, 1) tc_streamk_kernel(const __grid_constant__ CUtensorMap map_w,
                                                            const __grid_constant__ CUtensorMap map_a, GemmArgs args,
                                                            float* __restrict__ ws, int* __restrict__ tickets) {
  using L = SkSmem<NT, STAGES>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L::BAR_OFF);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2] MMA -> epilogue
  std::uint64_t* tempty = tfull + 2;      // [2] epilogue -> MMA
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = args.K / BK;
  const std::int64_t U = static_cast<std::int64_t>((args.N + BM - 1) / BM) * kblocks;
  const int G = gridDim.x, c = blockIdx.x;
  const std::int64_t u0 = sk_start(c, U, G), u1 = sk_start(c + 1, U, G);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_a)) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const std::uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the prologue above overlapped the predecessor kernel

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (std::int64_t u = u0; u < u1;) {
        const int t = static_cast<int>(u / kblocks), kb0 = static_cast<int>(u % kblocks);
        const int kb1 = static_cast<int>(kblocks < kb0 + (u1 - u) ? kblocks : kb0 + (u1 - u));
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int st = i % STAGES;
          if (i >= STAGES) mbar_wait(&empty[st], ((i / STAGES) - 1) & 1);
          unsigned char* sw = smem + st * L::STAGE_BYTES;
          mbar_expect_tx(&full[st], L::STAGE_BYTES);
          tma_load_2d(sw, &map_w, &full[st], 0, (t * kblocks + kb) * BM);  // one contiguous 16 KB tile
          tma_load_2d(sw + L::A_BYTES, &map_a, &full[st], kb * BK, 0);
        }
        u += kb1 - kb0;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = (1u << 4) | (static_cast<std::uint32_t>(NT >> 3) << 17) |
                                      (static_cast<std::uint32_t>(BM >> 4) << 24);
      int i = 0, seg = 0;
      for (std::int64_t u = u0; u < u1; ++seg) {
        const int kb0 = static_cast<int>(u % kblocks);
        const int kb1 = static_cast<int>(kblocks < kb0 + (u1 - u) ? kblocks : kb0 + (u1 - u));
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], ((seg / 2) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const std::uint32_t acc_tmem = tmem + buf * NT;
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int st = i % STAGES;
          mbar_wait(&full[st], (i / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const unsigned char* sw = smem + st * L::STAGE_BYTES;
          const std::uint64_t da = smem_desc(sw), db = smem_desc(sw + L::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const std::uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
                "}\n" ::"r"(acc_tmem),
                "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           su32(&empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&tfull[buf]))
                     : "memory");
        u += kb1 - kb0;
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4, row = q * 32 + lane;
    const int mcols = min(args.M, NT);
    int seg = 0;
    for (std::int64_t u = u0; u < u1; ++seg) {
      const int t = static_cast<int>(u / kblocks), kb0 = static_cast<int>(u % kblocks);
      const int kb1 = static_cast<int>(kblocks < kb0 + (u1 - u) ? kblocks : kb0 + (u1 - u));
      u += kb1 - kb0;
      const int buf = seg & 1;
      const int n = t * BM + row;
      mbar_wait(&tfull[buf], (seg / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const bool whole = kb0 == 0 && kb1 == kblocks;
      // Partial segments go to slot 0 (the CTA's first tile) or 1 (its last).
      float* part = ws + ((static_cast<std::int64_t>(c) * 2 + (seg == 0 ? 0 : 1)) * NT) * BM;
#pragma unroll 1
      for (int cc = 0; cc < mcols; cc += 16) {
        std::uint32_t r[16];
        tmem_ld16(tmem + buf * NT + (static_cast<std::uint32_t>(q * 32) << 16) + cc, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float v = __uint_as_float(r[j]);
          if (whole) epi_row(args, n, cc + j, v, lane);
          else if (cc + j < mcols) part[(cc + j) * BM + row] = v;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tempty[buf])) : "memory");
      if (whole) continue;
      // Ticket: the last of the tile's CTAs reduces.
      const int c_first = sk_owner(static_cast<std::int64_t>(t) * kblocks, U, G);
      const int c_last = sk_owner(static_cast<std::int64_t>(t) * kblocks + kblocks - 1, U, G);
      __threadfence();
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (row == 0) {
        const int prev = atomicAdd(&tickets[t], 1);
        const bool last = prev == c_last - c_first;
        if (last) tickets[t] = 0;  // ready for the next launch
        *last_flag = last ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (!*last_flag) continue;
      __threadfence();
      for (int m0 = 0; m0 < mcols; m0 += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.f;
        for (int o = c_first; o <= c_last; ++o) {
          // CTA o's segment of tile t is its first (slot 0) unless tile t is
          // not where o's range starts.
          const int slot = (sk_start(o, U, G) / kblocks == t) ? 0 : 1;
          const float* src = ws + ((static_cast<std::int64_t>(o) * 2 + slot) * NT) * BM;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (m0 + j < mcols) acc[j] += __ldcg(src + (m0 + j) * BM + row);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (m0 + j < mcols) epi_row(args, n, m0 + j, acc[j], lane);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(L::TMEM_COLS));
  }
}

// ---- host side ----------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    IB2_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw DeviceError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D f16 tensor map over [rows][K] (row stride ld elements), box 64 x box_rows.
CUtensorMap make_map(const void* base, std::int64_t rows, int K, int ld, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

struct MapKey {
  const void* p;
  std::int64_t rows;
  int K, box;
  bool operator==(const MapKey& o) const { return p == o.p && rows == o.rows && K == o.K && box == o.box; }
};
struct MapKeyHash {
  std::size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (static_cast<std::size_t>(k.rows) * 31u) ^ (static_cast<std::size_t>(k.K) << 7) ^
           static_cast<std::size_t>(k.box);
  }
};

// Tile-blocked weight [N][K] seen by TMA as [ceil(N/128)*128*K/64 rows][64].
const CUtensorMap& cached_wmap(const void* base, std::int64_t N, int K, int box_rows);

const CUtensorMap& cached_map(const void* base, std::int64_t rows, int K, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  std::lock_guard<std::mutex> g(mu);
  const MapKey key{base, rows, K, box_rows};
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, make_map(base, rows, K, K, box_rows)).first;
  return it->second;
}

const CUtensorMap& cached_wmap(const void* base, std::int64_t N, int K, int box_rows) {
  const std::int64_t phys_rows = (N + 127) / 128 * 128 * (K / BK);
  return cached_map(base, phys_rows, BK, box_rows);
}

std::int64_t g_a_rows_capacity = 0;  // rows of every activation buffer (set by the executor)

template <int BN, int STAGES>
void launch_tc(const GemmArgs& a, cudaStream_t s) {
  using L = TcSmem<BN, STAGES>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  const std::int64_t a_rows = g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M;
  const CUtensorMap& ma = cached_map(a.a, a_rows, a.K, BM);
  const CUtensorMap& mw = cached_wmap(a.w, a.N, a.K, BN == 256 ? 128 : BN);
  dim3 grid((a.M + BM - 1) / BM, (a.N + BN - 1) / BN);
  launch_pdl(tc_gemm_kernel<BN, STAGES>, grid, dim3(256), L::TOTAL, s, ma, mw, a);
}


int g_sms = 0;

// Stream-K workspace: 2 partial slots of [256][128] fp32 per CTA, and one
// ticket per weight tile (reset by the tile's reducer), per device.
struct StreamKWs {
  float* ws = nullptr;
  int* tickets = nullptr;
  int tiles = 0;
};
StreamKWs& streamk_ws(int tiles) {
  static std::mutex mu;
  static StreamKWs per_dev[16];
  int dev = 0;
  IB2_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  StreamKWs& w = per_dev[dev & 15];
  if (!w.ws) IB2_CUDA(cudaMalloc(&w.ws, static_cast<std::size_t>(g_sms) * 2 * 256 * BM * sizeof(float)));
  if (tiles > w.tiles) {
    if (w.tickets) IB2_CUDA(cudaFree(w.tickets));
    const int n = std::max(tiles, 1024);
    IB2_CUDA(cudaMalloc(&w.tickets, n * sizeof(int)));
    IB2_CUDA(cudaMemset(w.tickets, 0, n * sizeof(int)));
    w.tiles = n;
  }
  return w;
}

template <int NT, int STAGES>
void launch_skinny(const GemmArgs& a, cudaStream_t s) {
  using L = SkSmem<NT, STAGES>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(tc_streamk_kernel<NT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  L::TOTAL));
    configured = true;
  }
  const int tiles = static_cast<int>((a.N + BM - 1) / BM), kblocks = a.K / BK;
  const std::int64_t units = static_cast<std::int64_t>(tiles) * kblocks;
  // One CTA per SM, each streaming >= 4 k-blocks (64 KB of weights).
  const int ctas = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g_sms, units / 4)));
  StreamKWs& w = streamk_ws(tiles);
  const std::int64_t a_rows = g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M;
  const CUtensorMap& mw = cached_wmap(a.w, a.N, a.K, BM);
  const CUtensorMap& ma = cached_map(a.a, a_rows, a.K, NT);
  launch_pdl(tc_streamk_kernel<NT, STAGES>, dim3(ctas), dim3(256), L::TOTAL, s, mw, ma, a, w.ws, w.tickets);
}

bool skinny_ok(const GemmArgs& a) {
  static const bool off = getenv("IB2_NO_SKINNY") != nullptr;
  return !off && a.M <= 256 && a.K % BK == 0 && a.N % 2 == 0;
}

void launch_skinny_any(const GemmArgs& a, cudaStream_t s) {
  if (!g_sms) {
    int dev = 0;
    IB2_CUDA(cudaGetDevice(&dev));
    IB2_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  if (a.M <= 16) launch_skinny<16, 10>(a, s);
  else if (a.M <= 32) launch_skinny<32, 9>(a, s);
  else if (a.M <= 64) launch_skinny<64, 8>(a, s);
  else if (a.M <= 128) launch_skinny<128, 6>(a, s);
  else launch_skinny<256, 4>(a, s);
}

}  // namespace

void set_gemm_activation_rows(std::int64_t rows) { g_a_rows_capacity = rows; }

CUtensorMap make_tmap_2d(const void* base, std::int64_t inner, std::int64_t rows, std::int64_t row_stride_bytes,
                         int box_inner, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_bytes)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

bool gemm_uses_tcgen05() { return true; }

void launch_gemm(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  if (a.K % BK != 0 || a.N % 2 != 0) {  // N tails are masked; K must fill whole 64-wide blocks
    launch_gemm_simt(a, s);
    return;
  }
  if (skinny_ok(a)) {
    launch_skinny_any(a, s);
    return;
  }
  // Small M is weight-bandwidth bound: narrow N tiles put more SMs on the
  // weight stream.  Large M uses wide tiles for operand reuse.
  const std::int64_t tiles128 = static_cast<std::int64_t>((a.N + 127) / 128) * ((a.M + BM - 1) / BM);
  if (a.M > 512 && a.N >= 1024) launch_tc<256, 4>(a, s);
  else if (tiles128 >= 148) launch_tc<128, 6>(a, s);
  else launch_tc<64, 8>(a, s);
}

void debug_tile_weights(const void* src, void* dst, int N, int K, void* stream) {
  if (K % BK) throw DeviceError("debug_tile_weights: K must be a multiple of 64");
  launch_tile_weights(static_cast<const f16*>(src), static_cast<f16*>(dst), N, K, static_cast<cudaStream_t>(stream));
}

void debug_gemm(const void* a, const void* w, int M, int N, int K, int epi, const void* bias, void* out, int ldo,
                void* outf, int ldf, int flags, void* stream) {
  const bool force_simt = flags & 1;
  if (!(flags & 2)) {
  // The executor keeps weights tile-blocked; the hook takes row-major W.
  static f16* tiled = nullptr;
  static std::size_t tiled_elems = 0;
  const std::size_t need = static_cast<std::size_t>((N + 127) / 128 * 128) * K;
  if (need > tiled_elems) {
    if (tiled) cudaFree(tiled);
    IB2_CUDA(cudaMalloc(&tiled, need * sizeof(f16)));
    tiled_elems = need;
  }
  launch_tile_weights(static_cast<const f16*>(w), tiled, N, K, static_cast<cudaStream_t>(stream));
  w = tiled;
  }
  GemmArgs g{static_cast<const f16*>(a), static_cast<const f16*>(w), M, N, K, static_cast<Epi>(epi),
             static_cast<const f16*>(bias), static_cast<f16*>(out), ldo, static_cast<float*>(outf), ldf};
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const std::int64_t saved = g_a_rows_capacity;
  g_a_rows_capacity = 0;  // caller buffers are exactly M rows
  if (force_simt) launch_gemm_simt(g, s);
  else launch_gemm(g, s);
  g_a_rows_capacity = saved;
}

}  // namespace ib2
