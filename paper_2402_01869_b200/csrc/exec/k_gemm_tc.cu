// K3: projection GEMMs on 5th-generation tensor cores (sm_100a).
//
//   C[M][N] = A[M][K] . W[N][K]^T   (f16 in, fp32 accumulate in TMEM)
//
// Two warp-specialised kernels, both fed by TMA (128 B swizzle) through an
// mbarrier ring, one elected thread issuing tcgen05.mma, accumulators in TMEM
// drained by four epilogue warps with fused bias / GELU / SwiGLU / residual
// epilogues:
//   * tc_splitk_kernel (M <= 256, decode batches): swap-AB, weights on the
//     UMMA M side, cluster split-K with a DSMEM reduction;
//   * tc_gemm_pair_kernel (M > 256, chunk batches): CTA pair, cta_group::2,
//     256x256 tiles, persistent with double-buffered TMEM accumulators.
// Weights are stored tile-blocked (model.hpp weight_tile_offset): every TMA of
// a weight tile is one contiguous 16 KB run.  Tensor maps cover the full buffer
// capacity; TMA zero-fills rows past it and the epilogues mask rows >= M.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "gemm_epilogue.cuh"
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace ib2 {

void launch_gemm_simt(const GemmArgs& a, cudaStream_t s);

namespace {

constexpr int BM = 128, BK = 64, UMMA_K = 16;

using namespace tc;

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

// ---- small-M path: swap-AB, cluster split-K ----------------------------------
//
// Decode-dominated iterations have M (tokens) of 8..256 while the N x K
// weights are 17-134 MB per projection: the GEMM is a weight stream.  C^T =
// W A^T puts 128 weight rows on the UMMA M side (TMEM lanes) and the tokens on
// the UMMA N side (NT columns), so every weight byte is read exactly once.
//
// Work split so every SM streams about the same number of bytes: a cluster of
// S CTAs owns a contiguous run of T weight tiles and CTA rank r streams the
// k-slice r of each of them (S = 1: whole tiles).  Accumulators alternate
// between two TMEM buffers, so a tile's epilogue overlaps the next tile's
// MMAs and the TMA ring never drains.  With S > 1 each rank drops its fp32
// partial tile into one of two shared-memory slots, signals every rank's
// `ready` mbarrier over DSMEM, and rank r sums token columns
// [r*M/S, (r+1)*M/S) of all S partials in rank order (ld.shared::cluster;
// deterministic, no global workspace, no atomics) before the fused epilogue;
// `consumed` mbarriers hand the slot back.  Only the epilogue warps take part,
// so the weight stream never waits for the reduction.

template <int NT, int STAGES>
struct SkSmem {
  static constexpr int A_BYTES = BM * BK * 2;  // weights tile
  static constexpr int B_BYTES = NT * BK * 2;  // tokens tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // fp32 partial-tile slots next to the ring: two for NT <= 64 (a tile's
  // reduction overlaps the next tile's), one for NT = 128, none for 256.
  static constexpr int PART_SLOTS = NT <= 64 ? 2 : (NT == 128 ? 1 : 0);
  static constexpr bool SPLIT_OK = PART_SLOTS > 0;
  static constexpr int PART_BYTES = NT * BM * 4;  // one fp32 partial tile
  static constexpr int PART_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = PART_OFF + PART_SLOTS * PART_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 9) * 8 + 16 + 1024;
  // stream-K: an owner stages up to two fp32 pieces in its drained ring
  static_assert(NT > 128 || STAGES * STAGE_BYTES >= 2 * NT * BM * 4, "stream-K pieces fit in the ring");
  static constexpr int TMEM_COLS = 2 * NT < 32 ? 32 : 2 * NT;
  static_assert(TOTAL <= 232448, "shared memory budget");
};

// Epilogue of weight row n (this lane) for tokens m0..m0+15: every global
// load is issued before any store so the 16 residual read-modify-writes
// overlap instead of paying one memory latency each.
__device__ __forceinline__ void epi_rows16(const GemmArgs& a, int n, int m0, const float* v, int lane) {
  if (a.epi == Epi::QkvRopeKv) {
    // Thread = column n (fixed part / head / dim), 16 tokens.  Rotary pairs
    // are columns (2i, 2i+1): neighbouring lanes.
    const QkvWrite& w = a.qkv;
    const int D = w.H * w.hd;
    const int part = n >= D ? (n >= 2 * D ? 2 : 1) : 0;
    const int hn = n - part * D, h = hn / w.hd, d = hn - h * w.hd;
    const bool rot = part < 2 && d < w.rot;
    const float b = (a.bias && n < a.N) ? __half2float(a.bias[n]) : 0.f;
    float x[16], pr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = __half2float(__float2half_rn(v[j] + b));
#pragma unroll
    for (int j = 0; j < 16; ++j) pr[j] = __shfl_xor_sync(0xffffffffu, x[j], 1);
    if (n >= a.N) return;
    int pos[16];
    std::int32_t pb[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) pos[j] = m0 + j < a.M ? w.rows[m0 + j].pos : 0;
    if (part > 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        pb[j] = m0 + j < a.M ? w.table[static_cast<std::int64_t>(w.rows[m0 + j].slot) * w.max_lb + pos[j] / kBlockTokens]
                             : 0;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (m0 + j >= a.M) break;
      float y = x[j];
      if (rot) {
        const float2 cs = *reinterpret_cast<const float2*>(w.rope_cs + (static_cast<std::int64_t>(pos[j]) * (w.rot / 2) + d / 2) * 2);
        y = (d & 1) ? __fadd_rn(__fmul_rn(x[j], cs.x), __fmul_rn(pr[j], cs.y))
                    : __fsub_rn(__fmul_rn(x[j], cs.x), __fmul_rn(pr[j], cs.y));
      }
      const f16 hv = __float2half_rn(y);
      if (part == 0)
        a.out[static_cast<std::int64_t>(m0 + j) * a.ldo + n] = hv;
      else
        w.pool[w.layer_off + static_cast<std::int64_t>(pb[j]) * w.block_stride +
               ((static_cast<std::int64_t>(part - 1) * w.H + h) * kBlockTokens + pos[j] % kBlockTokens) * w.hd + d] = hv;
    }
    return;
  }
  if (a.epi == Epi::SwiGluF16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float up = __shfl_down_sync(0xffffffffu, v[j], 1);
      if (!(lane & 1) && m0 + j < a.M && n < a.N)
        a.out[static_cast<std::int64_t>(m0 + j) * a.ldo + n / 2] = __float2half_rn(silu(v[j]) * up);
    }
    return;
  }
  if (n >= a.N) return;
  const float b = a.bias ? __half2float(a.bias[n]) : 0.f;
  switch (a.epi) {
    case Epi::StoreF16:
    case Epi::GeluF16:
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (m0 + j < a.M) {
          const float x = v[j] + b;
          a.out[static_cast<std::int64_t>(m0 + j) * a.ldo + n] = __float2half_rn(a.epi == Epi::GeluF16 ? gelu_tanh(x) : x);
        }
      break;
    case Epi::ResidAdd: {
      float old[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) old[j] = m0 + j < a.M ? a.outf[static_cast<std::int64_t>(m0 + j) * a.ldf + n] : 0.f;
      float add[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        add[j] = (a.addf && m0 + j < a.M) ? a.addf[static_cast<std::int64_t>(m0 + j) * a.ldf + n] : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (m0 + j < a.M) {
          const float r = old[j] + (v[j] + b);
          a.outf[static_cast<std::int64_t>(m0 + j) * a.ldf + n] = a.addf ? r + add[j] : r;
        }
      break;
    }
    case Epi::StoreF32:
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (m0 + j < a.M) a.outf[static_cast<std::int64_t>(m0 + j) * a.ldf + n] = v[j] + b;
      break;
    default: break;
  }
}

__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, std::uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ std::uint32_t cluster_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ std::uint32_t map_to_rank(std::uint32_t local, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(std::uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void wait_cluster(std::uint64_t* b, std::uint32_t parity) { mbar_wait_cluster(b, parity); }

// Stream-K (S = 1, sk != nullptr): the (tile, k block) units are split
// evenly over the grid, so every SM streams the same number of weight bytes
// whatever the tile count (96 / 128 / 394 GPT-J tiles on 148 SMs).  A CTA's
// range is a run of segments: maybe the END of one tile (its first segment,
// kb > 0), whole tiles, maybe the START of a tile (its last segment).  The
// CTA holding a tile's k block 0 owns it and works on it last; the pieces of
// its other k blocks were produced FIRST by the following CTAs, which drop
// them (fp32) into their workspace slot and publish `epoch`.  The owner adds
// them in k order after its own partial (deterministic) and runs the fused
// epilogue, so the reduction never stalls the weight stream.
struct StreamK {
  float* ws;             // [grid][NT * BM] fp32 pieces
  std::int32_t* flags;   // [grid] epoch of the piece in the slot
  std::int32_t epoch;
};

__device__ __forceinline__ int sk_cta_of(long long u, long long total, int G) {
  // the CTA whose range [c*total/G, (c+1)*total/G) holds unit u
  int c = static_cast<int>(u * G / total);
  while (c + 1 < G && (static_cast<long long>(c + 1) * total) / G <= u) ++c;
  while (c > 0 && (static_cast<long long>(c) * total) / G > u) --c;
  return c;
}

template <int NT, int STAGES>
__global__ void __launch_bounds__(256, 1) tc_splitk_kernel(const __grid_constant__ CUtensorMap map_w,
                                                           const __grid_constant__ CUtensorMap map_a, GemmArgs args,
                                                           int S, StreamK sk) {
  using L = SkSmem<NT, STAGES>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L::BAR_OFF);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2] MMA -> epilogue
  std::uint64_t* tempty = tfull + 2;      // [2] epilogue -> MMA
  std::uint64_t* ready = tempty + 2;      // [2] all ranks' partials of a slot written
  std::uint64_t* consumed = ready + 2;    // [2] all ranks done reading a slot
  std::uint64_t* fixbar = consumed + 2;   // [1] stream-K pieces landed in the ring
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(fixbar + 1);
  float* parts = reinterpret_cast<float*>(smem + L::PART_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (args.N + BM - 1) / BM, kblocks = args.K / BK;
  const int rank = S > 1 ? static_cast<int>(cluster_rank()) : 0;
  const int n_clusters = gridDim.x / S, cid = blockIdx.x / S;
  const int t0 = static_cast<int>(static_cast<long long>(cid) * tiles / n_clusters);
  const int t1 = static_cast<int>(static_cast<long long>(cid + 1) * tiles / n_clusters);
  const int kb0 = rank * kblocks / S, kb1 = (rank + 1) * kblocks / S;
  // Segments of this CTA: (tile, [kb_a, kb_b)).  Cluster split-K / whole
  // tiles: t0..t1 with [kb0, kb1).  Stream-K: the unit range [u0, u1).
  const bool streamk = sk.ws != nullptr;
  const long long total_u = static_cast<long long>(tiles) * kblocks;
  const long long u0 = streamk ? static_cast<long long>(blockIdx.x) * total_u / gridDim.x : 0;
  const long long u1 = streamk ? static_cast<long long>(blockIdx.x + 1) * total_u / gridDim.x : 0;
  const int seg_first_t = streamk ? static_cast<int>(u0 / kblocks) : t0;
  const int seg_end_t = streamk ? (u1 > u0 ? static_cast<int>((u1 - 1) / kblocks) + 1 : seg_first_t) : t1;
  auto seg_kb = [&](int t, int& a, int& b) {
    if (!streamk) {
      a = kb0;
      b = kb1;
      return;
    }
    const long long lo = static_cast<long long>(t) * kblocks, hi = lo + kblocks;
    a = static_cast<int>((u0 > lo ? u0 : lo) - lo);
    b = static_cast<int>((u1 < hi ? u1 : hi) - lo);
  };

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
      mbar_init(&ready[i], 4 * S);
      mbar_init(&consumed[i], 4 * S);
    }
    mbar_init(fixbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (S > 1) {  // peers' barriers are initialised before anyone signals them
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const std::uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // Weights do not depend on the predecessor kernel: the first ring's
      // worth of weight tiles streams in while it is still finishing; the
      // activation tiles follow griddepcontrol.wait.
      int early_kb[STAGES];
      int early = 0;
      if (!args.no_early_w) {
        for (int t = seg_first_t; t < seg_end_t && early < STAGES; ++t) {
          int a, b;
          seg_kb(t, a, b);
          for (int kb = a; kb < b && early < STAGES; ++kb, ++early) {
            early_kb[early] = kb;
            mbar_expect_tx(&full[early], L::STAGE_BYTES);
            tma_load_2d(smem + early * L::STAGE_BYTES, &map_w, &full[early], 0, (t * kblocks + kb) * BM);
          }
        }
      }
      pdl_wait();
      for (int i = 0; i < early; ++i)
        tma_load_2d(smem + i * L::STAGE_BYTES + L::A_BYTES, &map_a, &full[i], early_kb[i] * BK, 0);
      int i = 0;
      for (int t = seg_first_t; t < seg_end_t; ++t) {
        int a, b;
        seg_kb(t, a, b);
        for (int kb = a; kb < b; ++kb, ++i) {
          if (i < early) continue;
          const int st = i % STAGES;
          mbar_wait(&empty[st], ((i / STAGES) - 1) & 1);
          unsigned char* sw = smem + st * L::STAGE_BYTES;
          mbar_expect_tx(&full[st], L::STAGE_BYTES);
          tma_load_2d(sw, &map_w, &full[st], 0, (t * kblocks + kb) * BM);  // one contiguous 16 KB tile
          tma_load_2d(sw + L::A_BYTES, &map_a, &full[st], kb * BK, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = (1u << 4) | (static_cast<std::uint32_t>(NT >> 3) << 17) |
                                      (static_cast<std::uint32_t>(BM >> 4) << 24);
      int i = 0;
      for (int t = seg_first_t, seg = 0; t < seg_end_t; ++t, ++seg) {
        const int buf = seg & 1;
        int ka, kbe;
        seg_kb(t, ka, kbe);
        if (seg >= 2) mbar_wait(&tempty[buf], ((seg / 2) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const std::uint32_t acc_tmem = tmem + buf * NT;
        for (int kb = ka; kb < kbe; ++kb, ++i) {
          const int st = i % STAGES;
          mbar_wait(&full[st], (i / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const unsigned char* sw = smem + st * L::STAGE_BYTES;
          const std::uint64_t da = smem_desc(sw), db = smem_desc(sw + L::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const std::uint32_t acc = (kb > ka || k > 0) ? 1u : 0u;
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
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // the epilogue reads / writes buffers of earlier kernels
    const int q = warp - 4, row = q * 32 + lane;
    const int mcols = min(args.M, NT);
    const int m_lo = rank * mcols / S, m_hi = (rank + 1) * mcols / S;
    for (int t = seg_first_t, seg = 0; t < seg_end_t; ++t, ++seg) {
      const int buf = seg & 1;
      const int n = t * BM + row;
      mbar_wait(&tfull[buf], (seg / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (streamk) {
        int ka, kbe;
        seg_kb(t, ka, kbe);
        float* mine = sk.ws + static_cast<std::int64_t>(blockIdx.x) * (NT * BM);
        if (ka > 0) {
          // A piece (end / middle of a tile owned by an earlier CTA): fp32 -> slot, then publish.
#pragma unroll 1
          for (int cc = 0; cc < mcols; cc += 16) {
            std::uint32_t r[16];
            tmem_ld16(tmem + buf * NT + (static_cast<std::uint32_t>(q * 32) << 16) + cc, r);
#pragma unroll
            for (int j = 0; j < 16; ++j) mine[(cc + j) * BM + row] = __uint_as_float(r[j]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __threadfence();
          asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the 4 epilogue warps
          if (q == 0 && lane == 0)
            asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(sk.flags + blockIdx.x), "r"(sk.epoch) : "memory");
        } else {
          // Whole tile, or the owner of a tile whose later k blocks are pieces of
          // the next CTAs (at most two): their fp32 slots are bulk-copied into
          // this CTA's drained stage ring (its last MMAs retired: tfull), then
          // added after this CTA's own partial, in k order.
          const int c_last = kbe < kblocks ? sk_cta_of(static_cast<long long>(t + 1) * kblocks - 1, total_u, gridDim.x)
                                           : static_cast<int>(blockIdx.x);
          const int npieces = c_last - static_cast<int>(blockIdx.x);
          if (npieces > 2) __trap();  // the grid planner keeps >= kblocks / 2 units per CTA
          if (npieces > 0) {
            if (q == 0 && lane == 0) {
              for (int p = blockIdx.x + 1; p <= c_last; ++p) {
                const long long t_start = clock64();
                while (true) {
                  std::int32_t e;
                  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(e) : "l"(sk.flags + p) : "memory");
                  if (e == sk.epoch) break;
                  if (clock64() - t_start > kWaitLimitCycles) {
                    printf("ib2 watchdog: stream-K piece of CTA %d (epoch %d) missing for CTA %d\n", p, sk.epoch,
                           blockIdx.x);
                    __trap();
                  }
                }
              }
              asm volatile("fence.proxy.async.global;\n" ::: "memory");
              constexpr std::uint32_t bytes = NT * BM * 4;
              mbar_expect_tx(fixbar, bytes * npieces);
              for (int k = 0; k < npieces; ++k)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        su32(smem + k * bytes)),
                    "l"(reinterpret_cast<std::uint64_t>(sk.ws + static_cast<std::int64_t>(blockIdx.x + 1 + k) * (NT * BM))),
                    "r"(bytes), "r"(su32(fixbar))
                    : "memory");
            }
            mbar_wait(fixbar, 0);  // once per kernel: a CTA owns at most one partial tile
          }
          const float* staged = reinterpret_cast<const float*>(smem);
#pragma unroll 1
          for (int cc = 0; cc < mcols; cc += 16) {
            std::uint32_t r[16];
            tmem_ld16(tmem + buf * NT + (static_cast<std::uint32_t>(q * 32) << 16) + cc, r);
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
            for (int k = 0; k < npieces; ++k) {
              const float* piece = staged + static_cast<std::int64_t>(k) * (NT * BM);
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] += piece[(cc + j) * BM + row];
            }
            epi_rows16(args, n, cc, v, lane);
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tempty[buf])) : "memory");
        continue;
      }
      constexpr int NS = L::PART_SLOTS > 0 ? L::PART_SLOTS : 1;
      const int slot = seg % NS;
      float* part = parts + slot * (NT * BM);
      if (S > 1 && seg >= NS) wait_cluster(&consumed[slot], ((seg / NS) - 1) & 1);
#pragma unroll 1
      for (int cc = 0; cc < mcols; cc += 16) {
        std::uint32_t r[16];
        tmem_ld16(tmem + buf * NT + (static_cast<std::uint32_t>(q * 32) << 16) + cc, r);
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        if (S == 1) {
          epi_rows16(args, n, cc, v, lane);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) part[(cc + j) * BM + row] = v[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tempty[buf])) : "memory");
      if (S == 1) continue;
      // Partials of this slot -> every rank; then reduce this rank's columns.
      // Every writer fences at cluster scope before its warp's lanes < S
      // signal the ranks (release by the signalling lane covers the warp's
      // writes through __syncwarp as well; the explicit fence states it).
      asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
      __syncwarp();
      if (lane < S) arrive_remote(map_to_rank(su32(&ready[slot]), lane));
      wait_cluster(&ready[slot], (seg / NS) & 1);
      const std::uint32_t local = su32(part) + row * 4;
      for (int m0 = m_lo; m0 < m_hi; m0 += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.f;
        for (int rr = 0; rr < S; ++rr) {
          const std::uint32_t peer = map_to_rank(local, rr);
          float x[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            x[j] = 0.f;
            if (m0 + j < m_hi)
              asm volatile("ld.shared::cluster.f32 %0, [%1];\n"
                           : "=f"(x[j])
                           : "r"(peer + static_cast<std::uint32_t>((m0 + j) * BM * 4)));
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += x[j];
        }
        // Columns past m_hi belong to the next rank: mask them out.
        GemmArgs a2 = args;
        a2.M = m_hi;
        epi_rows16(a2, n, m0, acc, lane);
      }
      __syncwarp();
      if (lane < S) arrive_remote(map_to_rank(su32(&consumed[slot]), lane));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (S > 1) {  // peers may still read this CTA's partial slots
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(L::TMEM_COLS));
  }
}

// ---- large-M path: CTA-pair (cta_group::2) persistent GEMM --------------------
//
// Chunk iterations (prefill / recompute, M ~ 0.3k-2k rows) are tensor-core
// bound.  A cluster of 2 CTAs on neighbouring SMs computes 256 x 256 output
// tiles with tcgen05.mma.cta_group::2 (M = 256 split over the pair's TMEM, N =
// 256): each CTA stages its 128 rows of A and its 128 rows of W per 64-wide k
// block, so shared-memory traffic per SM is 32 KB per 128x256x64 MMA instead
// of 48 KB.  Persistent over the tile list (M-fastest, so the pairs running
// together share weight tiles through L2); accumulators alternate between two
// 256-column TMEM buffers so a tile's epilogue (4 warps per CTA, 16-byte
// vector stores, fused bias / GELU / SwiGLU / residual) overlaps the next
// tile's MMAs.
//   warp 0      TMA producer (both CTAs; completion counted on the leader's
//               full barrier via .cta_group::2);
//   warp 1      MMA issuer (leader CTA only); commits multicast to both CTAs;
//   warp 2      TMEM allocator (cta_group::2, 512 columns);
//   warps 4-7   epilogue (both CTAs, own 128 rows).

constexpr int kPairStages = 6;
// BN: tile width (UMMA N of the pair); each CTA stages BN / 2 weight rows.
template <int BN>
struct PairSmem {
  static constexpr int STAGES = BN == 256 ? kPairStages : 8;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 5) * 8 + 16 + 1024;
  static_assert(STAGES * STAGE_BYTES >= 128 * BN * 4, "a split-tail piece is staged in the drained ring");
};

__device__ __forceinline__ std::uint32_t cta_rank_in_cluster() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ std::uint32_t mapa_rank(std::uint32_t local, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, std::uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

// 16 consecutive output columns n0.. of row m (vector stores when aligned).
__device__ __forceinline__ void epi_cols16(const GemmArgs& a, int m, int n0, float* v) {
  if (m >= a.M || n0 >= a.N) return;
  if (a.epi == Epi::QkvRopeKv) {  // 16 columns of one head part; rotary pairs inside
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      x[i] = __half2float(__float2half_rn(v[i] + (a.bias ? __half2float(a.bias[n0 + i]) : 0.f)));
    if (n0 + 16 <= a.N) qkv_store16(a, m, n0, x);
    return;
  }
  const bool full = n0 + 16 <= a.N;
  if (a.bias && a.epi != Epi::SwiGluF16) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (full || n0 + i < a.N) v[i] += __half2float(a.bias[n0 + i]);
  }
  switch (a.epi) {
    case Epi::StoreF16:
    case Epi::GeluF16: {
      if (a.epi == Epi::GeluF16) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = gelu_tanh(v[i]);
      }
      f16* o = a.out + static_cast<std::int64_t>(m) * a.ldo + n0;
      if (full && (a.ldo % 8) == 0) {
        uint4 w[2];
        std::uint32_t* u = reinterpret_cast<std::uint32_t*>(w);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          u[i] = *reinterpret_cast<const std::uint32_t*>(&h);
        }
        reinterpret_cast<uint4*>(o)[0] = w[0];
        reinterpret_cast<uint4*>(o)[1] = w[1];
      } else {
        for (int i = 0; i < 16 && n0 + i < a.N; ++i) o[i] = __float2half_rn(v[i]);
      }
      break;
    }
    case Epi::ResidAdd:
    case Epi::StoreF32: {
      float* o = a.outf + static_cast<std::int64_t>(m) * a.ldf + n0;
      if (full && (a.ldf % 4) == 0) {
        float4* o4 = reinterpret_cast<float4*>(o);
        if (a.epi == Epi::ResidAdd) {
          float4 r[4], ad[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) r[i] = o4[i];
          if (a.addf) {
            const float4* a4 = reinterpret_cast<const float4*>(a.addf + static_cast<std::int64_t>(m) * a.ldf + n0);
#pragma unroll
            for (int i = 0; i < 4; ++i) ad[i] = a4[i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o4[i] = make_float4((r[i].x + v[4 * i]) + ad[i].x, (r[i].y + v[4 * i + 1]) + ad[i].y,
                                  (r[i].z + v[4 * i + 2]) + ad[i].z, (r[i].w + v[4 * i + 3]) + ad[i].w);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o4[i] = make_float4(r[i].x + v[4 * i], r[i].y + v[4 * i + 1], r[i].z + v[4 * i + 2], r[i].w + v[4 * i + 3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      } else {
        for (int i = 0; i < 16 && n0 + i < a.N; ++i) {
          if (a.epi != Epi::ResidAdd) {
            o[i] = v[i];
            continue;
          }
          const float r = o[i] + v[i];
          o[i] = a.addf ? r + a.addf[static_cast<std::int64_t>(m) * a.ldf + n0 + i] : r;
        }
      }
      break;
    }
    case Epi::SwiGluF16: {
      f16* o = a.out + static_cast<std::int64_t>(m) * a.ldo + n0 / 2;
      if (full && (a.ldo % 8) == 0) {
        uint4 w;
        std::uint32_t* u = reinterpret_cast<std::uint32_t*>(&w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __half2 h = __floats2half2_rn(silu(v[4 * i]) * v[4 * i + 1], silu(v[4 * i + 2]) * v[4 * i + 3]);
          u[i] = *reinterpret_cast<const std::uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(o) = w;
      } else {
        for (int i = 0; i < 16 && n0 + i < a.N; i += 2) o[i / 2] = __float2half_rn(silu(v[i]) * v[i + 1]);
      }
      break;
    }
  }
}

// Work of one CTA pair: whole tiles in data-parallel rounds (t = pair,
// pair + npairs, ...) while every pair has one, then -- split tail (sk.ws
// set) -- each of the remaining T mod npairs tiles is shared by a pair of
// pairs (g = 2 when npairs >= 2 rem), each taking half of its k blocks,
// instead of one pair per tile while the rest idle through a last partial
// round.  The group's first pair owns the tile: it bulk-copies the other
// half's fp32 piece (computed at the same time) into its drained stage ring
// and adds it after its own (deterministic).  (Spreading a tail tile over every pair, classic
// stream-K, measured slower: the owner's read of ~17 pieces outweighed the
// saved k blocks.)
struct PairSegs {
  int pair, npairs, total, nk, dp_tiles, rem, g;
  int t, a, b;  // current segment
  int dp_next;
  bool tail_done;
  __device__ void init(int p, int np, int tot, int nkb, bool split_tail) {
    pair = p;
    npairs = np;
    total = tot;
    nk = nkb;
    dp_tiles = split_tail ? (tot / np) * np : tot;
    rem = tot - dp_tiles;
    g = rem > 0 ? np / rem : 1;
    g = g < 1 ? 1 : (g > 2 ? 2 : g);
    g = g > nk ? nk : g;
    dp_next = p;
    tail_done = false;
  }
  __device__ bool next() {
    if (dp_next < dp_tiles) {
      t = dp_next;
      a = 0;
      b = nk;
      dp_next += npairs;
      return true;
    }
    if (tail_done) return false;
    tail_done = true;
    if (pair >= rem * g) return false;
    const int part = pair % g;
    t = dp_tiles + pair / g;
    a = part * nk / g;
    b = (part + 1) * nk / g;
    return true;
  }
};

template <int BN>
__global__ void __launch_bounds__(256, 1) tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                                                              const __grid_constant__ CUtensorMap map_w,
                                                              GemmArgs args, StreamK sk) {
  using L = PairSmem<BN>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L::BAR_OFF);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2] MMA -> epilogues (multicast)
  std::uint64_t* tempty = tfull + 2;      // [2] epilogues of both CTAs -> MMA (leader's)
  std::uint64_t* fixbar = tempty + 2;     // [1] split-tail piece landed in shared memory
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(fixbar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cta_rank_in_cluster();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int MT = (args.M + 255) / 256, NTL = (args.N + BN - 1) / BN;
  const int total = MT * NTL;
  const int nk = args.K / BK;
  const bool streamk = sk.ws != nullptr;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_w)) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs
    }
    mbar_init(fixbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // Both CTAs of the pair must be running before the 2-CTA TMEM allocation:
  // its hand-shake signals the peer through shared memory, and a signal sent
  // before the peer CTA started is lost (observed: the peer's allocator warp
  // waiting forever while the leader sat in the cluster barrier below).
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const std::uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const std::uint32_t full0 = mapa_rank(su32(full), 0);  // leader's full barriers
      // The weight tiles of the first ring's worth of k blocks stream in
      // before griddepcontrol.wait (they do not depend on the predecessor).
      int pre = 0;
      // Row of this CTA's BN / 2 weight rows of tile ntl, k block kb, in the
      // tile-blocked [N / 128][K / 64][128][64] weight layout.
      auto wrow = [&](int ntl, int kb) {
        return BN == 256 ? ((ntl * 2 + static_cast<int>(rank)) * nk + kb) * 128
                         : (ntl * nk + kb) * 128 + static_cast<int>(rank) * 64;
      };
      PairSegs it;
      it.init(pair, npairs, total, nk, streamk);
      while (pre < STAGES && !args.no_early_w && it.next()) {
        for (int kb = it.a; kb < it.b && pre < STAGES; ++kb, ++pre) {
          if (leader) mbar_expect_tx(&full[pre], 2 * L::STAGE_BYTES);
          tma_load_2d_pair(smem + pre * L::STAGE_BYTES + L::A_BYTES, &map_w, full0 + pre * 8, 0, wrow(it.t / MT, kb));
        }
      }
      pdl_wait();
      int i = 0;
      it.init(pair, npairs, total, nk, streamk);
      while (it.next()) {
        const int t = it.t;
        const int mt = t % MT, ntl = t / MT;
        const int arow = mt * 256 + static_cast<int>(rank) * 128;
        for (int kb = it.a; kb < it.b; ++kb, ++i) {
          const int st = i % STAGES;
          unsigned char* sa = smem + st * L::STAGE_BYTES;
          const std::uint32_t bar = full0 + st * 8;
          if (i < pre) {  // weights already in flight
            tma_load_2d_pair(sa, &map_a, bar, kb * BK, arow);
            continue;
          }
          mbar_wait(&empty[st], ((i / STAGES) - 1) & 1);
          if (leader) mbar_expect_tx(&full[st], 2 * L::STAGE_BYTES);
          tma_load_2d_pair(sa, &map_a, bar, kb * BK, arow);
          tma_load_2d_pair(sa + L::A_BYTES, &map_w, bar, 0, wrow(ntl, kb));
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr std::uint32_t idesc = (1u << 4) | (static_cast<std::uint32_t>(BN >> 3) << 17) |
                                      (static_cast<std::uint32_t>(256 >> 4) << 24);
      int i = 0, seg = 0;
      PairSegs it;
      it.init(pair, npairs, total, nk, streamk);
      for (; it.next(); ++seg) {
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], ((seg / 2) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const std::uint32_t acc_tmem = tmem + buf * BN;
        const int ka = it.a;
        for (int kb = it.a; kb < it.b; ++kb, ++i) {
          const int st = i % STAGES;
          mbar_wait(&full[st], (i / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const unsigned char* sa = smem + st * L::STAGE_BYTES;
          const std::uint64_t da = smem_desc(sa), db = smem_desc(sa + L::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const std::uint32_t acc = (kb > ka || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
                "}\n" ::"r"(acc_tmem),
                "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                  su32(&empty[st])),
              "h"(static_cast<unsigned short>(3))
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                su32(&tfull[buf])),
            "h"(static_cast<unsigned short>(3))
            : "memory");
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // the epilogue reads / writes buffers of earlier kernels
    const int q = warp - 4;
    const std::uint32_t tempty0 = mapa_rank(su32(tempty), 0);
    int seg = 0;
    PairSegs it;
    it.init(pair, npairs, total, nk, streamk);
    const int row = q * 32 + lane;  // this thread's row of the CTA's 128
    for (; it.next(); ++seg) {
      const int t = it.t;
      const int buf = seg & 1;
      const int mt = t % MT, ntl = t / MT;
      const int m = mt * 256 + static_cast<int>(rank) * 128 + row;
      mbar_wait(&tfull[buf], (seg / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (it.a > 0) {
        // A piece of a tail tile owned by an earlier pair: fp32 -> this CTA's slot, publish.
        // Layout [column chunk][row][16]: the owner reads it back from shared
        // memory with few bank conflicts.
        float* mine = sk.ws + static_cast<std::int64_t>(blockIdx.x) * (128 * BN);
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          std::uint32_t r[16];
          tmem_ld16(tmem + buf * BN + (static_cast<std::uint32_t>(q * 32) << 16) + c, r);
          float4* d4 = reinterpret_cast<float4*>(mine + (static_cast<std::int64_t>(c / 16) * 128 + row) * 16);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                                __uint_as_float(r[4 * j + 3]));
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __threadfence();
        asm volatile("bar.sync 1, 128;\n" ::: "memory");  // this CTA's 4 epilogue warps
        if (q == 0 && lane == 0)
          asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(sk.flags + blockIdx.x), "r"(sk.epoch) : "memory");
      } else {
        // Whole tile, or owner of a split tail tile: wait for the other half's piece,
        // bulk-copy it into the drained stage ring (the last MMAs have retired:
        // tfull), add it after this pair's half.
        const bool owner = it.b < nk;
        const float* piece_s = reinterpret_cast<const float*>(smem);
        if (owner) {
          const int cta = 2 * (pair + 1) + static_cast<int>(rank);
          if (q == 0 && lane == 0) {
            const long long t_start = clock64();
            while (true) {
              std::int32_t e;
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(e) : "l"(sk.flags + cta) : "memory");
              if (e == sk.epoch) break;
              if (clock64() - t_start > kWaitLimitCycles) {
                printf("ib2 watchdog: split-tail piece of CTA %d (epoch %d) missing for CTA %d\n", cta, sk.epoch,
                       blockIdx.x);
                __trap();
              }
            }
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            constexpr std::uint32_t bytes = 128 * BN * 4, part = bytes / 4;
            mbar_expect_tx(fixbar, bytes);
            const float* src = sk.ws + static_cast<std::int64_t>(cta) * (128 * BN);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                      su32(smem + j * part)),
                  "l"(reinterpret_cast<std::uint64_t>(src) + j * part), "r"(part), "r"(su32(fixbar))
                  : "memory");
          }
          mbar_wait(fixbar, 0);  // used once per kernel: a CTA owns at most one split tail tile
        }
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          std::uint32_t r[16];
          tmem_ld16(tmem + buf * BN + (static_cast<std::uint32_t>(q * 32) << 16) + c, r);
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
          if (owner) {
            const float4* s4 = reinterpret_cast<const float4*>(piece_s + ((c / 16) * 128 + row) * 16);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 x = s4[j];
              v[4 * j] += x.x;
              v[4 * j + 1] += x.y;
              v[4 * j + 2] += x.z;
              v[4 * j + 3] += x.w;
            }
          }
          epi_cols16(args, m, ntl * BN + c, v);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(tempty0 + buf * 8)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
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



int g_sms = 0;

StreamK streamk_for(cudaStream_t s);

// GemmArgs::streamk_ok: 0 never, 1 if enabled, 2 forced (tests).  The pair
// GEMM's split tail is on by default (C4: 42.3 -> 41.9 ms per iteration, A/B
// in profiles/r2q; IB2_NO_SPLIT_TAIL=1 turns it off); the decode GEMM's
// stream-K is opt-in (IB2_STREAMK=1; measured slower, profiles/r2o).
bool streamk_enabled(const GemmArgs& a, bool pair_tail = false) {
  static const bool sk_on = getenv("IB2_STREAMK") != nullptr, tail_on = getenv("IB2_NO_SPLIT_TAIL") == nullptr;
  return a.streamk_ok == 2 || (a.streamk_ok == 1 && (pair_tail ? tail_on : sk_on));
}

template <int BN>
void launch_tc_pair_bn(const GemmArgs& a, cudaStream_t s) {
  using L = PairSmem<BN>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  const std::int64_t a_rows = a.a_rows > 0 ? a.a_rows : (g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M);
  const CUtensorMap& ma = cached_map(a.a, a_rows, a.K, 128);
  const CUtensorMap& mw = cached_wmap(a.w, a.N, a.K, BN / 2);
  const int tiles = ((a.M + 255) / 256) * ((a.N + BN - 1) / BN);
  // Tiles that do not divide into whole rounds over the pairs: split tail
  // (PairSegs; compute stream only, see StreamK).
  static const bool no_streamk = getenv("IB2_NO_STREAMK") != nullptr;  // diagnostics
  // Only for long k loops (K >= 8192: the MLP-down projections), where it
  // measured +11..14 %; at K <= 5120 it is neutral to -6 % and tiny GEMMs pay
  // the hand-off latency (C0: 0.20 -> 0.44 ms per iteration).
  // IB2_PAIR_MAX (diagnostics): cap the persistent grid, leaving SMs to
  // kernels of another stream (split_batch experiments); no split tail then.
  static const int pair_cap = getenv("IB2_PAIR_MAX") ? atoi(getenv("IB2_PAIR_MAX")) : 0;
  const bool use_sk = streamk_enabled(a, true) && !no_streamk && tiles % (g_sms / 2) != 0 &&
                      (a.streamk_ok == 2 ? a.K / BK >= 2 : a.K / BK >= 128) && pair_cap == 0;
  const StreamK sk = use_sk ? streamk_for(s) : StreamK{nullptr, nullptr, 0};
  const int max_pairs = pair_cap > 0 ? std::min(pair_cap, g_sms / 2) : g_sms / 2;
  const int pairs = use_sk ? g_sms / 2 : std::max(1, std::min(max_pairs, tiles));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  IB2_CUDA(cudaLaunchKernelEx(&cfg, tc_gemm_pair_kernel<BN>, ma, mw, a, sk));
}

int g_force_pair_bn = 0;  // isim_debug_gemm flags 4 / 8: force the 128 / 256 tile width

// Tile width.  256 x 256 always: the 256 x 128 tile was meant to cut wave
// quantisation (N = 5120 at M ~ 1200: 100 wide tiles on 74 pairs = 2 rounds,
// 68 % busy) but measured 30-45 % slower per GEMM on every 13B projection at
// M = 600 / 1218 / 2048 (profiles/r2g/gemm_tile_width.txt) -- a 256 x 128 k
// step halves the MMA work but not the per-stage barrier / TMA cost.  It stays
// selectable for tests (isim_debug_gemm flag 4) and diagnostics (IB2_PAIR_BN).
void launch_tc_pair(const GemmArgs& a, cudaStream_t s) {
  static const int env_force = getenv("IB2_PAIR_BN") ? atoi(getenv("IB2_PAIR_BN")) : 0;  // diagnostics
  const int force = g_force_pair_bn ? g_force_pair_bn : env_force;
  if (force == 128) launch_tc_pair_bn<128>(a, s);
  else launch_tc_pair_bn<256>(a, s);
}

// Work split of a decode-sized GEMM: clusters of S CTAs (K-slices) over T
// tiles each, chosen so the per-CTA weight stream ceil(tiles / clusters) *
// kblocks / S is smallest (ties: smaller S), one CTA per SM.
struct SplitPlan {
  int S, clusters;
};
// Clusters are placed within a GPC, so fewer than SMs / S clusters of S
// CTAs may be co-resident: ask the occupancy API (cached per kernel and S).
template <typename Kernel>
int max_clusters(Kernel kernel, int S, int smem) {
  static std::mutex mu;
  static std::unordered_map<long long, int> cache;
  const long long key = (reinterpret_cast<long long>(reinterpret_cast<const void*>(kernel)) << 4) ^ S;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g_sms / S * S);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = g_sms / S;
  }
  cache.emplace(key, n);
  return n;
}

// Many tiles (more than fit as 2-CTA clusters): whole tiles, one CTA per SM
// (more CTAs than that do not raise the weight stream rate).  Few tiles: one
// tile per cluster, the largest S <= 4 whose clusters are all co-resident.
template <typename Kernel>
SplitPlan plan_split(Kernel kernel, int smem, int tiles, int kblocks, bool split_ok) {
  if (!split_ok || tiles > max_clusters(kernel, 2, smem)) return {1, std::min(g_sms, tiles)};
  int S = 1;
  for (int s = 2; s <= 4; ++s)
    if (kblocks / s >= 4 && tiles <= max_clusters(kernel, s, smem)) S = s;
  return {S, tiles};
}

// Stream-K workspace, one per stream (GEMMs on different streams may run
// concurrently): a piece slot per CTA + its epoch flag.
StreamK streamk_for(cudaStream_t s) {
  struct Ws {
    float* ws = nullptr;
    std::int32_t* flags = nullptr;
    std::int32_t epoch = 0;
  };
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, Ws> pool;
  std::lock_guard<std::mutex> g(mu);
  Ws& w = pool[s];
  if (!w.ws) {
    IB2_CUDA(cudaMalloc(&w.ws, static_cast<std::size_t>(g_sms) * 256 * BM * sizeof(float)));
    IB2_CUDA(cudaMalloc(&w.flags, static_cast<std::size_t>(g_sms) * sizeof(std::int32_t)));
    IB2_CUDA(cudaMemset(w.flags, 0, static_cast<std::size_t>(g_sms) * sizeof(std::int32_t)));
  }
  w.epoch = w.epoch == 0x7fffffff ? 1 : w.epoch + 1;
  return StreamK{w.ws, w.flags, w.epoch};
}

template <int NT, int STAGES>
void launch_skinny(const GemmArgs& a, cudaStream_t s) {
  using L = SkSmem<NT, STAGES>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(tc_splitk_kernel<NT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    IB2_CUDA(cudaFuncSetAttribute(tc_splitk_kernel<NT, STAGES>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  const int tiles = static_cast<int>((a.N + BM - 1) / BM), kblocks = a.K / BK;
  static const int force_s = getenv("IB2_SPLIT_S") ? atoi(getenv("IB2_SPLIT_S")) : 0;  // diagnostics
  SplitPlan sp = plan_split(tc_splitk_kernel<NT, STAGES>, L::TOTAL, tiles, kblocks, L::SPLIT_OK);
  if (force_s > 0 && L::SPLIT_OK)
    sp = {force_s, std::max(1, std::min(max_clusters(tc_splitk_kernel<NT, STAGES>, force_s, L::TOTAL), tiles))};
  static const bool verbose = getenv("IB2_SPLIT_VERBOSE") != nullptr;
  // Whole tiles that do not fill the SMs evenly: stream-K over every SM.
  static const bool no_streamk = getenv("IB2_NO_STREAMK") != nullptr;  // diagnostics
  // Owners spin on pieces of later CTAs, so two stream-K GEMMs must never run
  // concurrently (each could hold SMs the other's pieces need): the executor
  // allows it on its compute stream only.  Opt-in (streamk_enabled): measured
  // per GEMM (profiles/r2o/streamk_per_gemm.txt) it wins on a few shapes
  // (GPT-J QKV at M = 32: +9 %) and loses on more (M = 108: -14..-26 %), and
  // C4 end to end ran 2.3 % slower with it.
  const bool use_sk = NT <= 128 && streamk_enabled(a) && sp.S == 1 && !no_streamk && tiles % g_sms != 0 &&
                      kblocks >= 2;
  StreamK sk{nullptr, nullptr, 0};
  if (use_sk) {
    sk = streamk_for(s);
    // at least kblocks / 2 units per CTA: a tile spans at most 3 CTAs (<= 2 pieces)
    sp.clusters = static_cast<int>(std::min<long long>(g_sms, (2LL * tiles * kblocks) / std::max(1, kblocks)));
  }
  if (verbose)
    fprintf(stderr, "splitk N=%d K=%d M=%d: S=%d clusters=%d%s\n", a.N, a.K, a.M, sp.S, sp.clusters,
            use_sk ? " stream-K" : "");
  const std::int64_t a_rows = a.a_rows > 0 ? a.a_rows : (g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M);
  const CUtensorMap& mw = cached_wmap(a.w, a.N, a.K, BM);
  const CUtensorMap& ma = cached_map(a.a, a_rows, a.K, NT);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sp.clusters * sp.S);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = sp.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  IB2_CUDA(cudaLaunchKernelEx(&cfg, tc_splitk_kernel<NT, STAGES>, mw, ma, a, sp.S, sk));
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
  // (Deeper weight rings -- 11 / 9 stages for M <= 16 / 32 -- measured
  // identical per GEMM: the ring is not what limits the weight stream.)
  if (a.M <= 16) launch_skinny<16, 10>(a, s);
  else if (a.M <= 32) launch_skinny<32, 8>(a, s);
  else if (a.M <= 64) launch_skinny<64, 6>(a, s);
  else if (a.M <= 128) launch_skinny<128, 5>(a, s);
  else if ((a.N + BM - 1) / BM * 2 <= g_sms && a.epi != Epi::QkvRopeKv) {
    // Few weight tiles (O-proj, MLP-out) and 129..256 tokens: the NT = 256
    // variant has no room for split-K partials and would run one CTA per tile
    // (32 of 148 SMs); two NT = 128 passes re-read the weights but use every SM.
    const std::int64_t cap = g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M;
    for (int m0 = 0; m0 < a.M; m0 += 128) {
      GemmArgs c = a;
      c.M = std::min(128, a.M - m0);
      c.a = a.a + static_cast<std::int64_t>(m0) * a.K;
      c.a_rows = (a.a_rows > 0 ? a.a_rows : cap) - m0;
      if (c.out) c.out = a.out + static_cast<std::int64_t>(m0) * a.ldo;
      if (c.outf) c.outf = a.outf + static_cast<std::int64_t>(m0) * a.ldf;
      if (c.addf) c.addf = a.addf + static_cast<std::int64_t>(m0) * a.ldf;
      launch_skinny<128, 5>(c, s);
    }
  } else {
    launch_skinny<256, 4>(a, s);
  }
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

void launch_gemm(const GemmArgs& a_in, cudaStream_t s) {
  if (a_in.M <= 0) return;
  static const bool no_early = getenv("IB2_NO_EARLY_W") != nullptr;  // diagnostics
  GemmArgs a = a_in;
  a.no_early_w = no_early ? 1 : 0;
  if (a.K % BK != 0 || a.N % 2 != 0) {  // N tails are masked; K must fill whole 64-wide blocks
    launch_gemm_simt(a, s);
    return;
  }
  if (skinny_ok(a)) {
    launch_skinny_any(a, s);
    return;
  }
  // M > 256: tensor-core bound, CTA-pair 256x256 tiles.
  if (!g_sms) {
    int dev = 0;
    IB2_CUDA(cudaGetDevice(&dev));
    IB2_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  launch_tc_pair(a, s);
}

void debug_tile_weights(const void* src, void* dst, int N, int K, void* stream) {
  if (K % BK) throw DeviceError("debug_tile_weights: K must be a multiple of 64");
  launch_tile_weights(static_cast<const f16*>(src), static_cast<f16*>(dst), N, K, static_cast<cudaStream_t>(stream));
}

void debug_gemm(const void* a, const void* w, int M, int N, int K, int epi, const void* bias, void* out, int ldo,
                void* outf, int ldf, int flags, void* stream) {
  const bool force_simt = flags & 1;
  g_force_pair_bn = (flags & 4) ? 128 : (flags & 8) ? 256 : 0;
  const int streamk_ok = (flags & 16) ? 0 : (flags & 32) ? 2 : 1;
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
  g.streamk_ok = streamk_ok;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const std::int64_t saved = g_a_rows_capacity;
  g_a_rows_capacity = 0;  // caller buffers are exactly M rows
  if (force_simt) launch_gemm_simt(g, s);
  else launch_gemm(g, s);
  g_a_rows_capacity = saved;
  g_force_pair_bn = 0;
}

}  // namespace ib2
