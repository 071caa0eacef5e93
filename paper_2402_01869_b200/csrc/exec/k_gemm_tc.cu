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
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
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

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        unsigned char* sa = smem + s * L::STAGE_BYTES;
        unsigned char* sb = sa + L::A_BYTES;
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        tma_load_2d(sa, &map_a, &full[s], kb * BK, m0);
        tma_load_2d(sb, &map_w, &full[s], kb * BK, n0);
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


// ---- small-M path: swap-AB + deterministic split-K ---------------------------
//
// Decode-dominated iterations have M (tokens) of 8..256 while N x K weights are
// 17-134 MB per projection: the GEMM is a weight stream.  Computing C^T = W A^T
// puts 128 weight rows on the UMMA M side (TMEM lanes) and the few tokens on
// the UMMA N side (NT columns), so every weight byte is read once and the
// token tile (NT x 64 per stage) is tiny.  Grid = (N/128 weight tiles) x
// (K splits) sized to ~2 CTAs per SM; each split writes fp32 partials and the
// last CTA of a tile (atomic ticket) reduces them in split order -- a fixed
// order, so results are deterministic -- then applies the fused epilogue.

template <int NT, int STAGES>
struct SkSmem {
  static constexpr int A_BYTES = BM * BK * 2;  // weights tile
  static constexpr int B_BYTES = NT * BK * 2;  // tokens tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 1) * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = NT < 32 ? 32 : NT;
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

// Epilogue for one weight row n (this lane) over tokens; SwiGLU pairs come
// from the neighbouring lane (gate = even row, up = odd row).
__device__ __forceinline__ void epi_row(const GemmArgs& a, int n, int m, float v, int lane) {
  if (a.epi == Epi::SwiGluF16) {
    const float up = __shfl_down_sync(0xffffffffu, v, 1);
    if (!(lane & 1) && m < a.M && n < a.N)
      a.out[static_cast<std::int64_t>(m) * a.ldo + n / 2] = __float2half_rn(silu(v) * up);
    return;
  }
  if (m < a.M && n < a.N) epi_one(a, m, n, v);
}

template <int NT, int STAGES>
__global__ void __launch_bounds__(256, 1) tc_skinny_kernel(const __grid_constant__ CUtensorMap map_w,
                                                           const __grid_constant__ CUtensorMap map_a, GemmArgs args,
                                                           float* __restrict__ ws, std::int32_t* __restrict__ tickets) {
  using L = SkSmem<NT, STAGES>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L::BAR_OFF);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* done = empty + STAGES;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(done + 1);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BM;
  const int split = blockIdx.y, splits = gridDim.y;
  const int nk = args.K / BK;
  const int kb0 = split * nk / splits, kb1 = (split + 1) * nk / splits;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&map_a)) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
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

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0; kb < kb1; ++kb) {
        const int i = kb - kb0, st = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[st], ((i / STAGES) - 1) & 1);
        unsigned char* sw = smem + st * L::STAGE_BYTES;
        mbar_expect_tx(&full[st], L::STAGE_BYTES);
        tma_load_2d(sw, &map_w, &full[st], kb * BK, n0);
        tma_load_2d(sw + L::A_BYTES, &map_a, &full[st], kb * BK, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = (1u << 4) | (static_cast<std::uint32_t>(NT >> 3) << 17) |
                                      (static_cast<std::uint32_t>(BM >> 4) << 24);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int i = kb - kb0, st = i % STAGES;
        mbar_wait(&full[st], (i / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const unsigned char* sw = smem + st * L::STAGE_BYTES;
        const std::uint64_t da = smem_desc(sw), db = smem_desc(sw + L::A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / UMMA_K; ++k) {
          const std::uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          asm volatile(
              "{\n"
              ".reg .pred p;\n"
              "setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
              "}\n" ::"r"(tmem),
              "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&empty[st]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(done))
                   : "memory");
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    const int n = n0 + q * 32 + lane;  // this lane's weight row
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    float* part = ws + (static_cast<std::int64_t>(split) * args.M) * args.N;
#pragma unroll 1
    for (int c = 0; c < NT; c += 16) {
      if (c >= args.M) break;
      std::uint32_t r[16];
      const std::uint32_t taddr = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = c + j;
        const float v = __uint_as_float(r[j]);
        if (splits == 1) epi_row(args, n, m, v, lane);
        else if (m < args.M && n < args.N) part[static_cast<std::int64_t>(m) * args.N + n] = v;
      }
    }
    if (splits > 1) {
      __threadfence();
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (q == 0 && lane == 0) {
        const int prev = atomicAdd(&tickets[blockIdx.x], 1);
        s_last = prev == splits - 1;
        if (s_last) tickets[blockIdx.x] = 0;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (s_last) {
        __threadfence();
        for (int m = 0; m < args.M; ++m) {
          float v = 0.f;
          if (n < args.N)
            for (int sp = 0; sp < splits; ++sp)
              v += __ldcg(ws + (static_cast<std::int64_t>(sp) * args.M + m) * args.N + n);
          epi_row(args, n, m, v, lane);
        }
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

const CUtensorMap& cached_map(const void* base, std::int64_t rows, int K, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  std::lock_guard<std::mutex> g(mu);
  const MapKey key{base, rows, K, box_rows};
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, make_map(base, rows, K, K, box_rows)).first;
  return it->second;
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
  const CUtensorMap& mw = cached_map(a.w, a.N, a.K, BN);
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  tc_gemm_kernel<BN, STAGES><<<grid, 256, L::TOTAL, s>>>(ma, mw, a);
  IB2_LAUNCH_CHECK();
}


float* g_ws = nullptr;
std::int32_t* g_tickets = nullptr;
std::size_t g_ws_bytes = 0;
int g_ws_device = -1;

template <int NT, int STAGES>
void launch_skinny(const GemmArgs& a, int splits, cudaStream_t s) {
  using L = SkSmem<NT, STAGES>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(tc_skinny_kernel<NT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  const std::int64_t a_rows = g_a_rows_capacity > a.M ? g_a_rows_capacity : a.M;
  const CUtensorMap& mw = cached_map(a.w, a.N, a.K, BM);
  const CUtensorMap& ma = cached_map(a.a, a_rows, a.K, NT);
  tc_skinny_kernel<NT, STAGES><<<dim3((a.N + BM - 1) / BM, splits), 256, L::TOTAL, s>>>(mw, ma, a, g_ws, g_tickets);
  IB2_LAUNCH_CHECK();
}

// Choose the split so that ~2 CTAs land on every SM, keeping >= 4 K blocks
// per split, and make sure the fp32 partial workspace is large enough.
int skinny_splits(const GemmArgs& a) {
  const int tiles = (a.N + BM - 1) / BM, kblocks = a.K / BK;
  int sp = (2 * 148 + tiles - 1) / tiles;
  sp = std::max(1, std::min({sp, kblocks / 4, 16}));
  const std::size_t need = static_cast<std::size_t>(sp) * a.M * a.N * 4;
  int dev = 0;
  IB2_CUDA(cudaGetDevice(&dev));
  if (sp > 1 && (need > g_ws_bytes || dev != g_ws_device)) {
    if (g_ws) cudaFree(g_ws);
    if (!g_tickets || dev != g_ws_device) {
      IB2_CUDA(cudaMalloc(&g_tickets, 65536 * 4));
      IB2_CUDA(cudaMemset(g_tickets, 0, 65536 * 4));
    }
    g_ws_bytes = std::max<std::size_t>(need, 64u << 20);
    IB2_CUDA(cudaMalloc(&g_ws, g_ws_bytes));
    g_ws_device = dev;
  }
  return sp;
}

bool skinny_ok(const GemmArgs& a) {
  static const bool off = getenv("IB2_NO_SKINNY") != nullptr;
  return !off && a.M <= 256 && a.K % BK == 0 && a.N % 2 == 0 && (a.N + BM - 1) / BM <= 65536;
}

void launch_skinny_any(const GemmArgs& a, cudaStream_t s) {
  const int sp = skinny_splits(a);
  if (a.M <= 16) launch_skinny<16, 8>(a, sp, s);
  else if (a.M <= 32) launch_skinny<32, 8>(a, sp, s);
  else if (a.M <= 64) launch_skinny<64, 8>(a, sp, s);
  else if (a.M <= 128) launch_skinny<128, 6>(a, sp, s);
  else launch_skinny<256, 4>(a, sp, s);
}

}  // namespace

void set_gemm_activation_rows(std::int64_t rows) { g_a_rows_capacity = rows; }

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

void debug_gemm(const void* a, const void* w, int M, int N, int K, int epi, const void* bias, void* out, int ldo,
                void* outf, int ldf, bool force_simt, void* stream) {
  GemmArgs g{static_cast<const f16*>(a), static_cast<const f16*>(w), M, N, K, static_cast<Epi>(epi),
             static_cast<const f16*>(bias), static_cast<f16*>(out), ldo, static_cast<float*>(outf), ldf};
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const std::int64_t saved = g_a_rows_capacity;
  g_a_rows_capacity = 0;  // caller buffers are exactly M rows
  if (force_simt) launch_gemm_simt(g, s);
  else launch_gemm(g, s);
  g_a_rows_capacity = saved;
  IB2_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ib2
