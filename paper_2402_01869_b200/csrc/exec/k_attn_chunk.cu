// K2: chunk attention (prefill / recompute / API-returned tokens) over the
// paged prefix on 5th-generation tensor cores.
//
// One CTA = one work item: a tile of up to 128 consecutive query rows of one
// request, one head, restricted to keys [kv_lo, kv_hi) (split-KV).  Flash
// attention with both contractions on tcgen05 and the accumulators in TMEM:
//
//   warp 0      TMA producer: the Q tile once ([128][hd] from the qkv
//               activations), then per key tile the K and V rows of BN/16 paged
//               blocks ([16][hd] each, contiguous in the pool) into a 2-stage
//               ring, 128-byte swizzle (64-key tiles);
//   warp 1      MMA issuer: S_t = Q K_t^T (M=128, N=BN, K=hd; both operands
//               K-major) into one of two TMEM S buffers, then O += P_{t-1} V_{t-1}
//               (M=128, N=hd, K=BN; P K-major from shared memory, V MN-major
//               straight from the TMA tile) -- S_t overlaps softmax(t-1);
//   warps 2-5   softmax (warp 2 also allocates TMEM: O = hd, S = 2 x BN
//               columns): thread = query row = TMEM lane.  Row max / exp2 / sum
//               are thread-local (no shuffles); P is written f16 into swizzled
//               shared memory; O is rescaled in TMEM only when the running max
//               grew by more than 2^8 (the exact max used is tracked, so the
//               final normalisation is exact); epilogue O / l -> f16 output, or
//               an fp32 partial (O, m, l) for the combine kernel.
//
// Keys are visited in ascending block order, like K1.  Tensor-core
// bound: 4 * rows * keys * hd FLOP per (item, head).
#include <cfloat>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace ib2 {

namespace {

using namespace tc;

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O when the max grew by > 2^8
// Six warps: 0 TMA producer, 1 MMA issuer, 2-5 softmax (2 also allocates
// TMEM).  192 threads x <= 128 registers lets two CTAs share an SM's 64K
// registers (256 threads did not: 1 resident CTA).
constexpr int kK2Threads = 192;

// Head dims 64 / 128 run two CTAs per SM (64-key tiles, 256 TMEM columns
// and <= 113 KB of shared memory each; head dim 128 with one P buffer): the
// two CTAs' softmax warps interleave on the SM while either one's MMAs run,
// which one CTA's four softmax warps cannot keep busy.  Head dim 256 (O alone
// takes 256 columns) keeps one CTA per SM with 64-key tiles.
template <int HD>
struct AttnCfg {
  static constexpr int BQ = 128;
  static constexpr int BN = 64;                     // keys per tile
  static constexpr int CTAS = HD == 256 ? 1 : 2;    // resident CTAs per SM
  static constexpr int NP = HD == 128 ? 1 : 2;      // P buffers
  static constexpr int NCH = HD / 64;               // 64-wide head-dim chunks (one 128 B swizzle row)
  static constexpr int STAGES = 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BN * HD * 2;  // K or V tile
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int P_BYTES = BQ * BN * 2;  // one P buffer
  static constexpr int KV_OFF = Q_BYTES;
  static constexpr int P_OFF = KV_OFF + STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = P_OFF + NP * P_BYTES;
  // Barriers + alignment slack.  Two CTAs per SM must fit in 228 KB minus
  // 1 KB reserved per CTA (115,712 B each): the slack assumes the dynamic
  // shared window starts at least 512 B aligned (checked in the kernel).
  static constexpr int SLACK = 512;
  static constexpr int TOTAL = BAR_OFF + 256 + SLACK;
  static constexpr int TMEM_COLS = CTAS == 2 ? 256 : 512;
  static constexpr int S_COL = HD;  // S buffers after O
  static_assert(HD + 2 * BN <= TMEM_COLS, "TMEM budget");
  static_assert(CTAS == 1 ? TOTAL <= 232448 : TOTAL <= 115712, "shared memory budget");
};

template <int HD>
__global__ void __launch_bounds__(kK2Threads, AttnCfg<HD>::CTAS) chunk_attn_tc_kernel(const __grid_constant__ CUtensorMap map_q,
                                                               const __grid_constant__ CUtensorMap map_kv,
                                                               const TileDesc* __restrict__ items,
                                                               const std::int32_t* __restrict__ table, int max_lb,
                                                               std::int64_t layer_row0, int H,
                                                               f16* __restrict__ out, float* __restrict__ ws_o,
                                                               float* __restrict__ ws_ml) {
  using C = AttnCfg<HD>;
  constexpr int BQ = C::BQ, BN = C::BN, NCH = C::NCH, STAGES = C::STAGES, NP = C::NP;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + C::BAR_OFF);
  std::uint64_t* qfull = bars;              // 1
  std::uint64_t* kfull = bars + 1;          // [STAGES] K half of a stage landed
  std::uint64_t* kempty = kfull + STAGES;   // [STAGES] S MMA done with it
  std::uint64_t* vfull = kempty + STAGES;   // [STAGES] V half landed
  std::uint64_t* vempty = vfull + STAGES;   // [STAGES] PV MMA done with it
  std::uint64_t* sfull = vempty + STAGES;   // [2]
  std::uint64_t* sfree = sfull + 2;         // [2]
  std::uint64_t* pfull = sfree + 2;         // [NP] P buffer written (4 warps)
  std::uint64_t* pvdone = pfull + 2;        // [NP] PV MMA of that P buffer done
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(pvdone + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;  // heads fastest: CTAs issue item by item (items are longest first)
  if (threadIdx.x == 0 && smem - smem_raw > C::SLACK) __trap();  // layout would overrun the allocation

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_q);
    prefetch_map(&map_kv);
    mbar_init(qfull, 1);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 4);  // one arrival per softmax warp
      mbar_init(&pfull[i], 4);
      mbar_init(&pvdone[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  fence_before();
  __syncthreads();
  fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // qkv, pool and block tables come from earlier kernels of this iteration
  items = after_wait(items);
  table = after_wait(table);

  const TileDesc td = items[blockIdx.y];
  const int last_pos = td.pos0 + td.nrows - 1;
  const int kv_hi = min(td.kv_hi, last_pos + 1);
  const int kt0 = td.kv_lo / BN;
  const int nt = (kv_hi + BN - 1) / BN - kt0;
  unsigned char* sQ = smem;
  unsigned char* sKV = smem + C::KV_OFF;
  unsigned char* sP = smem + C::P_OFF;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qfull, C::Q_BYTES);
#pragma unroll
      for (int j = 0; j < NCH; ++j) tma_load_2d(sQ + j * BQ * 128, &map_q, qfull, h * HD + 64 * j, td.row0);
      const std::int32_t* tab = table + static_cast<std::int64_t>(td.slot) * max_lb;
      const int lb_last = (kv_hi - 1) / kBlockTokens;
      // K runs one tile ahead of V: K(t) is released by S(t), V(t) only by PV(t).
      auto load = [&](int t, int kv) {
        const int st = t % STAGES;
        std::uint64_t* full = kv ? &vfull[st] : &kfull[st];
        if (t >= STAGES) mbar_wait(kv ? &vempty[st] : &kempty[st], ((t / STAGES) - 1) & 1);
        mbar_expect_tx(full, C::KV_BYTES);
        unsigned char* dst = sKV + st * C::STAGE_BYTES + kv * C::KV_BYTES;
#pragma unroll 1
        for (int b = 0; b < BN / kBlockTokens; ++b) {
          // Blocks past the key range re-load the last valid block (finite
          // values; their scores are masked to -inf, so P = 0 there).
          const int lb = min((kt0 + t) * (BN / kBlockTokens) + b, lb_last);
          const std::int64_t pb = tab[lb];
          const int row = static_cast<int>(layer_row0 + (pb * 2 + kv) * H * kBlockTokens + h * kBlockTokens);
#pragma unroll
          for (int j = 0; j < NCH; ++j)
            tma_load_2d(dst + j * BN * 128 + b * kBlockTokens * 128, &map_kv, full, 64 * j, row);
        }
      };
      load(0, 0);
      for (int t = 0; t < nt; ++t) {
        if (t + 1 < nt) load(t + 1, 0);
        load(t, 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc_s = idesc_f16(BQ, BN, false, false);
      constexpr std::uint32_t idesc_pv = idesc_f16(BQ, HD, false, true);
      const std::uint32_t q_base = su32(sQ), kv_base = su32(sKV), p_base = su32(sP);
      auto issue_pv = [&](int u) {
        const int pb = u % NP, st = u % STAGES;
        mbar_wait(&pfull[pb], (u / NP) & 1);
        mbar_wait(&vfull[st], (u / STAGES) & 1);
        fence_after();
        const std::uint32_t v_base = kv_base + st * C::STAGE_BYTES + C::KV_BYTES;
        const std::uint32_t pbuf = p_base + pb * C::P_BYTES;
#pragma unroll
        for (int k = 0; k < BN / 16; ++k) {
          const std::uint64_t da = desc_sw128(pbuf + (k / 4) * BQ * 128 + (k % 4) * 32, 16, 1024);
          const std::uint64_t db = desc_sw128(v_base + k * 16 * 128, BN * 128, 1024);
          mma_f16(tmem, da, db, idesc_pv, (u > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&pvdone[pb]);
        mma_commit(&vempty[st]);
      };
      mbar_wait(qfull, 0);
      for (int t = 0; t < nt; ++t) {
        const int st = t % STAGES, b = t & 1;
        mbar_wait(&kfull[st], (t / STAGES) & 1);
        if (t >= 2) mbar_wait(&sfree[b], ((t / 2) - 1) & 1);
        fence_after();
        const std::uint32_t k_base = kv_base + st * C::STAGE_BYTES;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const std::uint64_t da = desc_sw128(q_base + (k / 4) * BQ * 128 + (k % 4) * 32, 16, 1024);
          const std::uint64_t db = desc_sw128(k_base + (k / 4) * BN * 128 + (k % 4) * 32, 16, 1024);
          mma_f16(tmem + C::S_COL + b * BN, da, db, idesc_s, k > 0 ? 1u : 0u);
        }
        mma_commit(&sfull[b]);
        mma_commit(&kempty[st]);
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(nt - 1);
    }
  } else {
    // warps 2-5: TMEM lane quarter = warp % 4 (a warp reaches only lanes
    // 32 * (warp % 4) .. + 31), so the four quarters are 2, 3, 0, 1.
    const int q = warp & 3;
    const int r = q * 32 + lane;  // query row of this thread = TMEM lane
    const std::uint32_t lane_off = static_cast<std::uint32_t>(q * 32) << 16;
    const int qp = td.pos0 + min(r, td.nrows - 1);
    const float sc = rsqrtf(static_cast<float>(HD)) * kLog2e;
    float m_used = -FLT_MAX;  // max the exponentials are taken against (log2 units)
    float l = 0.f;
    for (int t = 0; t < nt; ++t) {
      const int b = t & 1;
      mbar_wait(&sfull[b], (t / 2) & 1);
      fence_after();
      float s[BN];
      {
        std::uint32_t raw[BN];
#pragma unroll
        for (int c = 0; c < BN; c += 16) tmem_ld16_nowait(tmem + lane_off + C::S_COL + b * BN + c, raw + c);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < BN; ++i) s[i] = __uint_as_float(raw[i]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[b]);

      const int k0 = (kt0 + t) * BN;
      float mx = -FLT_MAX;
      if (k0 >= td.kv_lo && k0 + BN <= kv_hi && k0 + BN - 1 <= qp) {  // whole tile visible to this row
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          s[i] *= sc;
          mx = fmaxf(mx, s[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const int kp = k0 + i;
          const bool ok = kp >= td.kv_lo && kp < kv_hi && kp <= qp;
          s[i] = ok ? s[i] * sc : -FLT_MAX;
          mx = fmaxf(mx, s[i]);
        }
      }
      float factor = 1.f;
      bool rescale = false;
      if (mx > -FLT_MAX) {
        if (m_used == -FLT_MAX) {
          m_used = mx;  // O holds only zero contributions so far
        } else if (mx > m_used + kRescaleThreshold) {
          factor = exp2f(m_used - mx);
          m_used = mx;
          rescale = true;
        }
      }
      l *= factor;
      // P = exp2(s - m_used) rounded to f16; the row sum uses the same rounded
      // values so numerator and denominator agree.
      std::uint32_t pk[BN / 2];
      // ex2.approx.ftz: masked scores (-FLT_MAX) give 0; results below 2^-126
      // flush to 0, as f16 rounding (smallest subnormal 2^-24) would anyway.
      // A row with nothing visible yet (m_used = -FLT_MAX) contributes 0.
      const float mrow = m_used == -FLT_MAX ? FLT_MAX : m_used;
#pragma unroll
      for (int i = 0; i < BN; i += 2) {
        const float e0 = ex2_approx(s[i] - mrow);
        const float e1 = ex2_approx(s[i + 1] - mrow);
        const __half2 hv = __floats2half2_rn(e0, e1);
        const float2 back = __half22float2(hv);
        l += back.x + back.y;
        pk[i / 2] = *reinterpret_cast<const std::uint32_t*>(&hv);
      }
      // P buffer t%NP is free once PV(t-NP) retired; O may only be rescaled
      // after PV(t-1) (which accumulates into it) and before PV(t).
      const int pbuf = t % NP;
      if (t >= NP) mbar_wait(&pvdone[pbuf], ((t - NP) / NP) & 1);
      if (__any_sync(0xffffffffu, rescale)) {
        if (t >= 1) mbar_wait(&pvdone[(t - 1) % NP], ((t - 1) / NP) & 1);
        fence_after();
#pragma unroll 1
        for (int c = 0; c < HD; c += 16) {
          std::uint32_t o[16];
          tmem_ld16_nowait(tmem + lane_off + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
          tmem_st16(tmem + lane_off + c, o);
        }
        tmem_wait_st();
      }
      // P row -> shared memory, K-major 128 B swizzle: 16 B unit u of row r
      // lands at unit u ^ (r & 7) of the row's 128 B line.
      unsigned char* pdst = sP + pbuf * C::P_BYTES;
#pragma unroll
      for (int u = 0; u < BN / 8; ++u) {
        const int ch = u / 8, uu = u % 8;
        uint4 v;
        v.x = pk[u * 4 + 0];
        v.y = pk[u * 4 + 1];
        v.z = pk[u * 4 + 2];
        v.w = pk[u * 4 + 3];
        *reinterpret_cast<uint4*>(pdst + ch * BQ * 128 + r * 128 + ((uu ^ (r & 7)) * 16)) = v;
      }
      fence_proxy_async();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[pbuf]);
    }
    // Epilogue.
    mbar_wait(&pvdone[(nt - 1) % NP], ((nt - 1) / NP) & 1);
    fence_after();
    if (td.part < 0) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      f16* dst = out + static_cast<std::int64_t>(td.row0 + r) * H * HD + h * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 16) {
        std::uint32_t o[16];
        tmem_ld16_nowait(tmem + lane_off + c, o);
        tmem_wait_ld();
        if (r < td.nrows) {
          uint4 v[2];
          std::uint32_t* w = reinterpret_cast<std::uint32_t*>(v);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const __half2 hv = __floats2half2_rn(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
            w[i] = *reinterpret_cast<const std::uint32_t*>(&hv);
          }
          *reinterpret_cast<uint4*>(dst + c) = v[0];
          *reinterpret_cast<uint4*>(dst + c + 8) = v[1];
        }
      }
    } else {
      const std::int64_t slot = (static_cast<std::int64_t>(td.part) * H + h) * BQ + r;
      float* dst = ws_o + slot * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 16) {
        std::uint32_t o[16];
        tmem_ld16_nowait(tmem + lane_off + c, o);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(dst + c + i) = make_float4(__uint_as_float(o[i]), __uint_as_float(o[i + 1]),
                                                                __uint_as_float(o[i + 2]), __uint_as_float(o[i + 3]));
      }
      ws_ml[slot * 2] = m_used;
      ws_ml[slot * 2 + 1] = l;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Merge the split-KV partials of one q-tile: one warp per (row, head); the
// lanes own hd/32 consecutive columns.
__global__ void __launch_bounds__(256) chunk_combine_kernel(const CombineDesc* __restrict__ cds, int H, int HD,
                                                            const float* __restrict__ ws_o,
                                                            const float* __restrict__ ws_ml, f16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const CombineDesc c = cds[blockIdx.x];
  const int h = blockIdx.y;
  const int r = blockIdx.z * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= c.nrows) return;
  float M = -FLT_MAX;
  for (int p = 0; p < c.nparts; ++p)
    M = fmaxf(M, ws_ml[((static_cast<std::int64_t>(c.part0 + p) * H + h) * kChunkTileRows + r) * 2]);
  const int per = HD / 32;  // 2, 4 or 8 columns per lane
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float L = 0.f;
  for (int p = 0; p < c.nparts; ++p) {
    const std::int64_t slot = (static_cast<std::int64_t>(c.part0 + p) * H + h) * kChunkTileRows + r;
    const float m = ws_ml[slot * 2];
    const float w = m == -FLT_MAX ? 0.f : exp2f(m - M);
    L += ws_ml[slot * 2 + 1] * w;
    const float* src = ws_o + slot * HD + lane * per;
    for (int i = 0; i < per; ++i) acc[i] += src[i] * w;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  f16* dst = out + static_cast<std::int64_t>(c.row0 + r) * H * HD + h * HD + lane * per;
  for (int i = 0; i < per; ++i) dst[i] = __float2half_rn(acc[i] * inv);
}

// Tensor maps are cached per (base, extent, geometry): executors created later
// may reuse a freed buffer address with a different shape.
const CUtensorMap& cached_tmap(const void* base, std::int64_t inner, std::int64_t rows, int box_rows) {
  struct Key {
    const void* p;
    std::int64_t inner, rows;
    int box;
    bool operator==(const Key& o) const { return p == o.p && inner == o.inner && rows == o.rows && box == o.box; }
  };
  struct Hash {
    std::size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.p) ^ (static_cast<std::size_t>(k.inner) << 20) ^
             (static_cast<std::size_t>(k.rows) * 0x9E3779B97F4A7C15ULL) ^ static_cast<std::size_t>(k.box);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  std::lock_guard<std::mutex> g(mu);
  const Key key{base, inner, rows, box_rows};
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, make_tmap_2d(base, inner, rows, inner * 2, 64, box_rows)).first;
  return it->second;
}

const CUtensorMap& q_map(const f16* qkv, int rows, int D) { return cached_tmap(qkv, 3LL * D, rows, 128); }

const CUtensorMap& kv_map(const KvGeom& g) {
  const std::int64_t rows = static_cast<std::int64_t>(g.layers) * g.num_blocks * 2 * g.heads * kBlockTokens;
  if (rows >= (1LL << 31)) throw DeviceError("KV pool too large for 32-bit TMA row coordinates");
  return cached_tmap(g.pool, g.head_dim, rows, kBlockTokens);
}

template <int HD>
void launch_chunk_hd(const f16* qkv, int qkv_rows, const TileDesc* items, int n_items, const KvGeom& g, int layer,
                     f16* out, float* ws_o, float* ws_ml, cudaStream_t s) {
  using C = AttnCfg<HD>;
  static bool configured = false;
  if (!configured) {
    IB2_CUDA(cudaFuncSetAttribute(chunk_attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL));
    // Two CTAs per SM need the whole 228 KB carve-out for shared memory.
    IB2_CUDA(cudaFuncSetAttribute(chunk_attn_tc_kernel<HD>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    // (cudaOccupancyMaxActiveBlocksPerMultiprocessor answers 1 for any kernel
    // that uses tcgen05.alloc, but the hardware co-schedules two such CTAs
    // per SM when their TMEM allocations fit: tools/occ/occ4.cu measured 148
    // of 148 SMs running two 256-column CTAs at once.)
    configured = true;
  }
  const std::int64_t layer_row0 = static_cast<std::int64_t>(layer) * g.num_blocks * 2 * g.heads * kBlockTokens;
  if (n_items > 65535) throw DeviceError("chunk attention: too many work items");
  launch_pdl(chunk_attn_tc_kernel<HD>, dim3(g.heads, n_items), dim3(kK2Threads), C::TOTAL, s, q_map(qkv, qkv_rows, g.heads * HD),
             kv_map(g), items, g.table, g.max_lblocks, layer_row0, g.heads, out, ws_o, ws_ml);
  IB2_LAUNCH_CHECK();
}

}  // namespace

int chunk_attention_ctas_per_sm(int head_dim) {
  switch (head_dim) {
    case 64: return AttnCfg<64>::CTAS;
    case 128: return AttnCfg<128>::CTAS;
    case 256: return AttnCfg<256>::CTAS;
    default: throw DeviceError("unsupported head_dim");
  }
}

int chunk_attention_key_tile(int head_dim) {
  switch (head_dim) {
    case 64: return AttnCfg<64>::BN;
    case 128: return AttnCfg<128>::BN;
    case 256: return AttnCfg<256>::BN;
    default: throw DeviceError("unsupported head_dim");
  }
}

void launch_chunk_attention(const f16* qkv, int qkv_rows, const TileDesc* items, int n_items,
                            const CombineDesc* combines, int n_combines, const KvGeom& g, int layer, f16* out,
                            float* ws_o, float* ws_ml, cudaStream_t s) {
  if (n_items <= 0) return;
  switch (g.head_dim) {
    case 64: launch_chunk_hd<64>(qkv, qkv_rows, items, n_items, g, layer, out, ws_o, ws_ml, s); break;
    case 128: launch_chunk_hd<128>(qkv, qkv_rows, items, n_items, g, layer, out, ws_o, ws_ml, s); break;
    case 256: launch_chunk_hd<256>(qkv, qkv_rows, items, n_items, g, layer, out, ws_o, ws_ml, s); break;
    default: throw DeviceError("unsupported head_dim");
  }
  if (n_combines > 0) {
    launch_pdl(chunk_combine_kernel, dim3(n_combines, g.heads, kChunkTileRows / 8), dim3(256), 0, s, combines, g.heads,
               g.head_dim, ws_o, ws_ml, out);
    IB2_LAUNCH_CHECK();
  }
}

}  // namespace ib2
