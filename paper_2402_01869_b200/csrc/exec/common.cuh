// Device-side vocabulary shared by the executor's kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <utility>

#include "../sched/base.hpp"

namespace ib2 {

using f16 = __half;  // activations, KV cache and weights; fp32 accumulation

#define IB2_CUDA(expr)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw ::ib2::DeviceError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " @" __FILE__); \
  } while (0)

#define IB2_LAUNCH_CHECK() IB2_CUDA(cudaGetLastError())

constexpr int kBlockTokens = 16;  // paged KV block = 16 token positions

// Programmatic dependent launch: every per-iteration kernel lets its successor
// launch immediately (its prologue overlaps this kernel's tail) and waits for
// its predecessor's completion before touching global memory it produced.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Loads through `const __restrict__` pointers become ld.global.nc, which the
// compiler treats as invariant and may hoist above griddepcontrol.wait (it
// did, in K1: the row descriptors of the previous iteration were read).
// Passing a pointer through an asm volatile after pdl_wait() makes every load
// through it depend on the wait.  tests/test_sass.py checks the .so.
template <typename T>
__device__ __forceinline__ T* after_wait(T* p) {
  asm volatile("" : "+l"(p));
  return p;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw DeviceError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// splitmix64 finalizer: the counter hash behind synthetic weights and ids.
__host__ __device__ inline std::uint64_t mix64(std::uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Uniform weight with std 0.02: u in [-1,1) on a 2^-23 grid times 0.02*sqrt(3).
__host__ __device__ inline float synth_weight(std::uint64_t seed, std::uint32_t tensor_id, std::uint64_t idx) {
  const std::uint64_t base = mix64(seed + 0x9E3779B97F4A7C15ULL * (static_cast<std::uint64_t>(tensor_id) + 1));
  const std::uint32_t u24 = static_cast<std::uint32_t>(mix64(base + idx) >> 40);
  const float u = static_cast<float>(u24) * 1.1920928955078125e-07f - 1.0f;
  return u * 0.034641016f;
}

// Synthetic prompt / API-returned token id at a position of a request.
__host__ __device__ inline std::int32_t synth_token(std::uint64_t seed, std::int64_t req_id, std::int64_t pos,
                                                   std::int32_t vocab) {
  const std::uint64_t base = mix64(seed + 0xD1B54A32D192ED03ULL * static_cast<std::uint64_t>(req_id + 1));
  return static_cast<std::int32_t>(mix64(base + static_cast<std::uint64_t>(pos)) % static_cast<std::uint64_t>(vocab));
}

// One query row of the batch.
struct RowDesc {
  std::int32_t slot;
  std::int32_t pos;
  std::int32_t synthetic;  // 1: input id is synthetic (fresh span), else history
  std::int32_t pad;
  std::int64_t req_id;
};

// A tile of consecutive chunk rows of one request for prefill attention,
// restricted to keys [kv_lo, kv_hi) (split-KV).  part < 0: the item covers
// all keys and writes the normalized output; else it writes an fp32 partial
// (o, m, l) into slot `part` for the combine pass.
struct TileDesc {
  std::int32_t row0;   // first batch row
  std::int32_t nrows;  // <= kChunkTileRows
  std::int32_t slot;
  std::int32_t pos0;   // position of row0
  std::int32_t kv_lo, kv_hi;
  std::int32_t part;
  std::int32_t pad;
};

// Split q-tiles whose partials must be merged.
struct CombineDesc {
  std::int32_t row0, nrows, part0, nparts;
};
constexpr int kChunkTileRows = 128;  // query rows per K2 item (UMMA M)
constexpr int kMaxChunkParts = 1024;  // (part, head) slots of the split-KV workspace

// Swap copy descriptor: positions [pos0, pos0+n) of a slot <-> staging rows.
struct SwapDesc {
  std::int32_t slot;
  std::int32_t pos0;
  std::int32_t n;
  std::int32_t ld;         // tokens per layer of the staging slab (0: n)
  std::int64_t stage_off;  // element offset of position pos0, layer 0, in a [L][ld][2D] slab
};

// Epilogue variants of the projection GEMMs.
enum class Epi : int {
  StoreF16 = 0,     // out = acc (+bias)
  GeluF16 = 1,      // out = gelu_tanh(acc + bias)
  ResidAdd = 2,      // resid(fp32) += acc (+bias)
  SwiGluF16 = 3,    // out[j] = silu(acc[2j]) * acc[2j+1]
  StoreF32 = 4,      // outf = acc (+bias)
  QkvRopeKv = 5      // fused K4: q -> out (RoPE), k (RoPE), v -> paged KV pool
};

// Epi::QkvRopeKv: the QKV projection's epilogue applies the interleaved
// (GPT-J) rotary embedding to q and k after the same f16 rounding as a
// separate pass would, stores q to `out`, and writes k and v of each row
// straight into its paged KV block.
struct QkvWrite {
  const RowDesc* rows;  // [M] slot, position of each row
  f16* pool;            // [L][blocks][2][H][16][hd]
  std::int64_t layer_off, block_stride;
  const std::int32_t* table;
  int max_lb;
  int H, hd, rot;        // rot: rotary dims (interleaved pairs), 0 = none
  const float* rope_cs;  // [pos][rot/2][cos, sin]
};

struct GemmArgs {
  const f16* a;       // [M][K] row-major (K contiguous)
  const f16* w;       // [N][K], tile-blocked (model.hpp weight_tile_offset)
  int M, N, K;
  Epi epi;
  const f16* bias;    // [N] or null
  f16* out;           // [M][ldo] f16 output
  int ldo;
  float* outf;         // fp32 output / residual stream
  int ldf;
  QkvWrite qkv;        // Epi::QkvRopeKv only
  int no_early_w;      // diagnostics: no weight prefetch before griddepcontrol.wait
  const float* addf;   // Epi::ResidAdd: if set, outf = (outf + acc) + addf (same [M][ldf] layout)
  std::int64_t a_rows;  // rows addressable from `a` for TMA bounds (0: the executor's buffer capacity)
  int streamk_ok;       // 0: no stream-K / split tail; 1: if enabled (IB2_STREAMK=1); 2: forced.  Only where no
                        // other stream-K GEMM can run concurrently (the executor's compute stream)
};

}  // namespace ib2
