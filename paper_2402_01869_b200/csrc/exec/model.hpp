// Random-init decoder families the executor serves:
//   tiny       GPT-2 style: 2 L, d=256, 4x64 heads, ffn 1024, learned positions
//   gptj-6b    GPT-J shape: 28 L, d=4096, 16x256 heads, ffn 16384, rotary 64,
//              parallel attention+MLP residual, one LayerNorm per block
//   vicuna-13b LLaMA shape: 40 L, d=5120, 40x128 heads, SwiGLU ffn 13824,
//              RMSNorm, full rotate-half RoPE
// Weights are f16, generated on the device from a counter hash (the CPU
// oracle regenerates the identical values); compute accumulates in fp32.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ib2 {

enum class Family { Gpt2 = 0, GptJ = 1, Llama = 2 };

struct ModelSpec {
  Family family = Family::Gpt2;
  int layers = 2, d_model = 256, heads = 4, ffn = 1024, vocab = 4096;
  int rotary_dim = 0;  // 0: none (learned positions)
  int max_pos = 4160;
  std::uint64_t weight_seed = 1234, token_seed = 99;
  double rope_theta = 10000.0;
  float norm_eps = 1e-5f;

  int head_dim() const { return d_model / heads; }
  int qkv_dim() const { return 3 * d_model; }
  // Width of the first MLP GEMM's output (SwiGLU computes gate and up).
  int ffn_in_width() const { return family == Family::Llama ? 2 * ffn : ffn; }
  bool has_bias() const { return family != Family::Llama; }
  bool qkv_bias() const { return family == Family::Gpt2; }
  bool lm_bias() const { return family == Family::GptJ; }
  bool parallel_residual() const { return family == Family::GptJ; }
  // KV bytes per token over all layers (the cost model's mem_per_token).
  std::int64_t kv_bytes_per_token() const { return 2LL * layers * d_model * 2; }
  std::int64_t param_count() const;
};

ModelSpec parse_model_json(const std::string& text);
std::string model_json(const ModelSpec& m);

// Element offsets (f16 units) of every tensor in the single weight arena.
struct LayerWeights {
  std::int64_t ln1_g, ln1_b, ln2_g, ln2_b;  // ln2 unused for GPT-J
  std::int64_t w_qkv, b_qkv, w_o, b_o;      // [3D][D], [D][D]
  std::int64_t w_in, b_in, w_out, b_out;    // [F or 2F][D], [D][F]
};
struct WeightLayout {
  std::int64_t tok_emb = 0, pos_emb = -1;   // [V][D], [P][D]
  std::vector<LayerWeights> layer;
  std::int64_t lnf_g = 0, lnf_b = 0, lm_w = 0, lm_b = -1;  // [V][D]
  std::int64_t total = 0;
  // (offset, count, tensor id, kind) for the device initializer; kind:
  // 0 = uniform(std 0.02), 1 = ones, 2 = zeros.  Projection weights [N][K]
  // are stored tile-blocked (tiled = true, see weight_tile_offset): every
  // 128-row x 64-column tile is one contiguous 16 KB run, so a TMA load of a
  // tile streams contiguous HBM.  N is padded to a multiple of 128 (zeros).
  struct Item {
    std::int64_t off, count;
    std::uint32_t id;
    int kind;
    std::int64_t rows = 0, cols = 0;
    bool tiled = false;
  };
  std::vector<Item> items;
};
WeightLayout layout_weights(const ModelSpec& m);

#ifdef __CUDACC__
#define IB2_HD __host__ __device__
#else
#define IB2_HD
#endif

// Element offset of logical (n, k) in a tile-blocked [N][K] weight.
constexpr int kWTileRows = 128, kWTileCols = 64;
IB2_HD inline std::int64_t weight_tile_offset(std::int64_t n, std::int64_t k, std::int64_t K) {
  return ((n / kWTileRows) * (K / kWTileCols) + k / kWTileCols) * (kWTileRows * kWTileCols) +
         (n % kWTileRows) * kWTileCols + k % kWTileCols;
}
inline std::int64_t tiled_weight_elems(std::int64_t N, std::int64_t K) {
  return (N + kWTileRows - 1) / kWTileRows * kWTileRows * K;
}

}  // namespace ib2
