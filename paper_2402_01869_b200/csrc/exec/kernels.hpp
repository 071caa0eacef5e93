// Host launchers of the executor's sm_100a kernels.  K-numbers follow
// SURVEY §2.3 (K1 paged decode attention, K2 chunk/prefill attention, K3
// projection GEMMs, K4 RoPE + paged KV write, K5 norms, K6 LM-head argmax,
// K7 swap gather/scatter, K8 block tables, K9 embeddings).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace ib2 {

struct KvGeom {
  f16* pool;         // [L][num_blocks][2][H][16][hd]
  std::int64_t num_blocks;
  int layers, heads, head_dim;
  const std::int32_t* table;  // [slots][max_lblocks]
  int max_lblocks;
  std::int64_t layer_stride() const { return num_blocks * 2LL * heads * kBlockTokens * head_dim; }
  std::int64_t block_stride() const { return 2LL * heads * kBlockTokens * head_dim; }
};

// init
void launch_init_tensor(f16* dst, std::int64_t count, std::uint64_t seed, std::uint32_t id, int kind,
                        std::int64_t rows, std::int64_t cols, bool tiled, cudaStream_t s);
void launch_tile_weights(const f16* src, f16* dst, std::int64_t N, std::int64_t K, cudaStream_t s);
void launch_iota_desc(std::int32_t* stack, std::int64_t n, cudaStream_t s);
void launch_fill_i32(std::int32_t* p, std::int64_t n, std::int32_t v, cudaStream_t s);

// K9: x[r] = E[tok] (+ P[pos]); history written for synthetic rows.
void launch_embed(const RowDesc* rows, int n, std::int32_t* hist, int hist_stride, const f16* tok_emb,
                  const f16* pos_emb, int D, std::uint64_t token_seed, int vocab, float* x, cudaStream_t s);

// K5: y = norm(x) (LayerNorm with bias, or RMSNorm when beta == null && rms)
void launch_norm(const float* x, int ldx, const std::int32_t* row_index, int n, int D, const f16* gamma,
                 const f16* beta, bool rms, float eps, f16* y, int ldy, cudaStream_t s);

// K4: RoPE on q,k in place + write k,v of every row into the paged pool.
void launch_rope_kv_write(f16* qkv, const RowDesc* rows, int n, const KvGeom& g, int layer, int rotary_dim,
                          bool interleaved, const float* rope_cs, cudaStream_t s);

// K1: split-KV paged decode attention for single rows.
void launch_decode_attention(const f16* qkv, const std::int32_t* drow, const RowDesc* rows, int n_drows,
                             const KvGeom& g, int layer, int max_pos_plus1, float* part_o, float* part_ml,
                             f16* out, std::int32_t* counters, cudaStream_t s);
// counters: n_rows x heads int32, zero before the first launch; K1 leaves them zero.

// K2: tiled causal attention over the paged prefix for chunk rows, split-KV
// items + combine pass for tiles whose keys were split.
// qkv_rows: row capacity of the qkv activation buffer (TMA bounds).
void launch_chunk_attention(const f16* qkv, int qkv_rows, const TileDesc* items, int n_items,
                            const CombineDesc* combines, int n_combines, const KvGeom& g, int layer, f16* out,
                            float* ws_o, float* ws_ml, cudaStream_t s);
// Keys per K2 tile for a head dim (split-KV ranges are aligned to it).
int chunk_attention_key_tile(int head_dim);
// Resident K2 CTAs per SM for a head dim (the split-KV planner's slot count).
int chunk_attention_ctas_per_sm(int head_dim);

// 2-D f16 TMA descriptor over [rows][inner] (row stride in bytes), box
// box_inner x box_rows, 128-byte swizzle.
CUtensorMap make_tmap_2d(const void* base, std::int64_t inner, std::int64_t rows, std::int64_t row_stride_bytes,
                         int box_inner, int box_rows);

// K3: projection GEMM with fused epilogue.
void launch_gemm(const GemmArgs& a, cudaStream_t s);
bool gemm_uses_tcgen05();

// K6: row argmax of fp32 logits, lowest index on ties; writes history.
// out_host: mapped pinned memory the ids are also stored to (may be null).
void launch_argmax(const float* logits, int n, int V, const std::int32_t* sample_rows, const RowDesc* rows,
                   std::int32_t* hist, int hist_stride, std::int32_t* out_tok, std::int32_t* out_host, cudaStream_t s);

// Small H2D copy performed by SMs from mapped pinned memory (bytes rounded up
// to 16; both buffers must have that slack).
void launch_copy_from_host(void* dst, const void* src_mapped, std::size_t bytes, cudaStream_t s);

void launch_gather_rows(const f16* src, int ld, const std::int32_t* rows, int n, int D, f16* dst,
                        cudaStream_t s);

// K8: block-table update: frees pushed (LIFO), then allocs popped.
void launch_block_update(std::int32_t* table, std::int32_t* stack, std::int32_t* top, std::int32_t* err,
                         const std::int32_t* frees, int nf, const std::int32_t* allocs, int na, cudaStream_t s);

// K7: swap gather (pool -> staging) / scatter (staging -> pool).
void launch_swap_copy(const SwapDesc* ops, const std::int32_t* tok_prefix, int n_ops, int total_tokens,
                      const KvGeom& g, f16* stage, bool to_stage, cudaStream_t s);

}  // namespace ib2
