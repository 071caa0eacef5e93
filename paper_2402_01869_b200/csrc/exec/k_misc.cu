#include <algorithm>
// Bandwidth-bound helper kernels: weight init, K9 embedding, K5 norms,
// K4 RoPE + paged KV write, K6 argmax, K8 block-table update, K7 swap copy.
// All are HBM/latency bound; they use 16-byte vector accesses where the row
// layout allows and size grids by rows (>= 148 CTAs for real batches).
#include <cfloat>

#include "kernels.hpp"

namespace ib2 {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}

// Values depend on the LOGICAL index only; tiled weights store logical
// (n, k) at its tile-blocked offset, padding rows are zero.
__global__ void init_tensor_kernel(f16* dst, std::int64_t count, std::uint64_t seed, std::uint32_t id, int kind,
                                   std::int64_t rows, std::int64_t cols, int tiled) {
  const std::int64_t kb = cols / 64;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    std::int64_t logical = i;
    bool pad = false;
    if (tiled) {
      const std::int64_t tile = i / 8192, rem = i % 8192;
      const std::int64_t n = (tile / kb) * 128 + rem / 64, k = (tile % kb) * 64 + rem % 64;
      pad = n >= rows;
      logical = n * cols + k;
    }
    const float v = pad ? 0.0f
                        : (kind == 1 ? 1.0f : (kind == 2 ? 0.0f : synth_weight(seed, id, static_cast<std::uint64_t>(logical))));
    dst[i] = __float2half_rn(v);
  }
}

// Row-major [N][K] -> tile-blocked (for the kernel test hook).
__global__ void tile_weights_kernel(const f16* __restrict__ src, f16* __restrict__ dst, std::int64_t N, std::int64_t K,
                                    std::int64_t count) {
  const std::int64_t kb = K / 64;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t tile = i / 8192, rem = i % 8192;
    const std::int64_t n = (tile / kb) * 128 + rem / 64, k = (tile % kb) * 64 + rem % 64;
    dst[i] = n < N ? src[n * K + k] : __float2half_rn(0.f);
  }
}

__global__ void iota_desc_kernel(std::int32_t* p, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<std::int32_t>(n - 1 - i);
}

__global__ void fill_kernel(std::int32_t* p, std::int64_t n, std::int32_t v) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void embed_kernel(const RowDesc* __restrict__ rows, std::int32_t* __restrict__ hist, int hist_stride,
                             const f16* __restrict__ tok_emb, const f16* __restrict__ pos_emb, int D,
                             std::uint64_t token_seed, int vocab, float* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const RowDesc d = rows[r];
  std::int32_t* h = hist + static_cast<std::int64_t>(d.slot) * hist_stride + d.pos;
  __shared__ std::int32_t tok_s;
  if (threadIdx.x == 0) {
    std::int32_t t;
    if (d.synthetic) {
      t = synth_token(token_seed, d.req_id, d.pos, vocab);
      *h = t;
    } else {
      t = *h;
    }
    tok_s = t;
  }
  __syncthreads();
  const f16* e = tok_emb + static_cast<std::int64_t>(tok_s) * D;
  const f16* p = pos_emb ? pos_emb + static_cast<std::int64_t>(d.pos) * D : nullptr;
  float* xr = x + static_cast<std::int64_t>(r) * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    float v = __half2float(e[i]);
    if (p) v = __fadd_rn(v, __half2float(p[i]));
    xr[i] = v;
  }
}

// One CTA per row; two-pass statistics from a register-resident row.
template <int NT, int PER>
__global__ void __launch_bounds__(NT) norm_kernel(const float* __restrict__ x, int ldx,
                                                  const std::int32_t* __restrict__ row_index, int D,
                                                  const f16* __restrict__ gamma, const f16* __restrict__ beta,
                                                  int rms, float eps, f16* __restrict__ y, int ldy) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[NT / 32];
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  const float* xr = x + static_cast<std::int64_t>(src) * ldx;
  float v[PER];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = threadIdx.x + i * NT;
    v[i] = c < D ? xr[c] : 0.f;
    s += v[i];
  }
  float mean = 0.f;
  if (!rms) mean = block_sum<NT>(s, red) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = threadIdx.x + i * NT;
    const float dv = c < D ? v[i] - mean : 0.f;
    q += dv * dv;
  }
  const float var = block_sum<NT>(q, red) / D;
  const float inv = rsqrtf(var + eps);
  f16* yr = y + static_cast<std::int64_t>(r) * ldy;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = threadIdx.x + i * NT;
    if (c < D) {
      float o = (v[i] - mean) * inv * __half2float(gamma[c]);
      if (beta) o += __half2float(beta[c]);
      yr[c] = __float2half_rn(o);
    }
  }
}

// Per row: rotate q and k of every head (fp32, no contraction, matching the
// oracle's float32 arithmetic), round to f16, and store k, v into the row's
// paged slot.
// K4: RoPE on q and k + k, v into the paged pool, 16-byte vectors.  Work
// items per row: q / k rotated vectors (rotate-half: one item = a vector of
// the first half and its partner in the second, so q can be updated in place;
// interleaved: one item = one vector of adjacent pairs), the unrotated k
// dims, and v.  k and v go straight to the pool (K1 / K2 read them there);
// only q is written back to the qkv rows.
__device__ __forceinline__ void rot_pair(float a, float b, float co, float si, float& ra, float& rb) {
  ra = __fsub_rn(__fmul_rn(a, co), __fmul_rn(b, si));
  rb = __fadd_rn(__fmul_rn(b, co), __fmul_rn(a, si));
}

__global__ void rope_kv_kernel(f16* __restrict__ qkv, const RowDesc* __restrict__ rows, f16* __restrict__ pool,
                               std::int64_t layer_off, std::int64_t block_stride, const std::int32_t* __restrict__ table,
                               int max_lb, int H, int hd, int rot, int interleaved, const float* __restrict__ cs) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const RowDesc d = rows[r];
  const int D = H * hd;
  f16* row = qkv + static_cast<std::int64_t>(r) * 3 * D;
  const int pb = table[static_cast<std::int64_t>(d.slot) * max_lb + d.pos / kBlockTokens];
  f16* blk = pool + layer_off + static_cast<std::int64_t>(pb) * block_stride;
  const int tok = d.pos % kBlockTokens;
  const float* c = cs + static_cast<std::int64_t>(d.pos) * rot;  // [rot/2][2] = (cos, sin)
  const int vec = hd / 8, rvec = rot / 8;             // 16 B vectors per head / rotated ones
  const int ritems = interleaved ? rvec : rvec / 2;   // rotation items per head
  auto kv_dst = [&](int kv, int h, int j) {
    return reinterpret_cast<uint4*>(blk + ((static_cast<std::int64_t>(kv) * H + h) * kBlockTokens + tok) * hd + j * 8);
  };
  const int n_rot = 2 * H * ritems;          // q and k rotation items
  const int n_kcopy = H * (vec - rvec);      // unrotated k vectors
  const int n_v = H * vec;
  for (int t = threadIdx.x; t < n_rot + n_kcopy + n_v; t += blockDim.x) {
    if (t < n_rot) {
      const int which = t / (H * ritems);  // 0 = q, 1 = k
      const int h = (t / ritems) % H, j = t % ritems;
      f16* head = row + which * D + h * hd;
      if (interleaved) {
        uint4 u = *reinterpret_cast<const uint4*>(head + j * 8);
        __half2* hp = reinterpret_cast<__half2*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = j * 4 + e;
          const float2 ab = __half22float2(hp[e]);
          float ra, rb;
          rot_pair(ab.x, ab.y, c[2 * i], c[2 * i + 1], ra, rb);
          hp[e] = __halves2half2(__float2half_rn(ra), __float2half_rn(rb));
        }
        if (which == 0) *reinterpret_cast<uint4*>(head + j * 8) = u;
        else *kv_dst(0, h, j) = u;
      } else {
        const int half = rot / 2, jb = j + half / 8;
        uint4 ua = *reinterpret_cast<const uint4*>(head + j * 8);
        uint4 ub = *reinterpret_cast<const uint4*>(head + jb * 8);
        __half* ha = reinterpret_cast<__half*>(&ua);
        __half* hb = reinterpret_cast<__half*>(&ub);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = j * 8 + e;
          float ra, rb;
          rot_pair(__half2float(ha[e]), __half2float(hb[e]), c[2 * i], c[2 * i + 1], ra, rb);
          ha[e] = __float2half_rn(ra);
          hb[e] = __float2half_rn(rb);
        }
        if (which == 0) {
          *reinterpret_cast<uint4*>(head + j * 8) = ua;
          *reinterpret_cast<uint4*>(head + jb * 8) = ub;
        } else {
          *kv_dst(0, h, j) = ua;
          *kv_dst(0, h, jb) = ub;
        }
      }
    } else if (t < n_rot + n_kcopy) {
      const int u = t - n_rot, nv = vec - rvec;
      const int h = u / nv, j = rvec + u % nv;
      *kv_dst(0, h, j) = *reinterpret_cast<const uint4*>(row + D + h * hd + j * 8);
    } else {
      const int u = t - n_rot - n_kcopy;
      const int h = u / vec, j = u % vec;
      *kv_dst(1, h, j) = *reinterpret_cast<const uint4*>(row + 2 * D + h * hd + j * 8);
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) argmax_kernel(const float* __restrict__ logits, int V,
                                                   const std::int32_t* __restrict__ sample_rows,
                                                   const RowDesc* __restrict__ rows, std::int32_t* __restrict__ hist,
                                                   int hist_stride, std::int32_t* __restrict__ out_tok,
                                                   std::int32_t* __restrict__ out_host) {
  pdl_trigger();
  pdl_wait();
  const int s = blockIdx.x;
  const float* l = logits + static_cast<std::int64_t>(s) * V;
  float best = -FLT_MAX;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += NT) {
    const float v = l[i];
    if (v > best) {
      best = v;
      idx = i;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  __shared__ float sb[NT / 32];
  __shared__ int si[NT / 32];
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < idx)) {
        best = sb[w];
        idx = si[w];
      }
    const RowDesc d = rows[sample_rows[s]];
    hist[static_cast<std::int64_t>(d.slot) * hist_stride + d.pos + 1] = idx;
    out_tok[s] = idx;
    if (out_host) out_host[s] = idx;
  }
}

__global__ void gather_rows_kernel(const f16* __restrict__ src, int ld, const std::int32_t* __restrict__ rows, int D,
                                   f16* __restrict__ dst) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<std::int64_t>(rows[r]) * ld);
  uint4* d = reinterpret_cast<uint4*>(dst + static_cast<std::int64_t>(r) * D);
  for (int i = threadIdx.x; i < D / 8; i += blockDim.x) d[i] = s[i];
}

// K8: single CTA, two phases separated by a barrier so pops may consume the
// blocks pushed by this launch (LIFO: the last freed block is reused first).
// A double free or an empty pool is a plan / sizing bug: the kernel records
// the code and traps, so the launch fails loudly before any later kernel of
// the iteration could use a -1 block id as a pool offset.
__global__ void __launch_bounds__(1024) block_update_kernel(std::int32_t* __restrict__ table,
                                                            std::int32_t* __restrict__ stack,
                                                            std::int32_t* __restrict__ top,
                                                            std::int32_t* __restrict__ err,
                                                            const std::int32_t* __restrict__ frees, int nf,
                                                            const std::int32_t* __restrict__ allocs, int na) {
  pdl_trigger();
  pdl_wait();
  const int t0 = *top;
  for (int k = threadIdx.x; k < nf; k += blockDim.x) {
    const int e = frees[k];
    const int pb = table[e];
    if (pb < 0) {
      atomicExch(err, 1);
      __trap();
    }
    stack[t0 + k] = pb;
    table[e] = -1;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < na; k += blockDim.x) {
    const int src = t0 + nf - 1 - k;
    const int e = allocs[k];
    if (src < 0 || table[e] >= 0) {
      atomicExch(err, 2);
      __trap();
    }
    table[e] = stack[src];
  }
  if (threadIdx.x == 0) *top = t0 + nf - na;
}

// K7: one CTA per (swap token, layer); moves the token's 2*D k/v elements
// between the paged pool and the op's [L][n][2D] staging slab.
__global__ void swap_copy_kernel(const SwapDesc* __restrict__ ops, const std::int32_t* __restrict__ prefix, int n_ops,
                                 f16* __restrict__ pool, std::int64_t layer_stride, std::int64_t block_stride,
                                 const std::int32_t* __restrict__ table, int max_lb, int H, int hd,
                                 f16* __restrict__ stage, int to_stage) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x, layer = blockIdx.y;
  int lo = 0, hi = n_ops;  // find op with prefix[op] <= t < prefix[op+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid;
  }
  const SwapDesc op = ops[lo];
  const int i = t - prefix[lo];
  const int pos = op.pos0 + i;
  const int D = H * hd;
  const int pb = table[static_cast<std::int64_t>(op.slot) * max_lb + pos / kBlockTokens];
  f16* blk = pool + layer * layer_stride + static_cast<std::int64_t>(pb) * block_stride;
  const int ld = op.ld > 0 ? op.ld : op.n;
  f16* srow = stage + op.stage_off + (static_cast<std::int64_t>(layer) * ld + i) * 2 * D;
  const int tok = pos % kBlockTokens;
  for (int v = threadIdx.x; v < 2 * D / 8; v += blockDim.x) {
    const int e = v * 8;
    const int kv = e / D, h = (e % D) / hd, dd = e % hd;
    uint4* p = reinterpret_cast<uint4*>(blk + ((static_cast<std::int64_t>(kv) * H + h) * kBlockTokens + tok) * hd + dd);
    uint4* q = reinterpret_cast<uint4*>(srow + e);
    if (to_stage) *q = *p;
    else *p = *q;
  }
}

int grid_for(std::int64_t n, int threads) {
  const std::int64_t g = (n + threads - 1) / threads;
  return static_cast<int>(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

void launch_init_tensor(f16* dst, std::int64_t count, std::uint64_t seed, std::uint32_t id, int kind,
                        std::int64_t rows, std::int64_t cols, bool tiled, cudaStream_t s) {
  init_tensor_kernel<<<grid_for(count, 256), 256, 0, s>>>(dst, count, seed, id, kind, rows, cols, tiled ? 1 : 0);
  IB2_LAUNCH_CHECK();
}

void launch_tile_weights(const f16* src, f16* dst, std::int64_t N, std::int64_t K, cudaStream_t s) {
  const std::int64_t count = (N + 127) / 128 * 128 * K;
  tile_weights_kernel<<<grid_for(count, 256), 256, 0, s>>>(src, dst, N, K, count);
  IB2_LAUNCH_CHECK();
}

void launch_iota_desc(std::int32_t* stack, std::int64_t n, cudaStream_t s) {
  iota_desc_kernel<<<grid_for(n, 256), 256, 0, s>>>(stack, n);
  IB2_LAUNCH_CHECK();
}

void launch_fill_i32(std::int32_t* p, std::int64_t n, std::int32_t v, cudaStream_t s) {
  fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, n, v);
  IB2_LAUNCH_CHECK();
}

void launch_embed(const RowDesc* rows, int n, std::int32_t* hist, int hist_stride, const f16* tok_emb,
                  const f16* pos_emb, int D, std::uint64_t token_seed, int vocab, float* x, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(embed_kernel, dim3(n), dim3(256), 0, s, rows, hist, hist_stride, tok_emb, pos_emb, D, token_seed, vocab, x);
  IB2_LAUNCH_CHECK();
}

void launch_norm(const float* x, int ldx, const std::int32_t* row_index, int n, int D, const f16* gamma,
                 const f16* beta, bool rms, float eps, f16* y, int ldy, cudaStream_t s) {
  if (n <= 0) return;
  if (D <= 1024) {
    launch_pdl(norm_kernel<256, 4>, dim3(n), dim3(256), 0, s, x, ldx, row_index, D, gamma, beta, static_cast<int>(rms), eps, y, ldy);
  } else if (D <= 4096) {
    launch_pdl(norm_kernel<512, 8>, dim3(n), dim3(512), 0, s, x, ldx, row_index, D, gamma, beta, static_cast<int>(rms), eps, y, ldy);
  } else {
    launch_pdl(norm_kernel<512, 16>, dim3(n), dim3(512), 0, s, x, ldx, row_index, D, gamma, beta, static_cast<int>(rms), eps, y, ldy);
  }
  IB2_LAUNCH_CHECK();
}

void launch_rope_kv_write(f16* qkv, const RowDesc* rows, int n, const KvGeom& g, int layer, int rotary_dim,
                          bool interleaved, const float* rope_cs, cudaStream_t s) {
  if (n <= 0) return;
  if (g.head_dim % 8 || rotary_dim % (interleaved ? 8 : 16) || rotary_dim > g.head_dim)
    throw DeviceError("rope_kv: head_dim / rotary_dim not a multiple of the 16-byte vector");
  launch_pdl(rope_kv_kernel, dim3(n), dim3(256), 0, s, qkv, rows, g.pool, layer * g.layer_stride(), g.block_stride(),
             g.table, g.max_lblocks, g.heads, g.head_dim, rotary_dim, interleaved ? 1 : 0, rope_cs);
  IB2_LAUNCH_CHECK();
}

void launch_argmax(const float* logits, int n, int V, const std::int32_t* sample_rows, const RowDesc* rows,
                   std::int32_t* hist, int hist_stride, std::int32_t* out_tok, std::int32_t* out_host, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(argmax_kernel<512>, dim3(n), dim3(512), 0, s, logits, V, sample_rows, rows, hist, hist_stride, out_tok,
             out_host);
  IB2_LAUNCH_CHECK();
}

// Small host -> device copies through the SMs from mapped pinned memory: the
// copy engines may be busy for milliseconds with swap transfers, and a
// cudaMemcpyAsync queued behind them would stall the compute stream.
__global__ void copy_from_host_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, std::int64_t n16) {
  pdl_trigger();
  pdl_wait();
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

void launch_copy_from_host(void* dst, const void* src_mapped, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  const std::int64_t n16 = static_cast<std::int64_t>((bytes + 15) / 16);
  const int blocks = static_cast<int>(std::min<std::int64_t>((n16 + 255) / 256, 64));
  launch_pdl(copy_from_host_kernel, dim3(blocks), dim3(256), 0, s, static_cast<uint4*>(dst),
             static_cast<const uint4*>(src_mapped), n16);
  IB2_LAUNCH_CHECK();
}

void launch_gather_rows(const f16* src, int ld, const std::int32_t* rows, int n, int D, f16* dst,
                        cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(gather_rows_kernel, dim3(n), dim3(256), 0, s, src, ld, rows, D, dst);
  IB2_LAUNCH_CHECK();
}

void launch_block_update(std::int32_t* table, std::int32_t* stack, std::int32_t* top, std::int32_t* err,
                         const std::int32_t* frees, int nf, const std::int32_t* allocs, int na, cudaStream_t s) {
  if (nf == 0 && na == 0) return;
  launch_pdl(block_update_kernel, dim3(1), dim3(1024), 0, s, table, stack, top, err, frees, nf, allocs, na);
  IB2_LAUNCH_CHECK();
}

void launch_swap_copy(const SwapDesc* ops, const std::int32_t* tok_prefix, int n_ops, int total_tokens,
                      const KvGeom& g, f16* stage, bool to_stage, cudaStream_t s) {
  if (total_tokens <= 0) return;
  dim3 grid(total_tokens, g.layers);
  launch_pdl(swap_copy_kernel, grid, dim3(256), 0, s, ops, tok_prefix, n_ops, g.pool, g.layer_stride(), g.block_stride(),
             g.table, g.max_lblocks, g.heads, g.head_dim, stage, to_stage ? 1 : 0);
  IB2_LAUNCH_CHECK();
}

}  // namespace ib2
