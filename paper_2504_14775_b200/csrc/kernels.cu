// Memory-bound kernels of the stage forward: metadata expansion + device slot
// mapping, embedding gather, RMSNorm, RoPE + paged KV write, SiLU*mul, argmax,
// sampled-token commit. All bf16 I/O is 16-byte vectorised.
//
// Per-sequence metadata (`seq_info`, int32 x 5 per sequence, plan order:
// decodes first, then prefill chunks, as `MicroBatchPlan` orders them):
//   [0] row      block-table / token-history row of the request
//   [1] start    tokens already in the KV cache (position of the first new token)
//   [2] n_new    tokens appended by this micro-batch (1 for a decode)
//   [3] tok_off  index of the sequence's first token in the packed token dim
//   [4] emit     index into the sampled-token list, or -1
#include <float.h>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

// ----------------------------------------------------------- metadata
// Bounds checks: the host is trusted for shapes but not for ids -- a row, page index, page id
// or position outside the stage's tables would silently corrupt another request's KV. Invalid
// entries are skipped (block-table deltas, prompt rows) or given slot -1 (tokens; the KV-writing
// epilogues skip those), and a bit is OR-ed into a host-mapped error word that the executor
// reads after every micro-batch (gllm_meta_errors) -- no extra sync or copy on the fast path.
static unsigned* g_err_host = nullptr;
static unsigned* g_err_dev = nullptr;

static unsigned* err_word() {
  if (g_err_dev == nullptr) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&g_err_host), sizeof(unsigned), cudaHostAllocMapped) != cudaSuccess)
      return nullptr;
    *g_err_host = 0;
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_err_dev), g_err_host, 0) != cudaSuccess) {
      g_err_dev = nullptr;
      return nullptr;
    }
  }
  return g_err_dev;
}

unsigned meta_errors(int reset) {
  if (g_err_host == nullptr) return 0;
  const unsigned v = *reinterpret_cast<volatile unsigned*>(g_err_host);
  if (reset) *reinterpret_cast<volatile unsigned*>(g_err_host) = 0;
  return v;
}

__device__ __forceinline__ void flag_error(unsigned* err, unsigned bit) {
  if (err != nullptr) atomicOr_system(err, bit);
#ifdef GLLM_DEBUG
  __trap();
#endif
}

// meta layout: deltas [n_deltas][3] = (row, page_index, page_id), then
// prompt headers [n_prompt_rows][3] = (row, length, offset into the token area),
// then the token area.
__global__ void apply_metadata_kernel(const int* __restrict__ meta, int n_deltas, int n_prompt_rows,
                                      int* __restrict__ block_table, int mpr, int* __restrict__ token_hist,
                                      int max_seq_len, int max_rows, int num_pages, unsigned* err) {
  const int* hdr = meta + 3 * n_deltas;
  const int* toks = hdr + 3 * n_prompt_rows;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < n_deltas; i += blockDim.x) {
      const int row = meta[3 * i], idx = meta[3 * i + 1], page = meta[3 * i + 2];
      if ((unsigned)row >= (unsigned)max_rows || (unsigned)idx >= (unsigned)mpr ||
          (unsigned)page >= (unsigned)num_pages) {
        flag_error(err, GLLM_META_BAD_DELTA);
        continue;
      }
      block_table[(size_t)row * mpr + idx] = page;
    }
  }
  for (int p = blockIdx.x; p < n_prompt_rows; p += gridDim.x) {
    const int row = hdr[3 * p], len = hdr[3 * p + 1], off = hdr[3 * p + 2];
    if ((unsigned)row >= (unsigned)max_rows || len < 0 || len > max_seq_len || off < 0) {
      if (threadIdx.x == 0) flag_error(err, GLLM_META_BAD_PROMPT);
      continue;
    }
    int* dst = token_hist + (size_t)row * max_seq_len;
    for (int t = threadIdx.x; t < len; t += blockDim.x) dst[t] = toks[off + t];
  }
}

int apply_batch_metadata(const int* meta, int n_deltas, int n_prompt_rows, int* block_table, int mpr,
                         int* token_hist, int max_seq_len, int max_rows, int num_pages, cudaStream_t st) {
  if (n_deltas == 0 && n_prompt_rows == 0) return 0;
  int blocks = n_prompt_rows > 0 ? (n_prompt_rows < 1024 ? n_prompt_rows : 1024) : 1;
  apply_metadata_kernel<<<blocks, 256, 0, st>>>(meta, n_deltas, n_prompt_rows, block_table, mpr, token_hist,
                                                  max_seq_len, max_rows, num_pages, err_word());
  return check_launch("apply_metadata");
}

// One warp per sequence writes its tokens' positions, slots (device slot mapping:
// slot = table[row][pos / ps] * ps + pos % ps) and token ids.
__global__ void expand_tokens_kernel(const int* __restrict__ seq_info, int n_seqs, const int* __restrict__ block_table,
                                     int mpr, const int* __restrict__ token_hist, int max_seq_len, int page_size,
                                     int* __restrict__ tok_pos, int* __restrict__ tok_slot, int* __restrict__ tok_id,
                                     int* __restrict__ emit_rows, int max_rows, int num_pages, unsigned* err) {
  const int s = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (s >= n_seqs) return;
  const int* si = seq_info + 5 * s;
  const int row = si[0], start = si[1], n = si[2], off = si[3], emit = si[4];
  const bool row_ok = (unsigned)row < (unsigned)max_rows && start >= 0 && n >= 0 && start + n <= max_seq_len &&
                      start + n <= mpr * page_size;
  if (!row_ok && lane == 0) flag_error(err, GLLM_META_BAD_SEQ);
  const int* table = block_table + (size_t)(row_ok ? row : 0) * mpr;
  const int* hist = token_hist != nullptr ? token_hist + (size_t)(row_ok ? row : 0) * max_seq_len : nullptr;
  for (int t = lane; t < n; t += 32) {
    const int pos = start + t;
    tok_pos[off + t] = row_ok ? pos : 0;
    int slot = -1;
    if (row_ok) {
      const int page = table[pos / page_size];
      if ((unsigned)page < (unsigned)num_pages) slot = page * page_size + pos % page_size;
      else flag_error(err, GLLM_META_BAD_PAGE);
    }
    tok_slot[off + t] = slot;
    if (tok_id != nullptr) tok_id[off + t] = row_ok ? hist[pos] : 0;
  }
  if (lane == 0 && emit >= 0 && emit_rows != nullptr) emit_rows[emit] = off + n - 1;
}

// Row gather of the embedding table; 16 bytes per thread.
__global__ void embed_kernel(const int* __restrict__ tok_id, const bf16* __restrict__ embed, int d,
                             bf16* __restrict__ out) {
  const int t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(embed + (size_t)tok_id[t] * d);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = src[i];
}

int expand_tokens(const int* seq_info, int n_seqs, const int* block_table, int mpr, const int* token_hist,
                  int max_seq_len, int page_size, int* tok_pos, int* tok_slot, int* tok_id, int* emit_rows,
                  const bf16* embed, int d, bf16* x_out, int max_rows, int num_pages, cudaStream_t st) {
  if (n_seqs <= 0) return 0;
  const int warps = 8;
  expand_tokens_kernel<<<(n_seqs + warps - 1) / warps, warps * 32, 0, st>>>(
      seq_info, n_seqs, block_table, mpr, token_hist, max_seq_len, page_size, tok_pos, tok_slot, tok_id, emit_rows,
      max_rows, num_pages, err_word());
  if (int rc = check_launch("expand_tokens")) return rc;
  return 0;
}

int embed_tokens(const int* tok_id, int n_tokens, const bf16* embed, int d, bf16* out, cudaStream_t st) {
  if (n_tokens <= 0) return 0;
  embed_kernel<<<n_tokens, 128, 0, st>>>(tok_id, embed, d, out);
  return check_launch("embed");
}

// ----------------------------------------------------------- RMSNorm
// out[r] = x[row(r)] * rsqrt(mean(x^2) + eps) * w ; one CTA per row, fp32 math.
template <int VEC_PER_THREAD>
__global__ void rmsnorm_kernel(const bf16* __restrict__ x, int ldx, const int* __restrict__ row_index,
                               const bf16* __restrict__ w, bf16* __restrict__ out, int d, float eps) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  const uint4* xp = reinterpret_cast<const uint4*>(x + (size_t)src * ldx);
  const uint4* wp = reinterpret_cast<const uint4*>(w);
  uint4* op = reinterpret_cast<uint4*>(out + (size_t)r * d);
  const int nvec = d / 8;
  float v[VEC_PER_THREAD][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VEC_PER_THREAD; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      uint4 u = xp[i];
      uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_bf16x2(a[j]);
        v[k][2 * j] = f.x;
        v[k][2 * j + 1] = f.y;
        ss += f.x * f.x + f.y * f.y;
      }
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)d + eps);
#pragma unroll
  for (int k = 0; k < VEC_PER_THREAD; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      uint4 g = wp[i];
      uint32_t ga[4] = {g.x, g.y, g.z, g.w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 gw = unpack_bf16x2(ga[j]);
        // HF order: normalise in fp32, round to the activation dtype, then scale by the weight.
        float a = bf2f(f2bf(v[k][2 * j] * inv)) * gw.x;
        float b = bf2f(f2bf(v[k][2 * j + 1] * inv)) * gw.y;
        o[j] = pack_bf16x2(a, b);
      }
      op[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

int rmsnorm(const bf16* x, int ldx, const int* row_index, const bf16* w, bf16* out, int rows, int d, float eps,
            cudaStream_t st) {
  if (rows <= 0) return 0;
  if (d % 8) return set_error(GLLM_ERR_INVALID, "rmsnorm needs d %% 8 == 0");
  const int nvec = d / 8;
  if (nvec <= 128) {
    cudaError_t e = launch_kernel(rmsnorm_kernel<1>, dim3(rows), dim3(128), 0, st, 1, x, ldx, row_index, w, out, d, eps);
    if (e != cudaSuccess) return set_cuda_error(e, "rmsnorm launch");
  } else if (nvec <= 1024) {
    const int threads = ((nvec + 3) / 4 + 31) / 32 * 32;
    cudaError_t e =
        launch_kernel(rmsnorm_kernel<4>, dim3(rows), dim3(threads), 0, st, 1, x, ldx, row_index, w, out, d, eps);
    if (e != cudaSuccess) return set_cuda_error(e, "rmsnorm launch");
  } else {
    return set_error(GLLM_ERR_INVALID, "rmsnorm d=%d too large", d);
  }
  return check_launch("rmsnorm");
}

// ----------------------------------------------------------- fused-norm statistics
// ss[g][r] = sum of x[r][64g .. 64g+64)^2 over the bf16 values (the layout the O / down GEMM
// epilogues write): a warp per row, lane = 8 columns, 8 lanes per group reduced by a butterfly.
__global__ void row_sumsq_kernel(const bf16* __restrict__ x, int ldx, int rows, int d, float* __restrict__ ss,
                                 int ld) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;  // whole warps
  const uint4* xp = reinterpret_cast<const uint4*>(x + (size_t)r * ldx);
  for (int i = lane; i < d / 8; i += 32) {
    const uint4 u = xp[i];
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(w4[j]);
      acc = fmaf(f.x, f.x, acc);
      acc = fmaf(f.y, f.y, acc);
    }
    for (int o = 1; o < 8; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((i & 7) == 0) ss[(size_t)(i / 8) * ld + r] = acc;
  }
}

int row_sumsq(const bf16* x, int ldx, int rows, int d, float* ss, int ld, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (d % 256 || ldx % 8) return set_error(GLLM_ERR_INVALID, "row_sumsq needs d %% 256 == 0 and ldx %% 8 == 0");
  cudaError_t e = launch_kernel(row_sumsq_kernel, dim3((rows + 7) / 8), dim3(256), 0, st, 1, x, ldx, rows, d, ss, ld);
  if (e != cudaSuccess) return set_cuda_error(e, "row_sumsq launch");
  return check_launch("row_sumsq");
}

// ----------------------------------------------------------- SiLU * mul
// gu rows hold [gate(d_ff) | up(d_ff)]; out = silu(gate) * up.
__global__ void silu_mul_kernel(const bf16* __restrict__ gu, int d_ff, bf16* __restrict__ out, size_t groups) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= groups) return;
  const int per_row = d_ff / 8;
  const size_t r = i / per_row;
  const int c = (int)(i % per_row) * 8;
  uint4 g = *reinterpret_cast<const uint4*>(gu + r * 2 * d_ff + c);
  uint4 u = *reinterpret_cast<const uint4*>(gu + r * 2 * d_ff + d_ff + c);
  uint32_t ga[4] = {g.x, g.y, g.z, g.w}, ua[4] = {u.x, u.y, u.z, u.w}, o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 a = unpack_bf16x2(ga[j]), b = unpack_bf16x2(ua[j]);
    float s0 = bf2f(f2bf(silu_f(a.x))), s1 = bf2f(f2bf(silu_f(a.y)));
    o[j] = pack_bf16x2(s0 * b.x, s1 * b.y);
  }
  *reinterpret_cast<uint4*>(out + r * d_ff + c) = make_uint4(o[0], o[1], o[2], o[3]);
}

int silu_mul(const bf16* gu, int d_ff, bf16* out, int rows, cudaStream_t st) {
  if (rows <= 0) return 0;
  const size_t groups = (size_t)rows * (d_ff / 8);
  silu_mul_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(gu, d_ff, out, groups);
  return check_launch("silu_mul");
}

// ----------------------------------------------------------- RoPE + paged KV write
// qkv row layout: [q heads | k heads | v heads], head_dim contiguous. Rotates q and k
// in place (rotate-half convention, fp32 math, cos/sin table [pos][hd/2][2]) and
// scatters k, v into the paged caches laid out [page][kv_head][slot_in_page][hd].
__global__ void rope_kv_kernel(bf16* __restrict__ qkv, int n_heads, int n_kv, int hd, const int* __restrict__ tok_pos,
                               const int* __restrict__ tok_slot, const float* __restrict__ rope,
                               bf16* __restrict__ k_cache, bf16* __restrict__ v_cache, int page_size) {
  const int t = blockIdx.x;
  const int pos = tok_pos[t];
  const int slot = tok_slot[t];
  const int page = slot / page_size, off = slot % page_size;
  const int half = hd / 2;
  const int width = (n_heads + 2 * n_kv) * hd;
  bf16* row = qkv + (size_t)t * width;
  const float2* cs = reinterpret_cast<const float2*>(rope + (size_t)pos * hd);  // [half] (cos, sin)
  // rotary pairs for q and k heads
  const int pairs = (n_heads + n_kv) * half;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int h = i / half, j = i % half;
    bf16* base = row + h * hd;
    const float x1 = bf2f(base[j]), x2 = bf2f(base[j + half]);
    const float2 c = cs[j];
    const bf16 y1 = f2bf(x1 * c.x - x2 * c.y);
    const bf16 y2 = f2bf(x2 * c.x + x1 * c.y);
    if (h < n_heads) {
      base[j] = y1;
      base[j + half] = y2;
    } else {
      base[j] = y1;
      base[j + half] = y2;
      if (slot < 0) continue;       // metadata failed the bounds check in expand_tokens
      const int kh = h - n_heads;
      bf16* dst = k_cache + (((size_t)page * n_kv + kh) * page_size + off) * hd;
      dst[j] = y1;
      dst[j + half] = y2;
    }
  }
  if (slot < 0) return;
  // v heads: straight copy, 16 bytes per thread
  const int vvec = n_kv * hd / 8;
  const uint4* vsrc = reinterpret_cast<const uint4*>(row + (n_heads + n_kv) * hd);
  for (int i = threadIdx.x; i < vvec; i += blockDim.x) {
    const int kh = (i * 8) / hd, d0 = (i * 8) % hd;
    uint4* dst = reinterpret_cast<uint4*>(v_cache + (((size_t)page * n_kv + kh) * page_size + off) * hd + d0);
    *dst = vsrc[i];
  }
}

int rope_kv_write(bf16* qkv, int n_tokens, int n_heads, int n_kv, int head_dim, const int* tok_pos,
                  const int* tok_slot, const float* rope, bf16* k_cache, bf16* v_cache, int page_size,
                  cudaStream_t st) {
  if (n_tokens <= 0) return 0;
  rope_kv_kernel<<<n_tokens, 256, 0, st>>>(qkv, n_heads, n_kv, head_dim, tok_pos, tok_slot, rope, k_cache, v_cache,
                                           page_size);
  return check_launch("rope_kv_write");
}

// ----------------------------------------------------------- argmax (sampling)
// One CTA per row; each thread scans 8 bf16 per 16-byte load; ties -> lowest index.
__global__ void argmax_kernel(const bf16* __restrict__ logits, int vocab, int* __restrict__ out) {
  const int r = blockIdx.x;
  const bf16* row = logits + (size_t)r * vocab;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  const int nvec = vocab / 8;
  const uint4* v = reinterpret_cast<const uint4*>(row);
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    uint4 u = v[i];
    uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(a[j]);
      const int idx = i * 8 + 2 * j;
      if (f.x > best) { best = f.x; bi = idx; }
      if (f.y > best) { best = f.y; bi = idx + 1; }
    }
  }
  for (int i = nvec * 8 + threadIdx.x; i < vocab; i += blockDim.x) {
    float f = bf2f(row[i]);
    if (f > best) { best = f; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sb[w] = best; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sb[k] > best || (sb[k] == best && si[k] < bi)) { best = sb[k]; bi = si[k]; }
    out[r] = bi;
  }
}

int argmax_rows(const bf16* logits, int rows, int vocab, int* out, cudaStream_t st) {
  if (rows <= 0) return 0;
  argmax_kernel<<<rows, 512, 0, st>>>(logits, vocab, out);
  return check_launch("argmax");
}

// ----------------------------------------------------------- commit sampled tokens
// The sampled token of an emitting sequence becomes its next input:
// token_hist[row][start + n_new] = sampled[emit].
__global__ void commit_tokens_kernel(const int* __restrict__ seq_info, int n_seqs, const int* __restrict__ sampled,
                                     int* __restrict__ token_hist, int max_seq_len) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seqs) return;
  const int* si = seq_info + 5 * s;
  const int emit = si[4];
  if (emit < 0) return;
  const int pos = si[1] + si[2];
  if (pos < max_seq_len) token_hist[(size_t)si[0] * max_seq_len + pos] = sampled[emit];
}

int commit_tokens(const int* seq_info, int n_seqs, const int* sampled, int* token_hist, int max_seq_len,
                  cudaStream_t st) {
  if (n_seqs <= 0) return 0;
  commit_tokens_kernel<<<(n_seqs + 127) / 128, 128, 0, st>>>(seq_info, n_seqs, sampled, token_hist, max_seq_len);
  return check_launch("commit_tokens");
}

}  // namespace gllm
