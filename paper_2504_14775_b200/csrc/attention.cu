// Mixed-batch paged attention: chunked-prefill chunks and decodes in ONE launch.
//
// Work item = (sequence, query tile, kv head). A query tile holds up to
// QT = 64 / G query tokens of one sequence times the G query heads that share
// the kv head (GQA), i.e. up to 64 (token, head) rows; a decode is one tile of
// G rows. Each CTA streams the sequence's K/V from the paged cache
// ([page][kv_head][slot][hd]) in 32-key blocks through a cp.async double
// buffer (16-byte loads, pages resolved through the device block table), keeps
// an fp32 online softmax per row, and writes the normalised output in bf16.
// Causal: query at absolute position p sees keys 0..p (its prefix plus the
// chunk's own earlier tokens).
//
// Work list (int32 x 2 per item, built by the host packer): (seq index, q_start).
#include <float.h>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

constexpr int HD = 128;
constexpr int KB = 32;          // keys per block
constexpr int KPAD = HD + 8;    // bf16 row pitch in smem (conflict-free 16 B loads)
constexpr int MAX_ROWS = 64;
constexpr int ATT_THREADS = 256;
constexpr int NW = ATT_THREADS / 32;
constexpr int RPW = MAX_ROWS / NW;  // rows per warp

struct AttnSmem {
  float q[MAX_ROWS][HD];
  bf16 k[2][KB][KPAD];
  bf16 v[2][KB][KPAD];
  float p[MAX_ROWS][KB];
};

GLLM_DEVICE void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
GLLM_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GLLM_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(ATT_THREADS)
attn_paged_kernel(const bf16* __restrict__ qkv, const int* __restrict__ seq_info, const int* __restrict__ work,
                  const int* __restrict__ block_table, int mpr, const bf16* __restrict__ k_cache,
                  const bf16* __restrict__ v_cache, int n_heads, int n_kv, int page_size, float scale_log2,
                  bf16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  AttnSmem& sm = *reinterpret_cast<AttnSmem*>(smem_raw);
  const int item = blockIdx.x;
  const int kvh = blockIdx.y;
  const int sidx = work[2 * item];
  const int q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int row_id = si[0], start = si[1], n_new = si[2], tok_off = si[3];
  const int G = n_heads / n_kv;
  const int QT = MAX_ROWS / G;
  const int nq = min(QT, n_new - q0);
  const int R = nq * G;
  const int kv_len = start + q0 + nq;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* table = block_table + (size_t)row_id * mpr;

  // Q rows -> smem fp32, pre-scaled so softmax uses exp2.
  for (int i = threadIdx.x; i < R * (HD / 8); i += ATT_THREADS) {
    const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
    const int qi = r / G, gh = r % G;
    const uint4 u = *reinterpret_cast<const uint4*>(qkv + (size_t)(tok_off + q0 + qi) * qkv_w + (kvh * G + gh) * HD + c);
    uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(a[j]);
      sm.q[r][c + 2 * j] = f.x * scale_log2;
      sm.q[r][c + 2 * j + 1] = f.y * scale_log2;
    }
  }

  const size_t head_stride = (size_t)page_size * HD;  // one (page, kv_head) block
  auto load_block = [&](int blk, int buf) {
    // 32 keys x 16 chunks of 16 B for K and for V.
#pragma unroll
    for (int i = 0; i < (KB * HD / 8) / ATT_THREADS; ++i) {
      const int idx = threadIdx.x + i * ATT_THREADS;
      const int kk = idx >> 4, c = (idx & 15) * 8;
      int key = blk * KB + kk;
      if (key >= kv_len) key = kv_len - 1;  // clamp: duplicated key is masked below
      const int page = table[key / page_size];
      const size_t off = ((size_t)page * n_kv + kvh) * head_stride + (size_t)(key % page_size) * HD + c;
      cp_async16(&sm.k[buf][kk][c], k_cache + off);
      cp_async16(&sm.v[buf][kk][c], v_cache + off);
    }
    cp_async_commit();
  };

  const int rows_per_warp = (R + NW - 1) / NW;  // rows r = warp + NW*i
  float m_run[RPW], l_run[RPW], acc[RPW][4];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    m_run[i] = -FLT_MAX;
    l_run[i] = 0.f;
    acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  }

  const int n_blocks = (kv_len + KB - 1) / KB;
  load_block(0, 0);
  for (int b = 0; b < n_blocks; ++b) {
    const int buf = b & 1;
    if (b + 1 < n_blocks) {
      load_block(b + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- scores: lane j owns key (b*KB + j); hold its K row in registers.
    const int key = b * KB + lane;
    uint32_t kr[HD / 2];
    {
      const uint4* kp = reinterpret_cast<const uint4*>(&sm.k[buf][lane][0]);
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        uint4 u = kp[c];
        kr[4 * c] = u.x; kr[4 * c + 1] = u.y; kr[4 * c + 2] = u.z; kr[4 * c + 3] = u.w;
      }
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      if (i >= rows_per_warp) break;
      const int r = warp + NW * i;
      if (r >= R) break;
      const int qpos = start + q0 + r / G;
      const float4* qp = reinterpret_cast<const float4*>(&sm.q[r][0]);
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < HD / 4; ++c) {
        const float4 qv = qp[c];
        const float2 k0 = unpack_bf16x2(kr[2 * c]), k1 = unpack_bf16x2(kr[2 * c + 1]);
        s = fmaf(qv.x, k0.x, s); s = fmaf(qv.y, k0.y, s); s = fmaf(qv.z, k1.x, s); s = fmaf(qv.w, k1.y, s);
      }
      if (key > qpos || key >= kv_len) s = -FLT_MAX;
      const float mb = warp_max(s);
      const float m_new = fmaxf(m_run[i], mb);
      const float p = (s == -FLT_MAX) ? 0.f : exp2f(s - m_new);
      const float corr = (m_run[i] == -FLT_MAX) ? 0.f : exp2f(m_run[i] - m_new);
      l_run[i] = l_run[i] * corr + warp_sum(p);
      m_run[i] = m_new;
      acc[i][0] *= corr; acc[i][1] *= corr; acc[i][2] *= corr; acc[i][3] *= corr;
      sm.p[r][lane] = p;
    }
    __syncwarp();
    // ---- O += P V: lane owns dims [4*lane, 4*lane+4) of each of its rows.
#pragma unroll 4
    for (int j = 0; j < KB; ++j) {
      const uint2 vv = *reinterpret_cast<const uint2*>(&sm.v[buf][j][4 * lane]);
      const float2 v0 = unpack_bf16x2(vv.x), v1 = unpack_bf16x2(vv.y);
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        if (i >= rows_per_warp) break;
        const int r = warp + NW * i;
        if (r >= R) break;
        const float p = sm.p[r][j];
        acc[i][0] = fmaf(p, v0.x, acc[i][0]); acc[i][1] = fmaf(p, v0.y, acc[i][1]);
        acc[i][2] = fmaf(p, v1.x, acc[i][2]); acc[i][3] = fmaf(p, v1.y, acc[i][3]);
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    if (i >= rows_per_warp) break;
    const int r = warp + NW * i;
    if (r >= R) break;
    const int qi = r / G, gh = r % G;
    const float inv = l_run[i] > 0.f ? 1.f / l_run[i] : 0.f;
    bf16* o = out + (size_t)(tok_off + q0 + qi) * (n_heads * HD) + (kvh * G + gh) * HD + 4 * lane;
    *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16x2(acc[i][0] * inv, acc[i][1] * inv),
                                              pack_bf16x2(acc[i][2] * inv, acc[i][3] * inv));
  }
}

int attention_q_tile(int n_heads, int n_kv) { return MAX_ROWS / (n_heads / n_kv); }

int attention_paged(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                    int mpr, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int head_dim,
                    int page_size, bf16* out, cudaStream_t st) {
  if (n_work <= 0) return 0;
  if (head_dim != HD) return set_error(GLLM_ERR_INVALID, "attention supports head_dim 128 only (got %d)", head_dim);
  if (n_heads % n_kv || n_heads / n_kv > MAX_ROWS) return set_error(GLLM_ERR_INVALID, "bad GQA grouping");
  static bool attr = false;
  const int smem = (int)sizeof(AttnSmem);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_paged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attention smem attribute");
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  dim3 grid(n_work, n_kv);
  attn_paged_kernel<<<grid, ATT_THREADS, smem, st>>>(qkv, seq_info, work, block_table, mpr, k_cache, v_cache, n_heads,
                                                     n_kv, page_size, scale_log2, out);
  return check_launch("attention_paged");
}

}  // namespace gllm
