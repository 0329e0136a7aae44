// Mixed-batch paged attention: chunked-prefill chunks and decodes in ONE launch.
//
// Work item = (sequence, q_start) x kv head (grid.y). The role is uniform per CTA:
//
//  * decode role (the item has one query token): the CTA streams the sequence's
//    K and V pages for its kv head straight from the paged cache with
//    cp.async.bulk (the 1-D TMA engine): one (page, kv head) block is a
//    contiguous page_size*256 B run, so each page costs two bulk copies and no
//    address math per element. Every warp owns a 2-stage page ring guarded by
//    mbarriers and walks pages w, w+4, ...; inside a warp LPK lanes cooperate on
//    one key (128-bit smem reads, shuffle-reduced dot products) and each key
//    group keeps its own online-softmax state, merged by shuffles and then
//    across warps through shared memory. HBM-bound by design.
//  * prefill role: up to 64 (token, head) rows of one chunk (QT = 64/G tokens x
//    the G heads sharing the kv head), K/V staged in 32-key blocks with a
//    cp.async double buffer, fp32 online softmax, causal mask against the
//    chunk's own earlier tokens and its cached prefix.
//
// Cache layout [page][kv_head][slot][hd] (stage.py); pages resolved through the
// device block table. Work list: int32 (seq index, q_start) pairs, host-packed.
#include <float.h>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

constexpr int HD = 128;
constexpr int ATT_THREADS = 128;
constexpr int NWARP = ATT_THREADS / 32;

// ---------------------------------------------------------------- prefill role
constexpr int KB = 32;          // keys per block
constexpr int KPAD = HD + 8;    // bf16 row pitch in smem (conflict-free 16 B loads)
constexpr int MAX_ROWS = 64;
constexpr int RPW = MAX_ROWS / NWARP;  // rows per warp

struct PrefillSmem {
  float q[MAX_ROWS][HD];
  bf16 k[2][KB][KPAD];
  bf16 v[2][KB][KPAD];
  float p[MAX_ROWS][KB];
};

// ---------------------------------------------------------------- decode role
constexpr int DEC_STAGES = 2;
constexpr int MAX_PAGE_BYTES = 16 * HD * 2;  // page_size <= 16 for the bulk ring
struct DecodeSmem {
  __align__(128) uint8_t kv[NWARP][DEC_STAGES][2][MAX_PAGE_BYTES];
  uint64_t full[NWARP][DEC_STAGES];
  float merge_m[NWARP][8];
  float merge_l[NWARP][8];
  float merge_acc[NWARP][8][HD];
};

constexpr size_t ATT_SMEM = sizeof(PrefillSmem) > sizeof(DecodeSmem) ? sizeof(PrefillSmem) : sizeof(DecodeSmem);

GLLM_DEVICE void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
GLLM_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GLLM_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

GLLM_DEVICE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
GLLM_DEVICE void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// G query heads share the kv head; LPK lanes cooperate on one key (DPL dims each).
template <int G, int LPK>
__device__ __forceinline__ void decode_role(uint8_t* smem_raw, const bf16* __restrict__ qkv, int tok, int kv_len,
                                            const int* __restrict__ table, const bf16* __restrict__ k_cache,
                                            const bf16* __restrict__ v_cache, int n_heads, int n_kv, int kvh,
                                            int page_size, float scale_log2, bf16* __restrict__ out) {
  constexpr int DPL = HD / LPK;       // dims per lane (16 or 8)
  constexpr int KPI = 32 / LPK;       // keys per warp iteration
  DecodeSmem& sm = *reinterpret_cast<DecodeSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane % LPK, grp = lane / LPK;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;
  const uint32_t page_bytes = (uint32_t)page_size * HD * 2;
  const size_t head_stride = (size_t)page_size * HD;
  const int n_pages = (kv_len + page_size - 1) / page_size;

  if (lane == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) mbar_init(&sm.full[warp][s], 1);
    fence_barrier_init();
  }
  __syncwarp();

  auto issue = [&](int p, int s) {
    const int page = table[p];
    const size_t off = ((size_t)page * n_kv + kvh) * head_stride;
    mbar_arrive_expect_tx(&sm.full[warp][s], 2 * page_bytes);
    bulk_g2s(sm.kv[warp][s][0], k_cache + off, page_bytes, &sm.full[warp][s]);
    bulk_g2s(sm.kv[warp][s][1], v_cache + off, page_bytes, &sm.full[warp][s]);
  };
  // prologue: first DEC_STAGES pages of this warp in flight
  if (lane == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) {
      const int p = warp + s * NWARP;
      if (p < n_pages) issue(p, s);
    }
  }

  // q slice of the G heads for this lane's dims, fp32, pre-scaled for exp2.
  float q[G][DPL];
  const bf16* qrow = qkv + (size_t)tok * qkv_w + (kvh * G) * HD + sub * DPL;
#pragma unroll
  for (int h = 0; h < G; ++h) {
#pragma unroll
    for (int c = 0; c < DPL; c += 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(qrow + h * HD + c);
      const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(a[j]);
        q[h][c + 2 * j] = f.x * scale_log2;
        q[h][c + 2 * j + 1] = f.y * scale_log2;
      }
    }
  }
  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m[h] = -FLT_MAX;
    l[h] = 0.f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[h][d] = 0.f;
  }

  int it = 0;
  for (int p = warp; p < n_pages; p += NWARP, ++it) {
    const int s = it % DEC_STAGES;
    mbar_wait(&sm.full[warp][s], (uint32_t)((it / DEC_STAGES) & 1));
    const bf16* kp = reinterpret_cast<const bf16*>(sm.kv[warp][s][0]);
    const bf16* vp = reinterpret_cast<const bf16*>(sm.kv[warp][s][1]);
    const int keys_here = min(page_size, kv_len - p * page_size);
    // scores for this lane group's keys of the page
    constexpr int MAXK = 16 / KPI > 0 ? 16 / KPI : 1;  // keys per lane group for page_size 16
    float sc[MAXK][G];
#pragma unroll
    for (int kk = 0; kk < MAXK; ++kk) {
      const int t = kk * KPI + grp;
      const bool valid = t < keys_here;
      float part[G];
#pragma unroll
      for (int h = 0; h < G; ++h) part[h] = 0.f;
      if (t < page_size) {
        const bf16* kr = kp + t * HD + sub * DPL;
#pragma unroll
        for (int c = 0; c < DPL; c += 8) {
          const uint4 u = *reinterpret_cast<const uint4*>(kr + c);
          const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(a[j]);
#pragma unroll
            for (int h = 0; h < G; ++h) part[h] = fmaf(q[h][c + 2 * j + 1], f.y, fmaf(q[h][c + 2 * j], f.x, part[h]));
          }
        }
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
#pragma unroll
        for (int o = LPK / 2; o > 0; o >>= 1) part[h] += __shfl_xor_sync(0xffffffffu, part[h], o);
        sc[kk][h] = valid ? part[h] : -FLT_MAX;
      }
    }
    // one rescale per page, then accumulate P.V for this group's keys
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float mx = m[h];
#pragma unroll
      for (int kk = 0; kk < MAXK; ++kk) mx = fmaxf(mx, sc[kk][h]);
      const float corr = (m[h] == -FLT_MAX) ? 0.f : exp2f(m[h] - mx);
      m[h] = mx;
      l[h] *= corr;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[h][d] *= corr;
#pragma unroll
      for (int kk = 0; kk < MAXK; ++kk) sc[kk][h] = (sc[kk][h] == -FLT_MAX) ? 0.f : exp2f(sc[kk][h] - mx);
    }
#pragma unroll
    for (int kk = 0; kk < MAXK; ++kk) {
      const int t = kk * KPI + grp;
      if (t >= page_size) continue;
      const bf16* vr = vp + t * HD + sub * DPL;
      float vv[DPL];
#pragma unroll
      for (int c = 0; c < DPL; c += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(vr + c);
        const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(a[j]);
          vv[c + 2 * j] = f.x;
          vv[c + 2 * j + 1] = f.y;
        }
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float pr = sc[kk][h];
        l[h] += pr;
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[h][d] = fmaf(pr, vv[d], acc[h][d]);
      }
    }
    __syncwarp();
    const int pn = p + DEC_STAGES * NWARP;
    if (lane == 0 && pn < n_pages) {
      fence_proxy_async();
      issue(pn, s);
    }
  }

  // merge the KPI key groups of this warp (lanes sub, sub+LPK, ...)
#pragma unroll
  for (int o = LPK; o < 32; o <<= 1) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float mo = __shfl_xor_sync(0xffffffffu, m[h], o);
      const float lo = __shfl_xor_sync(0xffffffffu, l[h], o);
      const float mn = fmaxf(m[h], mo);
      const float ca = (m[h] == -FLT_MAX) ? 0.f : exp2f(m[h] - mn);
      const float cb = (mo == -FLT_MAX) ? 0.f : exp2f(mo - mn);
      l[h] = l[h] * ca + lo * cb;
#pragma unroll
      for (int d = 0; d < DPL; ++d) {
        const float ao = __shfl_xor_sync(0xffffffffu, acc[h][d], o);
        acc[h][d] = acc[h][d] * ca + ao * cb;
      }
      m[h] = mn;
    }
  }
  // across warps through shared memory
  if (grp == 0) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      if (sub == 0) {
        sm.merge_m[warp][h] = m[h];
        sm.merge_l[warp][h] = l[h];
      }
#pragma unroll
      for (int d = 0; d < DPL; ++d) sm.merge_acc[warp][h][sub * DPL + d] = acc[h][d];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * HD; i += ATT_THREADS) {
    const int h = i / HD, d = i % HD;
    float mx = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) mx = fmaxf(mx, sm.merge_m[w][h]);
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
      const float mw = sm.merge_m[w][h];
      const float c = (mw == -FLT_MAX) ? 0.f : exp2f(mw - mx);
      num += sm.merge_acc[w][h][d] * c;
      den += sm.merge_l[w][h] * c;
    }
    out[(size_t)tok * (n_heads * HD) + (kvh * G + h) * HD + d] = f2bf(den > 0.f ? num / den : 0.f);
  }
}

__device__ __forceinline__ void prefill_role(uint8_t* smem_raw, const bf16* __restrict__ qkv, int tok_off,
                                             int start, int q0, int nq, const int* __restrict__ table,
                                             const bf16* __restrict__ k_cache, const bf16* __restrict__ v_cache,
                                             int n_heads, int n_kv, int kvh, int page_size, float scale_log2,
                                             bf16* __restrict__ out) {
  PrefillSmem& sm = *reinterpret_cast<PrefillSmem*>(smem_raw);
  const int G = n_heads / n_kv;
  const int R = nq * G;
  const int kv_len = start + q0 + nq;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

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
  const size_t head_stride = (size_t)page_size * HD;
  auto load_block = [&](int blk, int buf) {
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

  const int rows_per_warp = (R + NWARP - 1) / NWARP;
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
      const int r = warp + NWARP * i;
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
#pragma unroll 4
    for (int j = 0; j < KB; ++j) {
      const uint2 vv = *reinterpret_cast<const uint2*>(&sm.v[buf][j][4 * lane]);
      const float2 v0 = unpack_bf16x2(vv.x), v1 = unpack_bf16x2(vv.y);
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        if (i >= rows_per_warp) break;
        const int r = warp + NWARP * i;
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
    const int r = warp + NWARP * i;
    if (r >= R) break;
    const int qi = r / G, gh = r % G;
    const float inv = l_run[i] > 0.f ? 1.f / l_run[i] : 0.f;
    bf16* o = out + (size_t)(tok_off + q0 + qi) * (n_heads * HD) + (kvh * G + gh) * HD + 4 * lane;
    *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16x2(acc[i][0] * inv, acc[i][1] * inv),
                                              pack_bf16x2(acc[i][2] * inv, acc[i][3] * inv));
  }
}

template <int G>
__global__ void __launch_bounds__(ATT_THREADS, 2)
attn_mixed_kernel(const bf16* __restrict__ qkv, const int* __restrict__ seq_info, const int* __restrict__ work,
                  const int* __restrict__ block_table, int mpr, const bf16* __restrict__ k_cache,
                  const bf16* __restrict__ v_cache, int n_heads, int n_kv, int page_size, float scale_log2,
                  bf16* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int item = blockIdx.x;
  const int kvh = blockIdx.y;
  const int sidx = work[2 * item];
  const int q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int row_id = si[0], start = si[1], n_new = si[2], tok_off = si[3];
  const int* table = block_table + (size_t)row_id * mpr;
  const int QT = MAX_ROWS / G;
  const int nq = min(QT, n_new - q0);
  if (nq == 1 && page_size <= 16) {
    constexpr int LPK = G <= 4 ? 8 : 16;
    decode_role<G, LPK>(smem_raw, qkv, tok_off + q0, start + q0 + 1, table, k_cache, v_cache, n_heads, n_kv, kvh,
                        page_size, scale_log2, out);
  } else {
    prefill_role(smem_raw, qkv, tok_off, start, q0, nq, table, k_cache, v_cache, n_heads, n_kv, kvh, page_size,
                 scale_log2, out);
  }
}

int attention_q_tile(int n_heads, int n_kv) { return MAX_ROWS / (n_heads / n_kv); }

template <int G>
static int launch_attn(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                       int mpr, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int page_size,
                       float scale_log2, bf16* out, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_mixed_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ATT_SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "attention smem attribute");
    attr = true;
  }
  dim3 grid(n_work, n_kv);
  attn_mixed_kernel<G><<<grid, ATT_THREADS, ATT_SMEM, st>>>(qkv, seq_info, work, block_table, mpr, k_cache, v_cache,
                                                            n_heads, n_kv, page_size, scale_log2, out);
  return check_launch("attention_mixed");
}

int attention_paged(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                    int mpr, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int head_dim,
                    int page_size, bf16* out, cudaStream_t st) {
  if (n_work <= 0) return 0;
  if (head_dim != HD) return set_error(GLLM_ERR_INVALID, "attention supports head_dim 128 only (got %d)", head_dim);
  if (n_heads % n_kv) return set_error(GLLM_ERR_INVALID, "bad GQA grouping");
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  switch (n_heads / n_kv) {
    case 1: return launch_attn<1>(qkv, seq_info, work, n_work, block_table, mpr, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st);
    case 2: return launch_attn<2>(qkv, seq_info, work, n_work, block_table, mpr, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st);
    case 4: return launch_attn<4>(qkv, seq_info, work, n_work, block_table, mpr, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st);
    case 5: return launch_attn<5>(qkv, seq_info, work, n_work, block_table, mpr, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st);
    case 8: return launch_attn<8>(qkv, seq_info, work, n_work, block_table, mpr, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st);
    default: return set_error(GLLM_ERR_INVALID, "unsupported GQA group %d", n_heads / n_kv);
  }
}

}  // namespace gllm
