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
//  * prefill role (tensor cores): 128 (token, head) rows of one chunk
//    (QT = 128/G tokens x the G heads sharing the kv head) against its cached
//    prefix + its own earlier tokens in 64-key blocks. S = Q.K^T and O += P.V
//    are tcgen05.mma (M=128) with S and O accumulating in TMEM; each thread
//    owns one row (TMEM lane), so the causal mask and online softmax are
//    thread-local. Q/K/V/P are staged in 128B-swizzled smem (K-major for Q, K,
//    P; MN-major descriptor for V, which stays [key][dim] as the cache holds
//    it). K blocks are double-buffered with cp.async (prefetched two blocks
//    ahead), V single-buffered so two CTAs fit per SM; O is rescaled in TMEM only when a row's max grows by >8
//    (log2 units), the exact "lazy rescale" form of online softmax.
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
constexpr int PM = 128;        // query rows per CTA (MMA M)
constexpr int PBK = 64;        // keys per block (MMA N of S, K of P.V)
constexpr int TMEM_COLS = 256; // S: cols [0,64), O: cols [128,256)
constexpr float RESCALE_TH = 8.f;

struct PrefillSmem {
  __align__(1024) uint8_t q[2][PM * 128];        // two 64-dim halves, SW128 K-major
  __align__(1024) uint8_t k[2][2][PBK * 128];    // [buf][half]
  __align__(1024) uint8_t v[2][PBK * 128];       // [half] (single buffer: keeps 2 CTAs/SM)
  __align__(1024) uint8_t p[PM * 128];           // P [128 rows][64 keys] bf16, SW128 K-major
  uint64_t s_bar, pv_bar;
  uint32_t tmem_base;
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
      // Slots past kv_len hold stale pool bytes (possibly NaN/Inf): skip, never multiply by 0.
      if (t >= keys_here) continue;
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

// One 128-row query tile of a prefill chunk on the tensor cores (see file header).
template <int G>
__device__ __forceinline__ void prefill_role(uint8_t* smem_raw, const bf16* __restrict__ qkv, int tok_off, int start,
                                             int q0, int nq, const int* __restrict__ table,
                                             const bf16* __restrict__ k_cache, const bf16* __restrict__ v_cache,
                                             int n_heads, int n_kv, int kvh, int page_size, float scale_log2,
                                             bf16* __restrict__ out) {
  PrefillSmem& sm = *reinterpret_cast<PrefillSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int R = nq * G;
  const int kv_len = start + q0 + nq;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;
  const size_t head_stride = (size_t)page_size * HD;
  const int nb = (kv_len + PBK - 1) / PBK;

  if (tid == 0) {
    mbar_init(&sm.s_bar, 1);
    mbar_init(&sm.pv_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&sm.tmem_base, TMEM_COLS);

  // Q tile -> swizzled smem (rows >= R zero-filled).
  for (int i = tid; i < PM * 16; i += ATT_THREADS) {
    const int r = i >> 4, c16 = i & 15, half = c16 >> 3, c = c16 & 7;
    uint8_t* dst = sm.q[half] + sw128_off(r, c);
    if (r < R) {
      const int qi = r / G, gh = r % G;
      cp_async16(dst, qkv + (size_t)(tok_off + q0 + qi) * qkv_w + (kvh * G + gh) * HD + half * 64 + c * 8);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
  auto load_kv = [&](const bf16* cache, uint8_t (*buf)[PBK * 128], int blk) {
    // 64 keys x 16 chunks of 16 B; 8 per thread
#pragma unroll
    for (int j = 0; j < (PBK * 16) / ATT_THREADS; ++j) {
      const int i = tid + j * ATT_THREADS;
      const int kk = i >> 4, c16 = i & 15, half = c16 >> 3, c = c16 & 7;
      int key = blk * PBK + kk;
      if (key >= kv_len) key = kv_len - 1;  // clamped duplicate, masked in softmax
      const int page = table[key / page_size];
      const bf16* src = cache + ((size_t)page * n_kv + kvh) * head_stride + (size_t)(key % page_size) * HD + half * 64 + c * 8;
      cp_async16(buf[half] + sw128_off(kk, c), src);
    }
  };
  // prologue groups: [Q, K0], [K1]
  load_kv(k_cache, sm.k[0], 0);
  cp_async_commit();
  if (nb > 1) load_kv(k_cache, sm.k[1], 1);
  cp_async_commit();
  cp_async_wait<1>();
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t t_s = tmem, t_o = tmem + 128;
  constexpr uint32_t idesc_s = idesc_bf16_f32(PM, PBK);
  constexpr uint32_t idesc_o = idesc_bf16_f32(PM, HD, /*b_mn_major=*/true);

  auto issue_s = [&](int blk) {
    const int b = blk & 1;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int half = kk >> 2;
      const uint64_t da = smem_desc_sw128(sm.q[half]) + 2 * (kk & 3);
      const uint64_t db = smem_desc_sw128(sm.k[b][half]) + 2 * (kk & 3);
      mma_bf16_ss(t_s, da, db, idesc_s, kk > 0 ? 1u : 0u);
    }
    mma_commit(&sm.s_bar);
  };
  if (tid == 0) issue_s(0);

  // per-row state: this thread owns TMEM lane / query row `tid`
  const int row = tid;
  const int qpos = start + q0 + (row < R ? row / G : nq - 1);
  float m_ref = -FLT_MAX, l_sum = 0.f;

  for (int j = 0; j < nb; ++j) {
    mbar_wait(&sm.s_bar, j & 1);
    tc_fence_after();
    uint32_t s_raw[2][32];
    tmem_ld_32x32b_x32(t_s + ((uint32_t)(warp * 32) << 16), s_raw[0]);
    tmem_ld_32x32b_x32(t_s + ((uint32_t)(warp * 32) << 16) + 32, s_raw[1]);
    tmem_ld_wait();
    float s[PBK];
    float mb = -FLT_MAX;
#pragma unroll
    for (int c = 0; c < PBK; ++c) {
      const int kpos = j * PBK + c;
      float x = __uint_as_float(s_raw[c >> 5][c & 31]) * scale_log2;
      x = (kpos > qpos || kpos >= kv_len) ? -FLT_MAX : x;
      s[c] = x;
      mb = fmaxf(mb, x);
    }
    if (j > 0) mbar_wait(&sm.pv_bar, (j - 1) & 1);  // P smem free, O stable, V buffer free
    tc_fence_after();
    load_kv(v_cache, sm.v, j);
    cp_async_commit();
    // prefetch K for block j+2 into the buffer S_j just finished reading
    if (j + 2 < nb) load_kv(k_cache, sm.k[j & 1], j + 2);
    cp_async_commit();
    // lazy rescale: keep the reference max unless this block exceeds it by > RESCALE_TH.
    // The decision is per row, but tcgen05.ld/st are warp-collective, so the TMEM
    // round trip runs for the whole warp whenever any of its rows rescales.
    const bool grow = mb > m_ref + RESCALE_TH || m_ref == -FLT_MAX;
    float corr = 1.f;
    if (grow) {
      corr = (m_ref == -FLT_MAX) ? 0.f : exp2f(m_ref - mb);
      l_sum *= corr;
      m_ref = mb;
    }
    if (j > 0 && __any_sync(0xffffffffu, grow && corr != 1.f)) {
#pragma unroll
      for (int c = 0; c < HD; c += 32) {
        uint32_t o[32];
        const uint32_t ta = t_o + ((uint32_t)(warp * 32) << 16) + c;
        tmem_ld_32x32b_x32(ta, o);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
        tmem_st_32x32b_x32(ta, o);
      }
      tmem_st_wait();
    }
    // P = exp2(s - m_ref) -> bf16, swizzled K-major row of 64 keys
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float pv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float x = s[c * 8 + e];
        pv[e] = (x == -FLT_MAX) ? 0.f : exp2f(x - m_ref);
        l_sum += pv[e];
      }
      *reinterpret_cast<uint4*>(sm.p + sw128_off(row, c)) =
          make_uint4(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]), pack_bf16x2(pv[4], pv[5]),
                     pack_bf16x2(pv[6], pv[7]));
    }
    cp_async_wait<1>();  // V_j and K_{j+1} have landed (this thread's copies); K_{j+2} may fly
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < PBK / 16; ++kk) {
        const uint64_t da = smem_desc_sw128(sm.p) + 2 * kk;
        const uint64_t db = smem_desc_sw128_mn(sm.v[0] + kk * 2048, PBK * 128);
        mma_bf16_ss(t_o, da, db, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&sm.pv_bar);
      if (j + 1 < nb) issue_s(j + 1);
    }
  }
  mbar_wait(&sm.pv_bar, (nb - 1) & 1);
  tc_fence_after();
  const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
  const int qi = row / G, gh = row % G;
  bf16* o = out + (size_t)(tok_off + q0 + qi) * (n_heads * HD) + (kvh * G + gh) * HD;
#pragma unroll
  for (int c = 0; c < HD; c += 32) {
    uint32_t r32[32];
    tmem_ld_32x32b_x32(t_o + ((uint32_t)(warp * 32) << 16) + c, r32);  // warp-collective: all lanes
    tmem_ld_wait();
    if (row < R) {
#pragma unroll
      for (int e = 0; e < 32; e += 8)
        *reinterpret_cast<uint4*>(o + c + e) = make_uint4(
            pack_bf16x2(__uint_as_float(r32[e]) * inv, __uint_as_float(r32[e + 1]) * inv),
            pack_bf16x2(__uint_as_float(r32[e + 2]) * inv, __uint_as_float(r32[e + 3]) * inv),
            pack_bf16x2(__uint_as_float(r32[e + 4]) * inv, __uint_as_float(r32[e + 5]) * inv),
            pack_bf16x2(__uint_as_float(r32[e + 6]) * inv, __uint_as_float(r32[e + 7]) * inv));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TMEM_COLS);
}


template <int G>
__global__ void __launch_bounds__(ATT_THREADS, 2)
attn_mixed_kernel(const bf16* __restrict__ qkv, const int* __restrict__ seq_info, const int* __restrict__ work,
                  const int* __restrict__ block_table, int mpr, const bf16* __restrict__ k_cache,
                  const bf16* __restrict__ v_cache, int n_heads, int n_kv, int page_size, float scale_log2,
                  bf16* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  uint8_t* smem_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int item = blockIdx.x;
  const int kvh = blockIdx.y;
  const int sidx = work[2 * item];
  const int q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int row_id = si[0], start = si[1], n_new = si[2], tok_off = si[3];
  const int* table = block_table + (size_t)row_id * mpr;
  if (n_new == 1) {
    constexpr int LPK = G <= 4 ? 8 : 16;
    decode_role<G, LPK>(smem_raw, qkv, tok_off + q0, start + q0 + 1, table, k_cache, v_cache, n_heads, n_kv, kvh,
                        page_size, scale_log2, out);
  } else {
    const int nq = min(PM / G, n_new - q0);
    prefill_role<G>(smem_raw, qkv, tok_off, start, q0, nq, table, k_cache, v_cache, n_heads, n_kv, kvh, page_size,
                    scale_log2, out);
  }
}

// Query tokens per prefill work item (a decode, n_new == 1, is always one item).
int attention_q_tile(int n_heads, int n_kv) { return PM / (n_heads / n_kv); }

template <int G>
static int launch_attn(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                       int mpr, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int page_size,
                       float scale_log2, bf16* out, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_mixed_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ATT_SMEM + 1024);
    if (e != cudaSuccess) return set_cuda_error(e, "attention smem attribute");
    attr = true;
  }
  dim3 grid(n_work, n_kv);
  attn_mixed_kernel<G><<<grid, ATT_THREADS, ATT_SMEM + 1024, st>>>(qkv, seq_info, work, block_table, mpr, k_cache, v_cache,
                                                            n_heads, n_kv, page_size, scale_log2, out);
  return check_launch("attention_mixed");
}

int attention_paged(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                    int mpr, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int head_dim,
                    int page_size, bf16* out, cudaStream_t st) {
  if (n_work <= 0) return 0;
  if (head_dim != HD) return set_error(GLLM_ERR_INVALID, "attention supports head_dim 128 only (got %d)", head_dim);
  if (n_heads % n_kv) return set_error(GLLM_ERR_INVALID, "bad GQA grouping");
  if (page_size < 1 || page_size > 16) return set_error(GLLM_ERR_INVALID, "page_size must be in [1, 16]");
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
