// Mixed-batch paged attention: chunked-prefill chunks and decodes of one micro-batch,
// issued together (one call; two concurrent role launches, see AttnRoles).
//
// Work item = (sequence, q_start) x kv head (grid.x). The role is uniform per CTA:
//
//  * decode role (the item has one query token; `attn_decode_kernel<G, NW>`): NW = 4 or 8
//    warps each walk pages w, w+NW, ... of the sequence through a 3-stage ring filled by 2-D
//    TMA (one box per page and 64-dim half, 128B-swizzled so the ldmatrix fragment loads are
//    conflict-free); mma.sync m16n8k16 in transposed form (this GEMV-shaped work is too
//    small for a 128-row tcgen05 tile): S^T = K.Q^T and O^T += V^T.P^T with 16 keys / dims as
//    the MMA rows and the G <= 8 query heads as its 8 columns, online softmax across the
//    warp's 8 lane groups, warps merged through shared memory. HBM-bound by design. Pages before the last
//    one are fetched before griddepcontrol.wait (they predate this forward); a decode-only
//    launch of few long sequences splits each sequence's pages over a cluster of up to 4
//    CTAs whose partial (max, sum, O) rank 0 merges through distributed shared memory.
//  * prefill role (tensor cores, its own launch `attn_prefill_kernel`): a work
//    item is 2 x 128 (token, head) query rows of one chunk (2 x 128/G tokens x
//    the G heads sharing the kv head), attended against the cached prefix plus
//    the chunk's own earlier tokens in 128-key blocks, FlashAttention-style and
//    warp-specialised: warp 8 streams K/V blocks from the paged cache with 2-D
//    TMA (one box per page and 64-dim half, 128B-swizzled) into a 5-slot ring, one
//    lane per page with the page ids read a block ahead; warp 9 issues every
//    tcgen05.mma (S = Q.K^T with Q, K from smem; O += P.V with P read straight from
//    TMEM, V as an MN-major smem operand); warps 0-3 and 4-7 run the online softmax
//    of query tile 0 and 1, one thread per TMEM lane (= query row), with the row's
//    128 scores in registers (one TMEM read, 3-input max, MUFU exp2): setmaxnreg
//    moves registers from the producer warpgroup (warps 8-11) to the softmax ones.
//    The two tiles ping-pong: while one tile's softmax runs on the CUDA cores the
//    tensor core computes the other tile's P.V and next S. S/P (aliased, P as packed
//    bf16 over S's first 64 columns) and O take all 512 TMEM columns; O is rescaled
//    in TMEM only when a row's max grows by more than 8 (log2 units), the exact
//    "lazy rescale" form of online softmax.
//
// Cache layout [page][kv_head][slot][hd] (stage.py); pages resolved through the
// device block table. Work list: int32 (seq index, q_start) pairs, host-packed.
#include <float.h>
#include <stddef.h>
#include <stdlib.h>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

constexpr int HD = 128;

// ---------------------------------------------------------------- prefill role
constexpr int PM = 128;          // query rows per tile (MMA M = TMEM lanes)
constexpr int PTILES = 2;        // query tiles per CTA, ping-ponged on the tensor core
constexpr int PBK = 128;         // keys per block (MMA N of S, MMA K of P.V)
constexpr int PRING = 5;         // K/V block ring (K_j, V_j, K_j+1, ...): 2.5 blocks of prefetch
// warps 0-7 softmax (tile = warp / 4), warp 8 TMA, warp 9 MMA, warps 10-11 idle: a whole third
// warpgroup so it can hand registers to the softmax warpgroups (setmaxnreg: 3 warps per SM
// sub-partition share its 512 registers per lane, 224 + 224 + 56)
constexpr int PF_THREADS = 384;
constexpr int PF_REG_SOFTMAX = 200, PF_REG_PRODUCER = 96;
// the softmax warpgroups' increase must fit in what the producer warpgroup releases (launch: 168 each)
static_assert(2 * (PF_REG_SOFTMAX - 168) <= 168 - PF_REG_PRODUCER, "setmaxnreg.inc would wait forever");
constexpr int PF_TMEM_COLS = 512;
constexpr float RESCALE_TH = 8.f;
constexpr uint32_t PF_BLK_BYTES = PBK * HD * 2;  // one K or V block: two 64-dim SW128 halves

struct PrefillSmem {
  __align__(1024) uint8_t q[PTILES][2][PM * 128];   // [tile][64-dim half], SW128 K-major
  __align__(1024) uint8_t kv[PRING][2][PBK * 128];  // [slot][64-dim half], key rows
  uint64_t kv_full[PRING], kv_empty[PRING];
  uint64_t s_full[PTILES], p_full[PTILES], o_full[PTILES];
  uint32_t tmem_base;
};

// Timing experiments only (wrong results): MMA K-steps issued per S block / per P.V block.
#ifndef GLLM_PF_S_STEPS
#define GLLM_PF_S_STEPS 8
#endif
#ifndef GLLM_PF_PV_STEPS
#define GLLM_PF_PV_STEPS 8
#endif
#ifndef GLLM_PF_LOAD_PAGES
#define GLLM_PF_LOAD_PAGES 64
#endif
constexpr int PF_S_STEPS = GLLM_PF_S_STEPS, PF_PV_STEPS = GLLM_PF_PV_STEPS, PF_LOAD_PAGES = GLLM_PF_LOAD_PAGES;

// Debug builds (-DGLLM_TRACE, tools/attn_trace.py): clock64 stamps (relative to the CTA's start)
// of the prefill pipeline's phases for the first PF_TRACE_CTAS CTAs and PF_TRACE_BLK key blocks.
#ifdef GLLM_TRACE
constexpr int PF_TRACE_CTAS = 148, PF_TRACE_BLK = 64, PF_TRACE_EV = 12;
__device__ unsigned int g_pf_trace[PF_TRACE_CTAS][PF_TRACE_BLK][PF_TRACE_EV];
#define PF_TRACE(l, ev)                                                                                   \
  do {                                                                                                    \
    const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x;                                             \
    if (lin < PF_TRACE_CTAS && (l) < PF_TRACE_BLK)                                                        \
      g_pf_trace[lin][(l)][(ev)] = (unsigned)(clock64() - t_cta0);                                        \
  } while (0)
// decode role: per CTA (first DEC_TRACE_CTAS), warp, page iteration: [wait start, page ready, page done]
constexpr int DEC_TRACE_CTAS = 296, DEC_TRACE_IT = 32;
__device__ unsigned int g_dec_trace[DEC_TRACE_CTAS][8][DEC_TRACE_IT][3];
#define DEC_TRACE(it, ev)                                                                                 \
  do {                                                                                                    \
    const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x;                                             \
    if (lin < DEC_TRACE_CTAS && (it) < DEC_TRACE_IT && lane == 0)                                         \
      g_dec_trace[lin][warp][(it)][(ev)] = (unsigned)(clock64() - t_cta0);                                \
  } while (0)
#else
#define PF_TRACE(l, ev) ((void)0)
#define DEC_TRACE(it, ev) ((void)0)
#endif

// ---------------------------------------------------------------- decode role
constexpr int DEC_STAGES = 3;
constexpr int MAX_PAGE_BYTES = 16 * HD * 2;  // page_size <= 16 for the bulk ring
template <int NW, int ST = DEC_STAGES>  // streaming warps per CTA, page-ring stages per warp
struct DecodeSmem {
  union {
    __align__(128) uint8_t kv[NW][ST][2][MAX_PAGE_BYTES];
    float merge_acc[NW][8][HD];  // reused after every page has been consumed
  };
  uint64_t full[NW][ST];
  float merge_m[NW][8];
  float merge_l[NW][8];
};
// KV split over a cluster (decode-only launches): every rank's (max, sum, unnormalised O) of its
// page range lands in rank 0's copy of this block (DSMEM), placed after DecodeSmem.
constexpr int DEC_MAX_SPLIT = 4;
struct DecodeRed {
  float acc[DEC_MAX_SPLIT][8][HD];
  float m[DEC_MAX_SPLIT][8];
  float l[DEC_MAX_SPLIT][8];
};


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

GLLM_DEVICE void mma_16816_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
GLLM_DEVICE void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// 8x8 b16 matrix in the mma fragment layout (thread: row lane / 4, columns 2 (lane % 4) + {0, 1})
// -> its transpose in the same layout
GLLM_DEVICE uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
GLLM_DEVICE void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// Decode role: one query token, the G query heads of kv head `kvh` as the 8 columns of
// m16n8k16 MMAs. Each warp streams its pages (w, w+NW, ...) of [p_begin, p_end) through an
// ST-stage TMA ring and per 16-key page issues 8 HMMA for S^T = K.Q^T and 8 for
// O^T += V^T.P^T (P^T moved from the S^T accumulators into B fragments by movmatrix), with
// the online softmax of each head across the lane groups holding its 16 keys. Warps merge
// through smem; with a KV split (csize > 1) the ranks of the cluster then merge through rank 0's
// DecodeRed.
template <int G, int NW, int ST = DEC_STAGES>
__device__ __forceinline__ void decode_role(uint8_t* smem_raw, const bf16* __restrict__ qkv, int tok, int kv_len,
                                            const int* __restrict__ table, const CUtensorMap* k_map,
                                            const CUtensorMap* v_map, int n_heads, int n_kv, int kvh,
                                            int page_size, float scale_log2, bf16* __restrict__ out,
                                            int csize = 1, int crank = 0) {
  static_assert(G <= 8, "decode tile holds up to 8 query heads per kv head");
#ifdef GLLM_TRACE
  const long long t_cta0 = clock64();
#endif
  constexpr int HALF_BYTES = 16 * 128;  // one 64-dim box of a 16-slot page (8-slot pages use half)
  DecodeSmem<NW, ST>& sm = *reinterpret_cast<DecodeSmem<NW, ST>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;
  const uint32_t page_bytes = (uint32_t)page_size * HD * 2;
  const int n_pages_all = (kv_len + page_size - 1) / page_size;
  // this rank's contiguous page range (the whole sequence without a split)
  const int p_begin = crank * n_pages_all / csize, n_pages = (crank + 1) * n_pages_all / csize;
  const int nblk = page_size / 8;    // 8-key MMA n-blocks per page (1 or 2)

  if (lane == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&sm.full[warp][s], 1);
    fence_barrier_init();
    if (warp == 0) {  // the tensor maps' descriptors, fetched once per CTA ahead of the first TMA
      tma_prefetch_desc(k_map);
      tma_prefetch_desc(v_map);
    }
  }
  __syncwarp();
  // One page of one kv head = page_size rows x 128 dims; two 64-dim TMA boxes per tensor,
  // landing 128B-swizzled (row r, 16B chunk c at r*128 + ((c ^ r%8) << 4)) so the ldmatrix
  // fragment loads below are bank-conflict free.
  auto issue_page = [&](int page, int s) {
    const int row0 = (page * n_kv + kvh) * page_size;
    mbar_arrive_expect_tx(&sm.full[warp][s], 2 * page_bytes);
    tma_load_2d(k_map, &sm.full[warp][s], sm.kv[warp][s][0], 0, row0);
    tma_load_2d(k_map, &sm.full[warp][s], sm.kv[warp][s][0] + HALF_BYTES, 64, row0);
    tma_load_2d(v_map, &sm.full[warp][s], sm.kv[warp][s][1], 0, row0);
    tma_load_2d(v_map, &sm.full[warp][s], sm.kv[warp][s][1] + HALF_BYTES, 64, row0);
  };
  // Pages before the last one hold keys of earlier forwards and their block-table entries are
  // unchanged in this forward (a decode's row was assigned when it was prefilled; seq_info and
  // work arrive by a plain host copy ahead of the forward), so they are fetched before
  // griddepcontrol.wait, overlapping the QKV GEMM. The last page holds this token's K/V, written
  // by that GEMM's epilogue (and may be newly appended to the table): it waits, as does Q.
  const int p_last = n_pages_all - 1;
  // lane s reads the block-table entry of the warp's s-th page: one parallel round trip instead
  // of ST dependent ones before the first TMA
  int pre_page = 0;
  if (lane < ST) {
    const int p = p_begin + warp + lane * NW;
    if (p < n_pages && p < p_last) pre_page = table[p];
  }
  for (int s = 0; s < ST; ++s) {
    const int p = p_begin + warp + s * NW;
    const int pg = __shfl_sync(0xffffffffu, pre_page, s);
    if (lane == 0 && p < n_pages && p < p_last) issue_page(pg, s);
  }
  pdl_wait();
  if (lane == 0) {
    for (int s = 0; s < ST; ++s) {
      const int p = p_begin + warp + s * NW;
      if (p < n_pages && p == p_last) issue_page(table[p], s);
    }
  }
  // Transposed form, so the MMA's M (16 rows) runs over keys and its N (8) over the G <= 8
  // query heads instead of padding G heads to 16 rows: S^T = K . Q^T (A = a 16-key x 16-dim K
  // block via ldmatrix, B = Q^T from registers) and O^T += V^T . P^T (A = V^T via
  // ldmatrix.trans, B = P^T moved from the S^T accumulator layout by movmatrix.trans): 16
  // m16n8k16 MMAs per 16-key page instead of 32. Thread (gid = lane / 4, tid = lane % 4) holds
  // keys gid and gid + 8 of heads 2 tid and 2 tid + 1.
  const int gid = lane >> 2, tid = lane & 3;
  const int h0 = 2 * tid;
  // Q^T as B fragments (heads >= G are zero), 8 k-steps of 16 dims: head gid, dims 2 tid (+8)
  uint32_t qb[8][2];
  {
    const bool live = gid < G;
    const bf16* qrow = qkv + (size_t)tok * qkv_w + (kvh * G + (live ? gid : 0)) * HD;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qb[kk][0] = live ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + h0) : 0u;
      qb[kk][1] = live ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + h0) : 0u;
    }
  }
  float o[8][4];  // O^T: 16-dim tile mt; (dim 16 mt + gid, heads h0 / h0 + 1), (dim + 8, ...)
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  float m_run[2] = {-FLT_MAX, -FLT_MAX}, l_run[2] = {0.f, 0.f};   // heads h0, h0 + 1
  const int j = lane >> 3, r = lane & 7;  // ldmatrix: this lane addresses row r of matrix j

  int it = 0;
  for (int p = p_begin + warp; p < n_pages; p += NW, ++it) {
    const int s = it % ST;
    DEC_TRACE(it, 0);
    mbar_wait(&sm.full[warp][s], (uint32_t)((it / ST) & 1));
    DEC_TRACE(it, 1);
    uint8_t* kp = sm.kv[warp][s][0];
    uint8_t* vp = sm.kv[warp][s][1];
    const int keys_here = min(page_size, kv_len - p * page_size);
    if (keys_here < page_size) {
      // stale slots past kv_len may hold NaN/Inf bytes: zero their V rows (0 * NaN would poison O)
      for (int i = lane; i < (page_size - keys_here) * 16; i += 32)
        *reinterpret_cast<uint4*>(vp + (i & 8 ? HALF_BYTES : 0) + (keys_here + i / 16) * 128 + (i & 7) * 16) =
            make_uint4(0, 0, 0, 0);
      __syncwarp();
    }
    // ---- S^T = K . Q^T: 8 k-steps of 16 dims; matrix j = (keys 8 (j & 1).., dims 8 (j >> 1)..);
    // even / odd k-steps in two accumulators (two dependent MMA chains of 4, not one of 8)
    float sc[4] = {0.f, 0.f, 0.f, 0.f}, sc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int key = (j & 1) * 8 + r;
      const int c = (kk & 3) * 2 + (j >> 1);          // 16B chunk within the 64-dim half
      uint32_t ka[4];
      ldsm_x4(ka, kp + (kk >> 2) * HALF_BYTES + (key < page_size ? key : 0) * 128 + ((c ^ r) << 4));
      if (nblk < 2) { ka[1] = 0u; ka[3] = 0u; }      // 8-slot pages: keys 8-15 do not exist
      mma_16816_bf16(kk & 1 ? sc2 : sc, ka, qb[kk][0], qb[kk][1]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) sc[e] += sc2[e];
    // ---- online softmax per head over this page's 16 keys (8 lane groups x 2 keys)
    float x[2][2];   // [key gid / gid + 8][head h0 / h0 + 1]
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const bool valid = gid + 8 * k < keys_here;
#pragma unroll
      for (int h = 0; h < 2; ++h) x[k][h] = valid ? sc[2 * k + h] * scale_log2 : -FLT_MAX;
    }
    float mx[2], corr[2], ps[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(m_run[h], fmaxf(x[0][h], x[1][h]));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 4));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 8));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 16));
      corr[h] = (m_run[h] == -FLT_MAX) ? 0.f : exp2f(m_run[h] - mx[h]);
      m_run[h] = mx[h];
    }
    float pv[2][2];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int h = 0; h < 2; ++h) pv[k][h] = x[k][h] == -FLT_MAX ? 0.f : exp2f(x[k][h] - mx[h]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ps[h] = pv[0][h] + pv[1][h];
      ps[h] += __shfl_xor_sync(0xffffffffu, ps[h], 4);
      ps[h] += __shfl_xor_sync(0xffffffffu, ps[h], 8);
      ps[h] += __shfl_xor_sync(0xffffffffu, ps[h], 16);
      l_run[h] = l_run[h] * corr[h] + ps[h];
    }
    if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= corr[0];
        o[mt][1] *= corr[1];
        o[mt][2] *= corr[0];
        o[mt][3] *= corr[1];
      }
    }
    // P^T (keys x heads, accumulator layout) -> B fragments (k = keys, n = heads)
    const uint32_t pb0 = movmatrix_trans(pack_bf16x2(pv[0][0], pv[0][1]));   // keys 0-7
    const uint32_t pb1 = movmatrix_trans(pack_bf16x2(pv[1][0], pv[1][1]));   // keys 8-15
    // ---- O^T += V^T . P^T: 8 tiles of 16 dims; matrix j = (dims 8 (j & 1).., keys 8 (j >> 1)..)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int key = (j >> 1) * 8 + r;
      const int db = mt * 2 + (j & 1);                  // 8-dim block 0..15
      uint32_t va[4];
      ldsm_x4_t(va, vp + (db >> 3) * HALF_BYTES + (key < page_size ? key : 0) * 128 + (((db & 7) ^ r) << 4));
      if (nblk < 2) { va[2] = 0u; va[3] = 0u; }
      mma_16816_bf16(o[mt], va, pb0, pb1);
    }
    __syncwarp();
    const int pn = p + ST * NW;
    if (lane == 0 && pn < n_pages) {
      fence_proxy_async();
      issue_page(table[pn], s);
    }
    DEC_TRACE(it, 2);
  }
  // ---- merge the NW warps through smem (heads < G only); the ring is reused, so all
  // warps must be done with their pages first
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h0 + h >= G) continue;
    if (gid == 0) {
      sm.merge_m[warp][h0 + h] = m_run[h];
      sm.merge_l[warp][h0 + h] = l_run[h];
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      sm.merge_acc[warp][h0 + h][mt * 16 + gid] = o[mt][h];
      sm.merge_acc[warp][h0 + h][mt * 16 + 8 + gid] = o[mt][2 + h];
    }
  }
  __syncthreads();
  DecodeRed* red = reinterpret_cast<DecodeRed*>(smem_raw + ((sizeof(DecodeSmem<NW, ST>) + 127) & ~size_t(127)));
  const uint32_t red_leader = csize > 1 ? mapa_shared(smem_u32(red), 0) : 0u;
  for (int i = threadIdx.x; i < G * HD; i += NW * 32) {
    const int h = i / HD, d = i % HD;
    float mx = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, sm.merge_m[w][h]);
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = sm.merge_m[w][h];
      const float c = (mw == -FLT_MAX) ? 0.f : exp2f(mw - mx);
      num += sm.merge_acc[w][h][d] * c;
      den += sm.merge_l[w][h] * c;
    }
    if (csize == 1) {
      out[(size_t)tok * (n_heads * HD) + (kvh * G + h) * HD + d] = f2bf(den > 0.f ? num / den : 0.f);
    } else {
      // this rank's (max, sum, unnormalised O) into slot crank of rank 0's DecodeRed
      const uint32_t base = red_leader;
      st_shared_cluster_f32(base + (uint32_t)(offsetof(DecodeRed, acc) + ((crank * 8 + h) * HD + d) * 4), num);
      if (d == 0) {
        st_shared_cluster_f32(base + (uint32_t)(offsetof(DecodeRed, m) + (crank * 8 + h) * 4), mx);
        st_shared_cluster_f32(base + (uint32_t)(offsetof(DecodeRed, l) + (crank * 8 + h) * 4), den);
      }
    }
  }
  if (csize == 1) return;
  cluster_sync();  // release / acquire at cluster scope: every rank's slot is visible to rank 0
  if (crank != 0) return;
  for (int i = threadIdx.x; i < G * HD; i += NW * 32) {
    const int h = i / HD, d = i % HD;
    float mx = -FLT_MAX;
    for (int r = 0; r < csize; ++r) mx = fmaxf(mx, red->m[r][h]);
    float num = 0.f, den = 0.f;
    for (int r = 0; r < csize; ++r) {
      const float mr = red->m[r][h];
      const float c = (mr == -FLT_MAX) ? 0.f : exp2f(mr - mx);
      num += red->acc[r][h][d] * c;
      den += red->l[r][h] * c;
    }
    out[(size_t)tok * (n_heads * HD) + (kvh * G + h) * HD + d] = f2bf(den > 0.f ? num / den : 0.f);
  }
}


GLLM_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FFMA2 / FADD2 on sm_100): half the issue slots of scalar FFMA / FADD.
GLLM_DEVICE float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
GLLM_DEVICE float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

template <int N>
GLLM_DEVICE void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
GLLM_DEVICE void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

GLLM_DEVICE float fmax3(float a, float b, float c) {  // FMNMX3 on sm_100
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// P for keys [64h, 64h + 64) of this thread's row from the S values in registers: exp2(s * scale - m)
// packed to bf16 pairs into TMEM columns [32h, 32h + 32) (every S column was loaded before any P
// store). DIAG: keys c > kmax (after this row's token) are zeroed by position.
template <bool DIAG>
GLLM_DEVICE void softmax_p_half(uint32_t t_s, int h, const uint32_t (&s)[PBK], float2 sc2, float2 ng2, int kmax,
                                float2 (&acc)[2]) {
  uint32_t pk[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int c = h * 64 + 2 * e;
    const float2 x = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sc2, ng2);
    float a = ex2_approx(x.x), b = ex2_approx(x.y);
    if constexpr (DIAG) {
      a = c <= kmax ? a : 0.f;
      b = c + 1 <= kmax ? b : 0.f;
    }
    acc[e & 1] = fadd2(acc[e & 1], make_float2(a, b));
    pk[e] = pack_bf16x2(a, b);
  }
  tmem_st_32x32b_x32(t_s + h * 32, pk);
}

// D[tmem] (+)= A[tmem] * B[smem]: the A operand (P, 128 rows x K bf16, two per 32-bit column)
// is read from tensor memory.
GLLM_DEVICE void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Prefill chunks on the tensor cores (see the file header). Work item = (sequence, q0): query
// tokens [q0, q0 + 2*QT) of the chunk as two 128-row tiles; grid = (kv head, item).
template <int G>
__global__ void __launch_bounds__(PF_THREADS, 1)
attn_prefill_kernel(const __grid_constant__ CUtensorMap k_map, const __grid_constant__ CUtensorMap v_map,
                    const bf16* __restrict__ qkv, const int* __restrict__ seq_info, const int* __restrict__ work,
                    int n_work, const int* __restrict__ block_table, int mpr, int n_heads, int n_kv, int page_size,
                    float scale_log2, bf16* __restrict__ out, int n_split, float* __restrict__ part_o,
                    float* __restrict__ part_ml) {
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  PrefillSmem& sm =
      *reinterpret_cast<PrefillSmem*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  constexpr int QT = PM / G;  // query tokens per tile
#ifdef GLLM_TRACE
  const long long t_cta0 = clock64();
#endif
  pdl_trigger();
  pdl_wait();
  const int kvh = blockIdx.x;
  const int item = n_work - 1 - (int)blockIdx.y / n_split;  // a chunk's later (longer) tiles start first
  const int split = (int)blockIdx.y % n_split;
  const int sidx = work[2 * item], q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int row_id = si[0], start = si[1], n_new = si[2], tok_off = si[3];
  const int* table = block_table + (size_t)row_id * mpr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qkv_w = (n_heads + 2 * n_kv) * HD;

  int nq[PTILES], nblk[PTILES];
#pragma unroll
  for (int t = 0; t < PTILES; ++t) {
    nq[t] = max(0, min(QT, n_new - (q0 + t * QT)));
    nblk[t] = nq[t] > 0 ? (start + q0 + t * QT + nq[t] + PBK - 1) / PBK : 0;
  }
  const int kv_len = start + q0 + nq[0] + nq[1];  // keys of the item's last query
  const int nb = max(nblk[0], nblk[1]);
  // KV split (n_split > 1, few items): this CTA owns key blocks [jb, je) of the item and writes
  // an unnormalised partial (O, running max, row sum) that attn_split_combine merges
  const int per_split = (nb + n_split - 1) / n_split;
  const int jb = min(nb, split * per_split), je = min(nb, jb + per_split);
  const int nbl = je - jb;  // blocks this CTA loads
  int tb[PTILES];           // blocks of tile t in [jb, je)
#pragma unroll
  for (int t = 0; t < PTILES; ++t) tb[t] = max(0, min(je, nblk[t]) - jb);

  if (threadIdx.x == 0) {
    for (int s = 0; s < PRING; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int t = 0; t < PTILES; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 4);  // one arrival per softmax warp of the tile
      mbar_init(&sm.o_full[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&sm.tmem_base, PF_TMEM_COLS);
  if (warp < 8) {
    // Q tiles -> swizzled smem; tile row r = (token r / G, head r % G) of this kv head's group
    for (int i = threadIdx.x; i < PTILES * PM * 16; i += 256) {
      const int t = i / (PM * 16), r = (i >> 4) % PM, c16 = i & 15, half = c16 >> 3, c = c16 & 7;
      uint8_t* dst = sm.q[t][half] + sw128_off(r, c);
      if (r < nq[t] * G) {
        const int qi = r / G, gh = r % G;
        cp_async16(dst, qkv + (size_t)(tok_off + q0 + t * QT + qi) * qkv_w + (kvh * G + gh) * HD + half * 64 + c * 8);
      } else {
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (warp >= 8) {
  setmaxnreg_dec<PF_REG_PRODUCER>();
  if (warp == 8) {
    // ---- TMA producer: fill f = 2j loads K_j, f = 2j+1 loads V_j. Lane pl < ppb owns page pl of
    // every block and issues its two 64-dim boxes; its page id is read from the block table one
    // block ahead, so no table load sits between a slot's release and its refill.
    const int n_pages = (kv_len + page_size - 1) / page_size;
    const int ppb = PBK / page_size;
    const int ppl = min(ppb, PF_LOAD_PAGES);
    const uint32_t box_bytes = (uint32_t)page_size * 128;
    const uint64_t pol = policy_evict_last();  // every query tile of the sequence re-reads these pages
    // pages past the item's last key repeat its last page (never an unmapped table entry)
    auto page_row = [&](int j) {
      return lane < ppl ? (table[min(j * ppb + lane, n_pages - 1)] * n_kv + kvh) * page_size : 0;
    };
    int row_cur = nbl > 0 ? page_row(jb) : 0;
    int row_next = nbl > 1 ? page_row(jb + 1) : 0;
    for (int f = 0; f < 2 * nbl; ++f) {
      const int s = f % PRING;
      if (f >= PRING) mbar_wait(&sm.kv_empty[s], ((f / PRING) + 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&sm.kv_full[s], PF_BLK_BYTES / (ppb / ppl));
      __syncwarp();
      const CUtensorMap* m = (f & 1) ? &v_map : &k_map;
      if (lane < ppl) {
        tma_load_2d_hint(m, &sm.kv_full[s], sm.kv[s][0] + lane * box_bytes, 0, row_cur, pol);
        tma_load_2d_hint(m, &sm.kv_full[s], sm.kv[s][1] + lane * box_bytes, 64, row_cur, pol);
      }
      if (f & 1) {
        const int j = jb + (f >> 1);
        row_cur = row_next;
        row_next = j + 2 < jb + nbl ? page_row(j + 2) : 0;
      }
    }
  } else if (warp == 9) {
    // ---- MMA issuer: the warp walks the schedule, lane 0 issues
    constexpr uint32_t idesc_s = idesc_bf16_f32(PM, PBK);
    constexpr uint32_t idesc_o = idesc_bf16_f32(PM, HD, /*b_mn_major=*/true);
    auto wait_full = [&](int f) {
      mbar_wait(&sm.kv_full[f % PRING], (uint32_t)((f / PRING) & 1));
      tc_fence_after();
    };
    auto release = [&](int f) {
      if (lane == 0) mma_commit(&sm.kv_empty[f % PRING]);
      __syncwarp();
    };
    auto issue_s = [&](int t, int l) {  // S_t = Q_t . K^T of local block l
      const int s = (2 * l) % PRING;
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < PF_S_STEPS; ++kk) {
          const uint64_t da = smem_desc_sw128(sm.q[t][kk >> 2]) + 2 * (kk & 3);
          const uint64_t db = smem_desc_sw128(sm.kv[s][kk >> 2]) + 2 * (kk & 3);
          mma_bf16_ss(tmem + t * 256, da, db, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.s_full[t]);
      }
      __syncwarp();
    };
    // O_t += P_t . V of local block l, P (bf16) in S_t's first 64 columns
    auto issue_pv = [&](int t, int l) {
      const int s = (2 * l + 1) % PRING;
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < PF_PV_STEPS; ++kk) {
          const uint64_t db = smem_desc_sw128_mn(sm.kv[s][0] + kk * 2048, PBK * 128);
          mma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + kk * 8, db, idesc_o, (l > 0 || kk > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    if (nbl > 0) {
      wait_full(0);
      for (int t = 0; t < PTILES; ++t)
        if (tb[t] > 0) issue_s(t, 0);
      release(0);
    }
    for (int l = 0; l < nbl; ++l) {
      const int j = jb + l;
      if (lane == 0) PF_TRACE(l, 8);
      wait_full(2 * l + 1);
      if (lane == 0) PF_TRACE(l, 9);
      if (j == nb - 1 && kv_len < nb * PBK) {
        // keys past the item's last query are never attended, but stale cache slots may hold
        // NaN/Inf bytes and P = 0 times NaN would poison O: zero those V rows
        const int s = (2 * l + 1) % PRING;
        const int k0 = kv_len - j * PBK;
        for (int i = lane; i < (PBK - k0) * 16; i += 32) {
          const int r = k0 + (i >> 4), half = (i >> 3) & 1, c = i & 7;
          *reinterpret_cast<uint4*>(sm.kv[s][half] + sw128_off(r, c)) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async();
        __syncwarp();
      }
      const bool next = l + 1 < nbl;
      bool k_next = false;  // K_{l+1} is awaited only right before the first S that reads it
      for (int t = 0; t < PTILES; ++t) {
        if (l >= tb[t]) continue;
        mbar_wait(&sm.p_full[t], (uint32_t)(l & 1));
        tc_fence_after();
        if (lane == 0) PF_TRACE(l, 10 + t);
        issue_pv(t, l);
        if (l + 1 < tb[t]) {
          if (!k_next) {
            wait_full(2 * l + 2);
            k_next = true;
          }
          issue_s(t, l + 1);
          if (lane == 0 && t == 0) PF_TRACE(l, 6);
        } else {
          if (lane == 0) mma_commit(&sm.o_full[t]);
          __syncwarp();
        }
      }
      release(2 * l + 1);
      if (next) release(2 * l + 2);
      if (lane == 0) PF_TRACE(l, 7);
    }
  }
  } else {
    setmaxnreg_inc<PF_REG_SOFTMAX>();
    // ---- softmax + epilogue of tile t: this thread owns TMEM lane / query row `row`
    const int t = warp >> 2;
    const int tnq = t ? nq[1] : nq[0], tnb = t ? tb[1] : tb[0];
    if (tnq > 0) {
      const int row = (warp & 3) * 32 + lane;
      const uint32_t t_s = tmem + t * 256 + ((uint32_t)((warp & 3) * 32) << 16);
      const uint32_t t_o = t_s + 128;
      const int R = tnq * G;
      const int qfirst = start + q0 + t * QT;
      const int qpos = qfirst + (row < R ? row / G : tnq - 1);
      float m_ref = -FLT_MAX, l_sum = 0.f;
      for (int l = 0; l < tnb; ++l) {
        const int j = jb + l;
        mbar_wait(&sm.s_full[t], (uint32_t)(l & 1));
        tc_fence_after();
        if (row == 0) PF_TRACE(l, 3 * t);
        // one pass: the row's 128 S values in registers; diagonal blocks mask keys after this row's
        // token by position, so stale bytes in unattended slots never reach the max
        const bool diag = (j + 1) * PBK - 1 > qfirst;
        const int kmax = qpos - j * PBK;  // keys c <= kmax are attended
        uint32_t sv[PBK];
#pragma unroll
        for (int c = 0; c < PBK; c += 32) tmem_ld_32x32b_x32(t_s + c, *reinterpret_cast<uint32_t(*)[32]>(&sv[c]));
        tmem_ld_wait();
        if (diag) {
#pragma unroll
          for (int c = 0; c < PBK; ++c) sv[c] = c <= kmax ? sv[c] : __float_as_uint(-FLT_MAX);
        }
        // 4 independent 3-input max chains (one chain over 128 keys is latency-bound)
        float mx[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
        for (int c = 0; c < PBK; c += 8) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mx[k] = fmax3(mx[k], __uint_as_float(sv[c + 2 * k]), __uint_as_float(sv[c + 2 * k + 1]));
        }
        float mb = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        mb *= scale_log2;
        const bool grow = mb > m_ref + RESCALE_TH || m_ref == -FLT_MAX;
        float corr = 1.f;
        if (grow) {
          corr = (m_ref == -FLT_MAX) ? 0.f : ex2_approx(m_ref - mb);
          l_sum *= corr;
          m_ref = mb;
        }
        // O (complete through block j-1: S_t(j) was issued after P.V_t(j-1)) rescaled in TMEM;
        // tcgen05.ld/st are warp-collective, so the whole warp joins when any row grows
        if (l > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll 1
          for (int c = 0; c < HD; c += 32) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(t_o + c, o);
          }
        }
        if (row == 0) PF_TRACE(l, 3 * t + 1);
        // P = exp2(s * scale - m) as packed bf16 over S's first 64 columns, published per half
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(scale_log2, scale_log2), ng2 = make_float2(-m_ref, -m_ref);
        if (diag) {
          softmax_p_half<true>(t_s, 0, sv, sc2, ng2, kmax, acc);
          softmax_p_half<true>(t_s, 1, sv, sc2, ng2, kmax, acc);
        } else {
          softmax_p_half<false>(t_s, 0, sv, sc2, ng2, kmax, acc);
          softmax_p_half<false>(t_s, 1, sv, sc2, ng2, kmax, acc);
        }
        l_sum += (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
        // one arrival per warp once its lanes' P stores completed (4 arrivals, not 128)
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[t]);
        if (row == 0) PF_TRACE(l, 3 * t + 2);
      }
      if (n_split > 1) {
        // unnormalised partial: O (fp32), running max m (log2 units) and row sum of this split
        const size_t prow = ((((size_t)item * n_split + split) * n_kv + kvh) * PTILES + t) * PM + row;
        float* po = part_o + prow * HD;
        if (tnb > 0) {
          mbar_wait(&sm.o_full[t], 0);
          tc_fence_after();
        }
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t r32[32];
          if (tnb > 0) {
            tmem_ld_32x32b_x32(t_o + c, r32);  // warp-collective: all lanes
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) r32[e] = 0u;
          }
          if (row < R) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(po + c + e) =
                  make_float4(__uint_as_float(r32[e]), __uint_as_float(r32[e + 1]), __uint_as_float(r32[e + 2]),
                              __uint_as_float(r32[e + 3]));
          }
        }
        if (row < R) *reinterpret_cast<float2*>(part_ml + prow * 2) = make_float2(tnb > 0 ? m_ref : -FLT_MAX, l_sum);
      } else {
      mbar_wait(&sm.o_full[t], 0);
      tc_fence_after();
      const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
      const int qi = row / G, gh = row % G;
      bf16* o = out + (size_t)(tok_off + q0 + t * QT + qi) * (n_heads * HD) + (kvh * G + gh) * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t r32[32];
        tmem_ld_32x32b_x32(t_o + c, r32);
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
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, PF_TMEM_COLS);
}

// Merge the KV-split partials of every prefill row: m = max_s m_s, O = sum_s O_s 2^(m_s - m),
// l = sum_s l_s 2^(m_s - m), out = O / l. A warp per (item, kv head, query tile, row), 4 dims per lane.
constexpr int CMB_ROWS = 8;  // rows (warps) per combine CTA
template <int G>
__global__ void __launch_bounds__(32 * CMB_ROWS)
attn_split_combine(const int* __restrict__ seq_info, const int* __restrict__ work, int n_split, int n_heads, int n_kv,
                   const float* __restrict__ part_o, const float* __restrict__ part_ml, bf16* __restrict__ out) {
  constexpr int QT = PM / G;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * CMB_ROWS + (threadIdx.x >> 5);
  const int r = g % PM, tt = g / PM, t = tt % PTILES, kvh = (tt / PTILES) % n_kv, item = tt / PTILES / n_kv;
  const int sidx = work[2 * item], q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int n_new = si[2], tok_off = si[3];
  if (r >= max(0, min(QT, n_new - (q0 + t * QT))) * G) return;
  auto prow = [&](int s) { return ((((size_t)item * n_split + s) * n_kv + kvh) * PTILES + t) * PM + r; };
  float m = -FLT_MAX;
  for (int s = 0; s < n_split; ++s) m = fmaxf(m, part_ml[prow(s) * 2]);
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  float l = 0.f;
  for (int s = 0; s < n_split; ++s) {
    const float2 ml = *reinterpret_cast<const float2*>(part_ml + prow(s) * 2);
    if (ml.x == -FLT_MAX) continue;
    const float w = exp2f(ml.x - m);
    const float4 p = *reinterpret_cast<const float4*>(part_o + prow(s) * HD + lane * 4);
    l += ml.y * w;
    o.x += p.x * w;
    o.y += p.y * w;
    o.z += p.z * w;
    o.w += p.w * w;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  *reinterpret_cast<uint2*>(out + (size_t)(tok_off + q0 + t * QT + r / G) * (n_heads * HD) + (kvh * G + r % G) * HD +
                            lane * 4) = make_uint2(pack_bf16x2(o.x * inv, o.y * inv), pack_bf16x2(o.z * inv, o.w * inv));
}

// A mixed micro-batch is issued as two concurrent launches (prefill items on a forked side
// stream, decodes on the caller's stream, joined by an event): the prefill kernel takes all of
// an SM's TMEM and most of its smem, while decode CTAs want two per SM for bytes in flight.
// NW = 4 (two CTAs per SM) for large decode populations; NW = 8 (one CTA, twice the pages in
// flight per sequence) when all (sequence, kv head) items fit in one wave of SMs: small batches
// are latency-bound on each sequence's page stream.
template <int G, int NW, int ST = DEC_STAGES>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? (ST == DEC_STAGES ? 2 : 3) : 1)
attn_decode_kernel(const __grid_constant__ CUtensorMap k_map, const __grid_constant__ CUtensorMap v_map,
                   const bf16* __restrict__ qkv, const int* __restrict__ seq_info, const int* __restrict__ work,
                   const int* __restrict__ block_table, int mpr, int n_heads, int n_kv, int page_size,
                   float scale_log2, bf16* __restrict__ out, int csize) {
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  uint8_t* smem_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  pdl_trigger();  // decode_role waits (griddepcontrol.wait) after prefetching the settled pages
  // kv heads fastest: a work item's CTAs launch together; with a KV split the csize ranks of one
  // (item, kv head) are consecutive in x and form one cluster
  const int kvh = blockIdx.x / csize, crank = blockIdx.x % csize;
  const int item = blockIdx.y;
  const int sidx = work[2 * item];
  const int q0 = work[2 * item + 1];
  const int* si = seq_info + 5 * sidx;
  const int row_id = si[0], start = si[1], tok_off = si[3];
  const int* table = block_table + (size_t)row_id * mpr;
  decode_role<G, NW, ST>(smem_raw, qkv, tok_off + q0, start + q0 + 1, table, &k_map, &v_map, n_heads, n_kv, kvh,
                     page_size, scale_log2, out, csize, crank);
}

// Query tokens per prefill work item (a decode, n_new == 1, is always one item).
int attention_q_tile(int n_heads, int n_kv) { return PTILES * (PM / (n_heads / n_kv)); }

// KV split of the prefill items (n_split = 1: none); partials in caller-provided device memory
struct AttnSplit {
  int n_split = 1;
  float* part_o = nullptr;   // [items][n_split][n_kv][2 tiles][128 rows][128] fp32
  float* part_ml = nullptr;  // [items][n_split][n_kv][2 tiles][128 rows][2] (max, sum)
};

size_t attention_split_bytes(int n_items, int n_split, int n_kv) {
  return (size_t)n_items * n_split * n_kv * PTILES * PM * (HD + 2) * sizeof(float);
}

// Co-resident clusters of c 8-warp decode CTAs (cached per G and c).
template <int G>
static int decode_max_clusters(int c, size_t smem) {
  static int cache[DEC_MAX_SPLIT + 1] = {};
  if (cache[c] == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * device_sm_count());
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = c;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, attn_decode_kernel<G, 8>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[c] = n > 0 ? n : -1;
  }
  return cache[c];
}

template <bool PREFILL, int G>
static int launch_attn(const bf16* qkv, const int* seq_info, const int* work, int n_work, const int* block_table,
                       int mpr, int kv_pages, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int page_size,
                       float scale_log2, bf16* out, cudaStream_t st, const AttnSplit& sp = AttnSplit{},
                       int dec_pages = 0, int dec_mean_pages = 0) {
  constexpr size_t smem_pf = sizeof(PrefillSmem) + 1024;
  constexpr size_t smem4 = sizeof(DecodeSmem<4>) + 1024;
  constexpr size_t smem4s = sizeof(DecodeSmem<4, 2>) + 1024;   // 3 CTAs per SM
  constexpr size_t smem8 = ((sizeof(DecodeSmem<8>) + 127) & ~size_t(127)) + sizeof(DecodeRed) + 1024;
  static bool attr = false;
  if (!attr) {
    const void* fns[4] = {(const void*)attn_prefill_kernel<G>, (const void*)attn_decode_kernel<G, 4>,
                          (const void*)attn_decode_kernel<G, 8>, (const void*)attn_decode_kernel<G, 4, 2>};
    const size_t sm[4] = {smem_pf, smem4, smem8, smem4s};
    for (int i = PREFILL ? 0 : 1; i < (PREFILL ? 1 : 4); ++i) {
      cudaError_t e = cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm[i]);
      if (e != cudaSuccess) return set_cuda_error(e, "attention smem attribute");
      // all of the unified L1/smem as shared memory (decode: 8 streaming warps per SM)
      e = cudaFuncSetAttribute(fns[i], cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return set_cuda_error(e, "attention carveout attribute");
    }
    attr = true;
  }
  // the paged cache viewed as a 2-D [pages*kv_heads*page_size, 128] bf16 tensor: one TMA box per
  // (page, kv head, 64-dim half)
  CUtensorMap km, vm;
  if (int rc = make_tma_map_2d(&km, k_cache, (int64_t)kv_pages * n_kv * page_size, HD, HD, page_size)) return rc;
  if (int rc = make_tma_map_2d(&vm, v_cache, (int64_t)kv_pages * n_kv * page_size, HD, HD, page_size)) return rc;
  dim3 grid(n_kv, n_work);
  if constexpr (PREFILL) {
    grid.y = n_work * sp.n_split;
    attn_prefill_kernel<G><<<grid, PF_THREADS, smem_pf, st>>>(km, vm, qkv, seq_info, work, n_work, block_table, mpr,
                                                            n_heads, n_kv, page_size, scale_log2, out, sp.n_split,
                                                            sp.part_o, sp.part_ml);
    if (int rc = check_launch("attention_prefill")) return rc;
    if (sp.n_split > 1) {
      attn_split_combine<G><<<n_work * n_kv * PTILES * PM / CMB_ROWS, 32 * CMB_ROWS, 0, st>>>(
          seq_info, work, sp.n_split, n_heads, n_kv, sp.part_o, sp.part_ml, out);
      return check_launch("attention_split_combine");
    }
    return 0;
  } else {
    const int sms = device_sm_count();
    const long items = (long)n_work * n_kv;
    const bool wide = items <= sms;  // one wave of 8-warp CTAs
    // KV split (dec_pages = the longest decode's pages, 0 = unknown / not decode-only): the
    // fewest ranks that bring every warp to <= DEC_STAGES pages (one memory round trip), while
    // all clusters stay co-resident in one wave
    int csize = 1;
    if (wide && dec_pages > DEC_STAGES * 8) {
      static const int forced = [] {
        const char* e = getenv("GLLM_DECODE_SPLIT");  // 1 = off, 2..4 = forced where it fits (A/B)
        return e ? atoi(e) : 0;
      }();
      int want = (dec_pages + DEC_STAGES * 8 - 1) / (DEC_STAGES * 8);
      if (forced) want = forced;
      for (int c = want < DEC_MAX_SPLIT ? want : DEC_MAX_SPLIT; c >= 2; --c)
        if (items * c <= sms && items <= decode_max_clusters<G>(c, smem8)) {
          csize = c;
          break;
        }
    }
    grid.x = n_kv * csize;
    // Between one and 1.5 waves of two 4-warp CTAs per SM, three CTAs per SM with a 2-stage page
    // ring (the same pages in flight per SM) keep the items in one wave: e.g. 48-55 decodes with
    // 8 kv heads (384-440 items) against 296 two-per-SM slots.
    static const int three = [] {
      const char* e = getenv("GLLM_DECODE_3CTA");  // A/B switch (default on; 2 = at every population)
      return e ? atoi(e) : 1;
    }();
    // Beyond 1.5 waves too when the decodes are short (mean <= 64 pages, from the host metadata):
    // C2's 800 x ~500-token decodes 270 -> 262 us (0.965 of HBM); at 2000-4000 tokens the 2-stage
    // ring per warp loses 1-4%.
    const bool tri = !wide && three && items > 2L * sms &&
                     (items <= 3L * sms || three == 2 || (dec_mean_pages > 0 && dec_mean_pages <= 64));
    cudaError_t e = wide ? launch_kernel(attn_decode_kernel<G, 8>, grid, dim3(256), smem8, st, csize, km, vm, qkv,
                                         seq_info, work, block_table, mpr, n_heads, n_kv, page_size, scale_log2, out,
                                         csize)
                  : tri  ? launch_kernel(attn_decode_kernel<G, 4, 2>, grid, dim3(128), smem4s, st, 1, km, vm, qkv,
                                         seq_info, work, block_table, mpr, n_heads, n_kv, page_size, scale_log2, out, 1)
                         : launch_kernel(attn_decode_kernel<G, 4>, grid, dim3(128), smem4, st, 1, km, vm, qkv, seq_info,
                                         work, block_table, mpr, n_heads, n_kv, page_size, scale_log2, out, 1);
    if (e != cudaSuccess) return set_cuda_error(e, "attention_decode launch");
    return check_launch("attention_decode");
  }
}

struct AttnStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static int attn_streams(AttnStreams** out) {
  static AttnStreams s;
  static int dev = -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (s.side == nullptr || dev != cur) {
    cudaError_t e = cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming);
    if (e != cudaSuccess) return set_cuda_error(e, "attention side stream");
    dev = cur;
  }
  *out = &s;
  return 0;
}

// work[0, n_prefill_work) are prefill items, the rest decodes (host packer order).
template <int G>
static int launch_attn_g(int n_prefill_work, const bf16* qkv, const int* seq_info, const int* work, int n_work,
                         const int* block_table, int mpr, int kv_pages, const bf16* k_cache, const bf16* v_cache,
                         int n_heads, int n_kv, int page_size, float scale_log2, bf16* out, cudaStream_t st,
                         const AttnSplit& sp, int dec_pages, int dec_mean_pages) {
  const int n_dec = n_work - n_prefill_work;
  if (n_prefill_work == 0)
    return launch_attn<false, G>(qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads,
                                 n_kv, page_size, scale_log2, out, st, AttnSplit{}, dec_pages, dec_mean_pages);
  if (n_dec == 0)
    return launch_attn<true, G>(qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads,
                                n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
  AttnStreams* ss = nullptr;
  if (int rc = attn_streams(&ss)) return rc;
  cudaEventRecord(ss->fork, st);
  cudaStreamWaitEvent(ss->side, ss->fork, 0);
  int rc = launch_attn<true, G>(qkv, seq_info, work, n_prefill_work, block_table, mpr, kv_pages, k_cache, v_cache,
                                n_heads, n_kv, page_size, scale_log2, out, ss->side, sp);
  if (rc == 0)
    rc = launch_attn<false, G>(qkv, seq_info, work + 2 * n_prefill_work, n_dec, block_table, mpr, kv_pages, k_cache,
                               v_cache, n_heads, n_kv, page_size, scale_log2, out, st, AttnSplit{}, 0, dec_mean_pages);
  cudaEventRecord(ss->join, ss->side);
  cudaStreamWaitEvent(st, ss->join, 0);
  return rc;
}

// n_split: 0 = choose from the host copy of the metadata (when given) and the partial workspace;
// >= 1 = use that many key ranges per prefill item (1 = no split).
int attention_paged(const bf16* qkv, const int* seq_info, const int* work, int n_work, int n_prefill_work,
                    const int* block_table, int mpr, int kv_pages, const bf16* k_cache, const bf16* v_cache,
                    int n_heads, int n_kv, int head_dim, int page_size, bf16* out, cudaStream_t st, int n_split,
                    const int* host_seq_info, const int* host_work, void* part_ws, size_t part_bytes) {
  if (n_work <= 0) return 0;
  if (head_dim != HD) return set_error(GLLM_ERR_INVALID, "attention supports head_dim 128 only (got %d)", head_dim);
  if (n_heads % n_kv) return set_error(GLLM_ERR_INVALID, "bad GQA grouping");
  if (page_size != 8 && page_size != 16) return set_error(GLLM_ERR_INVALID, "page_size must be 8 or 16");
  if (n_prefill_work < 0 || n_prefill_work > n_work) return set_error(GLLM_ERR_INVALID, "bad n_prefill_work");
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  const int pf = n_prefill_work;
  AttnSplit sp;
  // Automatic KV split is opt-in (GLLM_ATTN_SPLIT=1): +8% on an isolated 640-token chunk after 6k
  // cached keys, but -7% on the prefill attention of the C5 serving bench, where the prefill
  // launch shares the SMs with the concurrent decode launch.
  static const bool auto_split = [] {
    const char* e = getenv("GLLM_ATTN_SPLIT");
    return e != nullptr && atoi(e) != 0;
  }();
  if (pf > 0 && n_split == 0 && auto_split && host_seq_info && host_work && part_ws) {
    // Few prefill CTAs (one per SM): cutting each item's key range into S parts trades wave
    // quantization for per-CTA fixed cost (Q load, pipeline fill, partial write + combine),
    // measured at ~8 key blocks. Pick S minimising waves(S) x (blocks per item / S + 8).
    const int sms = device_sm_count(), ctas = pf * n_kv;
    const int item_tokens = attention_q_tile(n_heads, n_kv);
    if (ctas < 2 * sms) {
      long blocks = 0;
      for (int i = 0; i < pf; ++i) {
        const int* si = host_seq_info + 5 * host_work[2 * i];
        const int last = min(si[2], host_work[2 * i + 1] + item_tokens);
        blocks += (si[1] + last + PBK - 1) / PBK;
      }
      const double per_item = (double)blocks / pf;
      double best = 0.0;
      for (int S = 1; S <= 8; ++S) {
        const double t = (double)((ctas * S + sms - 1) / sms) * (per_item / S + 8.0);
        if (S == 1 || t < best) {
          best = t;
          n_split = S;
        }
      }
    }
  }
  if (n_split > 1 && pf > 0) {
    while (n_split > 1 && attention_split_bytes(pf, n_split, n_kv) > part_bytes) --n_split;
    if (n_split > 1) {
      sp.n_split = n_split;
      sp.part_o = reinterpret_cast<float*>(part_ws);
      sp.part_ml = sp.part_o + (size_t)pf * n_split * n_kv * PTILES * PM * HD;
    }
  }
  // decode-only launch: the longest decode's page count lets the decode kernel pick a KV split;
  // any launch: the decodes' mean page count picks its CTA shape
  int dec_pages = 0, dec_mean_pages = 0;
  if (host_seq_info && host_work && n_work > pf) {
    long sum = 0;
    for (int i = pf; i < n_work; ++i) {
      const int* si = host_seq_info + 5 * host_work[2 * i];
      const int pages = (si[1] + host_work[2 * i + 1] + 1 + page_size - 1) / page_size;
      if (pf == 0) dec_pages = pages > dec_pages ? pages : dec_pages;
      sum += pages;
    }
    dec_mean_pages = (int)((sum + (n_work - pf) - 1) / (n_work - pf));
  }
  switch (n_heads / n_kv) {
    case 1: return launch_attn_g<1>(pf, qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
    case 2: return launch_attn_g<2>(pf, qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
    case 4: return launch_attn_g<4>(pf, qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
    case 5: return launch_attn_g<5>(pf, qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
    case 8: return launch_attn_g<8>(pf, qkv, seq_info, work, n_work, block_table, mpr, kv_pages, k_cache, v_cache, n_heads, n_kv, page_size, scale_log2, out, st, sp, dec_pages, dec_mean_pages);
    default: return set_error(GLLM_ERR_INVALID, "unsupported GQA group %d", n_heads / n_kv);
  }
}

}  // namespace gllm

#ifdef GLLM_TRACE
// debug builds only (not in include/gllm.h): copy the decode trace [296][8][32][3] u32 to host
extern "C" __attribute__((visibility("default"))) int gllm_debug_dec_trace_read(void* host, size_t bytes) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, gllm::g_dec_trace,
                              bytes < sizeof(gllm::g_dec_trace) ? bytes : sizeof(gllm::g_dec_trace)) == cudaSuccess ? 0 : -1;
}
// debug builds only (not in include/gllm.h): copy the prefill trace [148][64][12] u32 to host
extern "C" __attribute__((visibility("default"))) int gllm_debug_attn_trace_read(void* host, size_t bytes) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, gllm::g_pf_trace,
                              bytes < sizeof(gllm::g_pf_trace) ? bytes : sizeof(gllm::g_pf_trace)) == cudaSuccess ? 0 : -1;
}
#endif
