// Decode-sized GEMMs (M <= 32 tokens): Y[M, N] = X[M, K] . W[N, K]^T (+ fused epilogue).
//
// With a handful of tokens the projection is a weight stream: every byte of W is used once,
// so the only goal is HBM bandwidth. The 128-row tcgen05 tiles of gemm.cu pad M to 128 and
// need split-K + a reduce launch to reach all SMs; this kernel instead
//   * swaps A/B: the MMA's M (128 TMEM lanes) runs over output features (W rows) and its
//     N over the padded tokens (NT = 16 or 32), so a K-block is 16 KB of W + NT x 128 B of X;
//   * cuts the whole (tile, K-block) space into one contiguous range per persistent CTA
//     (stream-K): every SM streams the same number of W bytes, whatever N / K are. W is
//     read exactly once (no raster to preserve) and X stays L2-resident;
//   * fixes up tiles shared by several CTAs without waiting: each contributor writes its fp32
//     partial (M x 128, tiny at decode sizes), fences and bumps the tile counter; the last to
//     arrive sums the partials in contributor order (deterministic) and runs the epilogue.
// Cluster split-K (csize > 1, few output tiles): tile t is owned by a cluster of csize CTAs,
// rank r streaming K-blocks [r kbs / csize, (r+1) kbs / csize). Ranks 1.. write their fp32
// partials straight into rank 0's shared memory (DSMEM) and one cluster barrier publishes them:
// no global partials, fence, counter or L2 round trip in the launch's tail.
// Warp roles as in gemm.cu: warp 0 TMA producer (8-stage ring), warp 1 MMA issuer, warps 2-5
// epilogue (TMEM -> smem transpose -> bias / residual / SwiGLU / RoPE + paged KV write).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

namespace {

constexpr int W_ROWS = 128;  // output features per tile (MMA M)
constexpr int KB = 64;       // K per stage (one 128-byte swizzle atom of bf16)
constexpr int THREADS = 192;
constexpr int EPI_STORE = 0, EPI_SWIGLU = 2, EPI_QKV_ROPE = 3;

template <int NT>
struct SkSmem {
  static constexpr int STAGES = 8;  // 11 (more weights prefetched ahead of the PDL wait) measured neutral
  static constexpr int W_BYTES = W_ROWS * KB * 2;
  static constexpr int X_BYTES = NT * KB * 2;
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  static constexpr int ST_LD = W_ROWS + 4;  // fp32 transpose staging [NT][ST_LD]
  static constexpr int STAGE_OFF = 0;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int RS_OFF = EPI_OFF + NT * ST_LD * 4;  // fused-norm row scales [NT]
  static constexpr int MAX_CLUSTER = 4;
  static constexpr int RED_OFF = RS_OFF + NT * 4;  // cluster partials [MAX_CLUSTER - 1][NT][128] fp32
  static constexpr int BAR_OFF = RED_OFF + (MAX_CLUSTER - 1) * NT * W_ROWS * 4;
  static constexpr int TOTAL = 1024 + BAR_OFF + 256;
};

// Debug builds (-DGLLM_TRACE, tools/skinny_trace.py): %globaltimer stamps of each CTA's phases
// in a ring of TRACE_LAUNCHES launches, read back with gllm_debug_trace_read.
#ifdef GLLM_TRACE
constexpr int TRACE_LAUNCHES = 64, TRACE_CTAS = 160, TRACE_EV = 12;
__device__ unsigned long long g_trace[TRACE_LAUNCHES][TRACE_CTAS][TRACE_EV];
__device__ __forceinline__ void trace(int tag, int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (blockIdx.x < TRACE_CTAS) g_trace[tag % TRACE_LAUNCHES][blockIdx.x][ev] = t;
}
#define SK_TRACE(ev) trace(tag, ev)
#else
#define SK_TRACE(ev) ((void)tag)
#endif

GLLM_DEVICE void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Fused epilogue of one [M x 128] output tile staged in smem as fp32 st[m][f] (f = W row in tile).
template <int NT, int MODE>
__device__ __forceinline__ void skinny_epilogue(const float* st, int et, int t, int M, int N, bf16* __restrict__ C,
                                                int ldc, const bf16* __restrict__ bias,
                                                const bf16* __restrict__ residual, int ldr,
                                                const QkvRopeArgs& qa, const RowNorm& nm, const float* rs_sm) {
  constexpr int LD = SkSmem<NT>::ST_LD;
  // fused RMSNorm row scale of token m (1 without a norm), precomputed in smem by the caller
  auto row_scale = [&](int m) { return nm.ss_in != nullptr ? rs_sm[m] : 1.f; };
  if constexpr (MODE == EPI_STORE) {
    const int n0 = t * W_ROWS;
    // every lane runs the same trip count: 8 consecutive lanes = one 64-column group of a row,
    // reduced by a fixed butterfly for the fused-norm statistics
    for (int base = 0; base < M * 16; base += 128) {
      const int i = base + et;
      const bool live = i < M * 16;
      const int m = live ? i >> 4 : 0, c = (i & 15) * 8;
      float sq = 0.f;
      if (live) {
        const float rs = row_scale(m);
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = st[m * LD + c + j] * rs;
        if (bias != nullptr) {
          const uint4 u = *reinterpret_cast<const uint4*>(bias + n0 + c);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(w4[j]);
            v[2 * j] += f.x;
            v[2 * j + 1] += f.y;
          }
        }
        if (residual != nullptr) {
          // round the GEMM result to bf16 first, then add: same as bf16 "x + attn(x)"
          const uint4 u = *reinterpret_cast<const uint4*>(residual + (size_t)m * ldr + n0 + c);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(w4[j]);
            v[2 * j] = bf2f(f2bf(v[2 * j])) + f.x;
            v[2 * j + 1] = bf2f(f2bf(v[2 * j + 1])) + f.y;
          }
        }
        *reinterpret_cast<uint4*>(C + (size_t)m * ldc + n0 + c) =
            make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                       pack_bf16x2(v[6], v[7]));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float q = bf2f(f2bf(v[j]));
          sq = fmaf(q, q, sq);
        }
      }
      if (nm.ss_out != nullptr) {
        for (int o = 1; o < 8; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (live && (c & (NORM_GROUP - 1)) == 0) nm.ss_out[(size_t)((n0 + c) / NORM_GROUP) * nm.ld + m] = sq;
      }
    }
  } else if constexpr (MODE == EPI_SWIGLU) {
    // W rows interleave 64 gate / 64 up rows: tile t holds gate (f < 64) and up (f >= 64) of
    // output features [64t, 64t + 64); act = bf16(silu(bf16 g)) * bf16(u) as in gemm.cu
    for (int i = et; i < M * 8; i += 128) {
      const int m = i >> 3, c = (i & 7) * 8;
      const float rs = row_scale(m);
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float a0 = bf2f(f2bf(st[m * LD + c + 2 * j] * rs)), a1 = bf2f(f2bf(st[m * LD + c + 2 * j + 1] * rs));
        const float b0 = bf2f(f2bf(st[m * LD + 64 + c + 2 * j] * rs)),
                    b1 = bf2f(f2bf(st[m * LD + 64 + c + 2 * j + 1] * rs));
        a0 = bf2f(f2bf(silu_f(a0)));
        a1 = bf2f(f2bf(silu_f(a1)));
        pk[j] = pack_bf16x2(a0 * b0, a1 * b1);
      }
      *reinterpret_cast<uint4*>(C + (size_t)m * ldc + t * 64 + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  } else {
    // tile t = head t (128 dims): q heads rotated into C, k heads rotated and v heads copied into
    // the token's paged cache slot; same roundings as the 128-row QKV epilogue
    const int gh = t;
    for (int i = et; i < M * 8; i += 128) {
      const int m = i >> 3, c = (i & 7) * 8;
      const int pos = qa.tok_pos[m], slot = qa.tok_slot[m];
      const int page = slot / qa.page_size, off = slot % qa.page_size;
      const float2* cs = reinterpret_cast<const float2*>(qa.rope) + (size_t)pos * 64;
      const float rs = row_scale(m);
      float a[8], b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] = st[m * LD + c + j] * rs;
        b[j] = st[m * LD + 64 + c + j] * rs;
      }
      if (bias != nullptr) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a[j] += bf2f(bias[gh * 128 + c + j]);
          b[j] += bf2f(bias[gh * 128 + 64 + c + j]);
        }
      }
      uint32_t y1[4], y2[4];
      if (gh < qa.n_heads + qa.n_kv) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float p0 = bf2f(f2bf(a[j])), p1 = bf2f(f2bf(a[j + 1]));
          const float q0 = bf2f(f2bf(b[j])), q1 = bf2f(f2bf(b[j + 1]));
          const float2 c0 = cs[c + j], c1 = cs[c + j + 1];
          y1[j / 2] = pack_bf16x2(p0 * c0.x - q0 * c0.y, p1 * c1.x - q1 * c1.y);
          y2[j / 2] = pack_bf16x2(q0 * c0.x + p0 * c0.y, q1 * c1.x + p1 * c1.y);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          y1[j / 2] = pack_bf16x2(a[j], a[j + 1]);
          y2[j / 2] = pack_bf16x2(b[j], b[j + 1]);
        }
      }
      bf16* dst;
      if (gh < qa.n_heads) {
        dst = C + (size_t)m * ldc + gh * 128;
      } else {
        if (slot < 0) continue;     // metadata failed the bounds check in expand_tokens: no KV write
        const int kvh = gh < qa.n_heads + qa.n_kv ? gh - qa.n_heads : gh - qa.n_heads - qa.n_kv;
        bf16* cache = gh < qa.n_heads + qa.n_kv ? qa.k_cache : qa.v_cache;
        dst = cache + (((size_t)page * qa.n_kv + kvh) * qa.page_size + off) * 128;
      }
      *reinterpret_cast<uint4*>(dst + c) = make_uint4(y1[0], y1[1], y1[2], y1[3]);
      *reinterpret_cast<uint4*>(dst + 64 + c) = make_uint4(y2[0], y2[1], y2[2], y2[3]);
    }
  }
}

// Work = (tile t of 128 W rows, K-block kb), linearised t-major; CTA b owns [b*per, (b+1)*per).
template <int NT, int MODE>
__global__ void __launch_bounds__(THREADS, 1)
gemm_skinny_tcgen05(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, int M,
                    int N, int K, int per, bf16* __restrict__ C, int ldc, const bf16* __restrict__ bias,
                    const bf16* __restrict__ residual, int ldr, float* __restrict__ partial,
                    int* __restrict__ counters, const QkvRopeArgs qa, const RowNorm nm, int csize, int tag) {
  using L = SkSmem<NT>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* st = reinterpret_cast<float*>(smem + L::EPI_OFF);
  float* rs_sm = reinterpret_cast<float*>(smem + L::RS_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  volatile uint32_t* last_flag = tmem_slot + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SK_TRACE(0);
  pdl_trigger();
  const int kbs = K / KB;
  const int work = (N / W_ROWS) * kbs;
  int g_begin, g_end;
  if (csize > 1) {
    const int t = blockIdx.x / csize, r = blockIdx.x % csize;  // 1-D cluster: rank = blockIdx.x % csize
    g_begin = t * kbs + r * kbs / csize;
    g_end = t * kbs + (r + 1) * kbs / csize;
  } else {
    g_begin = blockIdx.x * per;
    g_end = min(g_begin + per, work);
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * NT < 32 ? 32 : 2 * NT);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) SK_TRACE(1);

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once per step
      const uint64_t pol_x = policy_evict_last();   // the activations are re-read by every CTA
      // The CTA's range is contiguous: iteration i is K-block (g_begin + i) % kbs of tile
      // (g_begin + i) / kbs. The weights of the first STAGES iterations are fetched before the
      // predecessor kernel has finished (PDL); only the activations wait for it.
      const int n_it = g_end - g_begin, pre = min(n_it, STAGES);
      for (int i = 0; i < pre; ++i) {
        const int g = g_begin + i, t = g / kbs;
        mbar_arrive_expect_tx(&full[i], L::STAGE_BYTES);
        tma_load_2d_hint(&map_w, &full[i], smem + i * L::STAGE_BYTES, (g - t * kbs) * KB, t * W_ROWS, pol_w);
      }
      pdl_wait();
      SK_TRACE(2);
      for (int i = 0; i < n_it; ++i) {
        const int g = g_begin + i, t = g / kbs, kc = (g - t * kbs) * KB;
        const int s = i % STAGES;
        uint8_t* sw = smem + s * L::STAGE_BYTES;
        if (i >= pre) {
          mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES);
          tma_load_2d_hint(&map_w, &full[s], sw, kc, t * W_ROWS, pol_w);
        }
        tma_load_2d_hint(&map_x, &full[s], sw + L::W_BYTES, kc, 0, pol_x);
      }
    }
    __syncwarp();
    if (csize > 1) {
      cluster_arrive_release();
      cluster_wait_acquire();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(W_ROWS, NT);
    int it = 0, lt = 0;
    for (int g = g_begin; g < g_end; ++lt) {
      const int t = g / kbs, kb0 = g - t * kbs, nkb = min(kbs - kb0, g_end - g);
      const int acc = lt & 1;
      mbar_wait(&acc_empty[acc], ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * NT);
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
#ifdef GLLM_TRACE
        if (it == 0 && lane == 0) SK_TRACE(3);
        if (it == STAGES && lane == 0) SK_TRACE(4);
#endif
        if (elect_one()) {
          const uint8_t* sw = smem + s * L::STAGE_BYTES;
          const uint64_t dw = smem_desc_sw128(sw);
          const uint64_t dx = smem_desc_sw128(sw + L::W_BYTES);
#pragma unroll
          for (int k = 0; k < KB / 16; ++k) mma_bf16_ss(d_tmem, dw + 2 * k, dx + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
          if (i == nkb - 1) mma_commit(&acc_full[acc]);
        }
        __syncwarp();
      }
      g += nkb;
    }
    __syncwarp();
    if (csize > 1) {
      cluster_arrive_release();
      cluster_wait_acquire();
    }
  } else {
    // epilogue warps 2-5: warp q = w % 4 reads TMEM lanes [32q, 32q + 32) = W rows of the tile
    pdl_wait();  // writes C / partials, reads the residual
    const int q = warp & 3, f = q * 32 + lane, et = threadIdx.x - 64;
    if (nm.ss_in != nullptr) {
      if (et < M) rs_sm[et] = row_norm_scale(nm, et);
      epi_bar();
    }
    int lt = 0;
    for (int g = g_begin; g < g_end; ++lt) {
      const int t = g / kbs, kb0 = g - t * kbs, nkb = min(kbs - kb0, g_end - g);
      g += nkb;
      const int acc = lt & 1;
      mbar_wait(&acc_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      if (et == 0) SK_TRACE(5);
      float v[NT];
      {
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NT);
        if constexpr (NT == 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(ta, r);
          tmem_ld_wait();
#pragma unroll
          for (int m = 0; m < 16; ++m) v[m] = __uint_as_float(r[m]);
        } else {
          uint32_t r[32];
          tmem_ld_32x32b_x32(ta, r);
          tmem_ld_wait();
#pragma unroll
          for (int m = 0; m < 32; ++m) v[m] = __uint_as_float(r[m]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);  // accumulator is in registers now
      if (et == 0) SK_TRACE(8);
      bool finish = true;
      if (csize > 1) {
        // cluster split-K: ranks >= 1 store their partial into rank 0's smem; the barrier
        // (release / acquire at cluster scope) publishes it; rank 0 sums ranks in order
        const int r = blockIdx.x % csize;
        float* red = reinterpret_cast<float*>(smem + L::RED_OFF);
        if (r != 0) {
          const uint32_t dst = mapa_shared(smem_u32(red + (size_t)(r - 1) * NT * W_ROWS + f), 0);
#pragma unroll
          for (int m = 0; m < NT; ++m)
            if (m < M) st_shared_cluster_f32(dst + (uint32_t)(m * W_ROWS * 4), v[m]);
        }
        cluster_arrive_release();
        cluster_wait_acquire();
        finish = r == 0;
        if (finish) {
          for (int j = 1; j < csize; ++j) {
            const float* p = red + (size_t)(j - 1) * NT * W_ROWS + f;
#pragma unroll
            for (int m = 0; m < NT; ++m)
              if (m < M) v[m] += p[m * W_ROWS];
          }
        }
      } else if (nkb != kbs) {
        // tile shared with other CTAs: publish, count in, the last contributor sums all
        const int first = (t * kbs) / per, last = (t * kbs + kbs - 1) / per;
        float* mine = partial + (size_t)(t + blockIdx.x) * NT * W_ROWS + f;
#pragma unroll
        for (int m = 0; m < NT; ++m)
          if (m < M) mine[m * W_ROWS] = v[m];
        __threadfence();
        epi_bar();
        if (et == 0) SK_TRACE(9);
        if (et == 0) {
          const int prev = atomicAdd(&counters[t], 1);
          const bool is_last = prev == last - first;
          if (is_last) counters[t] = 0;  // zero again for the next launch on this workspace
          *last_flag = is_last ? 1u : 0u;
        }
        epi_bar();
        if (et == 0) SK_TRACE(10);
        finish = *last_flag != 0;
        if (finish) {
          __threadfence();
          // contributors summed in order j = first..last (deterministic); the loads of a batch of
          // U partials are all issued before the adds, so the fix-up costs one L2 round trip per
          // batch instead of one per contributor
          constexpr int U = NT == 16 ? 4 : 2;
          float sum[NT];
#pragma unroll
          for (int m = 0; m < NT; ++m) sum[m] = 0.f;
          for (int j0 = first; j0 <= last; j0 += U) {
            float x[U][NT];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int j = j0 + u;
              const float* p = partial + (size_t)(t + j) * NT * W_ROWS + f;
              const bool ld = j <= last && j != (int)blockIdx.x;
#pragma unroll
              for (int m = 0; m < NT; ++m) x[u][m] = (ld && m < M) ? __ldcg(p + m * W_ROWS) : v[m];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (j0 + u <= last) {
#pragma unroll
                for (int m = 0; m < NT; ++m) sum[m] += x[u][m];
              }
          }
#pragma unroll
          for (int m = 0; m < NT; ++m) v[m] = sum[m];
          if (et == 0) SK_TRACE(11);
        }
      }
      if (finish) {
#pragma unroll
        for (int m = 0; m < NT; ++m) st[m * L::ST_LD + f] = v[m];
        epi_bar();
        skinny_epilogue<NT, MODE>(st, et, t, M, N, C, ldc, bias, residual, ldr, qa, nm, rs_sm);
        epi_bar();  // staging is reused by the next tile
      }
      if (et == 0) SK_TRACE(6);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 2 * NT < 32 ? 32 : 2 * NT);
  if (threadIdx.x == 0) SK_TRACE(7);
}

template <int NT, int MODE>
int launch_skinny(const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, int per, int grid, int csize,
                  bf16* C, int ldc, const bf16* bias, const bf16* res, int ldr, float* partial, int* counters,
                  const QkvRopeArgs& qa, const RowNorm& nm, cudaStream_t st) {
  constexpr int smem = SkSmem<NT>::TOTAL;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_skinny_tcgen05<NT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return set_cuda_error(e, "skinny gemm smem attribute");
    attr = true;
  }
  static int tag = 0;
  cudaError_t e = launch_kernel(gemm_skinny_tcgen05<NT, MODE>, dim3(grid), dim3(THREADS), smem, st, csize, mw, mx, M,
                                N, K, per, C, ldc, bias, res, ldr, partial, counters, qa, nm, csize, tag++);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm_skinny_tcgen05 launch");
  return check_launch("gemm_skinny_tcgen05");
}

// Co-resident clusters of c CTAs for this instantiation (GPC packing), cached per c.
template <int NT, int MODE>
int max_active_clusters(int c) {
  static int cache[SkSmem<NT>::MAX_CLUSTER + 1] = {};
  if (cache[c] == 0) {
    cudaFuncSetAttribute(gemm_skinny_tcgen05<NT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SkSmem<NT>::TOTAL);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * device_sm_count());
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SkSmem<NT>::TOTAL;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = c;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_skinny_tcgen05<NT, MODE>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[c] = n > 0 ? n : -1;
  }
  return cache[c];
}

// Cluster size for a skinny GEMM: the largest c <= 4 whose tiles x c CTAs are all co-resident and
// cover >= 3/5 of the SMs with >= 4 K-blocks each; 1 = stream-K (many tiles: it balances any N).
// Measured (tools/skinny_chain.py, M = 4): 40 tiles c=3 -13% vs stream-K, 32 tiles c=4 -17%,
// 48 tiles c=2 (65% of the SMs) -9%, 32 tiles c=2 (43%) +16%; 64 tiles c=2 even.
// GLLM_SKINNY_CLUSTER=1 forces stream-K, =2..4 forces c where it fits (A/B runs).
template <int NT, int MODE>
int pick_cluster(int tiles, int kbs) {
  static const int forced = [] {
    const char* e = getenv("GLLM_SKINNY_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  static const bool verbose = getenv("GLLM_SKINNY_VERBOSE") != nullptr;
  const int sms = device_sm_count();
  int pick = 1;
  for (int c = SkSmem<NT>::MAX_CLUSTER; c >= 2 && pick == 1; --c) {
    if (forced && c != forced) continue;
    if (kbs / c < 4 || tiles > max_active_clusters<NT, MODE>(c)) continue;
    if (forced || 5 * tiles * c >= 3 * sms) pick = c;
  }
  if (verbose)
    fprintf(stderr, "[gllm] skinny NT=%d mode=%d tiles=%d kbs=%d -> cluster %d (co-resident clusters c=2/3/4: %d/%d/%d)\n",
            NT, MODE, tiles, kbs, pick, max_active_clusters<NT, MODE>(2), max_active_clusters<NT, MODE>(3),
            max_active_clusters<NT, MODE>(4));
  return pick;
}

template <int NT, int MODE>
int run_skinny(const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, bf16* C, int ldc,
               const bf16* bias, const bf16* res, int ldr, float* partial, int* counters, const QkvRopeArgs& qa,
               const RowNorm& nm, cudaStream_t st) {
  const int sms = device_sm_count();
  const int tiles = N / W_ROWS, kbs = K / KB, work = tiles * kbs;
  const int csize = pick_cluster<NT, MODE>(tiles, kbs);
  int per = (work + sms - 1) / sms;
  if (per < 4) per = 4 < kbs ? 4 : kbs;  // >= 256 of K per CTA amortises the pipeline fill
  const int grid = csize > 1 ? tiles * csize : (work + per - 1) / per;
  return launch_skinny<NT, MODE>(mw, mx, M, N, K, per, grid, csize, C, ldc, bias, res, ldr, partial, counters, qa,
                                 nm, st);
}

thread_local const void* t_clean_ws = nullptr;

}  // namespace

constexpr size_t SKINNY_COUNTER_BYTES = GEMM_WS_HEAD_BYTES;

void gemm_ws_mark_clean(const void* workspace) { t_clean_ws = workspace; }

int gemm_ws_reset(void* workspace, cudaStream_t st) {
  if (workspace == nullptr) return 0;
  cudaError_t e = cudaMemsetAsync(workspace, 0, SKINNY_COUNTER_BYTES, st);
  if (e != cudaSuccess) return set_cuda_error(e, "skinny gemm counters");
  t_clean_ws = workspace;
  return 0;
}

bool gemm_skinny_eligible(int M, int N, int K) {
  static const int enabled = [] {
    const char* e = getenv("GLLM_GEMM_SKINNY");  // A/B switch (default on)
    return e ? atoi(e) : 1;
  }();
  return enabled && M >= 1 && M <= 32 && N % W_ROWS == 0 && K % KB == 0 && N / W_ROWS <= (int)(SKINNY_COUNTER_BYTES / 4);
}

size_t gemm_skinny_workspace_bytes(int M, int N, int K) {
  (void)K;
  const int nt = M <= 16 ? 16 : 32;
  return SKINNY_COUNTER_BYTES + (size_t)(N / W_ROWS + device_sm_count()) * nt * W_ROWS * sizeof(float);
}

int gemm_skinny(const bf16* A, int lda, int a_rows_alloc, const bf16* W, int ldw, bf16* C, int ldc, int M, int N,
                int K, int mode, const bf16* bias, const bf16* residual, int ldr, const QkvRopeArgs* qkv,
                void* workspace, size_t ws_bytes, cudaStream_t st, const RowNorm& nm) {
  const int nt = M <= 16 ? 16 : 32;
  const size_t need = gemm_skinny_workspace_bytes(M, N, K);
  if (workspace == nullptr || ws_bytes < need)
    return set_error(GLLM_ERR_INVALID, "skinny gemm workspace too small (%zu < %zu)", ws_bytes, need);
  if (t_clean_ws != workspace) {
    cudaError_t e = cudaMemsetAsync(workspace, 0, SKINNY_COUNTER_BYTES, st);
    if (e != cudaSuccess) return set_cuda_error(e, "skinny gemm counters");
  }
  int* counters = reinterpret_cast<int*>(workspace);
  float* partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + SKINNY_COUNTER_BYTES);
  CUtensorMap mw, mx;
  if (int rc = make_tma_map_2d(&mw, W, N, K, ldw, W_ROWS)) return rc;
  if (int rc = make_tma_map_2d(&mx, A, a_rows_alloc > M ? a_rows_alloc : M, K, lda, nt)) return rc;
  const QkvRopeArgs qa = qkv ? *qkv : QkvRopeArgs{};
#define GLLM_SKINNY(NTV)                                                                                     \
  if (mode == EPI_SWIGLU)                                                                                     \
    return run_skinny<NTV, EPI_SWIGLU>(mw, mx, M, N, K, C, ldc, nullptr, nullptr, 0, partial, counters, qa, nm, \
                                       st);                                                                     \
  if (mode == EPI_QKV_ROPE)                                                                                   \
    return run_skinny<NTV, EPI_QKV_ROPE>(mw, mx, M, N, K, C, ldc, bias, nullptr, 0, partial, counters, qa, nm, \
                                         st);                                                                   \
  return run_skinny<NTV, EPI_STORE>(mw, mx, M, N, K, C, ldc, bias, residual, ldr, partial, counters, qa, nm, st);
  if (nt == 16) {
    GLLM_SKINNY(16)
  } else {
    GLLM_SKINNY(32)
  }
#undef GLLM_SKINNY
}

}  // namespace gllm

#ifdef GLLM_TRACE
// debug builds only (not in include/gllm.h): copy the trace ring [64][160][12] u64 to host
extern "C" __attribute__((visibility("default"))) int gllm_debug_trace_read(void* host, size_t bytes) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, gllm::g_trace, bytes < sizeof(gllm::g_trace) ? bytes : sizeof(gllm::g_trace)) ==
                 cudaSuccess ? 0 : -1;
}
#endif
