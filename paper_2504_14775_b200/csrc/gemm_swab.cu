// Swap-AB 2-CTA tcgen05 GEMM for the residual projections (O, down) at medium / large M:
//
//   C[M, N] = A[M, K] . W[N, K]^T (+ bias[N]) (+ residual[M, N]),  fused-RMSNorm statistics out
//
// The weights take the MMA M axis and the tokens its N axis, so the token tile NT can be any
// multiple of 32 up to 256 instead of a multiple of the 256-row MMA: a token count like 2009
// becomes 9 tiles of 224 rather than 8 rows of 256, and the Llama-3-8B O / down projections at
// ~2k tokens are 144 units of 256 weights x 224 tokens over 74 clusters (two per cluster:
// 114,688 outputs on each) instead of 128 units of 256 x 256 (131,072 on the busiest) -- the tile
// shape cuBLAS's nvjet kernels pick for these shapes (profiles/r2/cublas_kernel_names.txt).
// Persistent like gemm.cu: a cluster of two CTAs walks its units (one token tile, every #clusters-
// per-tile-th weight tile; see the unit walk); per 64-wide K-block each CTA TMA-loads its 128 weight rows and half of the NT
// token rows, the leader issues one M=256, N=NT cta_group::2 MMA per K-step into one of two TMEM
// accumulators (columns 0 / 256), so the epilogue of unit i overlaps the MMAs of unit i+1.
//
// Epilogue (warps 2-5): TMEM lane = weight row, columns = tokens. Each warp writes its 32 rows x NT
// accumulators (+ bias) as bf16 into a [token][128 weights] smem staging tile and releases the TMEM
// buffer; then the 128 threads walk token rows, 16 threads per row and 8 consecutive outputs per
// thread: + residual (after the bf16 rounding, as gemm.cu's epilogue), one 16-byte store, and the
// sum of squares of each 64-column RMSNorm group over 8 lanes (fixed order: deterministic).
#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {
namespace {

constexpr int SW_BK = 64;
constexpr int SW_WROWS = 128;  // weight rows per CTA and unit (256 per cluster)
constexpr int SW_THREADS = 192;
constexpr int SW_SMEM_MAX = 227 * 1024;

template <int NT, bool QKV = false>
struct SwSmem {
  static constexpr int A_BYTES = SW_WROWS * SW_BK * 2;  // 16 KB weight box
  static constexpr int B_BYTES = (NT / 2) * SW_BK * 2;  // this CTA's half of the token box
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGING = NT * SW_WROWS * 2;     // bf16 [NT][128] epilogue staging
  // fp32 row scales of the unit's tokens (+ their positions and KV slots for the QKV epilogue)
  static constexpr int ROWSCALE = (QKV ? 3 : 1) * 256 * 4;
  static constexpr int STAGES_FIT = (SW_SMEM_MAX - 1024 - 256 - ROWSCALE - STAGING) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr int RING = STAGES * STAGE;
  static constexpr int TOTAL = 1024 + RING + STAGING + ROWSCALE + 256;
};

GLLM_DEVICE void sw_epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

enum : int { SW_STORE = 0, SW_SWIGLU = 2, SW_QKV_ROPE = 3 };  // gemm.cu's EPI_* numbering

template <int NT, int MODE>
__global__ void __launch_bounds__(SW_THREADS, 1)
gemm_swab_tcgen05(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, int M,
                  int N, int K, bf16* __restrict__ C, int ldc, const bf16* __restrict__ bias,
                  const bf16* __restrict__ residual, int ldr, const RowNorm nm, const QkvRopeArgs qa) {
  static_assert(NT % 32 == 0 && NT <= 256, "token tile: multiple of 32, at most 256");
  using L = SwSmem<NT, MODE == SW_QKV_ROPE>;
  constexpr int ST = L::STAGES;
  static_assert(ST >= 3, "smem ring too shallow");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  bf16* stg = reinterpret_cast<bf16*>(smem + L::RING);   // [NT][128]
  float* rs_s = reinterpret_cast<float*>(smem + L::RING + L::STAGING);  // [NT] row scales
  int* pos_s = reinterpret_cast<int*>(rs_s + 256);                       // [NT] (QKV) token positions
  int* slot_s = pos_s + 256;                                             // [NT] (QKV) KV slots
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::RING + L::STAGING + L::ROWSCALE);
  uint64_t* empty = full + ST;
  uint64_t* acc_full = empty + ST;   // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;  // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  const uint32_t rank = cluster_ctarank();
  const int m_tiles = (M + NT - 1) / NT;
  const int units = m_tiles * (N / (2 * SW_WROWS));
  const int unit0 = blockIdx.x >> 1, ustride = gridDim.x >> 1;
  const int nkb = K / SW_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 8);  // one arrival per epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg<2>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Unit walk. With at least one cluster per token tile, cluster c keeps token tile c % m_tiles for
  // its whole run and steps over the weight tiles (c / m_tiles) + k x (clusters of that token
  // tile): its per-token values (fused-norm row scales, positions, slots) are read once, and the
  // clusters at step k of all token tiles share the same few weight tiles in L2. Otherwise (fewer
  // units than clusters: one unit each, or when the token tiles' cluster counts do not divide the
  // weight tiles evenly enough) units are dealt token-tile-fastest.
  const int n_wt = N / (2 * SW_WROWS);
  // (only when it costs no extra wave: the token tile with the fewest clusters sets the length)
  const bool tt_major = ustride >= m_tiles &&
                        (n_wt + ustride / m_tiles - 1) / (ustride / m_tiles) <= (units + ustride - 1) / ustride;
  const int my_tt = unit0 % m_tiles, my_r = unit0 / m_tiles;
  const int my_cpt = tt_major ? (ustride - 1 - my_tt) / m_tiles + 1 : 1;
  const int my_units = tt_major ? (my_r < n_wt ? (n_wt - my_r + my_cpt - 1) / my_cpt : 0)
                                : (unit0 < units ? (units - unit0 + ustride - 1) / ustride : 0);
  auto coords = [&](int k, int& m0, int& n0) {
    if (tt_major) {
      m0 = my_tt * NT;
      n0 = (my_r + k * my_cpt) * (2 * SW_WROWS);
    } else {
      const int u = unit0 + k * ustride;
      m0 = (u % m_tiles) * NT;
      n0 = (u / m_tiles) * (2 * SW_WROWS);
    }
  };

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint32_t full_leader = mapa_shared(smem_u32(full), 0);
      auto expect = [&](int s) {
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * L::STAGE);
      };
      int pre = 0;
      if (my_units > 0) {  // the first unit's weights do not depend on the predecessor kernel
        int m0, n0;
        coords(0, m0, n0);
        pre = min(nkb, ST);
        for (int i = 0; i < pre; ++i) {
          expect(i);
          tma_load_2d_cg2(&map_w, full_leader + (uint32_t)(i * 8), smem + i * L::STAGE, i * SW_BK,
                          n0 + (int)rank * SW_WROWS, pol_w);
        }
      }
      pdl_wait();  // the activations are the predecessor's output
      int it = 0;
      for (int k = 0; k < my_units; ++k) {
        int m0, n0;
        coords(k, m0, n0);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1;
          uint8_t* sa = smem + s * L::STAGE;
          if (it >= pre) {
            mbar_wait(&empty[s], ph ^ 1);
            expect(s);
            tma_load_2d_cg2(&map_w, full_leader + (uint32_t)(s * 8), sa, i * SW_BK, n0 + (int)rank * SW_WROWS, pol_w);
          }
          tma_load_2d_cg2(&map_x, full_leader + (uint32_t)(s * 8), sa + L::A_BYTES, i * SW_BK,
                          m0 + (int)rank * (NT / 2), policy_evict_last());
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, NT);
      int it = 0, lt = 0;
      for (int k = 0; k < my_units; ++k, ++lt) {
        const int acc = lt & 1;
        mbar_wait(&acc_empty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 256);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint8_t* sa = smem + s * L::STAGE;
            const uint64_t da = smem_desc_sw128(sa);
            const uint64_t db = smem_desc_sw128(sa + L::A_BYTES);
#pragma unroll
            for (int k = 0; k < SW_BK / 16; ++k)
              mma_bf16_ss_cg<2>(d_tmem, da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
            mma_commit_cg<2>(&empty[s]);
            if (i == nkb - 1) mma_commit_cg<2>(&acc_full[acc]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    pdl_wait();  // C / residual / statistics are shared with the predecessor
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int t = (int)threadIdx.x - 64;  // 0..127
    const int c8 = t & 15;                // this thread's 8 output columns of a token row
    const uint32_t acc_empty_leader = mapa_shared(smem_u32(acc_empty), 0);
    int lt = 0;
    for (int k = 0; k < my_units; ++k, ++lt) {
      int m0, n0;
      coords(k, m0, n0);
      const int acc = lt & 1;
      const int wrow = n0 + (int)rank * SW_WROWS;   // this CTA's first weight row / output column
      const float b_mine = bias != nullptr ? bf2f(bias[wrow + q * 32 + lane]) : 0.f;
      if ((nm.ss_in != nullptr || MODE == SW_QKV_ROPE) && (k == 0 || !tt_major)) {
        // per-token values of this unit, read once (overlapping its MMAs): fused-RMSNorm row
        // scales, and for the QKV epilogue the positions and paged KV slots
        for (int j = t; j < NT; j += 128) {
          const int m = m0 + j;
          if (nm.ss_in != nullptr) rs_s[j] = m < M ? row_norm_scale(nm, m) : 1.f;
          if constexpr (MODE == SW_QKV_ROPE) {
            pos_s[j] = m < M ? qa.tok_pos[m] : 0;
            slot_s[j] = m < M ? qa.tok_slot[m] : -1;
          }
        }
        sw_epi_bar();
      }
      mbar_wait(&acc_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      // TMEM (weight row = lane, token = column) -> bf16(acc * row scale + bias) staged as
      // [token][weight] (the roundings of gemm.cu's epilogues)
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256);
#pragma unroll 1
      for (int j0 = 0; j0 < NT; j0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tb + (uint32_t)j0, r);
        tmem_ld_wait();
        if (nm.ss_in != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            stg[(j0 + j) * SW_WROWS + q * 32 + lane] = f2bf(__uint_as_float(r[j]) * rs_s[j0 + j] + b_mine);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[(j0 + j) * SW_WROWS + q * 32 + lane] = f2bf(__uint_as_float(r[j]) + b_mine);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc_empty_leader + (uint32_t)(acc * 8));  // TMEM buffer free
      sw_epi_bar();
      if constexpr (MODE == SW_STORE) {
      const int col = wrow + 8 * c8;
      // 4 token rows per pass (rows j, j+8, j+16, j+24): their residual loads are in flight together
      constexpr int R = 4;
#pragma unroll 1
      for (int jb = t >> 4; jb < NT; jb += 8 * R) {  // both half-warps run NT / 32 passes (shuffles below)
        uint4 sv[R], rv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int j = jb + 8 * r;
          sv[r] = *reinterpret_cast<const uint4*>(stg + j * SW_WROWS + 8 * c8);
          rv[r] = make_uint4(0, 0, 0, 0);
          if (residual != nullptr && m0 + j < M) rv[r] = *reinterpret_cast<const uint4*>(residual + (size_t)(m0 + j) * ldr + col);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = m0 + jb + 8 * r;
          const bool live = m < M;
          uint4 o = sv[r];
          if (residual != nullptr) {
            // the staged value is already bf16(acc + bias): add the residual, round once more
            const float2 g0 = unpack_bf16x2(o.x), g1 = unpack_bf16x2(o.y), g2 = unpack_bf16x2(o.z),
                         g3 = unpack_bf16x2(o.w);
            const float2 a = unpack_bf16x2(rv[r].x), b = unpack_bf16x2(rv[r].y), c = unpack_bf16x2(rv[r].z),
                         d = unpack_bf16x2(rv[r].w);
            o = make_uint4(pack_bf16x2(g0.x + a.x, g0.y + a.y), pack_bf16x2(g1.x + b.x, g1.y + b.y),
                           pack_bf16x2(g2.x + c.x, g2.y + c.y), pack_bf16x2(g3.x + d.x, g3.y + d.y));
          }
          if (live) *reinterpret_cast<uint4*>(C + (size_t)m * ldc + col) = o;
          if (nm.ss_out != nullptr) {
            const float2 h0 = unpack_bf16x2(o.x), h1 = unpack_bf16x2(o.y), h2 = unpack_bf16x2(o.z),
                         h3 = unpack_bf16x2(o.w);
            const float f[8] = {h0.x, h0.y, h1.x, h1.y, h2.x, h2.y, h3.x, h3.y};
            float ss = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
            // lanes 8g .. 8g+7 of this half-warp hold the 64 columns of one RMSNorm group of row m
            ss += __shfl_xor_sync(0xffffffffu, ss, 1);
            ss += __shfl_xor_sync(0xffffffffu, ss, 2);
            ss += __shfl_xor_sync(0xffffffffu, ss, 4);
            if (live && (c8 & 7) == 0) nm.ss_out[(size_t)(col / NORM_GROUP) * nm.ld + m] = ss;
          }
        }
      }
      } else if constexpr (MODE == SW_SWIGLU) {
        // the CTA's 128 weight rows are 64 gate rows then the 64 matching up rows (interleaved
        // weight): lanes with c8 < 8 write act = bf16(silu(g)) * u for 8 output columns
        const int ocol = (wrow >> 1) + 8 * (c8 & 7);
#pragma unroll 2
        for (int j = t >> 4; j < NT; j += 8) {
          const int m = m0 + j;
          if (c8 >= 8 || m >= M) continue;
          const uint4 gv = *reinterpret_cast<const uint4*>(stg + j * SW_WROWS + 8 * c8);
          const uint4 uv = *reinterpret_cast<const uint4*>(stg + j * SW_WROWS + 64 + 8 * c8);
          const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w}, uw[4] = {uv.x, uv.y, uv.z, uv.w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 g = unpack_bf16x2(gw[e]), u = unpack_bf16x2(uw[e]);
            const float a0 = bf2f(f2bf(silu_f(g.x))), a1 = bf2f(f2bf(silu_f(g.y)));
            o[e] = pack_bf16x2(a0 * u.x, a1 * u.y);
          }
          *reinterpret_cast<uint4*>(C + (size_t)m * ldc + ocol) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      } else {
        // QKV + RoPE + paged K/V write: the CTA's 128 weight rows are one whole head gh; lanes
        // c8 < 8 hold dims d = 8 c8.. of the first half, c8 >= 8 the matching second half, and each
        // reads its rotate-half partner from the staging tile
        const int gh = wrow >> 7;
        const int half = c8 >> 3, d0 = 8 * (c8 & 7);
        const bool rotate = gh < qa.n_heads + qa.n_kv;
        const bool is_q = gh < qa.n_heads, is_k = !is_q && rotate;
        const int kvh = is_k ? gh - qa.n_heads : gh - qa.n_heads - qa.n_kv;
        bf16* cache = is_k ? qa.k_cache : qa.v_cache;
        constexpr int R = 4;  // token rows per pass: their (cos, sin) loads are in flight together
#pragma unroll 1
        for (int jb = t >> 4; jb < NT; jb += 8 * R) {
          float4 cs[R][4];
          if (rotate) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const float4* src = reinterpret_cast<const float4*>(qa.rope + ((size_t)pos_s[jb + 8 * r] * 64 + d0) * 2);
#pragma unroll
              for (int e = 0; e < 4; ++e) cs[r][e] = src[e];   // (cos, sin) of dims d0 + 2e, d0 + 2e + 1
            }
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int j = jb + 8 * r, m = m0 + j;
            if (m >= M) continue;
            const uint4 xv = *reinterpret_cast<const uint4*>(stg + j * SW_WROWS + 8 * c8);
            uint4 out = xv;
            if (rotate) {
              const uint4 pv = *reinterpret_cast<const uint4*>(stg + j * SW_WROWS + 8 * (c8 ^ 8));
              const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, pw[4] = {pv.x, pv.y, pv.z, pv.w};
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 x = unpack_bf16x2(xw[e]), pr = unpack_bf16x2(pw[e]);
                const float4 c = cs[r][e];  // (cos, sin) of dim d0 + 2e, then of d0 + 2e + 1
                // first half: p c - q s; second half: q c + p s (p = first-half value, q = second)
                o[e] = half == 0 ? pack_bf16x2(x.x * c.x - pr.x * c.y, x.y * c.z - pr.y * c.w)
                                 : pack_bf16x2(x.x * c.x + pr.x * c.y, x.y * c.z + pr.y * c.w);
              }
              out = make_uint4(o[0], o[1], o[2], o[3]);
            }
            bf16* dst;
            if (is_q) {
              dst = C + (size_t)m * ldc + gh * 128;
            } else {
              const int slot = slot_s[j];
              if (slot < 0) continue;  // metadata failed the bounds check in expand_tokens: no KV write
              const int page = slot / qa.page_size, off = slot % qa.page_size;
              dst = cache + (((size_t)page * qa.n_kv + kvh) * qa.page_size + off) * 128;
            }
            *reinterpret_cast<uint4*>(dst + 8 * c8) = out;
          }
        }
      }
      sw_epi_bar();  // staging is reused by the next unit
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's MMAs, TMEM reads and remote arrivals are done
  if (warp == 1) tmem_dealloc_cg<2>(tmem_base, 512);
}

template <int NT, int MODE>
int launch_swab(const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, bf16* C, int ldc,
                const bf16* bias, const bf16* res, int ldr, const RowNorm& nm, const QkvRopeArgs& qa, cudaStream_t st) {
  constexpr int smem = SwSmem<NT, MODE == SW_QKV_ROPE>::TOTAL;
  auto kern = gemm_swab_tcgen05<NT, MODE>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "swab gemm smem attribute");
    attr_done = true;
  }
  const long units = (long)(N / (2 * SW_WROWS)) * ((M + NT - 1) / NT);
  const long slots = device_sm_count() / 2;
  const int clusters = (int)(units < slots ? units : slots);
  cudaError_t e = launch_kernel(kern, dim3(2 * clusters), dim3(SW_THREADS), smem, st, 2, mw, mx, M, N, K, C, ldc, bias,
                                res, ldr, nm, qa);
  if (e != cudaSuccess) return set_cuda_error(e, "swab gemm launch");
  return check_launch("gemm_swab_tcgen05");
}

}  // namespace

// Token width NT (multiple of 32, 128..256) minimising the per-cluster work waves x NT (ties to
// the wider tile); *work_per_sm = that work in outputs per SM (256 x NT x waves / 2).
int gemm_swab_tile(int M, int N, int K, double* work_per_sm) {
  static const int enabled = [] {
    const char* e = getenv("GLLM_GEMM_SWAB");  // A/B switch (default on)
    return e ? atoi(e) : 1;
  }();
  if (!enabled || M <= 0 || N % (2 * SW_WROWS) || K % SW_BK) return 0;
  const long slots = device_sm_count() / 2;
  int best_nt = 0;
  long best_w = 0;
  for (int nt = 256; nt >= 128; nt -= 32) {  // 64 / 96 measured slower than the 2-CTA tiles
    const long units = (long)(N / (2 * SW_WROWS)) * ((M + nt - 1) / nt);
    const long w = (units + slots - 1) / slots * nt;
    if (best_nt == 0 || w < best_w) {
      best_w = w;
      best_nt = nt;
    }
  }
  // modelled MMA efficiency falls with the token width like the 2-CTA tiles' with BN (256: 0.85,
  // 128: 0.75): the work is returned already divided by it, relative to 0.85
  if (work_per_sm) *work_per_sm = 128.0 * (double)best_w * 0.85 / (0.65 + 0.2 * best_nt / 256.0);
  return best_nt;
}

template <int NT>
int launch_mode(int mode, const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, bf16* C, int ldc,
                const bf16* bias, const bf16* res, int ldr, const RowNorm& nm, const QkvRopeArgs* qa, cudaStream_t st) {
  if (mode == SW_SWIGLU) return launch_swab<NT, SW_SWIGLU>(mw, mx, M, N, K, C, ldc, nullptr, nullptr, 0, nm, QkvRopeArgs{}, st);
  if (mode == SW_QKV_ROPE) return launch_swab<NT, SW_QKV_ROPE>(mw, mx, M, N, K, C, ldc, bias, nullptr, 0, nm, *qa, st);
  return launch_swab<NT, SW_STORE>(mw, mx, M, N, K, C, ldc, bias, res, ldr, nm, QkvRopeArgs{}, st);
}

int gemm_swab(const bf16* A, int lda, int a_rows_alloc, const bf16* W, int ldw, bf16* C, int ldc, int M, int N,
              int K, int nt, int mode, const bf16* bias, const bf16* residual, int ldr, const QkvRopeArgs* qa,
              cudaStream_t st, const RowNorm& nm) {
  if (ldc % 8 || (residual && ldr % 8)) return set_error(GLLM_ERR_INVALID, "gemm output pitch must be a multiple of 8");
  if (mode == SW_QKV_ROPE && qa == nullptr) return set_error(GLLM_ERR_INVALID, "swab gemm: QKV mode needs its args");
  CUtensorMap mw, mx;
  if (int rc = make_tma_map_2d(&mw, W, N, K, ldw, SW_WROWS)) return rc;
  if (int rc = make_tma_map_2d(&mx, A, a_rows_alloc > M ? a_rows_alloc : M, K, lda, nt / 2)) return rc;
  switch (nt) {
    case 128: return launch_mode<128>(mode, mw, mx, M, N, K, C, ldc, bias, residual, ldr, nm, qa, st);
    case 160: return launch_mode<160>(mode, mw, mx, M, N, K, C, ldc, bias, residual, ldr, nm, qa, st);
    case 192: return launch_mode<192>(mode, mw, mx, M, N, K, C, ldc, bias, residual, ldr, nm, qa, st);
    case 224: return launch_mode<224>(mode, mw, mx, M, N, K, C, ldc, bias, residual, ldr, nm, qa, st);
    case 256: return launch_mode<256>(mode, mw, mx, M, N, K, C, ldc, bias, residual, ldr, nm, qa, st);
    default: return set_error(GLLM_ERR_INVALID, "swab gemm: bad token tile %d", nt);
  }
}

}  // namespace gllm
