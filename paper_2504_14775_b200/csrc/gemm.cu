// tcgen05 + TMA bf16 GEMM for the stage projections (QKV, O, gate-up, down, LM head).
//
//   C[M, N] = A[M, K] . B[N, K]^T  (+ bias[N]) (+ residual[M, N])
//
// A = activations (tokens x K), B = weights (out_features x K); both K-major
// row-major bf16, exactly how the stage stores them, so no transposes.
// Persistent (one CTA per SM) over 128 x BN output tiles (optionally K-slices, split-K):
//   warp 0  : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1  : TMEM allocator + MMA issuer (one lane), tcgen05.mma M=128,N=BN,K=16 into
//             one of two TMEM accumulators (the epilogue drains the other)
//   warps 2-5: epilogue, tcgen05.ld 32 lanes x 32 cols -> bf16 (+bias/+residual, or fused
//             SiLU*mul for the interleaved gate-up weight)
// CG = 2: a cluster of two CTAs (one TPC) computes a 256 x BN tile with tcgen05.mma
// cta_group::2, each CTA loading its 128 A rows and half of the BN weight rows.
// Rows past M are zero-filled by TMA on load and masked on store. Tiling per call
// (gemm_impl): M <= 32 goes to the swap-AB decode kernel (gemm_skinny.cu); short-K GEMMs
// with few output tiles run whole-K narrow / 2-CTA tiles; other <= 4-row-tile GEMMs
// split K (fp32 partials + a reduce with the fused epilogue) to spread the weight stream
// over all 148 SMs; large M picks (CG, BN) by a modelled time.
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int GEMM_THREADS = 192;

// A rows per TMA box: 64 for a single 1-CTA row tile of <= 64 tokens, else the full 128
__host__ __device__ constexpr int a_box_rows(int M, int cg) { return (cg == 1 && M <= 64) ? 64 : BM; }

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TOTAL = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers, TMEM slot*/;
};

enum : int { EPI_STORE = 0, EPI_PARTIAL_F32 = 1, EPI_SWIGLU = 2, EPI_QKV_ROPE = 3 };


// Epilogue of one 128 x BN output tile held in TMEM columns [acc_col, acc_col + BN):
// warp (w % 4) reads TMEM lanes [32q, 32q+32), i.e. output rows m0 + 32q + lane.
template <int BN, int MODE>
__device__ __forceinline__ void epilogue_tile(uint32_t tmem_lane_base, int row, int n0, int split, int M, int N,
                                              bf16* __restrict__ C, int ldc, const bf16* __restrict__ bias,
                                              const bf16* __restrict__ residual, int ldr,
                                              float* __restrict__ partial, const QkvRopeArgs& qa,
                                              const RowNorm& nm) {
  // fused RMSNorm: this row's scale for the GEMM output (ss_in), and its output statistics (ss_out)
  const float rs = (nm.ss_in != nullptr && row < M) ? row_norm_scale(nm, row) : 1.f;
  if constexpr (MODE == EPI_QKV_ROPE) {
    // Head-aligned tile: columns [128h, 128h+128) are one whole head of this token row, so the
    // rotate-half pairs (d, d+64) are thread-local. q heads are rotated and written back to C;
    // k heads rotated and v heads copied straight into the paged cache slot of the token.
    const bool live = row < M;
    const int pos = live ? qa.tok_pos[row] : 0;
    const int slot = live ? qa.tok_slot[row] : 0;
    const int page = slot / qa.page_size, off = slot % qa.page_size;
    const float2* cs = reinterpret_cast<const float2*>(qa.rope) + (size_t)pos * 64;
#pragma unroll 1
    for (int hl = 0; hl < BN / 128; ++hl) {
      const int gh = (n0 >> 7) + hl;
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t x1[32], x2[32];
        tmem_ld_32x32b_x32(tmem_lane_base + (uint32_t)(128 * hl + c), x1);
        tmem_ld_32x32b_x32(tmem_lane_base + (uint32_t)(128 * hl + 64 + c), x2);
        tmem_ld_wait();
        if (!live) continue;
        const int col1 = gh * 128 + c;
        float a[32], b[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          a[j] = __uint_as_float(x1[j]) * rs;
          b[j] = __uint_as_float(x2[j]) * rs;
        }
        if (bias != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            a[j] += bf2f(bias[col1 + j]);
            b[j] += bf2f(bias[col1 + 64 + j]);
          }
        }
        uint32_t y1[16], y2[16];
        if (gh < qa.n_heads + qa.n_kv) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            // same roundings as GEMM -> bf16 -> RoPE kernel
            const float p0 = bf2f(f2bf(a[j])), p1 = bf2f(f2bf(a[j + 1]));
            const float q0 = bf2f(f2bf(b[j])), q1 = bf2f(f2bf(b[j + 1]));
            const float2 c0 = cs[c + j], c1 = cs[c + j + 1];
            y1[j / 2] = pack_bf16x2(p0 * c0.x - q0 * c0.y, p1 * c1.x - q1 * c1.y);
            y2[j / 2] = pack_bf16x2(q0 * c0.x + p0 * c0.y, q1 * c1.x + p1 * c1.y);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            y1[j / 2] = pack_bf16x2(a[j], a[j + 1]);
            y2[j / 2] = pack_bf16x2(b[j], b[j + 1]);
          }
        }
        bf16* dst;
        if (gh < qa.n_heads) {
          dst = C + (size_t)row * ldc + gh * 128;
        } else {
          if (slot < 0) continue;   // metadata failed the bounds check in expand_tokens: no KV write
          const int kvh = gh < qa.n_heads + qa.n_kv ? gh - qa.n_heads : gh - qa.n_heads - qa.n_kv;
          bf16* cache = gh < qa.n_heads + qa.n_kv ? qa.k_cache : qa.v_cache;
          dst = cache + (((size_t)page * qa.n_kv + kvh) * qa.page_size + off) * 128;
        }
        uint4* d1 = reinterpret_cast<uint4*>(dst + c);
        uint4* d2 = reinterpret_cast<uint4*>(dst + 64 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          d1[j] = make_uint4(y1[4 * j], y1[4 * j + 1], y1[4 * j + 2], y1[4 * j + 3]);
          d2[j] = make_uint4(y2[4 * j], y2[4 * j + 1], y2[4 * j + 2], y2[4 * j + 3]);
        }
      }
    }
  } else if constexpr (MODE == EPI_SWIGLU) {
    // B rows interleave 64 gate / 64 up rows, so TMEM columns [128p, 128p+64) are gate
    // and [128p+64, 128p+128) the matching up outputs of this thread's token row:
    // act = bf16(silu(bf16 g)) * bf16(u), the same roundings as a separate SiLU kernel.
#pragma unroll 1
    for (int p = 0; p < BN / 128; ++p) {
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t g[32], u[32];
        tmem_ld_32x32b_x32(tmem_lane_base + (uint32_t)(128 * p + c), g);
        tmem_ld_32x32b_x32(tmem_lane_base + (uint32_t)(128 * p + 64 + c), u);
        tmem_ld_wait();
        const int ocol = (n0 >> 1) + 64 * p + c;
        if (row >= M || ocol >= (N >> 1)) continue;
        uint32_t packed[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float a0 = bf2f(f2bf(__uint_as_float(g[2 * j]) * rs)), a1 = bf2f(f2bf(__uint_as_float(g[2 * j + 1]) * rs));
          const float b0 = bf2f(f2bf(__uint_as_float(u[2 * j]) * rs)), b1 = bf2f(f2bf(__uint_as_float(u[2 * j + 1]) * rs));
          a0 = bf2f(f2bf(silu_f(a0)));
          a1 = bf2f(f2bf(silu_f(a1)));
          packed[j] = pack_bf16x2(a0 * b0, a1 * b1);
        }
        uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ldc + ocol);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
      }
    }
  } else {
    float ss = 0.f;  // sum of squares of this row's bf16 outputs (fused-norm statistics)
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_lane_base + (uint32_t)c, r);
      tmem_ld_wait();
      const int col = n0 + c;
      if (row >= M || col >= N) continue;
      if constexpr (MODE == EPI_PARTIAL_F32) {
        float4* dst = reinterpret_cast<float4*>(partial + ((size_t)split * M + row) * N + col);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      } else {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * rs;
        if (bias != nullptr) {
          const uint4* bp = reinterpret_cast<const uint4*>(bias + col);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u = bp[j];
            float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), cc = unpack_bf16x2(u.z), d = unpack_bf16x2(u.w);
            v[8 * j + 0] += a.x; v[8 * j + 1] += a.y; v[8 * j + 2] += b.x; v[8 * j + 3] += b.y;
            v[8 * j + 4] += cc.x; v[8 * j + 5] += cc.y; v[8 * j + 6] += d.x; v[8 * j + 7] += d.y;
          }
        }
        if (residual != nullptr) {
          const uint4* rp = reinterpret_cast<const uint4*>(residual + (size_t)row * ldr + col);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u = rp[j];
            float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), cc = unpack_bf16x2(u.z), d = unpack_bf16x2(u.w);
            // round the GEMM result to bf16 first, then add: same as bf16 "x + attn(x)".
            v[8 * j + 0] = bf2f(f2bf(v[8 * j + 0])) + a.x; v[8 * j + 1] = bf2f(f2bf(v[8 * j + 1])) + a.y;
            v[8 * j + 2] = bf2f(f2bf(v[8 * j + 2])) + b.x; v[8 * j + 3] = bf2f(f2bf(v[8 * j + 3])) + b.y;
            v[8 * j + 4] = bf2f(f2bf(v[8 * j + 4])) + cc.x; v[8 * j + 5] = bf2f(f2bf(v[8 * j + 5])) + cc.y;
            v[8 * j + 6] = bf2f(f2bf(v[8 * j + 6])) + d.x; v[8 * j + 7] = bf2f(f2bf(v[8 * j + 7])) + d.y;
          }
        }
        uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ldc + col);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                              pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
        if (nm.ss_out != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float q = bf2f(f2bf(v[j]));
            ss = fmaf(q, q, ss);
          }
          if (c & 32) {  // end of a 64-column group
            nm.ss_out[(size_t)((col & ~(NORM_GROUP - 1)) / NORM_GROUP) * nm.ld + row] = ss;
            ss = 0.f;
          }
        }
      }
    }
  }
}

// Persistent: one CTA (CG = 1) or one CTA pair (CG = 2, a 2-CTA cluster on one TPC) per SM / SM
// pair walks work units u = cluster id, +#clusters, ... where a unit is (m-tile, n-tile, K-split)
// with the m-tile fastest, so the CTAs running at the same time share each weight (B) tile
// through L2 and the weight matrix streams from HBM ~once per GEMM.
//
// CG = 2 (tcgen05 cta_group::2): a unit is a 256 x BN tile. Each CTA of the pair TMA-loads its
// own 128 A rows and HALF of the B tile (BN/2 rows) into its smem; the leader CTA issues
// M=256 MMAs that read A and B from both CTAs' smem and accumulate each CTA's 128 rows in that
// CTA's TMEM. Per SM and K-block that is 16 KB (A) + BN/2 x 128 B (B) instead of 16 KB + BN x
// 128 B: at BN = 256 a third less smem/L2 traffic per MMA, which is what keeps the tensor pipe
// fed (the 1-CTA kernel is smem-bandwidth bound at ~2/3 of MMA peak). Both CTAs' TMA loads
// complete on the leader's `full` barrier; the leader's commits multicast `empty` / `acc_full`
// to both CTAs; both CTAs' epilogue warps arrive on the leader's `acc_empty`.
// The accumulator is double-buffered in TMEM (2 x BN columns): the epilogue of unit i overlaps
// the MMAs of unit i+1; the smem ring's phases continue across units.
template <int BN, int STAGES, int MODE, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  int M, int N, int K, int k_blocks_per_split, int n_splits, bf16* __restrict__ C, int ldc,
                  const bf16* __restrict__ bias, const bf16* __restrict__ residual, int ldr,
                  float* __restrict__ partial, const QkvRopeArgs qa, const RowNorm nm) {
  static_assert(CG == 1 || CG == 2, "cta_group 1 or 2");
  using L = GemmSmem<BN / CG, STAGES>;   // per-CTA stage: 128 A rows + BN/CG B rows
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;    // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;     // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  constexpr int TM = BM * CG;           // rows per unit
  const int m_tiles = (M + TM - 1) / TM;
  const int n_tiles = N / BN;
  const int units = m_tiles * n_tiles * n_splits;
  const int total_kb = K / BK;
  const int unit0 = blockIdx.x / CG, ustride = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4 * CG);   // one arrival per epilogue warp of every CTA
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg<CG>(tmem_slot, 2 * BN);
  // M <= 64 (one row tile, 1-CTA): TMA loads only the first 64 A rows of each stage (a_box_rows,
  // same rule as the host's tensor map); the other 64 rows of every stage are zeroed once here
  // and never written again, so the A bytes each K-block moves into smem halve
  const int a_box = a_box_rows(M, CG);
  if (a_box < BM) {
    for (int s = 0; s < STAGES; ++s) {
      uint4* z = reinterpret_cast<uint4*>(smem + s * L::STAGE_BYTES + a_box * BK * 2);
      for (int i = threadIdx.x; i < (BM - a_box) * BK * 2 / 16; i += GEMM_THREADS) z[i] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core's operand reads
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised, TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto unit_coords = [&](int u, int& m0, int& n0, int& split, int& kb0, int& nkb) {
    const int mt = u % m_tiles;
    const int rest = u / m_tiles;
    const int nt = rest % n_tiles;
    split = rest / n_tiles;
    m0 = mt * TM;
    n0 = nt * BN;
    kb0 = split * k_blocks_per_split;
    nkb = min(total_kb, kb0 + k_blocks_per_split) - kb0;
  };

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream through once per step
      // both CTAs' loads complete on the leader's `full` barrier (CG = 2)
      const uint32_t full_leader = CG == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
      auto expect = [&](int s) {
        if constexpr (CG == 1) mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES - (BM - a_box) * BK * 2);
        else if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * L::STAGE_BYTES);
      };
      auto load_b = [&](int s, int kc, int bn) {
        uint8_t* sb = smem + s * L::STAGE_BYTES + L::A_BYTES;
        if constexpr (CG == 1) tma_load_2d_hint(&map_b, &full[s], sb, kc, bn, pol_w);
        else tma_load_2d_cg2(&map_b, full_leader + (uint32_t)(s * 8), sb, kc, bn, pol_w);
      };
      // The weights (B) do not depend on the predecessor kernel: the first ring's worth of this
      // CTA's first unit is fetched before griddepcontrol.wait, so the weight stream overlaps the
      // predecessor's tail; only the activations (A) wait for it.
      int pre = 0;
      if (unit0 < units) {
        int m0, n0, split, kb0, nkb;
        unit_coords(unit0, m0, n0, split, kb0, nkb);
        pre = min(nkb, STAGES);
        for (int i = 0; i < pre; ++i) {
          expect(i);
          load_b(i, (kb0 + i) * BK, n0 + (int)rank * (BN / CG));
        }
      }
      pdl_wait();  // A is the predecessor's output
      int it = 0;
      for (int u = unit0; u < units; u += ustride) {
        int m0, n0, split, kb0, nkb;
        unit_coords(u, m0, n0, split, kb0, nkb);
        const int am = m0 + (int)rank * BM, bn = n0 + (int)rank * (BN / CG);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          const int kc = (kb0 + i) * BK;
          if (it >= pre) {
            mbar_wait(&empty[s], ph ^ 1);
            expect(s);
            load_b(s, kc, bn);
          }
          if constexpr (CG == 1) tma_load_2d(&map_a, &full[s], sa, kc, am);
          else tma_load_2d_cg2(&map_a, full_leader + (uint32_t)(s * 8), sa, kc, am, policy_evict_last());
        }
      }
    }
  } else if (warp == 1) {
    if (CG == 1 || rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(TM, BN);
      int it = 0, lt = 0;
      for (int u = unit0; u < units; u += ustride, ++lt) {
        int m0, n0, split, kb0, nkb;
        unit_coords(u, m0, n0, split, kb0, nkb);
        const int acc = lt & 1;
        mbar_wait(&acc_empty[acc], ((lt >> 1) & 1) ^ 1);   // every epilogue drained this buffer
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint8_t* sa = smem + s * L::STAGE_BYTES;
            const uint8_t* sb = sa + L::A_BYTES;
            const uint64_t da = smem_desc_sw128(sa);
            const uint64_t db = smem_desc_sw128(sb);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // +32 B along K inside the swizzle atom = +2 in the 16-byte address field.
              mma_bf16_ss_cg<CG>(d_tmem, da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit_cg<CG>(&empty[s]);
            if (i == nkb - 1) mma_commit_cg<CG>(&acc_full[acc]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // Epilogue warps 2-5: warp (w % 4) may only touch TMEM lanes [32*(w%4), 32*(w%4)+32).
    pdl_wait();  // C / residual / KV cache are shared with the predecessor
    const int q = warp & 3;
    const uint32_t acc_empty_leader = CG == 2 ? mapa_shared(smem_u32(acc_empty), 0) : 0u;
    int lt = 0;
    for (int u = unit0; u < units; u += ustride, ++lt) {
      int m0, n0, split, kb0, nkb;
      unit_coords(u, m0, n0, split, kb0, nkb);
      const int acc = lt & 1;
      mbar_wait(&acc_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      epilogue_tile<BN, MODE>(lane_base, m0 + (int)rank * BM + q * 32 + lane, n0, split, M, N, C, ldc, bias,
                              residual, ldr, partial, qa, nm);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(acc_empty_leader + (uint32_t)(acc * 8));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the peer's MMAs / remote arrivals are done
  if (warp == 1) tmem_dealloc_cg<CG>(tmem_base, 2 * BN);
}

// Sum split-K partials [splits, M, N] fp32 and apply the epilogue; 8 columns per thread.
__global__ void splitk_reduce(const float* __restrict__ partial, int splits, int M, int N, bf16* __restrict__ C,
                              int ldc, const bf16* __restrict__ bias, const bf16* __restrict__ residual, int ldr,
                              const RowNorm nm) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t groups = (size_t)M * (N / 8);
  // (lanes past the end stay for the column-group shuffle below; M * N / 8 is a multiple of 8)
  if (idx >= groups) {
    if (nm.ss_out != nullptr) {
      float z = 0.f;
      for (int o = 1; o < 8; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    return;
  }
  const int row = (int)(idx / (N / 8));
  const int col = (int)(idx % (N / 8)) * 8;
  float v[8];
  {
    const float4* p = reinterpret_cast<const float4*>(partial + (size_t)row * N + col);
    float4 a = p[0], b = p[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  for (int s = 1; s < splits; ++s) {
    const float4* p = reinterpret_cast<const float4*>(partial + ((size_t)s * M + row) * N + col);
    float4 a = p[0], b = p[1];
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w; v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
  }
  if (nm.ss_in != nullptr) {
    const float rs = row_norm_scale(nm, row);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= rs;
  }
  if (bias != nullptr) {
    uint4 u = *reinterpret_cast<const uint4*>(bias + col);
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(w[j]);
      v[2 * j] += f.x;
      v[2 * j + 1] += f.y;
    }
  }
  if (residual != nullptr) {
    uint4 u = *reinterpret_cast<const uint4*>(residual + (size_t)row * ldr + col);
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(w[j]);
      v[2 * j] = bf2f(f2bf(v[2 * j])) + f.x;
      v[2 * j + 1] = bf2f(f2bf(v[2 * j + 1])) + f.y;
    }
  }
  *reinterpret_cast<uint4*>(C + (size_t)row * ldc + col) =
      make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
  if (nm.ss_out != nullptr) {
    // the 8 consecutive lanes of a 64-column group reduce in a fixed butterfly order
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float q = bf2f(f2bf(v[j]));
      ss = fmaf(q, q, ss);
    }
    for (int o = 1; o < 8; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((col & (NORM_GROUP - 1)) == 0) nm.ss_out[(size_t)(col / NORM_GROUP) * nm.ld + row] = ss;
  }
}

// Split-K reduce for the SwiGLU GEMM: N = 2*d_ff interleaved columns -> act[M, d_ff].
// Output column o reads gate column 128*(o/64) + o%64 and up column gate + 64.
__global__ void splitk_reduce_swiglu(const float* __restrict__ partial, int splits, int M, int N,
                                     bf16* __restrict__ C, int ldc, const RowNorm nm) {
  const int half = N / 2;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)M * (half / 8)) return;
  const int row = (int)(idx / (half / 8));
  const int o = (int)(idx % (half / 8)) * 8;
  const int gcol = 128 * (o / 64) + o % 64;
  float g[8], u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) g[j] = u[j] = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float* base = partial + ((size_t)s * M + row) * N;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      g[j] += base[gcol + j];
      u[j] += base[gcol + 64 + j];
    }
  }
  const float rs = nm.ss_in != nullptr ? row_norm_scale(nm, row) : 1.f;
  uint32_t pk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float a0 = bf2f(f2bf(g[2 * j] * rs)), a1 = bf2f(f2bf(g[2 * j + 1] * rs));
    a0 = bf2f(f2bf(silu_f(a0)));
    a1 = bf2f(f2bf(silu_f(a1)));
    pk[j] = pack_bf16x2(a0 * bf2f(f2bf(u[2 * j] * rs)), a1 * bf2f(f2bf(u[2 * j + 1] * rs)));
  }
  *reinterpret_cast<uint4*>(C + (size_t)row * ldc + o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
}

// ------------------------------------------------------------------ host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int64_t rows, cols, ld;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull + (size_t)k.cols * 0xC2B2AE3D27D4EB4Full + (size_t)k.ld * 31 +
         (size_t)k.box_rows;
    return h;
  }
};

// bf16 [rows, cols] row-major with leading dimension ld (elements); box = 64 cols x box_rows, 128B swizzle.
static int make_map(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return 0;
    }
  }
  PFN_encodeTiled enc = get_encoder();
  if (!enc) return set_error(GLLM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16)
    return set_error(GLLM_ERR_INVALID, "TMA operand must be 16-byte aligned with 16-byte row pitch");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(GLLM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return 0;
}

int make_tma_map_2d(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return make_map(out, ptr, rows, cols, ld, box_rows);
}

template <int BN, int STAGES, int MODE, int CG = 1>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, int splits, int kbps,
                       bf16* C, int ldc, const bf16* bias, const bf16* res, int ldr, float* partial,
                       cudaStream_t st, const RowNorm& nm, const QkvRopeArgs& qa = QkvRopeArgs{}) {
  constexpr int smem = GemmSmem<BN / CG, STAGES>::TOTAL;
  auto kern = gemm_bf16_tcgen05<BN, STAGES, MODE, CG>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm smem attribute");
    attr_done = true;
  }
  const long units = (long)((M + BM * CG - 1) / (BM * CG)) * (N / BN) * splits;
  const long slots = device_sm_count() / CG;
  const int clusters = (int)(units < slots ? units : slots);
  cudaError_t e = launch_kernel(kern, dim3(CG * clusters), dim3(GEMM_THREADS), smem, st, CG, ma, mb, M, N, K, kbps,
                                splits, C, ldc, bias, res, ldr, partial, qa, nm);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  return check_launch("gemm_bf16_tcgen05");
}

// The SwiGLU and QKV + RoPE epilogues of the swap-AB units are opt-in (GLLM_GEMM_SWAB_SWIGLU=1,
// GLLM_GEMM_SWAB_QKV=1): faster in isolated microbenchmarks (gate-up 299 -> 292 us, fused QKV 86
// -> 79 us at 2009 tokens) but 3-5% slower in the C2 step's ncu launch list, where their
// epilogues also compute the fused-RMSNorm row scales (profiles/r2/launches_c2_swab_all.txt).
static bool swab_mode_off(bool swiglu, bool qkv) {
  static const bool sw = [] {
    const char* e = getenv("GLLM_GEMM_SWAB_SWIGLU");
    return e != nullptr && atoi(e) != 0;
  }();
  static const bool qk = [] {
    const char* e = getenv("GLLM_GEMM_SWAB_QKV");
    return e != nullptr && atoi(e) != 0;
  }();
  return (swiglu && !sw) || (qkv && !qk);
}

// swiglu != 0: B is the 64-row-interleaved [gate|up] weight (N = 2*d_ff) and C receives
// act = silu(gate) * up as [M, N/2]; tiles must cover whole 128-row gate/up pairs (BN >= 128).
static int gemm_impl(const bf16* A, int lda, const bf16* B, int ldb, bf16* C, int ldc, int M, int N, int K,
                     const bf16* bias, const bf16* residual, int ldr, int a_rows_alloc, int force_bn,
                     int force_splits, int swiglu, void* workspace, size_t ws_bytes, cudaStream_t st,
                     const QkvRopeArgs* qkv, const RowNorm& nm) {
  if (M <= 0) return 0;
  if (K % BK != 0 || N % 64 != 0) return set_error(GLLM_ERR_INVALID, "gemm needs K %% 64 == 0 and N %% 64 == 0 (K=%d N=%d)", K, N);
  // decode-sized M: swap-AB stream-K weight streaming (gemm_skinny.cu)
  if (force_splits == 0 && force_bn == 0 && gemm_skinny_eligible(M, N, K) &&
      ws_bytes >= gemm_skinny_workspace_bytes(M, N, K) && !(swiglu && (bias || residual)))
    return gemm_skinny(A, lda, a_rows_alloc, B, ldb, C, ldc, M, N, K, swiglu ? EPI_SWIGLU : (qkv ? EPI_QKV_ROPE : EPI_STORE),
                       bias, residual, ldr, qkv, workspace, ws_bytes, st, nm);
  if (ldc % 8 || (residual && ldr % 8)) return set_error(GLLM_ERR_INVALID, "gemm output pitch must be a multiple of 8");
  if (swiglu && (N % 128 || bias || residual)) return set_error(GLLM_ERR_INVALID, "swiglu gemm needs N %% 128 == 0, no bias/residual");
  const int num_sms = device_sm_count();
  const int m_tiles = (M + BM - 1) / BM;
  const int min_bn = (swiglu || qkv) ? 128 : 64;
  // Tile width. Up to 4 row tiles (M <= 512) the GEMM streams its weights and every CTA must
  // also ingest its A rows once per N tile: keep BN = 256 (A re-read by the fewest N tiles) and
  // fill the machine with split-K below. Beyond that: widest BN that still yields one wave.
  // Beyond 4 row tiles the GEMM is compute-bound: pick (cta_group, BN) by modelled time = waves x
  // per-SM tile work / relative MMA efficiency, the efficiency set by the smem operand traffic
  // per MMA cycle (1-CTA BN=256: 96 B/clk; 2-CTA BN=256: 64 B/clk; 1-CTA BN=128: 128 B/clk).
  static const int cg_pref = [] {
    const char* e = getenv("GLLM_GEMM_CG");  // GLLM_GEMM_CG=1 forces 1-CTA tiles (A/B runs)
    return e ? atoi(e) : 2;
  }();
  int bn = force_bn, cg_pick = 0;
  bool whole_k = false;  // medium M, short K: one wave of 2-CTA BN=128 tiles, no split-K
  if (bn == 0) {
    bn = 256;
    // 2 or 4 row tiles (M in 129-256 / 385-512) with few output tiles: when every 256-row x
    // 128-column tile pair fits one wave and K is short, whole-K 2-CTA tiles beat split-K
    // (no partials, no reduce launch, fused QKV epilogue kept). Measured at M = 214: QKV
    // 7168x5120 39.9 -> 28.7 us, O 5120x5120 35.8 -> 26.7 us; at K = 27648 split-K stays ahead
    // (87 vs 92 us: 80 CTAs cannot stream the weights alone).
    if (m_tiles <= 4 && m_tiles % 2 == 0 && force_splits == 0 && cg_pref == 2 && N % 128 == 0 && K <= 8192 &&
        (long)(m_tiles / 2) * (N / 128) * 2 <= num_sms) {
      bn = 128;
      cg_pick = 2;
      whole_k = true;
    }
    // 2 or 4 row tiles beyond that: whole-K 2-CTA tiles of the width with the least
    // wave-quantised work (waves x BN, ties to the wider tile) beat split-K + reduce while the
    // pairs keep half the SMs busy (M = 256, 10240 x 8192: BN 256 55.4 us vs split-K 3 68.6 us;
    // M = 512: BN 128 80.0 vs 94.2 us; M = 512, 5120 x 13824: 83.9 vs 87.0 us), and for K > 16384
    // when they fill >= 80% of the SMs in one wave (M = 256, 8192 x 28672: BN 128 104.4 vs
    // 119.9 us; at 54% busy, 5120 x 27648, split-K stays ahead).
    if (!whole_k && m_tiles <= 4 && m_tiles % 2 == 0 && force_splits == 0 && cg_pref == 2) {
      const long slots2 = num_sms / 2;
      long best_w = 0;
      int best_bn = 0;
      for (int cand : {256, 128}) {
        if (N % cand || cand < min_bn) continue;
        const long units = (long)(m_tiles / 2) * (N / cand);
        const long w = (units + slots2 - 1) / slots2 * cand;
        if (best_bn == 0 || w < best_w) {
          best_w = w;
          best_bn = cand;
        }
      }
      const long ctas = best_bn ? (long)(m_tiles / 2) * (N / best_bn) * 2 : 0;
      const bool fits = K <= 16384 ? ctas * 2 >= num_sms : (ctas <= num_sms && ctas * 5 >= 4L * num_sms);
      if (best_bn && fits) {
        bn = best_bn;
        cg_pick = 2;
        whole_k = true;
      }
    }
    // 2 or 4 row tiles on whole-K 2-CTA tiles: swap-AB units instead when they put less work on
    // each SM -- their free token width fills more clusters (M = 512, 5120 x 5120: 60 units of
    // 256 weights x 192 tokens instead of 40 of 256 x 256)
    if (whole_k && cg_pick == 2 && m_tiles <= 4 && force_bn == 0 && !qkv && !swab_mode_off(swiglu, false)) {
      const long units = (long)(m_tiles / 2) * (N / bn), slots2 = num_sms / 2;
      const double cur = (double)((units + slots2 - 1) / slots2) * 128.0 * bn / (bn == 256 ? 0.85 : 0.75);
      double w_swab = 0;
      const int nt = gemm_swab_tile(M, N, K, &w_swab);
      if (nt && w_swab / 0.85 < 0.98 * cur)
        return gemm_swab(A, lda, a_rows_alloc, B, ldb, C, ldc, M, N, K, nt, swiglu ? 2 : (qkv ? 3 : 0), bias, residual, ldr,
                         qkv, st, nm);
    }
    // One row tile (33-128 tokens past the decode kernel), short K: whole-K tiles of the
    // narrowest width the epilogue allows when they fill >= 1/4 of one wave (in a PDL chain at
    // M = 100: QKV 7168x5120 27.4 -> 21.7 us, 6144x4096 24.2 -> 18.2 us; K = 14336 stays split).
    // SwiGLU (gate-up, 200+ tiles of 128) too: the persistent CTAs stream their second tiles
    // behind the first (M = 128, 27648x5120: 91.1 -> 75.8 us; M = 100, 28672x4096: 75.7 -> 65.5).
    if (m_tiles == 1 && force_splits == 0 && K <= 8192 && N % min_bn == 0 &&
        (N / min_bn <= num_sms || swiglu) && 4 * (N / min_bn) >= num_sms) {
      bn = min_bn;
      whole_k = true;
    }
    if (m_tiles > 4 && force_splits == 0) {
      struct Cand { int cg, bn; double eff; };
      const Cand cands[] = {{2, 256, 0.85}, {2, 128, 0.75}, {1, 256, 0.75}, {1, 128, 0.55}, {1, 64, 0.37}};
      double best = 1e30;  // waves x BN / efficiency: per-SM work in units of 128 rows
      for (const Cand& c : cands) {
        if (N % c.bn || c.bn < min_bn || (c.cg == 2 && cg_pref != 2)) continue;
        const long units = (long)((M + BM * c.cg - 1) / (BM * c.cg)) * (N / c.bn);
        const long slots = num_sms / c.cg;
        const double t = (double)((units + slots - 1) / slots) * c.bn / c.eff;
        if (t < best) {
          best = t;
          bn = c.bn;
          cg_pick = c.cg;
        }
      }
      // swap-AB units (256 weights x a free token width; gemm_swab.cu, every fused epilogue) when
      // they put less work on each SM: 128 x NT x waves against 128 x BN x waves
      if (cg_pref == 2 && !swab_mode_off(swiglu, qkv != nullptr)) {
        double w_swab = 0;
        const int nt = gemm_swab_tile(M, N, K, &w_swab);
        if (nt && w_swab / 0.85 < 0.98 * 128.0 * best)
          return gemm_swab(A, lda, a_rows_alloc, B, ldb, C, ldc, M, N, K, nt, swiglu ? 2 : (qkv ? 3 : 0), bias, residual, ldr,
                         qkv, st, nm);
      }
    }
    while (bn > min_bn && N % bn) bn >>= 1;
    if (N % bn) bn = (N % 128 == 0) ? 128 : 64;
  }
  if ((swiglu || qkv) && bn < 128) return set_error(GLLM_ERR_INVALID, "swiglu/qkv gemm needs BN >= 128");
  const int n_tiles = N / bn;
  const int total_kb = K / BK;
  int splits = force_splits;
  if (splits == 0) {
    splits = 1;
    const long tiles = whole_k ? num_sms : (long)n_tiles * m_tiles;
    // Split K only when one wave is not filled (HBM-bound weight streaming for small M). The
    // split count minimises waves(s) / s -- the time of a wave shrinks with 1/s -- plus the fp32
    // partials (written and re-read: 8 B per output per split, against the 2 B per weight the
    // GEMM streams anyway): 40 tiles -> 3 splits (1 wave of 1/3 tiles) rather than 4 (160
    // units = 2 waves of 1/4 tiles).
    if (tiles < num_sms) {
      double best = 1e30;
      const double partial_cost = 2.0 * M / K;  // partial bytes per split / weight bytes
      for (int s = 1; s <= 16 && total_kb / s >= 4; ++s) {
        if (s > 1 && (workspace == nullptr || ws_bytes < GEMM_WS_HEAD_BYTES + (size_t)s * M * N * sizeof(float))) break;
        const double c = (double)((tiles * s + num_sms - 1) / num_sms) / s + (s > 1 ? s * partial_cost : 0.0);
        if (c < best) {
          best = c;
          splits = s;
        }
      }
    }
  }
  splits = splits < 1 ? 1 : (splits > total_kb ? total_kb : splits);
  const int kbps = (total_kb + splits - 1) / splits;
  splits = (total_kb + kbps - 1) / kbps;
  float* partial = nullptr;
  if (splits > 1) {
    // split-K partials live after the skinny kernel's tile counters (which must stay zero)
    size_t need = GEMM_WS_HEAD_BYTES + (size_t)splits * M * N * sizeof(float);
    if (workspace == nullptr || ws_bytes < need)
      return set_error(GLLM_ERR_INVALID, "gemm split-K workspace too small (%zu < %zu)", ws_bytes, need);
    partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + GEMM_WS_HEAD_BYTES);
  }
  // 2-CTA (cta_group::2) tiles: the modelled pick above, else (forced tiles, <= 4 row tiles
  // without split-K) whenever the 128-row tiles pair up evenly.
  const int cg = splits > 1 ? 1
                 : cg_pick    ? cg_pick
                              : ((cg_pref == 2 && m_tiles >= 2 && bn >= 128 && m_tiles % 2 == 0) ? 2 : 1);
  CUtensorMap ma, mb;
  const int a_rows = a_rows_alloc > M ? a_rows_alloc : M;
  if (int rc = make_map(&ma, A, a_rows, K, lda, a_box_rows(M, cg))) return rc;
  if (int rc = make_map(&mb, B, N, K, ldb, bn / cg)) return rc;
  int rc = 0;
  if (qkv && splits > 1) {
    // small-M QKV: split-K plain GEMM, then the standalone RoPE + KV-write kernel
    int rc = gemm_impl(A, lda, B, ldb, C, ldc, M, N, K, bias, nullptr, 0, a_rows_alloc, force_bn, splits, 0,
                       workspace, ws_bytes, st, nullptr, nm);
    if (rc) return rc;
    return rope_kv_write(C, M, qkv->n_heads, qkv->n_kv, 128, qkv->tok_pos, qkv->tok_slot, qkv->rope, qkv->k_cache,
                         qkv->v_cache, qkv->page_size, st);
  }
  const int mode = splits > 1 ? EPI_PARTIAL_F32 : (swiglu ? EPI_SWIGLU : (qkv ? EPI_QKV_ROPE : EPI_STORE));
#define GLLM_GEMM_CASE(BNV, ST)                                                                              \
  if (bn == BNV) {                                                                                           \
    if (mode == EPI_STORE)                                                                                   \
      rc = launch_gemm<BNV, ST, EPI_STORE>(ma, mb, M, N, K, splits, kbps, C, ldc, bias, residual, ldr,       \
                                           nullptr, st, nm);                                                     \
    else if (mode == EPI_PARTIAL_F32)                                                                        \
      rc = launch_gemm<BNV, ST, EPI_PARTIAL_F32>(ma, mb, M, N, K, splits, kbps, C, ldc, nullptr, nullptr, 0, \
                                                 partial, st, nm);                                               \
    else if (mode == EPI_SWIGLU)                                                                             \
      rc = launch_gemm<BNV, ST, EPI_SWIGLU>(ma, mb, M, N, K, splits, kbps, C, ldc, nullptr, nullptr, 0,      \
                                            nullptr, st, nm);                                                    \
    else                                                                                                     \
      rc = launch_gemm<BNV, ST, EPI_QKV_ROPE>(ma, mb, M, N, K, splits, kbps, C, ldc, bias, nullptr, 0,       \
                                              nullptr, st, nm, *qkv);                                            \
  }
#define GLLM_GEMM_CASE2(BNV, ST)                                                                              \
  if (bn == BNV) {                                                                                            \
    if (mode == EPI_STORE)                                                                                    \
      rc = launch_gemm<BNV, ST, EPI_STORE, 2>(ma, mb, M, N, K, splits, kbps, C, ldc, bias, residual, ldr,     \
                                              nullptr, st, nm);                                                   \
    else if (mode == EPI_SWIGLU)                                                                              \
      rc = launch_gemm<BNV, ST, EPI_SWIGLU, 2>(ma, mb, M, N, K, splits, kbps, C, ldc, nullptr, nullptr, 0,    \
                                               nullptr, st, nm);                                                  \
    else                                                                                                      \
      rc = launch_gemm<BNV, ST, EPI_QKV_ROPE, 2>(ma, mb, M, N, K, splits, kbps, C, ldc, bias, nullptr, 0,     \
                                                 nullptr, st, nm, *qkv);                                          \
  }
  if (cg == 2) {
    GLLM_GEMM_CASE2(256, 6)
    else GLLM_GEMM_CASE2(128, 8) else return set_error(GLLM_ERR_INVALID, "bad BN %d for 2-CTA tiles", bn);
  } else
  GLLM_GEMM_CASE(256, 4)
  else GLLM_GEMM_CASE(128, 6) else if (bn == 64 && !swiglu && !qkv) {
    rc = mode == EPI_STORE ? launch_gemm<64, 8, EPI_STORE>(ma, mb, M, N, K, splits, kbps, C, ldc, bias, residual,
                                                           ldr, nullptr, st, nm)
                           : launch_gemm<64, 8, EPI_PARTIAL_F32>(ma, mb, M, N, K, splits, kbps, C, ldc, nullptr,
                                                                 nullptr, 0, partial, st, nm);
  } else return set_error(GLLM_ERR_INVALID, "bad BN %d (swiglu/qkv need >= 128)", bn);
#undef GLLM_GEMM_CASE
#undef GLLM_GEMM_CASE2
  if (rc) return rc;
  if (splits > 1) {
    const int threads = 256;
    if (swiglu) {
      const size_t groups = (size_t)M * (N / 2 / 8);
      splitk_reduce_swiglu<<<(unsigned)((groups + threads - 1) / threads), threads, 0, st>>>(partial, splits, M, N,
                                                                                             C, ldc, nm);
      rc = check_launch("splitk_reduce_swiglu");
    } else {
      const size_t groups = (size_t)M * (N / 8);
      splitk_reduce<<<(unsigned)((groups + threads - 1) / threads), threads, 0, st>>>(partial, splits, M, N, C, ldc,
                                                                                     bias, residual, ldr, nm);
      rc = check_launch("splitk_reduce");
    }
  }
  return rc;
}

int gemm_bf16(const bf16* A, int lda, const bf16* B, int ldb, bf16* C, int ldc, int M, int N, int K,
              const bf16* bias, const bf16* residual, int ldr, int a_rows_alloc, int force_bn, int force_splits,
              void* workspace, size_t ws_bytes, cudaStream_t st, const RowNorm& norm) {
  return gemm_impl(A, lda, B, ldb, C, ldc, M, N, K, bias, residual, ldr, a_rows_alloc, force_bn, force_splits, 0,
                   workspace, ws_bytes, st, nullptr, norm);
}

int gemm_swiglu_bf16(const bf16* A, int lda, const bf16* B, int ldb, bf16* C, int ldc, int M, int d_ff, int K,
                     int a_rows_alloc, int force_bn, int force_splits, void* workspace, size_t ws_bytes,
                     cudaStream_t st, const RowNorm& norm) {
  return gemm_impl(A, lda, B, ldb, C, ldc, M, 2 * d_ff, K, nullptr, nullptr, 0, a_rows_alloc, force_bn, force_splits,
                   1, workspace, ws_bytes, st, nullptr, norm);
}

int gemm_qkv_rope_bf16(const bf16* A, int lda, const bf16* W, int ldb, const bf16* bias, bf16* qkv, int M, int K,
                       int n_heads, int n_kv, const int* tok_pos, const int* tok_slot, const float* rope,
                       bf16* k_cache, bf16* v_cache, int page_size, int a_rows_alloc, int force_bn,
                       int force_splits, void* workspace, size_t ws_bytes, cudaStream_t st,
                       const RowNorm& norm) {
  const int N = (n_heads + 2 * n_kv) * 128;
  QkvRopeArgs qa{tok_pos, tok_slot, rope, k_cache, v_cache, n_heads, n_kv, page_size};
  return gemm_impl(A, lda, W, ldb, qkv, N, M, N, K, bias, nullptr, 0, a_rows_alloc, force_bn, force_splits, 0,
                   workspace, ws_bytes, st, &qa, norm);
}

size_t gemm_workspace_bytes(int M, int N, int K) {
  // Upper bound used by the stage allocator: at most 16 splits.
  (void)K;
  return (size_t)16 * M * N * sizeof(float);
}

}  // namespace gllm
