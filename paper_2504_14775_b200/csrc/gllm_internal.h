// Internal declarations shared by the CUDA translation units (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/gllm.h"

namespace gllm {

typedef __nv_bfloat16 bf16;

int set_error(int code, const char* fmt, ...);

// Programmatic dependent launch on (default on; GLLM_PDL=0 turns it off for A/B runs).
bool pdl_enabled();

// cudaLaunchKernelEx with programmatic stream serialization (when enabled) and an optional
// cluster: the kernel must call pdl_wait() before touching its predecessor's memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster_x,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
int set_cuda_error(cudaError_t e, const char* what);
int check_launch(const char* what);
int device_sm_count();

// Extra epilogue operands of the fused QKV GEMM (RoPE on q/k + paged KV-cache write).
struct QkvRopeArgs {
  const int* tok_pos;    // [M] absolute position of each token row
  const int* tok_slot;   // [M] paged slot: page * page_size + offset
  const float* rope;     // [max_pos][64][2] (cos, sin)
  bf16* k_cache;         // this layer's [pages][n_kv][page_size][128]
  bf16* v_cache;
  int n_heads, n_kv, page_size;
};

// Fused RMSNorm (gllm_dims.fused_norm): the norm weight is folded into the consumer GEMM's weight
// columns, the GEMM reads the raw residual stream x, and its epilogue scales output row m by
// rsqrt(sum_g ss_in[g][m] / d + eps). The producers of x (the O / down GEMMs with the residual
// add) write ss_out[g][m] = sum of the squares of their bf16 outputs in column group g (64
// columns): plain stores of fixed-order sums, so the statistics are deterministic (no atomics).
constexpr int NORM_GROUP = 64;
struct RowNorm {
  const float* ss_in = nullptr;  // [d / 64][ld]
  float* ss_out = nullptr;       // [d / 64][ld]
  int ld = 0;
  int d = 0;
  float eps = 0.f;
};
#ifdef __CUDACC__
__device__ __forceinline__ float row_norm_scale(const RowNorm& nm, int row) {
  // d / 64 partials (64-128 for the served models): loads issued 16 at a time, summed in g order
  // (the same value as a plain sequential loop, in ~5 memory round trips instead of one per group)
  const int G = nm.d / NORM_GROUP;
  const float* p = nm.ss_in + row;
  float s = 0.f;
  int g = 0;
  for (; g + 16 <= G; g += 16) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = p[(size_t)(g + j) * nm.ld];
#pragma unroll
    for (int j = 0; j < 16; ++j) s += v[j];
  }
  for (; g < G; ++g) s += p[(size_t)g * nm.ld];
  return rsqrtf(s / nm.d + nm.eps);
}
#endif

// gemm.cu
int gemm_bf16(const bf16* A, int lda, const bf16* B, int ldb, bf16* C, int ldc, int M, int N, int K, const bf16* bias,
              const bf16* residual, int ldr, int a_rows_alloc, int force_bn, int force_splits, void* workspace,
              size_t ws_bytes, cudaStream_t st, const RowNorm& norm = RowNorm{});
// act[M, d_ff] = silu(A W_g^T) * (A W_u^T) with W = the 64-row-interleaved [gate|up] weight [2 d_ff, K]
int gemm_swiglu_bf16(const bf16* A, int lda, const bf16* B, int ldb, bf16* C, int ldc, int M, int d_ff, int K,
                     int a_rows_alloc, int force_bn, int force_splits, void* workspace, size_t ws_bytes,
                     cudaStream_t st, const RowNorm& norm = RowNorm{});
// qkv = A W^T (+bias) with RoPE on q/k and the k/v heads scattered to the paged cache, fused in
// the GEMM epilogue (q heads land in qkv rows; k/v columns of qkv are left unwritten)
int gemm_qkv_rope_bf16(const bf16* A, int lda, const bf16* W, int ldb, const bf16* bias, bf16* qkv, int M, int K,
                       int n_heads, int n_kv, const int* tok_pos, const int* tok_slot, const float* rope,
                       bf16* k_cache, bf16* v_cache, int page_size, int a_rows_alloc, int force_bn,
                       int force_splits, void* workspace, size_t ws_bytes, cudaStream_t st,
                       const RowNorm& norm = RowNorm{});
size_t gemm_workspace_bytes(int M, int N, int K);

// gemm_skinny.cu: M <= 32 (decode) GEMMs; mode 0 store (+bias/+residual), 2 SwiGLU, 3 QKV+RoPE+KV write.
// The workspace head holds tile counters that must be zero at launch: the stage zeroes them once
// per forward (gemm_ws_reset) and every launch leaves them zero; other callers get a memset per call.
constexpr size_t GEMM_WS_HEAD_BYTES = 16384;  // skinny tile counters at the head of every GEMM workspace
// gemm_swab.cu: swap-AB 2-CTA units of 256 weight rows x NT tokens for the store / residual
// epilogue; gemm_swab_tile returns the token width NT (0 = not applicable) and its per-SM work.
int gemm_swab_tile(int M, int N, int K, double* work_per_sm);
// mode: 0 store (+bias/+residual, statistics out), 2 SwiGLU (interleaved gate/up), 3 QKV + RoPE + KV write
int gemm_swab(const bf16* A, int lda, int a_rows_alloc, const bf16* W, int ldw, bf16* C, int ldc, int M, int N,
              int K, int nt, int mode, const bf16* bias, const bf16* residual, int ldr, const QkvRopeArgs* qa,
              cudaStream_t st, const RowNorm& nm);
bool gemm_skinny_eligible(int M, int N, int K);
size_t gemm_skinny_workspace_bytes(int M, int N, int K);
int gemm_skinny(const bf16* A, int lda, int a_rows_alloc, const bf16* W, int ldw, bf16* C, int ldc, int M, int N,
                int K, int mode, const bf16* bias, const bf16* residual, int ldr, const QkvRopeArgs* qkv,
                void* workspace, size_t ws_bytes, cudaStream_t st, const RowNorm& norm = RowNorm{});
int gemm_ws_reset(void* workspace, cudaStream_t st);
void gemm_ws_mark_clean(const void* workspace);
// bf16 [rows, cols] (leading dim ld) as a TMA map with 64-col x box_rows boxes, 128B swizzle (cached)
int make_tma_map_2d(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

// kernels.cu
int rmsnorm(const bf16* x, int ldx, const int* row_index, const bf16* w, bf16* out, int rows, int d, float eps,
            cudaStream_t st);
// fused-norm statistics of a stage's input rows: ss[g][r] = sum of x[r][64g, 64g+64)^2 (bf16 values)
int row_sumsq(const bf16* x, int ldx, int rows, int d, float* ss, int ld, cudaStream_t st);
int silu_mul(const bf16* gu, int d_ff, bf16* out, int rows, cudaStream_t st);
int rope_kv_write(bf16* qkv, int n_tokens, int n_heads, int n_kv, int head_dim, const int* tok_pos,
                  const int* tok_slot, const float* rope, bf16* k_cache, bf16* v_cache, int page_size,
                  cudaStream_t st);
// bounds-checked (see kernels.cu): invalid ids are skipped / get slot -1 and set GLLM_META_* bits
int apply_batch_metadata(const int* meta, int n_deltas, int n_prompt_rows, int* block_table, int max_pages_per_row,
                         int* token_hist, int max_seq_len, int max_rows, int num_pages, cudaStream_t st);
int expand_tokens(const int* seq_info, int n_seqs, const int* block_table, int max_pages_per_row,
                  const int* token_hist, int max_seq_len, int page_size, int* tok_pos, int* tok_slot, int* tok_id,
                  int* emit_rows, const bf16* embed, int d, bf16* x_out, int max_rows, int num_pages,
                  cudaStream_t st);
unsigned meta_errors(int reset);
int embed_tokens(const int* tok_id, int n_tokens, const bf16* embed, int d, bf16* out, cudaStream_t st);
int argmax_rows(const bf16* logits, int rows, int vocab, int* out, cudaStream_t st);
int commit_tokens(const int* seq_info, int n_seqs, const int* sampled, int* token_hist, int max_seq_len,
                  cudaStream_t st);

// attention.cu
int attention_q_tile(int n_heads, int n_kv);
// n_split: 0 = auto (needs host_seq_info / host_work and part_ws), 1 = no KV split, >1 = forced
int attention_paged(const bf16* qkv, const int* seq_info, const int* work, int n_work, int n_prefill_work,
                    const int* block_table, int mpr, int kv_pages, const bf16* k_cache, const bf16* v_cache, int n_heads, int n_kv, int head_dim,
                    int page_size, bf16* out, cudaStream_t st, int n_split = 1, const int* host_seq_info = nullptr,
                    const int* host_work = nullptr, void* part_ws = nullptr, size_t part_bytes = 0);
size_t attention_split_bytes(int n_items, int n_split, int n_kv);

}  // namespace gllm
