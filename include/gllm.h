/*
 * gllm.h — C-ABI of the B200 per-iteration path (libgllm.so, sm_100a).
 *
 * This boundary replaces the reference's two stage stand-ins and its count-only
 * KV bookkeeping with device work:
 *   stage_time(plan, cost)     pkg/src/tokensim/engine.py:96-100  -> gllm_stage_forward
 *   transfer_time(plan, comm)  pkg/src/tokensim/engine.py:103-105 -> activations in
 *                              gllm_batch.hidden, moved by NCCL send/recv (host runtime)
 *   KvCacheState counts        pkg/src/tokensim/kvcache.py:46-95  -> device block table,
 *                              updated by gllm_prepare_batch from the host page deltas
 *   commit "generated += 1"    pkg/src/tokensim/engine.py:338-358 -> gllm_argmax +
 *                              gllm_commit_tokens (sampled token becomes next input)
 *
 * Conventions: plain pointers and sizes only; every device pointer is caller-owned
 * (allocated by PyTorch); nothing here calls cudaMalloc or synchronises the host;
 * every call is stream-ordered on the stream passed in. Return value 0 = success,
 * otherwise a GLLM_ERR_* code with a message from gllm_last_error() (thread-local).
 * bf16 tensors are row-major; "ld" arguments are leading dimensions in elements.
 */
#ifndef GLLM_H_
#define GLLM_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GLLM_API __attribute__((visibility("default")))
#else
#define GLLM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gllm_stream_t; /* == cudaStream_t */

enum {
  GLLM_OK = 0,
  GLLM_ERR_INVALID = 1, /* bad argument / unsupported shape */
  GLLM_ERR_CUDA = 2     /* CUDA runtime or driver error */
};

/* Per-sequence metadata, int32 x GLLM_SEQ_FIELDS per sequence, in plan order
 * (decodes then prefill chunks, as MicroBatchPlan, sched.py:112-133):
 *   row      block-table / token-history row of the request
 *   start    tokens already cached (position of the first new token)
 *   n_new    tokens appended by this micro-batch (1 for a decode)
 *   tok_off  first token's index in the packed token dimension
 *   emit     index in the sampled-token output, or -1 (no token sampled) */
#define GLLM_SEQ_FIELDS 5

/* Metadata bounds-check bits (gllm_meta_errors): ids outside the stage's tables are never
 * written through -- deltas / prompt rows are skipped, tokens get slot -1 (no KV write). */
#define GLLM_META_BAD_DELTA 1u  /* block-table delta row / page index / page id out of range */
#define GLLM_META_BAD_PROMPT 2u /* prompt header row / length out of range */
#define GLLM_META_BAD_SEQ 4u    /* seq_info row out of range or start + n_new > max_seq_len */
#define GLLM_META_BAD_PAGE 8u   /* block-table entry of a token's position is not a valid page */

/* Model/stage dimensions (Llama / Qwen2 decoder, head_dim 128). */
typedef struct gllm_dims {
  int n_layers;     /* layers held by this stage */
  int d_model;
  int n_heads;
  int n_kv_heads;
  int head_dim;
  int d_ff;
  int vocab;
  int qkv_bias;     /* 1 for Qwen2 */
  float rms_eps;
  int page_size;
  int num_pages;    /* KV pages per layer */
  int max_rows;     /* block-table / token-history rows */
  int max_pages_per_row;
  int max_seq_len;  /* token-history row length */
  int max_tokens;   /* packed tokens per micro-batch (workspace sizing) */
  int max_emit;     /* sampled rows per micro-batch (workspace sizing) */
  int fused_norm;   /* 1: attn_norm / mlp_norm are folded into the columns of w_qkv / w_gate_up (the
                       norm vectors are ignored): no RMSNorm launches, the row scale is applied in the
                       QKV / gate-up GEMM epilogues and its statistics are accumulated by the O / down
                       GEMM epilogues. 0: separate RMSNorm kernels. */
} gllm_dims;

typedef struct gllm_layer {
  const void* attn_norm;  /* bf16 [d] */
  const void* w_qkv;      /* bf16 [(n_heads + 2 n_kv) * hd, d]: q | k | v rows */
  const void* b_qkv;      /* bf16 [(n_heads + 2 n_kv) * hd] or NULL */
  const void* w_o;        /* bf16 [d, n_heads * hd] */
  const void* mlp_norm;   /* bf16 [d] */
  const void* w_gate_up;  /* bf16 [2 d_ff, d]: 64-row blocks alternating gate / up (rows 128j..128j+63 =
                             gate rows 64j.., rows 128j+64.. = up rows 64j..), so a GEMM tile holds
                             matching gate/up outputs and SiLU*mul runs in its epilogue */
  const void* w_down;     /* bf16 [d, d_ff] */
} gllm_layer;

typedef struct gllm_stage {
  gllm_dims dims;
  int is_first;               /* embeds tokens, owns token history */
  int is_last;                /* final norm, LM head, argmax */
  const void* embed;          /* bf16 [vocab, d] (first stage) */
  const void* final_norm;     /* bf16 [d] (last stage) */
  const void* lm_head;        /* bf16 [vocab, d] (last stage) */
  const gllm_layer* layers;   /* HOST array [n_layers] */
  void* k_cache;              /* bf16 [n_layers][num_pages][n_kv][page_size][hd] */
  void* v_cache;              /* same shape */
  int32_t* block_table;       /* [max_rows][max_pages_per_row] */
  int32_t* token_hist;        /* [max_rows][max_seq_len] (first stage; NULL elsewhere) */
  const float* rope;          /* [max_seq_len][hd/2][2] (cos, sin) */
  void* workspace;            /* >= gllm_stage_workspace_bytes(&dims) */
  size_t workspace_bytes;
} gllm_stage;

/* One micro-batch. `meta` is ONE device int32 buffer holding, back to back:
 *   seq_info [n_seqs][5] | attention work [n_work][2] = (seq, q_start), the n_prefill_work
 *     prefill tiles (gllm_attention_q_tile tokens each) FIRST, then one item per decode
 *   | page deltas [n_deltas][3] = (row, page_index, page_id)
 *   | prompt headers [n_prompts][3] = (row, length, token offset) | prompt tokens */
typedef struct gllm_batch {
  int n_seqs;
  int n_tokens;
  int n_emit;
  int n_work;
  int n_prefill_work;   /* work items with more than one query token (0 => all-decode launch) */
  int n_deltas;
  int n_prompts;
  const int32_t* meta;  /* device */
  void* hidden;         /* bf16 [n_tokens, d]: residual stream in (non-first) / out (non-last) */
  int32_t* sampled;     /* int32 [n_emit] (last stage) */
  void* logits;         /* bf16 [n_emit, vocab] or NULL (workspace) */
  const int32_t* host_seq_info; /* optional HOST copy of seq_info (profiler byte/FLOP accounting) */
} gllm_batch;

/* Profiler record: one kernel class, aggregated over the launches captured between
 * gllm_profile_begin and gllm_profile_end (CUDA events on the launching stream). */
typedef struct gllm_profile_entry {
  char name[32];
  int launches;
  double total_ms;   /* sum of per-launch event durations */
  double flops;      /* algorithmic FLOPs (sum over launches) */
  double bytes;      /* algorithmic DRAM bytes (sum over launches) */
} gllm_profile_entry;

/* ---- library ---- */
GLLM_API int gllm_version(void);
GLLM_API const char* gllm_last_error(void);
GLLM_API int gllm_attention_q_tile(int n_heads, int n_kv_heads);
GLLM_API size_t gllm_stage_workspace_bytes(const gllm_dims* dims);

/* ---- stage: one micro-batch through this stage's layers (replaces stage_time) ---- */
GLLM_API int gllm_stage_forward(const gllm_stage* stage, const gllm_batch* batch, gllm_stream_t stream);
/* first stage: write sampled tokens back as the next inputs (after the last stage's argmax) */
GLLM_API int gllm_commit_tokens(const gllm_stage* stage, const gllm_batch* batch, const int32_t* sampled,
                       gllm_stream_t stream);

/* ---- individual kernels (tests, custom stages) ----
 * GEMM tiling is chosen per call: M <= 32 -> swap-AB stream-K "skinny" kernel (decode);
 * more than one 128-row tile and no split -> 2-CTA (cta_group::2) 256 x BN tiles; otherwise
 * 1-CTA 128 x BN tiles, split-K when one wave is not filled. force_bn / force_splits != 0 pin
 * the 1-/2-CTA tile path (force_splits = 1: whole tiles, >= 2: split-K). The workspace head
 * (16 KB) holds tile counters that must be zero between calls; these entry points zero them
 * themselves (gllm_stage_forward once per forward). workspace >= 16 KB + 42 MB covers every
 * shape a stage issues. */
/* Zero the workspace head once and let the following GEMM calls on this host thread that pass
 * the same workspace skip their own zeroing (every launch leaves the counters zero): for chains
 * of individual GEMMs. The caller must not write the workspace between those calls. */
GLLM_API int gllm_gemm_workspace_reset(void* workspace, gllm_stream_t stream);
GLLM_API int gllm_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N, int K,
                   const void* bias, const void* residual, int ldr, int force_bn, int force_splits,
                   void* workspace, size_t workspace_bytes, gllm_stream_t stream);
/* act[M, d_ff] = silu(A . W_gate^T) * (A . W_up^T), W in the interleaved w_gate_up layout above */
GLLM_API int gllm_gemm_swiglu_bf16(const void* A, int lda, const void* B_interleaved, int ldb, void* act, int ldc,
                                   int M, int d_ff, int K, int force_bn, int force_splits, void* workspace,
                                   size_t workspace_bytes, gllm_stream_t stream);
/* QKV projection with RoPE + paged KV write fused into the GEMM epilogue: q heads of
 * A . W^T (+bias) are rotated and written to qkv[M][(H+2KV)*128] (k/v columns untouched);
 * k heads are rotated and k/v written to the paged cache slot tok_slot[row] of each token */
GLLM_API int gllm_gemm_qkv_rope_bf16(const void* A, int lda, const void* W, int ldb, const void* bias, void* qkv,
                                     int M, int K, int n_heads, int n_kv_heads, const int32_t* tok_pos,
                                     const int32_t* tok_slot, const float* rope, void* k_cache, void* v_cache,
                                     int page_size, int force_bn, int force_splits, void* workspace,
                                     size_t workspace_bytes, gllm_stream_t stream);
GLLM_API int gllm_rmsnorm(const void* x, int ldx, const int32_t* row_index, const void* weight, void* out, int rows, int d,
                 float eps, gllm_stream_t stream);
GLLM_API int gllm_silu_mul(const void* gate_up, int d_ff, void* out, int rows, gllm_stream_t stream);
/* OR of GLLM_META_* bits raised by any micro-batch since the last reset (a host-mapped word the
 * kernels write only on a violation: reading it needs no sync). `reset` != 0 clears it.
 * The host runtime checks it after every retired micro-batch. */
GLLM_API uint32_t gllm_meta_errors(int reset);

GLLM_API int gllm_prepare_batch(const gllm_stage* stage, const gllm_batch* batch, int32_t* tok_pos, int32_t* tok_slot,
                       int32_t* tok_id, int32_t* emit_rows, gllm_stream_t stream);
GLLM_API int gllm_embed(const int32_t* tok_id, int n_tokens, const void* embed, int d, void* out, gllm_stream_t stream);
GLLM_API int gllm_rope_kv_write(void* qkv, int n_tokens, int n_heads, int n_kv_heads, int head_dim, const int32_t* tok_pos,
                       const int32_t* tok_slot, const float* rope, void* k_cache, void* v_cache, int page_size,
                       gllm_stream_t stream);
GLLM_API int gllm_attn_mixed_paged(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                          int n_prefill_work, const int32_t* block_table, int max_pages_per_row, int kv_pages,
                          const void* k_cache,
                          const void* v_cache, int n_heads, int n_kv_heads, int head_dim, int page_size, void* out,
                          gllm_stream_t stream);
/* same, with each prefill item's key range cut into n_split parts (more CTAs when a micro-batch has
 * few long chunks), merged by a combine pass; workspace >= gllm_attn_split_workspace_bytes(...).
 * gllm_stage_forward picks n_split itself from the host metadata. */
GLLM_API int gllm_attn_mixed_paged_split(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                                         int n_prefill_work, const int32_t* block_table, int max_pages_per_row,
                                         int kv_pages, const void* k_cache, const void* v_cache, int n_heads,
                                         int n_kv_heads, int head_dim, int page_size, void* out, int n_split,
                                         void* workspace, size_t workspace_bytes, gllm_stream_t stream);
GLLM_API size_t gllm_attn_split_workspace_bytes(int n_prefill_work, int n_split, int n_kv_heads);
/* same, with the splits chosen as gllm_stage_forward chooses them from host copies of seq_info
 * and work: a decode-only launch of few sequences splits each sequence's pages over a cluster of
 * up to 4 CTAs merged through distributed shared memory (no workspace); prefill KV splits follow
 * GLLM_ATTN_SPLIT and use the workspace (may be NULL / 0 to disable them). */
GLLM_API int gllm_attn_mixed_paged_auto(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                                        int n_prefill_work, const int32_t* block_table, int max_pages_per_row,
                                        int kv_pages, const void* k_cache, const void* v_cache, int n_heads,
                                        int n_kv_heads, int head_dim, int page_size, void* out,
                                        const int32_t* host_seq_info, const int32_t* host_work, void* workspace,
                                        size_t workspace_bytes, gllm_stream_t stream);
GLLM_API int gllm_argmax(const void* logits, int rows, int vocab, int32_t* out, gllm_stream_t stream);

/* ---- measurement ---- */
GLLM_API unsigned long long gllm_launch_count(void); /* kernels launched by this library so far */
GLLM_API int gllm_profile_begin(void);
/* synchronises the recorded events; fills up to max_entries, sets *n_entries */
GLLM_API int gllm_profile_end(gllm_profile_entry* out, int max_entries, int* n_entries);

#ifdef __cplusplus
}
#endif
#endif /* GLLM_H_ */
