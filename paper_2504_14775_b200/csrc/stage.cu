// C-ABI exports (include/gllm.h) and the stage orchestrator.
//
// gllm_stage_forward runs one micro-batch through this stage's layers with
// one host call (no per-kernel Python round trips): metadata apply + device
// slot mapping, embedding (first stage), then per layer
//   RMSNorm -> QKV GEMM(+bias, RoPE + paged KV write fused in its epilogue) -> mixed paged attention
//   -> O GEMM(+residual) -> RMSNorm -> gate-up GEMM with fused SiLU*mul -> down GEMM(+residual)
// and on the last stage final RMSNorm of the emitting rows -> LM head GEMM -> argmax.
// This is the real work behind the reference's `stage_time()` stand-in
// (`pkg/src/tokensim/engine.py:96-100`).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "gllm_internal.h"

namespace gllm {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
int set_cuda_error(cudaError_t e, const char* what) {
  return set_error(GLLM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
static std::atomic<unsigned long long> g_launches{0};

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, what);
}

// ------------------------------------------------------------------ profiler
// Kernel classes of the stage forward; each capture = (class, start/end event, algorithmic FLOPs, bytes).
enum ProfCat {
  P_META, P_EMBED, P_RMSNORM, P_GEMM_QKV, P_ROPE_KV, P_ATTN, P_GEMM_O, P_GEMM_GU, P_SILU, P_GEMM_DOWN,
  P_GEMM_LM, P_ARGMAX, P_COMMIT, P_NCAT
};
static const char* kProfNames[P_NCAT] = {"metadata", "embed", "rmsnorm", "gemm_qkv", "rope_kv_write",
                                          "attention", "gemm_o", "gemm_gate_up", "silu_mul", "gemm_down",
                                          "gemm_lm_head", "argmax", "commit_tokens"};
struct ProfRec {
  int cat;
  cudaEvent_t a, b;
  double flops, bytes;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_pool;
static size_t g_pool_next = 0;

static cudaEvent_t pool_event() {
  if (g_pool_next == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  return g_pool[g_pool_next++];
}

template <typename F>
static int prof_call(int cat, double flops, double bytes, cudaStream_t st, F&& fn) {
  if (!g_prof_on) return fn();
  cudaEvent_t a = pool_event(), b = pool_event();
  cudaEventRecord(a, st);
  int rc = fn();
  cudaEventRecord(b, st);
  g_prof.push_back({cat, a, b, flops, bytes});
  return rc;
}

// ---------------------------------------------------------------- debug: GLLM_CHECK_FINITE=1
__global__ void count_nonfinite_kernel(const bf16* __restrict__ x, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = __bfloat162float(x[i]);
    if (!isfinite(v)) ++c;
  }
  if (c) atomicAdd(out, c);
}
static bool check_finite_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("GLLM_CHECK_FINITE");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}
static int check_finite(const bf16* x, size_t n, const char* what, int layer, cudaStream_t st) {
  static unsigned long long* d = nullptr;
  if (!d) cudaMalloc(&d, sizeof(*d));
  cudaMemsetAsync(d, 0, sizeof(*d), st);
  count_nonfinite_kernel<<<256, 256, 0, st>>>(x, n, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (h) {
    fprintf(stderr, "[gllm] non-finite output: %s layer %d: %llu of %zu\n", what, layer, h, n);
    return set_error(GLLM_ERR_CUDA, "non-finite output of %s (layer %d)", what, layer);
  }
  return 0;
}
#define GLLM_CHECK(ptr, n, what, layer) \
  if (check_finite_enabled()) { if (int rc_ = check_finite((ptr), (n), (what), (layer), st)) return rc_; }

static double gemm_bytes(double M, double N, double K, bool residual, bool bias) {
  return 2.0 * (M * K + N * K + M * N) + (residual ? 2.0 * M * N : 0.0) + (bias ? 2.0 * N : 0.0);
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GLLM_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
}
int device_sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

struct StageWs {
  bf16 *x, *h, *qkv, *attn, *gu, *act, *hf, *logits;
  int *tok_pos, *tok_slot, *tok_id, *emit_rows;
  float* gemm;
  size_t gemm_bytes;
  void* attn_part;  // prefill KV-split partials
  size_t attn_part_bytes;
  float *ss_a, *ss_m;  // fused-norm row statistics (attention / MLP norm inputs)
  size_t total;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static StageWs carve(const gllm_dims& d, uint8_t* base) {
  StageWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  const size_t T = (size_t)d.max_tokens, E = (size_t)(d.max_emit > 0 ? d.max_emit : 1);
  const size_t qkv_w = (size_t)(d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
  w.x = (bf16*)take(T * d.d_model * 2);
  w.h = (bf16*)take(T * d.d_model * 2);
  w.qkv = (bf16*)take(T * qkv_w * 2);
  w.attn = (bf16*)take(T * (size_t)d.n_heads * d.head_dim * 2);
  w.gu = (bf16*)take(T * 2 * (size_t)d.d_ff * 2);
  w.act = (bf16*)take(T * (size_t)d.d_ff * 2);
  w.hf = (bf16*)take(E * d.d_model * 2);
  w.logits = (bf16*)take(E * (size_t)d.vocab * 2);
  w.tok_pos = (int*)take(T * 4);
  w.tok_slot = (int*)take(T * 4);
  w.tok_id = (int*)take(T * 4);
  w.emit_rows = (int*)take(E * 4);
  // split-K partials: splits * tiles <= 2 * SMs, tile <= 128 x 256 fp32
  w.gemm_bytes = 16384 + (size_t)3 * 160 * 128 * 256 * 4;
  w.gemm = (float*)take(w.gemm_bytes);
  // KV-split partials: splitting only happens below two waves of prefill CTAs (< 2 x 148 items x kv
  // heads) and keeps items x kv heads x splits <= 2 x 148 + items x kv heads
  w.attn_part_bytes = attention_split_bytes(4 * 160, 1, 1);
  w.attn_part = take(w.attn_part_bytes);
  w.ss_a = (float*)take(T * (d.d_model / NORM_GROUP) * 4);
  w.ss_m = (float*)take(T * (d.d_model / NORM_GROUP) * 4);
  w.total = off;
  return w;
}

struct MetaView {
  const int *seq_info, *work, *deltas, *prompts;
};
static MetaView meta_view(const gllm_batch& b) {
  MetaView v;
  v.seq_info = b.meta;
  v.work = v.seq_info + GLLM_SEQ_FIELDS * b.n_seqs;
  v.deltas = v.work + 2 * b.n_work;
  v.prompts = v.deltas + 3 * b.n_deltas;
  return v;
}

static int prepare(const gllm_stage& S, const gllm_batch& B, int* tok_pos, int* tok_slot, int* tok_id,
                   int* emit_rows, cudaStream_t st) {
  const gllm_dims& d = S.dims;
  MetaView mv = meta_view(B);
  if (int rc = apply_batch_metadata(mv.deltas, B.n_deltas, S.token_hist ? B.n_prompts : 0, S.block_table,
                                    d.max_pages_per_row, S.token_hist, d.max_seq_len, d.max_rows, d.num_pages, st))
    return rc;
  return expand_tokens(mv.seq_info, B.n_seqs, S.block_table, d.max_pages_per_row, S.is_first ? S.token_hist : nullptr,
                       d.max_seq_len, d.page_size, tok_pos, tok_slot, S.is_first ? tok_id : nullptr,
                       S.is_last ? emit_rows : nullptr, nullptr, d.d_model, nullptr, d.max_rows, d.num_pages, st);
}

static int validate(const gllm_stage* S, const gllm_batch* B) {
  if (!S || !B) return set_error(GLLM_ERR_INVALID, "null stage or batch");
  const gllm_dims& d = S->dims;
  if (B->n_tokens > d.max_tokens) return set_error(GLLM_ERR_INVALID, "n_tokens %d > max_tokens %d", B->n_tokens, d.max_tokens);
  if (B->n_emit > d.max_emit) return set_error(GLLM_ERR_INVALID, "n_emit %d > max_emit %d", B->n_emit, d.max_emit);
  if (d.head_dim != 128) return set_error(GLLM_ERR_INVALID, "head_dim must be 128");
  if (S->workspace_bytes < carve(d, nullptr).total)
    return set_error(GLLM_ERR_INVALID, "stage workspace too small (%zu < %zu)", S->workspace_bytes, carve(d, nullptr).total);
  if (S->is_first && (!S->embed || !S->token_hist)) return set_error(GLLM_ERR_INVALID, "first stage needs embed + token_hist");
  if (S->is_last && (!S->final_norm || !S->lm_head)) return set_error(GLLM_ERR_INVALID, "last stage needs final_norm + lm_head");
  if (!S->is_first && !B->hidden) return set_error(GLLM_ERR_INVALID, "non-first stage needs batch.hidden input");
  return 0;
}

static int forward(const gllm_stage& S, const gllm_batch& B, cudaStream_t st) {
  const gllm_dims& d = S.dims;
  StageWs w = carve(d, reinterpret_cast<uint8_t*>(S.workspace));
  const int T = B.n_tokens;
  const int D = d.d_model, H = d.n_heads, KV = d.n_kv_heads, HDIM = d.head_dim;
  const int qkv_w = (H + 2 * KV) * HDIM;
  MetaView mv = meta_view(B);
  bf16* x = B.hidden ? reinterpret_cast<bf16*>(B.hidden) : w.x;
  const int maxT = d.max_tokens;
  // skinny-GEMM tile counters zeroed once per forward; every GEMM leaves them zero again
  struct CleanGuard {
    ~CleanGuard() { gemm_ws_mark_clean(nullptr); }
  } clean_guard;
  if (int rc = gemm_ws_reset(w.gemm, st)) return rc;

  // Algorithmic attention work of this batch (profiler only; needs the host seq_info copy).
  double att_flops = 0, att_bytes = 0;
  if (g_prof_on && B.host_seq_info) {
    for (int i = 0; i < B.n_seqs; ++i) {
      const int32_t* si = B.host_seq_info + GLLM_SEQ_FIELDS * i;
      const double start = si[1], n = si[2];
      att_bytes += (start + n) * KV * HDIM * 2.0 * 2.0 + n * H * HDIM * 2.0 * 2.0;
      att_flops += 4.0 * H * HDIM * (n * start + n * (n + 1) / 2.0);
    }
  }
  const double Td = T, Dd = D, Fd = d.d_ff, Qd = qkv_w, Od = (double)H * HDIM;
  if (int rc = prof_call(P_META, 0, 0, st, [&] { return prepare(S, B, w.tok_pos, w.tok_slot, w.tok_id, w.emit_rows, st); }))
    return rc;
  GLLM_CHECK(x, (size_t)T * D * (S.is_first ? 0 : 1), "stage_input", -1);
  if (S.is_first)
    if (int rc = prof_call(P_EMBED, 0, 4.0 * Td * Dd, st,
                           [&] { return embed_tokens(w.tok_id, T, reinterpret_cast<const bf16*>(S.embed), D, x, st); }))
      return rc;

  const size_t layer_kv = (size_t)d.num_pages * KV * d.page_size * HDIM;
  // Fused RMSNorm (d.fused_norm): the norm weights live in w_qkv / w_gate_up, the QKV and gate-up
  // GEMMs read x itself and scale their output rows by rsqrt(mean(x^2) + eps); the O / down GEMMs
  // write the next norm's per-64-column sums of squares (ss_m, ss_a) while writing x. The stage
  // input's statistics come from one row_sumsq pass.
  const bool fused = d.fused_norm != 0;
  if (fused && D % 256) return set_error(GLLM_ERR_INVALID, "fused_norm needs d_model %% 256 == 0");
  if (fused)
    if (int rc = prof_call(P_RMSNORM, 0, 2.0 * Td * Dd, st, [&] { return row_sumsq(x, D, T, D, w.ss_a, maxT, st); }))
      return rc;
  RowNorm nm_qkv, nm_o, nm_gu, nm_down;
  if (fused) {
    nm_qkv.ss_in = w.ss_a;
    nm_o.ss_out = w.ss_m;
    nm_gu.ss_in = w.ss_m;
    nm_down.ss_out = w.ss_a;
    for (RowNorm* n : {&nm_qkv, &nm_o, &nm_gu, &nm_down}) {
      n->ld = maxT;
      n->d = D;
      n->eps = d.rms_eps;
    }
  }
  const bf16* h_in = fused ? x : w.h;  // A operand of the QKV / gate-up GEMMs
  for (int l = 0; l < d.n_layers; ++l) {
    const gllm_layer& L = S.layers[l];
    bf16* kc = reinterpret_cast<bf16*>(S.k_cache) + (size_t)l * layer_kv;
    bf16* vc = reinterpret_cast<bf16*>(S.v_cache) + (size_t)l * layer_kv;
    int rc;
    if (!fused)
      if ((rc = prof_call(P_RMSNORM, 0, 4.0 * Td * Dd, st,
                          [&] { return rmsnorm(x, D, nullptr, (const bf16*)L.attn_norm, w.h, T, D, d.rms_eps, st); })))
        return rc;
    // QKV GEMM (+bias) with RoPE and the paged K/V write fused into its epilogue
    if ((rc = prof_call(P_GEMM_QKV, 2.0 * Td * Qd * Dd,
                        gemm_bytes(Td, Qd, Dd, false, L.b_qkv != nullptr) + Td * 2.0 * KV * HDIM * 2.0, st, [&] {
           return gemm_qkv_rope_bf16(h_in, D, (const bf16*)L.w_qkv, D, (const bf16*)L.b_qkv, w.qkv, T, D, H, KV,
                                     w.tok_pos, w.tok_slot, S.rope, kc, vc, d.page_size, maxT, 0, 0, w.gemm,
                                     w.gemm_bytes, st, nm_qkv);
         })))
      return rc;
    if ((rc = prof_call(P_ATTN, att_flops, att_bytes, st, [&] {
           return attention_paged(w.qkv, mv.seq_info, mv.work, B.n_work, B.n_prefill_work, S.block_table,
                                  d.max_pages_per_row, d.num_pages, kc, vc, H, KV, HDIM, d.page_size, w.attn, st,
                                  /*n_split=*/0, B.host_seq_info,
                                  B.host_seq_info ? B.host_seq_info + GLLM_SEQ_FIELDS * B.n_seqs : nullptr,
                                  w.attn_part, w.attn_part_bytes);
         })))
      return rc;
    GLLM_CHECK(w.attn, (size_t)T * H * HDIM, "attention", l);
    if ((rc = prof_call(P_GEMM_O, 2.0 * Td * Dd * Od, gemm_bytes(Td, Dd, Od, true, false), st, [&] {
           return gemm_bf16(w.attn, H * HDIM, (const bf16*)L.w_o, H * HDIM, x, D, T, D, H * HDIM, nullptr, x, D, maxT,
                            0, 0, w.gemm, w.gemm_bytes, st, nm_o);
         })))
      return rc;
    GLLM_CHECK(x, (size_t)T * D, "gemm_o", l);
    if (!fused)
      if ((rc = prof_call(P_RMSNORM, 0, 4.0 * Td * Dd, st,
                          [&] { return rmsnorm(x, D, nullptr, (const bf16*)L.mlp_norm, w.h, T, D, d.rms_eps, st); })))
        return rc;
    // gate-up GEMM with SiLU*mul fused into its epilogue: writes act [T, d_ff] directly
    if ((rc = prof_call(P_GEMM_GU, 2.0 * Td * 2 * Fd * Dd,
                        2.0 * (Td * Dd + 2 * Fd * Dd + Td * Fd), st, [&] {
           return gemm_swiglu_bf16(h_in, D, (const bf16*)L.w_gate_up, D, w.act, d.d_ff, T, d.d_ff, D, maxT, 0, 0,
                                   w.gemm, w.gemm_bytes, st, nm_gu);
         })))
      return rc;
    GLLM_CHECK(w.act, (size_t)T * d.d_ff, "gemm_gate_up_swiglu", l);
    if ((rc = prof_call(P_GEMM_DOWN, 2.0 * Td * Dd * Fd, gemm_bytes(Td, Dd, Fd, true, false), st, [&] {
           return gemm_bf16(w.act, d.d_ff, (const bf16*)L.w_down, d.d_ff, x, D, T, D, d.d_ff, nullptr, x, D, maxT, 0,
                            0, w.gemm, w.gemm_bytes, st, nm_down);
         })))
      return rc;
    GLLM_CHECK(x, (size_t)T * D, "gemm_down", l);
  }
  if (S.is_last && B.n_emit > 0) {
    bf16* logits = B.logits ? reinterpret_cast<bf16*>(B.logits) : w.logits;
    const double E = B.n_emit, V = d.vocab;
    int rc;
    if ((rc = prof_call(P_RMSNORM, 0, 4.0 * E * Dd, st, [&] {
           return rmsnorm(x, D, w.emit_rows, (const bf16*)S.final_norm, w.hf, B.n_emit, D, d.rms_eps, st);
         })))
      return rc;
    if ((rc = prof_call(P_GEMM_LM, 2.0 * E * V * Dd, gemm_bytes(E, V, Dd, false, false), st, [&] {
           return gemm_bf16(w.hf, D, (const bf16*)S.lm_head, D, logits, d.vocab, B.n_emit, d.vocab, D, nullptr,
                            nullptr, 0, d.max_emit, 0, 0, w.gemm, w.gemm_bytes, st);
         })))
      return rc;
    if ((rc = prof_call(P_ARGMAX, 0, 2.0 * E * V, st, [&] { return argmax_rows(logits, B.n_emit, d.vocab, B.sampled, st); })))
      return rc;
    if (S.is_first)
      if ((rc = prof_call(P_COMMIT, 0, 0, st, [&] {
             return commit_tokens(mv.seq_info, B.n_seqs, B.sampled, S.token_hist, d.max_seq_len, st);
           })))
        return rc;
  }
  return 0;
}

}  // namespace gllm

using namespace gllm;

extern "C" {

int gllm_version(void) { return 1; }
const char* gllm_last_error(void) { return g_err; }
int gllm_attention_q_tile(int n_heads, int n_kv_heads) {
  if (n_kv_heads <= 0 || n_heads % n_kv_heads) return -1;
  return attention_q_tile(n_heads, n_kv_heads);
}
size_t gllm_stage_workspace_bytes(const gllm_dims* dims) { return dims ? carve(*dims, nullptr).total : 0; }

int gllm_stage_forward(const gllm_stage* stage, const gllm_batch* batch, gllm_stream_t stream) {
  if (int rc = validate(stage, batch)) return rc;
  return forward(*stage, *batch, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_commit_tokens(const gllm_stage* stage, const gllm_batch* batch, const int32_t* sampled,
                       gllm_stream_t stream) {
  if (!stage || !batch || !stage->token_hist) return set_error(GLLM_ERR_INVALID, "commit needs the first stage");
  return commit_tokens(batch->meta, batch->n_seqs, sampled, stage->token_hist, stage->dims.max_seq_len,
                       reinterpret_cast<cudaStream_t>(stream));
}

int gllm_gemm_workspace_reset(void* workspace, gllm_stream_t stream) {
  if (workspace == nullptr) return set_error(GLLM_ERR_INVALID, "null GEMM workspace");
  return gemm_ws_reset(workspace, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N, int K,
                   const void* bias, const void* residual, int ldr, int force_bn, int force_splits, void* workspace,
                   size_t workspace_bytes, gllm_stream_t stream) {
  return gemm_bf16((const bf16*)A, lda, (const bf16*)B, ldb, (bf16*)C, ldc, M, N, K, (const bf16*)bias,
                   (const bf16*)residual, ldr, M, force_bn, force_splits, workspace, workspace_bytes,
                   reinterpret_cast<cudaStream_t>(stream));
}

int gllm_gemm_swiglu_bf16(const void* A, int lda, const void* B_interleaved, int ldb, void* act, int ldc, int M,
                          int d_ff, int K, int force_bn, int force_splits, void* workspace, size_t workspace_bytes,
                          gllm_stream_t stream) {
  return gemm_swiglu_bf16((const bf16*)A, lda, (const bf16*)B_interleaved, ldb, (bf16*)act, ldc, M, d_ff, K, M,
                          force_bn, force_splits, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_gemm_qkv_rope_bf16(const void* A, int lda, const void* W, int ldb, const void* bias, void* qkv, int M, int K,
                            int n_heads, int n_kv_heads, const int32_t* tok_pos, const int32_t* tok_slot,
                            const float* rope, void* k_cache, void* v_cache, int page_size, int force_bn,
                            int force_splits, void* workspace, size_t workspace_bytes, gllm_stream_t stream) {
  return gemm_qkv_rope_bf16((const bf16*)A, lda, (const bf16*)W, ldb, (const bf16*)bias, (bf16*)qkv, M, K, n_heads,
                            n_kv_heads, tok_pos, tok_slot, rope, (bf16*)k_cache, (bf16*)v_cache, page_size, M,
                            force_bn, force_splits, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_rmsnorm(const void* x, int ldx, const int32_t* row_index, const void* weight, void* out, int rows, int d,
                 float eps, gllm_stream_t stream) {
  return rmsnorm((const bf16*)x, ldx, row_index, (const bf16*)weight, (bf16*)out, rows, d, eps,
                 reinterpret_cast<cudaStream_t>(stream));
}

int gllm_silu_mul(const void* gate_up, int d_ff, void* out, int rows, gllm_stream_t stream) {
  return silu_mul((const bf16*)gate_up, d_ff, (bf16*)out, rows, reinterpret_cast<cudaStream_t>(stream));
}

uint32_t gllm_meta_errors(int reset) { return meta_errors(reset); }

int gllm_prepare_batch(const gllm_stage* stage, const gllm_batch* batch, int32_t* tok_pos, int32_t* tok_slot,
                       int32_t* tok_id, int32_t* emit_rows, gllm_stream_t stream) {
  if (!stage || !batch) return set_error(GLLM_ERR_INVALID, "null stage or batch");
  return prepare(*stage, *batch, tok_pos, tok_slot, tok_id, emit_rows, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_embed(const int32_t* tok_id, int n_tokens, const void* embed, int d, void* out, gllm_stream_t stream) {
  return embed_tokens(tok_id, n_tokens, (const bf16*)embed, d, (bf16*)out, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_rope_kv_write(void* qkv, int n_tokens, int n_heads, int n_kv_heads, int head_dim, const int32_t* tok_pos,
                       const int32_t* tok_slot, const float* rope, void* k_cache, void* v_cache, int page_size,
                       gllm_stream_t stream) {
  return rope_kv_write((bf16*)qkv, n_tokens, n_heads, n_kv_heads, head_dim, tok_pos, tok_slot, rope, (bf16*)k_cache,
                       (bf16*)v_cache, page_size, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_attn_mixed_paged(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                          int n_prefill_work, const int32_t* block_table, int max_pages_per_row, int kv_pages,
                          const void* k_cache,
                          const void* v_cache, int n_heads, int n_kv_heads, int head_dim, int page_size, void* out,
                          gllm_stream_t stream) {
  return attention_paged((const bf16*)qkv, seq_info, work, n_work, n_prefill_work, block_table, max_pages_per_row,
                         kv_pages,
                         (const bf16*)k_cache, (const bf16*)v_cache, n_heads, n_kv_heads, head_dim, page_size,
                         (bf16*)out, reinterpret_cast<cudaStream_t>(stream));
}

int gllm_attn_mixed_paged_auto(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                               int n_prefill_work, const int32_t* block_table, int max_pages_per_row, int kv_pages,
                               const void* k_cache, const void* v_cache, int n_heads, int n_kv_heads, int head_dim,
                               int page_size, void* out, const int32_t* host_seq_info, const int32_t* host_work,
                               void* workspace, size_t workspace_bytes, gllm_stream_t stream) {
  if (!host_seq_info || !host_work) return set_error(GLLM_ERR_INVALID, "host seq_info / work copies required");
  return attention_paged((const bf16*)qkv, seq_info, work, n_work, n_prefill_work, block_table, max_pages_per_row,
                         kv_pages, (const bf16*)k_cache, (const bf16*)v_cache, n_heads, n_kv_heads, head_dim,
                         page_size, (bf16*)out, reinterpret_cast<cudaStream_t>(stream), /*n_split=*/0, host_seq_info,
                         host_work, workspace, workspace_bytes);
}

int gllm_attn_mixed_paged_split(const void* qkv, const int32_t* seq_info, const int32_t* work, int n_work,
                                int n_prefill_work, const int32_t* block_table, int max_pages_per_row, int kv_pages,
                                const void* k_cache, const void* v_cache, int n_heads, int n_kv_heads, int head_dim,
                                int page_size, void* out, int n_split, void* workspace, size_t workspace_bytes,
                                gllm_stream_t stream) {
  if (n_split < 1) return set_error(GLLM_ERR_INVALID, "n_split must be >= 1");
  if (n_split > 1 && workspace_bytes < attention_split_bytes(n_prefill_work, n_split, n_kv_heads))
    return set_error(GLLM_ERR_INVALID, "attention split workspace too small");
  return attention_paged((const bf16*)qkv, seq_info, work, n_work, n_prefill_work, block_table, max_pages_per_row,
                         kv_pages, (const bf16*)k_cache, (const bf16*)v_cache, n_heads, n_kv_heads, head_dim,
                         page_size, (bf16*)out, reinterpret_cast<cudaStream_t>(stream), n_split, nullptr, nullptr,
                         workspace, workspace_bytes);
}

size_t gllm_attn_split_workspace_bytes(int n_prefill_work, int n_split, int n_kv_heads) {
  return attention_split_bytes(n_prefill_work, n_split, n_kv_heads);
}

int gllm_argmax(const void* logits, int rows, int vocab, int32_t* out, gllm_stream_t stream) {
  return argmax_rows((const bf16*)logits, rows, vocab, out, reinterpret_cast<cudaStream_t>(stream));
}

unsigned long long gllm_launch_count(void) { return g_launches.load(); }

int gllm_profile_begin(void) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof.clear();
  g_pool_next = 0;
  g_prof_on = true;
  return 0;
}

int gllm_profile_end(gllm_profile_entry* out, int max_entries, int* n_entries) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = false;
  gllm_profile_entry agg[P_NCAT];
  memset(agg, 0, sizeof(agg));
  for (const ProfRec& r : g_prof) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return set_cuda_error(e, "profile event");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    gllm_profile_entry& a = agg[r.cat];
    a.launches += 1;
    a.total_ms += ms;
    a.flops += r.flops;
    a.bytes += r.bytes;
  }
  int n = 0;
  for (int c = 0; c < P_NCAT && n < max_entries; ++c) {
    if (agg[c].launches == 0) continue;
    out[n] = agg[c];
    snprintf(out[n].name, sizeof(out[n].name), "%s", kProfNames[c]);
    ++n;
  }
  if (n_entries) *n_entries = n;
  g_prof.clear();
  return 0;
}

}  // extern "C"
