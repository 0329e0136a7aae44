"""Stage workers: device-resident weights, paged KV pool, block table, token history.

A `StageWorker` holds one pipeline stage (a contiguous layer range) on one GPU
and runs micro-batches through it with a single C-ABI call
(`gllm_stage_forward`). `pack_batch` turns the engine's `BatchMeta` (the
paper's pre-broadcast per-iteration metadata, `PAPER.md:262`) into the one
int32 buffer the device expects (layout in include/gllm.h).

HBM layout per stage (SURVEY §8(d) notation):
  k_cache, v_cache : bf16 [L_s][num_pages][n_kv][page_size][head_dim]
                     -> one (page, kv head) is a contiguous page_size*256 B block
  block_table      : int32 [max_rows][ceil(max_seq_len / page_size)]
  token_hist       : int32 [max_rows][max_seq_len]   (first stage: prompt + sampled tokens)
  workspace        : activations for max_tokens tokens + split-K partials
"""

from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native
from .modelspec import ModelSpec, deinterleave_gate_up, init_embed, init_layer, interleave_gate_up, rope_table
from .workload import prompt_token_ids


@dataclass
class PackedBatch:
    seq: int
    n_seqs: int
    n_tokens: int
    n_emit: int
    n_work: int
    n_prefill_work: int
    n_deltas: int
    n_prompts: int
    data: np.ndarray             # int32 packed metadata (host)
    emit_ids: list[int]          # request id of each sampled row
    emit_pos: list[int]          # token position each sampled row predicts
    flags: int = 0               # runtime flags carried in the PP metadata header (bit 0: profile)


def pack_batch(meta, q_tile: int, prompt_source) -> PackedBatch:
    """Pack `engine.BatchMeta` into the device metadata layout (vectorised over sequences).

    `prompt_source(request_id) -> np.int32 array` supplies prompt tokens of
    requests that got a block-table row in this batch.
    """
    n = len(meta.ids)
    n_new = np.asarray(meta.n_new, dtype=np.int32).reshape(-1)
    starts = np.asarray(meta.starts, dtype=np.int32).reshape(-1)
    emits = np.asarray(meta.emits, dtype=bool).reshape(-1)
    off = np.zeros(n, dtype=np.int32)
    if n:
        np.cumsum(n_new[:-1], out=off[1:])
    emit_idx = np.where(emits, np.cumsum(emits) - 1, -1).astype(np.int32)
    info = np.stack([np.asarray(meta.rows, dtype=np.int32).reshape(-1), starts, n_new, off, emit_idx], axis=1)
    eidx = np.flatnonzero(emits)
    emit_ids = [meta.ids[i] for i in eidx.tolist()]
    emit_pos = (starts[eidx] + n_new[eidx]).tolist()
    # attention work: prefill tiles first (heavy CTAs launch first), then one item per decode
    pf = np.flatnonzero(n_new > 1)
    tiles = (n_new[pf] + q_tile - 1) // q_tile
    total = int(tiles.sum())
    first = np.zeros(len(pf), dtype=np.int64)
    if len(pf):
        np.cumsum(tiles[:-1], out=first[1:])
    pf_seq = np.repeat(pf, tiles)
    pf_q0 = (np.arange(total) - np.repeat(first, tiles)) * q_tile
    dec = np.flatnonzero(n_new == 1)
    work_a = np.concatenate([np.stack([pf_seq, pf_q0], axis=1).reshape(-1, 2),
                             np.stack([dec, np.zeros_like(dec)], axis=1).reshape(-1, 2)]).astype(np.int32)
    deltas = np.asarray(meta.page_deltas, dtype=np.int32).reshape(-1, 3)
    hdrs, toks = [], []
    toff = 0
    for rid, row in meta.new_prompts:
        t = np.asarray(prompt_source(rid), dtype=np.int32)
        hdrs.append((row, len(t), toff))
        toks.append(t)
        toff += len(t)
    hdr_a = np.asarray(hdrs, dtype=np.int32).reshape(-1, 3)
    data = np.concatenate([info.ravel(), work_a.ravel(), deltas.ravel(), hdr_a.ravel()] + toks).astype(np.int32)
    return PackedBatch(meta.seq, n, int(n_new.sum()), len(emit_ids), len(work_a), total, len(deltas), len(hdrs),
                       data, emit_ids, emit_pos)


class StageWorker:
    """One pipeline stage (layers `layers` of `spec`) resident on `device`."""

    def __init__(self, spec: ModelSpec, layers: range, *, is_first: bool, is_last: bool, num_pages: int,
                 page_size: int, max_rows: int, max_seq_len: int, max_tokens: int, max_emit: int,
                 seed: int = 0, device="cuda", fused_norm: bool | None = None, scratch: bool = False):
        """`scratch`: one extra block-table row and KV page past the engine's (max_rows, num_pages),
        the target of the padding sequences of CUDA-graph decode batches (`executor.LocalExecutor`)."""
        import torch

        lib = native.load()
        self.spec = spec
        self.layer_ids = list(layers)
        self.is_first, self.is_last = is_first, is_last
        self.device = torch.device(device)
        self.page_size = page_size
        self.num_pages = num_pages
        self.max_rows = max_rows
        self.max_seq_len = max_seq_len
        self.max_tokens = max_tokens
        self.max_emit = max_emit
        self.q_tile = lib.gllm_attention_q_tile(spec.n_heads, spec.n_kv_heads)
        dev = self.device
        self.layers = [init_layer(spec, l, seed, dev) for l in self.layer_ids]
        # Fused RMSNorm (include/gllm.h, gllm_dims.fused_norm): fold each norm weight into the columns
        # of the projection it feeds, W' = W diag(w), and keep unit norm vectors -- the same model
        # (RMSNorm(x) * w) W^T == RMSNorm(x) W'^T, so the fp32 oracle sees identical math.
        self.fused_norm = fused_norm if fused_norm is not None else os.environ.get("GLLM_FUSED_NORM", "1") != "0"
        for w in self.layers:   # device layout for the fused SwiGLU epilogue (see include/gllm.h)
            w["w_gate_up"] = interleave_gate_up(w["w_gate_up"], spec.d_ff).contiguous()
        if self.fused_norm:
            self._fold_norms()
        self.embed = init_embed(spec, seed, dev, "embed") if is_first else None
        self.final_norm = init_embed(spec, seed, dev, "final_norm") if is_last else None
        self.lm_head = init_embed(spec, seed, dev, "lm_head") if is_last else None
        L = len(self.layer_ids)
        self.scratch_row = max_rows if scratch else None
        self.scratch_page = num_pages if scratch else None
        if scratch:
            max_rows, num_pages = max_rows + 1, num_pages + 1
        kv_shape = (L, num_pages, spec.n_kv_heads, page_size, spec.head_dim)
        self.k_cache = torch.empty(kv_shape, dtype=torch.bfloat16, device=dev)
        self.v_cache = torch.empty(kv_shape, dtype=torch.bfloat16, device=dev)
        self.max_pages_per_row = -(-max_seq_len // page_size)
        # -1 = unmapped: a position whose page was never delivered fails the device bounds check
        self.block_table = torch.full((max_rows, self.max_pages_per_row), -1, dtype=torch.int32, device=dev)
        if scratch:
            self.block_table[self.scratch_row, 0] = self.scratch_page
        self.token_hist = torch.zeros((max_rows, max_seq_len), dtype=torch.int32, device=dev) if is_first else None
        self.rope = torch.from_numpy(rope_table(spec, max_seq_len)).to(dev)
        self.dims = native.Dims(L, spec.d_model, spec.n_heads, spec.n_kv_heads, spec.head_dim, spec.d_ff, spec.vocab,
                                int(spec.qkv_bias), spec.rms_eps, page_size, num_pages, max_rows,
                                self.max_pages_per_row, max_seq_len, max_tokens, max_emit, int(self.fused_norm))
        ws = lib.gllm_stage_workspace_bytes(C.byref(self.dims))
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
        self._layer_arr = (native.Layer * max(L, 1))()
        for i, w in enumerate(self.layers):
            self._layer_arr[i] = native.Layer(*(native.ptr(w[k]) for k in
                                                ("attn_norm", "w_qkv", "b_qkv", "w_o", "mlp_norm", "w_gate_up", "w_down")))
        self.cstage = native.Stage(self.dims, int(is_first), int(is_last), native.ptr(self.embed),
                                   native.ptr(self.final_norm), native.ptr(self.lm_head), self._layer_arr,
                                   native.ptr(self.k_cache), native.ptr(self.v_cache), native.ptr(self.block_table),
                                   native.ptr(self.token_hist), native.ptr(self.rope), native.ptr(self.workspace), ws)

    def _fold_norms(self) -> None:
        """W <- W diag(norm), norm <- 1, in place (device pointers unchanged)."""
        for w in self.layers:
            for norm, proj in (("attn_norm", "w_qkv"), ("mlp_norm", "w_gate_up")):
                w[proj].copy_((w[proj].float() * w[norm].float()[None, :]).to(w[proj].dtype))
                w[norm].fill_(1.0)

    def refold_norms(self) -> None:
        """Switch to the fused-norm path, folding the current norm weights (tests set non-unit ones)."""
        self._fold_norms()
        self.fused_norm = True
        self.dims.fused_norm = 1
        self.cstage.dims.fused_norm = 1

    def canonical_layers(self) -> list[dict]:
        """Layer weights in the plain [gate; up] layout (for the fp32 oracle)."""
        out = []
        for w in self.layers:
            c = dict(w)
            c["w_gate_up"] = deinterleave_gate_up(w["w_gate_up"], self.spec.d_ff)
            out.append(c)
        return out

    def cbatch(self, pb: PackedBatch, meta_dev, hidden=None, sampled=None, logits=None) -> native.Batch:
        # host seq_info view for the profiler's byte/FLOP accounting (first n_seqs*5 ints)
        return native.Batch(pb.n_seqs, pb.n_tokens, pb.n_emit, pb.n_work, pb.n_prefill_work, pb.n_deltas, pb.n_prompts,
                            native.ptr(meta_dev), native.ptr(hidden), native.ptr(sampled), native.ptr(logits),
                            pb.data.ctypes.data)

    def forward(self, pb: PackedBatch, meta_dev, hidden=None, sampled=None, logits=None, stream=None) -> None:
        """Enqueue this stage's forward for one packed micro-batch on `stream` (no host sync)."""
        b = self.cbatch(pb, meta_dev, hidden, sampled, logits)
        native.call("gllm_stage_forward", C.byref(self.cstage), C.byref(b), native.stream_handle(stream))

    def commit_tokens(self, pb: PackedBatch, meta_dev, sampled, stream=None) -> None:
        b = self.cbatch(pb, meta_dev)
        native.call("gllm_commit_tokens", C.byref(self.cstage), C.byref(b), native.ptr(sampled),
                    native.stream_handle(stream))


def pad_decode_batch(pb: PackedBatch, bucket: int, scratch_row: int, scratch_page: int) -> PackedBatch:
    """A decode-only batch padded to `bucket` sequences for a captured CUDA graph: the padding
    sequences decode token 0 of the scratch row (its one KV page is the scratch page) and the
    block-table deltas are padded with the scratch row's own (idempotent) entry, so every count
    the device sees is fixed per bucket. Sampled rows past pb.n_emit are ignored by the caller."""
    n, nd = pb.n_seqs, pb.n_deltas
    d = pb.data
    info = d[:5 * n].reshape(n, 5)
    work = d[5 * n:7 * n].reshape(n, 2)
    deltas = d[7 * n:7 * n + 3 * nd].reshape(nd, 3)
    pad = bucket - n
    j = np.arange(n, bucket, dtype=np.int32)
    pinfo = np.stack([np.full(pad, scratch_row, np.int32), np.zeros(pad, np.int32), np.ones(pad, np.int32), j, j], axis=1)
    pwork = np.stack([j, np.zeros(pad, np.int32)], axis=1)
    pdel = np.tile(np.asarray([[scratch_row, 0, scratch_page]], np.int32), (bucket - nd, 1))
    data = np.concatenate([info.ravel(), pinfo.ravel(), work.ravel(), pwork.ravel(), deltas.ravel(),
                           pdel.ravel()]).astype(np.int32)
    return PackedBatch(pb.seq, bucket, bucket, bucket, bucket, 0, bucket, 0, data, pb.emit_ids, pb.emit_pos, pb.flags)


def default_prompt_source(specs_by_id: dict, vocab: int):
    """Seeded synthetic prompts (PCG64(1000 + id), or the trace's `token_seed`)."""
    def src(rid: int) -> np.ndarray:
        r = specs_by_id[rid]
        return prompt_token_ids(rid, r.input_tokens, vocab, getattr(r, "token_seed", None))
    return src


def prompt_source_with(prompts: dict, specs_by_id: dict, vocab: int):
    """Prompt tokens a caller submitted (`EngineCore.submit(spec, prompt_ids)`) take precedence over
    the seeded synthetic ones."""
    synth = default_prompt_source(specs_by_id, vocab)

    def src(rid: int) -> np.ndarray:
        t = prompts.get(rid)
        return t if t is not None else synth(rid)
    return src


def default_max_rows(requests, num_pages: int) -> int:
    """Block-table / token-history rows: bounded by concurrency, not by the trace length. A row is
    bound while its request holds KV (>= 1 page), so `num_pages` rows always suffice for the
    requests the KV cache can hold; a short trace needs no more rows than it has requests."""
    return max(1, min(len(requests) or num_pages, num_pages))


def default_max_seq_len(requests, floor: int = 16) -> int:
    """Longest prompt + output of the trace (+1 for the slot of the last sampled token)."""
    return max([r.input_tokens + r.output_tokens + 1 for r in requests] + [floor])
