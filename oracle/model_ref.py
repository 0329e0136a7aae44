"""fp32 CPU reference decoder (TEST INFRASTRUCTURE — never on the product path).

Independent of the paged design: every call recomputes full causal attention
over the whole token sequence with dense per-request K/V, no block tables,
no chunking. Numerics are plain fp32 (no bf16 rounding of activations); the
only shared input with the GPU path is the bf16 weight values (upcast), so
disagreement isolates kernel error. The RoPE table is the oracle's own
(`rope_table_ref`, restating HF's default / llama3 frequency rules), pinned to
`transformers`' rotary embedding and to full HF Llama/Qwen2 forwards by
tests/test_oracle_hf.py -- not the product's `modelspec.rope_table`.

Runs on any torch device: the CPU for small cases, or a GPU in fp32 (TF32
disabled) as the "plain torch fp32 reference" for full-depth / long-prompt
parity, where a CPU pass over 8-70B-parameter stages would take minutes.

The reference simulator has no model (`SPEC.md:20`); this restates the
standard Llama/Qwen2 decoder the north star names:
  h = x + Wo . attn(rope(Wq rms(x)), rope(Wk rms(x)), Wv rms(x))
  y = h + Wd . (silu(Wg rms(h)) * Wu rms(h))
  logits = Wlm . rms(y_L)
"""

from __future__ import annotations

import numpy as np
import torch


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    # x [T, H, hd]; cos/sin [T, hd/2]; rotate-half convention
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def inv_freq_ref(spec) -> np.ndarray:
    """RoPE inverse frequencies theta^(-2i/hd), with llama3 band scaling when `spec.rope_scaling`
    is set (restates `transformers.modeling_rope_utils` "default" / "llama3" rules): wavelengths
    above orig/low_freq_factor are divided by `factor`, below orig/high_freq_factor kept, and
    in between blended by smooth = (orig/wavelen - low)/(high - low)."""
    hd = spec.head_dim
    base = np.array([spec.rope_theta ** (-(2.0 * i) / hd) for i in range(hd // 2)], dtype=np.float64)
    sc = spec.rope_scaling
    if not sc:
        return base
    out = np.empty_like(base)
    orig = float(sc["original_max_position_embeddings"])
    lo_f, hi_f, factor = float(sc["low_freq_factor"]), float(sc["high_freq_factor"]), float(sc["factor"])
    for i, f in enumerate(base):
        wavelen = 2.0 * np.pi / f
        if wavelen < orig / hi_f:
            out[i] = f
        elif wavelen > orig / lo_f:
            out[i] = f / factor
        else:
            smooth = (orig / wavelen - lo_f) / (hi_f - lo_f)
            out[i] = (1.0 - smooth) * f / factor + smooth * f
    return out


def rope_table_ref(spec, max_pos: int) -> np.ndarray:
    """float32 [max_pos, hd/2, 2] = (cos, sin)(pos * inv_freq), rotate-half convention."""
    ang = np.outer(np.arange(max_pos, dtype=np.float64), inv_freq_ref(spec))
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


class RefDecoder:
    """fp32 decoder over a stage's (or the whole model's) weights on `device`.

    Weights are kept as given (bf16 on the GPU stage, typically) and upcast one layer at a time,
    so a full-depth 8B or 10-layer 70B reference fits beside the product's own copy.
    """

    def __init__(self, spec, layers: list[dict], rope: np.ndarray | None = None, embed=None, final_norm=None,
                 lm_head=None, device="cpu", max_pos: int = 16384):
        self.device = torch.device(device)
        f = lambda t: None if t is None else t.detach().to(self.device)
        self.spec = spec
        self.layers = [{k: f(v) for k, v in L.items()} for L in layers]
        rope = rope_table_ref(spec, max_pos) if rope is None else rope
        self.rope = torch.from_numpy(np.asarray(rope, dtype=np.float32)).to(self.device)
        self.embed = f(embed)
        self.final_norm = f(final_norm)
        self.lm_head = f(lm_head)
        self.emulate: frozenset = frozenset()   # diagnostics only: bf16 rounding points, see _r

    def _r(self, tag: str, t: torch.Tensor) -> torch.Tensor:
        """Round to bf16 where a bf16 implementation would (tags: "in" = GEMM inputs, "qkv", "p" =
        attention probabilities, "resid" = residual stream). Off by default: the oracle is fp32;
        tools/precision_probe.py uses it to attribute bf16-vs-fp32 drift."""
        return t.bfloat16().float() if tag in self.emulate else t

    def layer(self, L: dict, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        L = {k: None if v is None else v.float() for k, v in L.items()}
        s = self.spec
        T = x.shape[0]
        hd, H, KV = s.head_dim, s.n_heads, s.n_kv_heads
        r = self._r
        h = _rms(x, L["attn_norm"], s.rms_eps)
        qkv = r("in", h) @ L["w_qkv"].T
        if L.get("b_qkv") is not None:
            qkv = qkv + L["b_qkv"]
        qkv = r("qkv", qkv)
        q = qkv[:, : H * hd].view(T, H, hd)
        k = qkv[:, H * hd: (H + KV) * hd].view(T, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        cs = self.rope[pos]
        q = _rope(q, cs[..., 0], cs[..., 1])
        k = _rope(k, cs[..., 0], cs[..., 1])
        g = H // KV
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
        o = torch.empty(T, H, hd, dtype=x.dtype, device=x.device)
        qc = max(1, (1 << 26) // max(1, H * T))     # query rows per block: att block <= 256 MB fp32
        for t0 in range(0, T, qc):
            t1 = min(T, t0 + qc)
            att = torch.einsum("thd,shd->hts", q[t0:t1], k) / np.sqrt(hd)
            mask = pos[None, t0:t1, None] < pos[None, None, :]
            att = att.masked_fill(mask, float("-inf")).softmax(-1)
            o[t0:t1] = torch.einsum("hts,shd->thd", r("p", att), v)
        o = o.reshape(T, H * hd)
        x = r("resid", x + r("in", o) @ L["w_o"].T)
        h = _rms(x, L["mlp_norm"], s.rms_eps)
        gu = r("in", h) @ L["w_gate_up"].T
        a = torch.nn.functional.silu(gu[:, : s.d_ff]) * gu[:, s.d_ff:]
        return r("resid", x + r("in", a) @ L["w_down"].T)

    @torch.no_grad()
    def hidden(self, tokens=None, x: torch.Tensor | None = None) -> torch.Tensor:
        """Run the held layers over one full sequence (positions 0..T-1)."""
        if x is None:
            x = self.embed[torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=self.device)].float()
        x = x.to(self.device, torch.float32)
        pos = torch.arange(x.shape[0], device=self.device)
        for L in self.layers:
            x = self.layer(L, x, pos)
        return x

    @torch.no_grad()
    def logits(self, tokens) -> torch.Tensor:
        """fp32 logits [T, vocab] for every position of one sequence (teacher forcing)."""
        x = self.hidden(tokens)
        return _rms(x, self.final_norm.float(), self.spec.rms_eps) @ self.lm_head.float().T

    @torch.no_grad()
    def logits_at(self, tokens, positions) -> torch.Tensor:
        """fp32 logits at the given positions only (the LM head over a long prompt is skipped)."""
        x = self.hidden(tokens)[torch.as_tensor(list(positions), device=self.device)]
        return _rms(x, self.final_norm.float(), self.spec.rms_eps) @ self.lm_head.float().T


def from_stage_workers(workers, device="cpu", max_pos: int | None = None) -> RefDecoder:
    """Oracle over the same bf16 weights the GPU stage workers hold; RoPE from `rope_table_ref`."""
    spec = workers[0].spec
    layers = [L for w in workers for L in w.canonical_layers()]
    first, last = workers[0], workers[-1]
    return RefDecoder(spec, layers, None, first.embed, last.final_norm, last.lm_head, device=device,
                      max_pos=max_pos or first.max_seq_len + 1)
