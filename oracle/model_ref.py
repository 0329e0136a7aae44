"""fp32 CPU reference decoder (TEST INFRASTRUCTURE — never on the product path).

Independent of the paged design: every call recomputes full causal attention
over the whole token sequence with dense per-request K/V, no block tables,
no chunking. Numerics are plain fp32 (no bf16 rounding of activations); the
only shared inputs with the GPU path are the bf16 weight values (upcast) and
the RoPE table (`modelspec.rope_table`), so disagreement isolates kernel error.

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


class RefDecoder:
    """fp32 copy of a stage's (or the whole model's) weights on the CPU."""

    def __init__(self, spec, layers: list[dict], rope: np.ndarray, embed=None, final_norm=None, lm_head=None):
        f = lambda t: None if t is None else t.detach().to("cpu", torch.float32)
        self.spec = spec
        self.layers = [{k: f(v) for k, v in L.items()} for L in layers]
        self.rope = torch.from_numpy(np.asarray(rope, dtype=np.float32))
        self.embed = f(embed)
        self.final_norm = f(final_norm)
        self.lm_head = f(lm_head)

    def layer(self, L: dict, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        s = self.spec
        T = x.shape[0]
        hd, H, KV = s.head_dim, s.n_heads, s.n_kv_heads
        h = _rms(x, L["attn_norm"], s.rms_eps)
        qkv = h @ L["w_qkv"].T
        if L.get("b_qkv") is not None:
            qkv = qkv + L["b_qkv"]
        q = qkv[:, : H * hd].view(T, H, hd)
        k = qkv[:, H * hd: (H + KV) * hd].view(T, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        cs = self.rope[pos]
        q = _rope(q, cs[..., 0], cs[..., 1])
        k = _rope(k, cs[..., 0], cs[..., 1])
        g = H // KV
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
        att = torch.einsum("thd,shd->hts", q, k) / np.sqrt(hd)
        mask = pos[None, :, None] < pos[None, None, :]
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        o = torch.einsum("hts,shd->thd", att, v).reshape(T, H * hd)
        x = x + o @ L["w_o"].T
        h = _rms(x, L["mlp_norm"], s.rms_eps)
        gu = h @ L["w_gate_up"].T
        a = torch.nn.functional.silu(gu[:, : s.d_ff]) * gu[:, s.d_ff:]
        return x + a @ L["w_down"].T

    @torch.no_grad()
    def hidden(self, tokens=None, x: torch.Tensor | None = None) -> torch.Tensor:
        """Run the held layers over one full sequence (positions 0..T-1)."""
        if x is None:
            x = self.embed[torch.as_tensor(np.asarray(tokens, dtype=np.int64))]
        pos = torch.arange(x.shape[0])
        for L in self.layers:
            x = self.layer(L, x, pos)
        return x

    @torch.no_grad()
    def logits(self, tokens) -> torch.Tensor:
        """fp32 logits [T, vocab] for every position of one sequence (teacher forcing)."""
        x = self.hidden(tokens)
        return _rms(x, self.final_norm, self.spec.rms_eps) @ self.lm_head.T


def from_stage_workers(workers) -> RefDecoder:
    """Oracle over the same bf16 weights the GPU stage workers hold (read back once)."""
    spec = workers[0].spec
    layers = [L for w in workers for L in w.canonical_layers()]
    first, last = workers[0], workers[-1]
    return RefDecoder(spec, layers, first.rope.cpu().numpy(), first.embed, last.final_norm, last.lm_head)
