"""Model shapes for the BASELINE configs, seeded random-init weights, RoPE tables.

Shapes are the public HF configs; the reference has no
model at all (`SPEC.md:20`), so these only need to be self-consistent between
the B200 path and the fp32 oracle (`oracle/model_ref.py`).

Weights: seeded N(0, 0.02), output projections (o, down) scaled by 1/sqrt(2L),
norm weights 1. Generated directly in bf16 on the device that
will hold them; the oracle reads back the same bf16 values and upcasts.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    qkv_bias: bool = False
    rope_theta: float = 10000.0
    rope_scaling: dict | None = None
    rms_eps: float = 1e-5

    @property
    def qkv_width(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def kv_bytes_per_token_layer(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * 2

    @property
    def params_per_layer(self) -> int:
        d, hd = self.d_model, self.head_dim
        return d * self.qkv_width + self.n_heads * hd * d + 2 * self.d_ff * d + self.d_ff * d

    def with_layers(self, n: int) -> "ModelSpec":
        return replace(self, n_layers=n)


_LLAMA3_SCALING = {"factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                   "original_max_position_embeddings": 8192}

MODELS: dict[str, ModelSpec] = {
    # C1: BASELINE fixes L=4, d=256; head_dim 128 so one kernel specialisation covers every config.
    "tiny": ModelSpec("tiny", 4, 256, 2, 1, 128, 768, 32000),
    "llama3-8b": ModelSpec("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, rope_theta=500000.0),
    "qwen2.5-14b": ModelSpec("qwen2.5-14b", 48, 5120, 40, 8, 128, 13824, 152064, qkv_bias=True,
                             rope_theta=1000000.0, rms_eps=1e-6),
    "qwen2.5-32b": ModelSpec("qwen2.5-32b", 64, 5120, 40, 8, 128, 27648, 152064, qkv_bias=True,
                             rope_theta=1000000.0, rms_eps=1e-6),
    "llama3.1-70b": ModelSpec("llama3.1-70b", 80, 8192, 64, 8, 128, 28672, 128256, rope_theta=500000.0,
                              rope_scaling=_LLAMA3_SCALING),
}


def stage_layers(n_layers: int, pp: int, stage: int) -> range:
    """Contiguous ceil(L/PP) layer ranges."""
    per = -(-n_layers // pp)
    lo = min(stage * per, n_layers)
    return range(lo, min(lo + per, n_layers))


def inv_freq(spec: ModelSpec) -> np.ndarray:
    hd = spec.head_dim
    f = 1.0 / (spec.rope_theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd))
    sc = spec.rope_scaling
    if sc:
        # llama3 frequency-dependent scaling
        factor, lo, hi = sc["factor"], sc["low_freq_factor"], sc["high_freq_factor"]
        old = sc["original_max_position_embeddings"]
        low_wl, high_wl = old / lo, old / hi
        wl = 2 * math.pi / f
        smooth = (old / wl - lo) / (hi - lo)
        scaled = np.where(wl > low_wl, f / factor, f)
        mid = (wl <= low_wl) & (wl >= high_wl)
        scaled = np.where(mid, (1 - smooth) * f / factor + smooth * f, scaled)
        f = scaled
    return f


def rope_table(spec: ModelSpec, max_pos: int) -> np.ndarray:
    """float32 [max_pos, head_dim/2, 2] of (cos, sin) for the rotate-half convention."""
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv_freq(spec)[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


# Weight tensors of one decoder layer, in generation order.
LAYER_TENSORS = ("attn_norm", "w_qkv", "b_qkv", "w_o", "mlp_norm", "w_gate_up", "w_down")


def layer_shapes(spec: ModelSpec) -> dict[str, tuple[int, ...] | None]:
    d, hd = spec.d_model, spec.head_dim
    return {
        "attn_norm": (d,),
        "w_qkv": (spec.qkv_width, d),
        "b_qkv": (spec.qkv_width,) if spec.qkv_bias else None,
        "w_o": (d, spec.n_heads * hd),
        "mlp_norm": (d,),
        "w_gate_up": (2 * spec.d_ff, d),
        "w_down": (d, spec.d_ff),
    }


def init_layer(spec: ModelSpec, layer: int, seed: int, device) -> dict:
    """Seeded bf16 weights of one layer on `device` (torch); tensor k of layer l uses seed (seed, l, k)."""
    import torch

    out = {}
    out_scale = 1.0 / math.sqrt(2.0 * spec.n_layers)
    for k, name in enumerate(LAYER_TENSORS):
        shape = layer_shapes(spec)[name]
        if shape is None:
            out[name] = None
            continue
        if name.endswith("norm"):
            out[name] = torch.ones(shape, dtype=torch.bfloat16, device=device)
            continue
        g = torch.Generator(device=device)
        g.manual_seed(_mix(seed, layer, k))
        std = 0.02 * (out_scale if name in ("w_o", "w_down") else 1.0)
        t = torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std
        out[name] = t.to(torch.bfloat16)
    return out


def interleave_gate_up(w, d_ff: int, block: int = 64):
    """[gate; up] ([2 d_ff, d]) -> 64-row alternating gate/up blocks (the fused-SwiGLU GEMM layout)."""
    d = w.shape[-1]
    return w.view(2, d_ff // block, block, d).transpose(0, 1).reshape(2 * d_ff, d)


def deinterleave_gate_up(w, d_ff: int, block: int = 64):
    """Inverse of `interleave_gate_up`."""
    d = w.shape[-1]
    return w.view(d_ff // block, 2, block, d).transpose(0, 1).reshape(2 * d_ff, d)


def init_embed(spec: ModelSpec, seed: int, device, which: str):
    """`embed` ([vocab, d]), `lm_head` ([vocab, d]) or `final_norm` ([d])."""
    import torch

    if which == "final_norm":
        return torch.ones(spec.d_model, dtype=torch.bfloat16, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(_mix(seed, 10_000 + (0 if which == "embed" else 1), 0))
    t = torch.randn((spec.vocab, spec.d_model), generator=g, device=device, dtype=torch.float32) * 0.02
    return t.to(torch.bfloat16)


def _mix(seed: int, a: int, b: int) -> int:
    return (seed * 1_000_003 + a * 7919 + b * 104_729) % (2 ** 62)
