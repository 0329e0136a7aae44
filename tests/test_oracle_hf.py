"""Pin the fp32 oracle decoder (oracle/model_ref.py) to an independent implementation:
HF `transformers` LlamaForCausalLM / Qwen2ForCausalLM (CPU, fp32, eager attention).

* RoPE: `rope_table_ref` (the oracle's own restatement) equals HF's rotary embedding for the
  exact rope settings of every BASELINE model (default theta 5e5 / 1e6, llama3 band scaling
  of Llama-3.1-70B) up to position 9000; the product's `modelspec.rope_table` agrees too.
* Full forward: the oracle, fed HF's weights and HF's cos/sin table, reproduces HF logits on
  2-layer models with the BASELINE attention geometry (head_dim 128, GQA, QKV bias for Qwen2,
  llama3 scaling), non-unit RMSNorm weights.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from oracle.model_ref import RefDecoder, inv_freq_ref, rope_table_ref  # noqa: E402
from paper_2504_14775_b200.modelspec import MODELS, ModelSpec, rope_table  # noqa: E402


def _rope_params(spec):
    p = {"rope_theta": spec.rope_theta, "rope_type": "default"}
    if spec.rope_scaling:
        p = {"rope_theta": spec.rope_theta, "rope_type": "llama3", **spec.rope_scaling}
    return p


def _hf_config(spec, n_layers, vocab):
    kw = dict(vocab_size=vocab, hidden_size=spec.d_model, intermediate_size=spec.d_ff, num_hidden_layers=n_layers,
              num_attention_heads=spec.n_heads, num_key_value_heads=spec.n_kv_heads, head_dim=spec.head_dim,
              rms_norm_eps=spec.rms_eps, max_position_embeddings=131072, tie_word_embeddings=False,
              rope_parameters=_rope_params(spec))
    if spec.qkv_bias:
        cfg = transformers.Qwen2Config(**kw)
    else:
        cfg = transformers.LlamaConfig(attention_bias=False, mlp_bias=False, **kw)
    cfg._attn_implementation = "eager"
    return cfg


def _hf_cos_sin(model, n):
    rot = model.model.rotary_emb
    x = torch.zeros(1, n, 8, dtype=torch.float32)
    cos, sin = rot(x, torch.arange(n)[None, :])
    hd2 = cos.shape[-1] // 2
    return cos[0, :, :hd2].double().numpy(), sin[0, :, :hd2].double().numpy(), rot.inv_freq.double().numpy()


@pytest.mark.parametrize("name", ["llama3-8b", "qwen2.5-14b", "llama3.1-70b", "tiny"])
def test_rope_table_matches_hf(name):
    spec = MODELS[name]
    model = transformers.AutoModelForCausalLM.from_config(_hf_config(spec.with_layers(1), 1, 64))
    n = 9000
    cos, sin, inv = _hf_cos_sin(model, n)
    np.testing.assert_allclose(inv_freq_ref(spec), inv, rtol=2e-6, atol=0)
    ours = rope_table_ref(spec, n).astype(np.float64)
    prod = rope_table(spec, n).astype(np.float64)
    # HF forms pos * inv_freq in fp32: angle error ~ pos * 2^-24, so compare with that bound
    tol = 4e-7 * np.arange(n)[:, None] + 2e-6
    for tab in (ours, prod):
        assert (np.abs(tab[..., 0] - cos) <= tol).all()
        assert (np.abs(tab[..., 1] - sin) <= tol).all()
    np.testing.assert_allclose(ours, prod, atol=1e-6)


GEOMS = {
    # BASELINE attention geometry at a small width: (base model, d, heads, kv heads, d_ff)
    "llama3-8b": ("llama3-8b", 256, 4, 1, 384),
    "qwen2.5-14b": ("qwen2.5-14b", 320, 5, 1, 448),
    "llama3.1-70b": ("llama3.1-70b", 256, 8, 1, 512),
}


@pytest.mark.parametrize("name", list(GEOMS))
def test_oracle_matches_hf_forward(name):
    base, d, H, KV, dff = GEOMS[name]
    spec = ModelSpec(name, 2, d, H, KV, 128, dff, 777, MODELS[base].qkv_bias, MODELS[base].rope_theta,
                     MODELS[base].rope_scaling, MODELS[base].rms_eps)
    torch.manual_seed(5)
    model = transformers.AutoModelForCausalLM.from_config(_hf_config(spec, 2, spec.vocab)).float().eval()
    with torch.no_grad():
        for n, p in model.named_parameters():
            if "norm" in n:
                p.copy_(1.0 + 0.3 * torch.randn_like(p))
            elif n.endswith("bias"):
                p.copy_(0.5 * torch.randn_like(p))
            else:
                p.copy_(0.05 * torch.randn_like(p))
    m = model.model
    layers = []
    for blk in m.layers:
        a, mlp = blk.self_attn, blk.mlp
        layers.append({
            "attn_norm": blk.input_layernorm.weight,
            "w_qkv": torch.cat([a.q_proj.weight, a.k_proj.weight, a.v_proj.weight]),
            "b_qkv": torch.cat([a.q_proj.bias, a.k_proj.bias, a.v_proj.bias]) if spec.qkv_bias else None,
            "w_o": a.o_proj.weight,
            "mlp_norm": blk.post_attention_layernorm.weight,
            "w_gate_up": torch.cat([mlp.gate_proj.weight, mlp.up_proj.weight]),
            "w_down": mlp.down_proj.weight,
        })
    T = 61
    cos, sin, _ = _hf_cos_sin(model, T)
    hf_rope = np.stack([cos, sin], axis=-1).astype(np.float32)
    ref = RefDecoder(spec, layers, hf_rope, m.embed_tokens.weight, m.norm.weight, model.lm_head.weight)
    toks = np.random.default_rng(3).integers(0, spec.vocab, T)
    with torch.no_grad():
        want = model(torch.as_tensor(toks)[None, :]).logits[0].double()
    got = ref.logits(toks).double()
    rel = ((got - want).norm() / want.norm()).item()
    print(f"{name}: oracle vs HF rel err {rel:.2e}")
    assert rel < 1e-5, rel
    # and with the oracle's own RoPE table
    got2 = RefDecoder(spec, layers, None, m.embed_tokens.weight, m.norm.weight, model.lm_head.weight,
                      max_pos=T).logits(toks).double()
    assert ((got2 - want).norm() / want.norm()).item() < 1e-5
