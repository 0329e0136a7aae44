"""Attribute bf16-vs-fp32 logits drift at depth (GPU box): serve a few requests through the engine,
then compare the GPU logits and several oracle variants (fp32; bf16 rounding emulated at GEMM
inputs / residual stream / attention P) against each other, and the fp32 oracle's sensitivity to a
1e-3 relative perturbation of the embeddings (does the random-init network amplify noise?).

    python tools/precision_probe.py llama3-8b 32
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.model_ref import from_stage_workers  # noqa: E402
from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig  # noqa: E402
from paper_2504_14775_b200.executor import LocalExecutor  # noqa: E402
from paper_2504_14775_b200.modelspec import MODELS  # noqa: E402
from paper_2504_14775_b200.workload import prompt_token_ids  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
layers_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,8,32").split(",")]
torch.backends.cuda.matmul.allow_tf32 = False
for L in layers_list:
    spec = MODELS[name].with_layers(L)
    reqs = [RequestSpec(0, 0.0, 300, 4), RequestSpec(1, 0.3, 77, 3)]
    ex = LocalExecutor(spec, reqs, num_pages=256, page_size=16, max_tokens=2048, max_emit=32,
                       record_logits=True, seed=11)
    Engine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(256, 16),
           throttle=ThrottleConfig(T=2, min_p=16), executor=ex).run()
    orc = from_stage_workers(ex.stages, device="cuda")
    rid = 0
    seq = np.concatenate([prompt_token_ids(rid, 300, spec.vocab), np.asarray(ex.outputs[rid], np.int32)])
    items = [(pos, lg) for r, pos, lg in ex.logits if r == rid]
    last = max(p for p, _ in items)
    gpu = torch.tensor(np.stack([lg for _, lg in items])).cuda()
    pos = [p - 1 for p, _ in items]

    def run(em):
        orc.emulate = frozenset(em)
        return orc.logits_at(seq[:last], pos)

    def rel(a, b):
        return ((a - b).norm(dim=-1) / b.norm(dim=-1)).max().item()

    f32 = run(())
    out = {"gpu": rel(gpu, f32)}
    for em in (("in",), ("resid",), ("in", "resid"), ("in", "resid", "qkv", "p")):
        e = run(em)
        out["+".join(em)] = (rel(e, f32), rel(gpu, e))
    orc.emulate = frozenset()
    x = orc.embed[torch.as_tensor(seq[:last].astype(np.int64), device="cuda")].float()
    xp = x * (1 + 1e-3 * torch.randn_like(x))
    hp = orc.hidden(x=xp)[torch.as_tensor(pos, device="cuda")]
    from oracle.model_ref import _rms
    lp = _rms(hp, orc.final_norm.float(), spec.rms_eps) @ orc.lm_head.float().T
    out["sens_1e-3_embed"] = rel(lp, f32)
    print(f"{name} L={L}: gpu-vs-fp32 {out['gpu']:.3e}; emulated (vs fp32, gpu-vs-emulated): " +
          "; ".join(f"{k} ({v[0]:.3e}, {v[1]:.3e})" for k, v in out.items() if isinstance(v, tuple)) +
          f"; fp32 sensitivity to 1e-3 embed noise {out['sens_1e-3_embed']:.3e}", flush=True)
    del ex, orc
    torch.cuda.empty_cache()
