"""Stage forward at every BASELINE model shape (2-layer slices) vs the fp32 oracle under teacher forcing.

Covers what the 8B bench path does not: QKV bias + GQA group 5 (Qwen2.5-14B/32B),
GQA group 8 + llama3 RoPE scaling + d=8192 (Llama-3.1-70B), a PP=2 split of the
layers on one GPU, and Sarathi scheduling through the same executor.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig  # noqa: E402
from paper_2504_14775_b200.workload import prompt_token_ids  # noqa: E402

pytestmark = pytest.mark.gpu


def _check(name, n_stages=1, scheduler="throttle", reqs=None, watch=None, pages=256):
    from oracle.model_ref import from_stage_workers
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    spec = MODELS[name].with_layers(2)
    reqs = reqs or [RequestSpec(0, 0.0, 90, 4), RequestSpec(1, 0.2, 33, 3), RequestSpec(2, 1.0, 150, 2)]
    ex = LocalExecutor(spec, reqs, num_pages=pages, page_size=16, n_stages=n_stages, max_tokens=2048,
                       max_emit=max(32, len(reqs)), record_logits=True, seed=11)
    Engine(reqs, scheduler=scheduler, pipeline=PipelineConfig(depth=n_stages), kv_config=KvConfig(pages, 16),
           throttle=ThrottleConfig(T=2, min_p=16), token_budget=64, executor=ex).run()
    oracle = from_stage_workers(ex.stages)
    worst = 0.0
    for rid, pos, lg in ex.logits:
        if watch is not None and rid not in watch:
            continue
        r = reqs[rid]
        seq = np.concatenate([prompt_token_ids(rid, r.input_tokens, spec.vocab),
                              np.asarray(ex.outputs[rid], dtype=np.int32)])[:pos]
        want = oracle.logits(seq)[pos - 1].numpy()
        worst = max(worst, float(np.linalg.norm(lg - want) / np.linalg.norm(want)))
    for r in reqs:
        assert len(ex.outputs[r.id]) == r.output_tokens
    assert worst < 2e-2, (name, worst)
    return worst


@pytest.mark.parametrize("name", ["qwen2.5-14b", "qwen2.5-32b", "llama3.1-70b", "llama3-8b"])
def test_model_shape_logits(cuda_ok, name):
    _check(name)


def test_two_stage_split_and_sarathi(cuda_ok):
    _check("qwen2.5-14b", n_stages=2, scheduler="sarathi")


@pytest.mark.parametrize("name,n_req", [("llama3-8b", 40), ("qwen2.5-14b", 100)])
def test_wide_decode_batches(cuda_ok, name, n_req):
    """Decode steps of 33-128 sequences (128-row tiles with split-K or whole-K tiles, the split-K
    QKV path with its separate RoPE + KV-write pass, fused-norm row scales in the split-K reduce)
    vs the fp32 oracle."""
    reqs = [RequestSpec(i, 0.0, 12 + (7 * i) % 29, 3) for i in range(n_req)]
    _check(name, reqs=reqs, watch={0, 17, n_req - 1}, pages=1024)
