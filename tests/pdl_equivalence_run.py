"""Helper for test_pdl_bit_identical (run in a subprocess: GLLM_* switches are read once per process).

Serves a seeded trace on a 2-layer Llama-3-8B-shaped stage (prefill chunks up to 2048 tokens,
medium and decode-sized batches: 2-CTA, split-K, skinny GEMMs, both attention roles) and prints
every sampled token plus a digest of the recorded logits as JSON.
"""
import dataclasses
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, ThrottleConfig
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.workload import ArrivalProcess, builtin_length_table, synthesize_requests

    spec = dataclasses.replace(MODELS["llama3-8b"], n_layers=2)
    reqs = synthesize_requests(ArrivalProcess.poisson(400.0, 3), builtin_length_table("sharegpt-like"), 48)
    reqs = [dataclasses.replace(r, output_tokens=min(r.output_tokens, 12)) for r in reqs]
    pages = sum(-(-(r.input_tokens + r.output_tokens) // 16) for r in reqs) + 64
    ex = LocalExecutor(spec, reqs, num_pages=pages, page_size=16, max_tokens=2560, max_emit=64, record_logits=True,
                       record_ids=[0, 7, 21], seed=5)
    Engine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(pages, 16), throttle=ThrottleConfig(),
           executor=ex).run()
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for rid, pos, lg in ex.logits:
        h.update(np.asarray([rid, pos], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(lg, dtype=np.float32).tobytes())
    print(json.dumps({"tokens": {str(k): v for k, v in sorted(ex.outputs.items())}, "logits_sha256": h.hexdigest(),
                      "launches": ex.launches}))


if __name__ == "__main__":
    main()
