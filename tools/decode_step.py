"""Decode-only step time at a fixed batch size (the low-load TPOT regime), on one B200.

    python tools/decode_step.py --model qwen2.5-14b --batch 4 [--ctx 512] [--steps 30]

N requests (prompt --ctx tokens, long outputs) all arrive at t=0; the virtual-clock engine
(reference scheduling) drives LocalExecutor until every request decodes, then the device time
of each decode-only micro-batch (N tokens, no prefill) is read from CUDA events. Prints the
median ms per step and its ratio to the HBM floor (stage weights + the batch's KV-cache reads at
the mid-window context, over the measured HBM bandwidth). Run under `ncu --nvtx --nvtx-include decode_timed/` for a per-kernel split.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-14b")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--cuda-graphs", action="store_true", help="decode-only batches as captured CUDA graphs")
    ap.add_argument("--profile", action="store_true",
                    help="per-kernel-class device time of the timed steps (native CUDA-event profiler; "
                         "its events serialise the launches, so ms_per_step is then not the clean figure)")
    a = ap.parse_args()

    import torch

    from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig, native
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    spec = MODELS[a.model]
    warm = 40
    # the first prompts finish prefill up to ~batch*ctx/2048 iterations before the last, plus the
    # throttled tail (#P = #WP/T once #WP < T*MaxP: ~T*ln(T*MaxP/MinP) more iterations): their
    # outputs must outlast that, or the batch never runs full decode-only steps
    pf_iters = -(-a.batch * a.ctx // 2048) + 96
    reqs = [RequestSpec(i, 0.0, a.ctx, warm + a.steps + 8 + pf_iters) for i in range(a.batch)]
    pages = a.batch * (-(-(a.ctx + warm + a.steps + 16 + pf_iters) // 16)) + 64
    ex = LocalExecutor(spec, reqs, num_pages=pages, page_size=16, max_tokens=2048, max_emit=max(a.batch, 32), seed=0,
                       cuda_graphs=a.cuda_graphs)
    eng = Engine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(pages, 16), throttle=ThrottleConfig(),
                 executor=ex)
    decode_only, ranged, wall = [], False, []
    while eng.step():
        its = eng._iters
        if its and its[-1].prefill_tokens == 0 and its[-1].decode_tokens == a.batch:
            decode_only.append(its[-1].batch_seq)
            wall.append(time.perf_counter())
            if len(decode_only) == warm // 2 and not ranged:
                torch.cuda.synchronize()
                torch.cuda.nvtx.range_push("decode_timed")
                if a.profile:
                    native.profile_begin()
                ranged = True
            if len(decode_only) >= warm // 2 + a.steps:
                break
    torch.cuda.synchronize()
    prof = native.profile_end() if (ranged and a.profile) else None
    if ranged:
        torch.cuda.nvtx.range_pop()
    for _ in range(8):  # retire the last timed batches (their device times are read at retirement)
        if not eng.step():
            break
    torch.cuda.synchronize()
    dev = ex.batch_device_ms()
    ms = [dev[s] for s in decode_only[warm // 2:] if s in dev]
    w_bytes = spec.n_layers * spec.params_per_layer * 2 + spec.vocab * spec.d_model * 2
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        hbm = 6650.0
    # every decode also reads its KV cache: batch x context (mid-window) x layers x KV bytes
    ctx_mid = a.ctx + pf_iters // 2 + warm // 2 + a.steps // 2
    kv_bytes = a.batch * ctx_mid * spec.n_layers * spec.kv_bytes_per_token_layer
    floor_ms = (w_bytes + kv_bytes) / (hbm * 1e9) * 1e3
    med = statistics.median(ms)
    # host wall time per decode step through the engine (planning, packing, launches, token read-back)
    gaps = [b - a_ for a_, b in zip(wall[warm // 2:], wall[warm // 2 + 1:])]
    wall_ms = statistics.median(gaps) * 1e3 if gaps else None
    print(json.dumps({"model": a.model, "batch": a.batch, "ctx": a.ctx, "cuda_graphs": a.cuda_graphs,
                      "graph_replays": ex.graph_replays, "steps": len(ms), "ms_per_step": round(med, 3),
                      "wall_ms_per_step": round(wall_ms, 3) if wall_ms else None,
                      "floor_ms": round(floor_ms, 3), "kv_gb": round(kv_bytes / 1e9, 2),
                      "frac_of_floor": round(floor_ms / med, 3)}))
    if prof:
        n = max(1, len(decode_only) - warm // 2)
        for name, e in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"]):
            us = e["total_ms"] * 1e3 / max(1, e["launches"])
            gbs = e["bytes"] / (e["total_ms"] * 1e6) if e["total_ms"] else 0.0
            print(f"  {name:14s} {e['total_ms'] / n:7.3f} ms/step  {e['launches'] // n:4d} launches/step  "
                  f"{us:8.1f} us/launch  {gbs:7.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
