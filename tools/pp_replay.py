"""PP=N serving on ONE B200 by measured-time replay (BASELINE configs 3-5 and the C4 ablation).

    python tools/pp_replay.py --model qwen2.5-32b --pp 4 --rates 8,16,32 --schedulers throttle,sarathi \
        [--trace sharegpt|c5] [--n-requests 1000] [--out profiles/r2/pp_replay_c4.jsonl]

What it measures. The whole trace is served by the virtual-clock `Engine` (the reference's event
loop, `engine.py:265-330`: in-order stage admission, depth-gated scheduling, last-stage commit)
with `measured_stage_times=True`: every micro-batch really runs on the GPU, stage by stage
(ceil(L/PP) layers each, `stage_layers`), and each stage's duration in the pipeline timeline is
that stage's CUDA-event device time for that micro-batch, not the cost model. Only the
inter-stage hop is modelled (`CommModel`: latency + N_tok * d * 2 B / bandwidth, the NVLink
send/recv of the activations). Stages execute one at a time on one GPU (the host waits for each
micro-batch), so each stage's time is measured without contention, as on its own GPU of a PP=N
box; the host enqueue is hidden behind a GPU sleep so launch gaps are not timed.

Differences from a real PP=N box, stated on every row: (1) the KV pool is what fits next to
ALL stages' weights on this one GPU (a real box has N x the HBM); (2) the hops are modelled;
(3) host scheduling time is not on the timeline (the reference's simulator convention).

Reported per (scheduler, rate): whole-trace output tokens/s (finished output tokens / (last
completion - first arrival), `metrics.output_throughput`), p50/mean TTFT and TPOT, per-stage
bubble over [0, makespan] (`engine.py:108-125`), per-iteration token stddev (the paper's
balance metric), preemptions, and the trace hash (both schedulers serve the identical trace).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def trace_hash(reqs) -> str:
    h = hashlib.sha256()
    for r in reqs:
        h.update(f"{r.id},{r.arrival_ms!r},{r.input_tokens},{r.output_tokens};".encode())
    return h.hexdigest()[:16]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-32b")
    ap.add_argument("--pp", type=int, default=4)
    ap.add_argument("--rates", default="8,16,32")
    ap.add_argument("--schedulers", default="throttle,sarathi")
    ap.add_argument("--trace", default="sharegpt", choices=["sharegpt", "c5", "azure"])
    ap.add_argument("--n-requests", type=int, default=1000)
    ap.add_argument("--hop-latency-ms", type=float, default=0.02)
    ap.add_argument("--hop-gbs", type=float, default=400.0, help="effective NVLink send/recv GB/s per hop")
    ap.add_argument("--layers", type=int, default=0, help="test only: truncate the model")
    ap.add_argument("--max-pages", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--max-wall-s", type=float, default=0.0,
                    help="stop a run cleanly after this much host time (the row is marked truncated)")
    a = ap.parse_args()

    import torch

    from paper_2504_14775_b200 import (CommModel, Engine, KvConfig, PipelineConfig, ThrottleConfig,
                                       build_report)
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.workload import (ArrivalProcess, LengthDistribution, builtin_length_table,
                                                synthesize_requests)

    spec = MODELS[a.model]
    if a.layers:
        spec = spec.with_layers(a.layers)
    if a.trace == "c5":
        dist = LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)])
    else:
        dist = builtin_length_table("azure-like" if a.trace == "azure" else "sharegpt-like")
    rates = [float(r) for r in a.rates.split(",")]
    traces = {r: synthesize_requests(ArrivalProcess.poisson(r, 0), dist, a.n_requests) for r in rates}
    base = traces[rates[0]]
    page = 16
    need = sum(-(-(q.input_tokens + q.output_tokens) // page) for q in base)
    max_tokens = (2048 + a.n_requests + 255) // 256 * 256
    free, _ = torch.cuda.mem_get_info()
    w_bytes = spec.n_layers * spec.params_per_layer * 2 + 2 * spec.vocab * spec.d_model * 2
    page_bytes = spec.n_layers * spec.kv_bytes_per_token_layer * page
    ws = a.pp * max_tokens * (6 * spec.d_model + 3 * spec.qkv_width + 6 * spec.d_ff) * 2
    fit = int((free - w_bytes - ws - a.n_requests * spec.vocab * 2 - (8 << 30)) // page_bytes)
    num_pages = max(1024, min(need, fit))
    if a.max_pages:
        num_pages = min(num_pages, a.max_pages)

    class ReplayExecutor(LocalExecutor):
        """LocalExecutor whose launch first parks the stream in a GPU sleep, so the host's kernel
        enqueue for the micro-batch finishes before the first stage's start event fires."""

        def launch(self, meta) -> None:
            with torch.cuda.stream(self.stream):
                torch.cuda._sleep(4_000_000)
            super().launch(meta)

    ex = ReplayExecutor(spec, base, num_pages=num_pages, page_size=page, n_stages=a.pp,
                        max_tokens=max_tokens, max_emit=a.n_requests, seed=0)
    comm = CommModel(a.hop_latency_ms, spec.d_model * 2.0, a.hop_gbs * 1e6)
    rows = []
    for sched in a.schedulers.split(","):
        for r in rates:
            reqs = traces[r]
            ex.outputs.clear()
            ex.timings.clear()
            eng = Engine(reqs, scheduler=sched, pipeline=PipelineConfig(depth=a.pp, comm=comm),
                         kv_config=KvConfig(num_pages, page), throttle=ThrottleConfig(), executor=ex,
                         measured_stage_times=True)
            t0 = time.perf_counter()
            truncated = False
            if a.max_wall_s:
                while eng.step():
                    if time.perf_counter() - t0 > a.max_wall_s:
                        truncated = True
                        break
                torch.cuda.synchronize()
                raw = eng.raw_data()
            else:
                raw = eng.run()
            wall = time.perf_counter() - t0
            rep = build_report(raw)
            stage_busy = [sum(b - s for s, b in ivs) for ivs in raw.busy_intervals]
            row = {"model": a.model + (f"[{a.layers} layers]" if a.layers else ""), "pp": a.pp,
                   "scheduler": sched, "token_budget": 2048 if sched == "sarathi" else None,
                   "throttle": "T=8 MaxP=2048 MinP=32 thr=0.05", "trace": a.trace, "rate_per_s": r,
                   "n_requests": len(reqs), "trace_hash": trace_hash(reqs),
                   "finished": rep.finished_requests, "output_tok_s": rep.output_tokens_per_s,
                   "p50_ttft_ms": rep.ttft_p50_ms, "p50_tpot_ms": rep.tpot_p50_ms,
                   "mean_ttft_ms": rep.ttft_mean_ms, "mean_tpot_ms": rep.tpot_mean_ms,
                   "bubble_per_stage": [round(x, 4) for x in rep.bubble_fractions],
                   "bubble_mean": rep.bubble_mean, "token_mean": rep.token_mean,
                   "token_stddev": rep.token_stddev, "iterations": len(raw.iterations),
                   "preemptions": rep.preemptions, "makespan_ms": rep.makespan_ms,
                   "stage_busy_ms": [round(x, 1) for x in stage_busy], "kv_pages": num_pages,
                   "hop": f"modelled {a.hop_latency_ms} ms + N_tok*{spec.d_model * 2} B / {a.hop_gbs} GB/s",
                   "method": "measured-time replay on 1 B200: every stage executed and CUDA-event timed; "
                             "pipeline timeline = reference event loop over the measured stage times",
                   "host_wall_s": round(wall, 1), "truncated": truncated}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "a") as fh:
            for row in rows:
                fh.write(json.dumps(row) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
