"""Request-rate sweep of the wall-clock serving path on one B200 (BASELINE config 3: rate sweep).

    python tools/sweep.py --model qwen2.5-14b --rates 4,16,64 --n-requests 300 \
        [--scheduler throttle|sarathi] [--out profiles/r1b_sweep_c3.csv]
        [--trace-file trace.jsonl|azure.csv]   # replay a recorded trace, arrivals resampled per rate

For each rate: the same ShareGPT-like trace (`workload.py:27-38`, lengths seed 1) with
Poisson(rate, seed 0) arrivals is served end to end by `ServingEngine` (Token Throttling
T=8 / MaxP=2048 / MinP=32 / thr=0.05, page 16) on real weights (random init). Reported per
rate: output tokens/s over the run, p50 and mean TTFT / TPOT, GPU idle fraction (the
bubble of the single stage, `engine.py:108-125` on CUDA-event busy intervals).

Next to each measured row, the reference's cost model is fitted to this run's measured
micro-batch times (`calibration.fit_stage_cost`) and the virtual-clock
engine (the reference's event loop, bit-exact with `tokensim`) replays the same trace with
it: the sim_* columns are what the reference simulator predicts once calibrated to B200.
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-14b")
    ap.add_argument("--rates", default="4,16,64")
    ap.add_argument("--n-requests", type=int, default=300)
    ap.add_argument("--scheduler", default="throttle", choices=["throttle", "sarathi"])
    ap.add_argument("--out", default="")
    ap.add_argument("--trace-file", default="", help="JSONL trace or Azure-style CSV; its first --n-requests "
                    "requests are replayed at each rate (Poisson arrivals, seed 0, as resample_rate_per_s)")
    a = ap.parse_args()

    import torch

    from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, ThrottleConfig, build_report
    from paper_2504_14775_b200.calibration import fit_stage_cost
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.serving import ServingEngine
    from paper_2504_14775_b200.workload import (ArrivalProcess, builtin_length_table, load_azure_trace, load_trace,
                                                resample_arrivals, synthesize_requests)

    spec = MODELS[a.model]
    rates = [float(r) for r in a.rates.split(",")]
    dist = builtin_length_table("sharegpt-like")
    if a.trace_file:
        rec = (load_azure_trace if a.trace_file.endswith(".csv") else load_trace)(a.trace_file)[:a.n_requests]
        rec = [dataclasses.replace(q, id=i) for i, q in enumerate(rec)]  # ids 0..n-1 in arrival order
        traces = {r: resample_arrivals(rec, r, 0) for r in rates}
    else:
        traces = {r: synthesize_requests(ArrivalProcess.poisson(r, 0), dist, a.n_requests) for r in rates}
    base = traces[rates[0]]   # lengths are identical across rates (length seed = arrival seed + 1)
    page = 16
    need_pages = sum(-(-(q.input_tokens + q.output_tokens) // page) for q in base)
    max_tokens = (2048 + a.n_requests + 255) // 256 * 256
    free, _ = torch.cuda.mem_get_info()
    w_bytes = spec.n_layers * spec.params_per_layer * 2 + 2 * spec.vocab * spec.d_model * 2
    page_bytes = spec.n_layers * spec.kv_bytes_per_token_layer * page
    fit = int((free - w_bytes - max_tokens * (6 * spec.d_model + 3 * spec.qkv_width + 6 * spec.d_ff) * 2
               - a.n_requests * spec.vocab * 2 - (8 << 30)) // page_bytes)
    num_pages = max(1024, min(need_pages, fit))
    ex = LocalExecutor(spec, base, num_pages=num_pages, page_size=page, max_tokens=max_tokens,
                       max_emit=a.n_requests, seed=0)
    rows = []
    for r in rates:
        reqs = traces[r]
        ex.outputs.clear()
        ex.timings.clear()
        eng = ServingEngine(reqs, scheduler=a.scheduler, pipeline=PipelineConfig(depth=1),
                            kv_config=KvConfig(num_pages, page), throttle=ThrottleConfig(), executor=ex,
                            lookahead=True)
        t0 = time.perf_counter()
        raw = eng.run()
        wall = time.perf_counter() - t0
        rep = build_report(raw)
        dev = ex.batch_device_ms()
        its = {it.batch_seq: it for it in raw.iterations}
        seqs = [s for s in dev if s in its and s in eng._ctx_log]
        model, diag = fit_stage_cost([its[s].total_tokens for s in seqs], [eng._ctx_log[s] for s in seqs],
                                     [dev[s] for s in seqs])
        sim = build_report(Engine(reqs, scheduler=a.scheduler, pipeline=PipelineConfig(depth=1, cost=model),
                                  kv_config=KvConfig(num_pages, page), throttle=ThrottleConfig()).run())
        row = {"model": a.model, "pp": 1, "scheduler": a.scheduler, "rate_per_s": r, "n_requests": len(reqs),
               "finished": rep.finished_requests, "output_tok_s": rep.output_tokens_per_s,
               "p50_ttft_ms": rep.ttft_p50_ms, "p50_tpot_ms": rep.tpot_p50_ms,
               "mean_ttft_ms": rep.ttft_mean_ms, "mean_tpot_ms": rep.tpot_mean_ms,
               "gpu_idle_frac": rep.bubble_mean, "iterations": len(raw.iterations),
               "token_stddev": rep.token_stddev, "preemptions": rep.preemptions, "wall_s": round(wall, 2),
               "fit_c0": model.c0, "fit_c_tok": model.c_tok, "fit_c_ctx": model.c_ctx, "fit_r2": diag["r2"],
               "sim_p50_ttft_ms": sim.ttft_p50_ms, "sim_p50_tpot_ms": sim.tpot_p50_ms,
               "sim_output_tok_s": sim.output_tokens_per_s, "sim_idle_frac": sim.bubble_mean}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(rows[0]))
            w.writeheader()
            for row in rows:
                w.writerow({k: (f"{v:.6g}" if isinstance(v, float) else v) for k, v in row.items()})
    return 0


if __name__ == "__main__":
    sys.exit(main())
