"""Benchmark: output tokens/s of the per-iteration serving path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE config 2 — Llama-3-8B-shaped random-init bf16, PP=1 on
one B200, ShareGPT-like lengths (`workload.py:27-38`) with Poisson arrivals,
Token Throttling T=8 / MaxP=2048 / MinP=32 / KV_thresh=0.05, page size 16.
A "step" is one engine iteration: schedule -> KV apply -> metadata -> stage
forward -> argmax -> commit. Before the W warm-up steps the engine is warmed
in (untimed) until the decode population reaches steady state, so the K timed
steps measure the saturated serving regime.

Reported (one JSON line on rank 0):
  value       output tokens / sum of device time of the K micro-batches
              (CUDA events on the launch stream; metadata already in HBM)
  e2e         same tokens / wall time of the K steps through the public API
              (host scheduling + pinned H2D metadata + forward + D2H tokens); the
              serving loop plans batch i+1 while batch i runs (lookahead, serving.py)
  roofline    dominant kernel class from a profiled pass (native CUDA-event profiler)
  cpu_baseline the oracle CPU port (oracle/cpu_path.py) on this host
With N>1 under torchrun the stages are split across ranks (PP=N, pipeline.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="llama3-8b")
    p.add_argument("--n-requests", type=int, default=2000)
    p.add_argument("--rate", type=float, default=2000.0, help="Poisson arrivals per second")
    p.add_argument("--scheduler", default="throttle", choices=["throttle", "sarathi"])
    p.add_argument("--trace", default="sharegpt", choices=["sharegpt", "azure", "c5"],
                   help="length distribution: ShareGPT-like (C2-C4), Azure-like, or C5 long prompts (4-8k)")
    p.add_argument("--warm-decodes", type=int, default=1024, help="untimed warm-in until this many decodes run")
    p.add_argument("--warm-max-iters", type=int, default=400)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-profile", action="store_true")
    p.add_argument("--cpu-sample-layers", type=int, default=2)
    p.add_argument("--no-lookahead", action="store_true", help="wait for each commit before planning the next batch")
    p.add_argument("--report-dir", default="", help="write report.json / requests.csv / iterations.csv of the GPU run")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        self.file.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.file:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.file.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_trace(args):
    from paper_2504_14775_b200.workload import (ArrivalProcess, LengthDistribution, builtin_length_table,
                                                synthesize_requests)
    if args.trace == "c5":   # prompts 4096..8192 step 128, outputs 100..500
        dist = LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)])
    else:
        dist = builtin_length_table("azure-like" if args.trace == "azure" else "sharegpt-like")
    return synthesize_requests(ArrivalProcess.poisson(args.rate, 0), dist, args.n_requests)


def roofline(profile: dict, peaks: dict) -> dict:
    """Dominant kernel class by total device time; bound from its algorithmic intensity."""
    name, e = max(profile.items(), key=lambda kv: kv[1]["total_ms"])
    per_launch_ms = e["total_ms"] / e["launches"]
    ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    intensity = e["flops"] / e["bytes"] if e["bytes"] else float("inf")
    if e["flops"] > 0 and intensity >= ridge:
        achieved = e["flops"] / e["launches"] / (per_launch_ms * 1e-3) / 1e12
        peak = peaks["bf16_tflops_sustained"]
        out = {"bound": "tensor", "unit": "TFLOP/s", "algorithmic_per_launch": e["flops"] / e["launches"]}
    else:
        achieved = e["bytes"] / e["launches"] / (per_launch_ms * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        out = {"bound": "hbm", "unit": "GB/s", "algorithmic_per_launch": e["bytes"] / e["launches"]}
    traffic, traffic_src = None, None
    try:  # DRAM bytes per launch of this kernel class from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            t = json.load(fh).get(name)
        if t:
            traffic = t["dram_bytes_per_launch"]
            traffic_src = f"profiles/ncu_traffic.json ({t['shape']})"
    except OSError:
        pass
    # both resources at once: a class mixing bandwidth- and compute-bound work (the attention call
    # runs decode and prefill launches concurrently) is judged against bytes/HBM + FLOPs/tensor
    t_ideal = e["bytes"] / (peaks["hbm_gbs"] * 1e9) + e["flops"] / (peaks["bf16_tflops_sustained"] * 1e12)
    out["frac_bytes_plus_flops"] = round(t_ideal / (e["total_ms"] * 1e-3), 4)
    out.update({"kernel": name, "achieved": round(achieved, 2), "peak": peak, "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_src": traffic_src, "launches": e["launches"],
                "avg_launch_ms": round(per_launch_ms, 4),
                "peak_src": peaks["src"] + (" sustained" if out["bound"] == "tensor" else "")})
    return out


def run_ours(args):
    import torch

    from paper_2504_14775_b200 import KvConfig, PipelineConfig, ThrottleConfig, build_report, native
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.serving import ServingEngine

    spec = MODELS[args.model]
    reqs = make_trace(args)
    page_size = 16
    max_tokens = 2048 + args.n_requests
    max_tokens = (max_tokens + 255) // 256 * 256
    # KV pool: what the trace could ever need, capped by free HBM after weights + workspace (8 GB slack).
    need_pages = sum(-(-(r.input_tokens + r.output_tokens) // page_size) for r in reqs)
    weight_bytes = spec.n_layers * spec.params_per_layer * 2 + 2 * spec.vocab * spec.d_model * 2
    free, _ = torch.cuda.mem_get_info()
    page_bytes = spec.n_layers * spec.kv_bytes_per_token_layer * page_size
    ws_guess = max_tokens * (6 * spec.d_model + 3 * spec.qkv_width + 6 * spec.d_ff) * 2 + args.n_requests * spec.vocab * 2
    fit_pages = int((free - weight_bytes - ws_guess - (8 << 30)) // page_bytes)
    num_pages = max(1024, min(need_pages, fit_pages))
    t_init = time.time()
    ex = LocalExecutor(spec, reqs, num_pages=num_pages, page_size=page_size, max_tokens=max_tokens,
                       max_emit=args.n_requests, seed=0)
    torch.cuda.synchronize()
    init_s = time.time() - t_init
    eng = ServingEngine(reqs, scheduler=args.scheduler, pipeline=PipelineConfig(depth=1),
                        kv_config=KvConfig(num_pages, page_size), throttle=ThrottleConfig(), executor=ex,
                        lookahead=not args.no_lookahead)

    state = {"phase": "warm", "timed_start": None, "timed": [], "commits": 0, "stop": False,
             "warm_iters": 0, "launch0": 0}
    clocks = ClockSampler()
    W, K = args.warmup, args.steps

    def on_commit(seq, t, n_out):
        st = state
        if st["phase"] == "warm":
            st["warm_iters"] += 1
            if eng._rd >= args.warm_decodes or st["warm_iters"] >= args.warm_max_iters:
                st["phase"], st["count"] = "warmup", 0
                clocks.start()   # sampler running before (and throughout) the timed region
            return
        if st["phase"] == "warmup":
            st["count"] += 1
            if st["count"] >= W:
                # timed region starts here: drain the device (with lookahead one batch is already
                # queued; its commit is skipped below so only batches launched after t0 count)
                torch.cuda.synchronize()
                st["phase"] = "timed"
                st["skip"] = 0 if args.no_lookahead else 1
                st["timed_start"] = time.perf_counter()
                st["t_engine"] = t
                st["launch0"] = native.launch_count()
                torch.cuda.nvtx.range_push("bench_timed")   # ncu --nvtx --nvtx-include bench_timed/
            return
        if st["phase"] == "timed":
            if st["skip"]:
                st["skip"] -= 1
                return
            st["timed"].append((seq, t, n_out))
            if len(st["timed"]) >= K:
                # the K-th timed batch is complete (its commit waited on its event); read the clock
                # before synchronizing, which would also wait for the next, untimed, queued batch
                st["timed_end"] = time.perf_counter()
                st["launch1"] = native.launch_count()
                torch.cuda.synchronize()
                torch.cuda.nvtx.range_pop()
                st["clocks"] = clocks.stop()
                st["phase"] = "profile"
                if args.no_profile:
                    st["stop"] = True
                    return
                native.profile_begin()
                st["pcount"] = 0
            return
        if st["phase"] == "profile":
            st["pcount"] += 1
            if st["pcount"] >= max(3, min(K, 10)):
                torch.cuda.synchronize()
                st["profile"] = native.profile_end()
                st["stop"] = True

    class _Stop(Exception):
        pass

    def hook(seq, t, n_out):
        on_commit(seq, t, n_out)
        if state["stop"]:
            raise _Stop

    try:
        eng.run(on_commit=hook)
    except _Stop:
        ex.synchronize()
        eng._busy = ex.stage_busy_intervals()
        eng.makespan_ms = eng.now_ms()
    timed = state["timed"]
    if len(timed) < K:
        raise RuntimeError(f"trace exhausted before {K} timed steps (got {len(timed)})")
    dev_ms = ex.batch_device_ms()
    out_tokens = sum(n for _, _, n in timed)
    device_s = sum(dev_ms[s] for s, _, _ in timed) / 1000.0
    wall_s = state["timed_end"] - state["timed_start"]
    tokens_per_step = [eng._iters[s].prefill_tokens + eng._iters[s].decode_tokens for s, _, _ in timed]
    raw = eng.raw_data()
    rep = build_report(raw)
    res = {
        "value": out_tokens / device_s, "wall_s": wall_s, "device_s": device_s, "out_tokens": out_tokens,
        "e2e": out_tokens / wall_s, "tokens_per_step": statistics.mean(tokens_per_step),
        "decodes_per_step": statistics.mean(eng._iters[s].decode_tokens for s, _, _ in timed),
        "init_s": init_s, "num_pages": num_pages, "warm_iters": state["warm_iters"],
        "launches": state["launch1"] - state["launch0"], "clocks": state["clocks"],
        "profile": state.get("profile"), "report": rep, "bubble": raw.bubble_fractions(),
        "h2d_bytes_per_step": ex.h2d_bytes_total_for([s for s, _, _ in timed]) / K,
        "d2h_bytes_per_step": 4.0 * out_tokens / K,
    }
    # cost-model calibration: fit the reference StageCostModel to measured stages
    from paper_2504_14775_b200.calibration import fit_stage_cost
    its = {it.batch_seq: it for it in raw.iterations}
    seqs = [s for s in dev_ms if s in its and s in eng._ctx_log]
    if len(seqs) >= 3:
        model, diag = fit_stage_cost([its[s].total_tokens for s in seqs], [eng._ctx_log[s] for s in seqs],
                                     [dev_ms[s] for s in seqs])
        res["calibration"] = {"c0": model.c0, "c_tok": model.c_tok, "c_ctx": model.c_ctx, **diag}
    if args.report_dir:
        from paper_2504_14775_b200.metrics import write_report
        write_report(rep, args.report_dir, extended=True)
    return res, spec


def cpu_baseline(args, spec):
    from oracle.cpu_path import run_cpu_path
    from paper_2504_14775_b200.workload import ArrivalProcess, builtin_length_table, synthesize_requests
    reqs = make_trace(args)
    return run_cpu_path(spec, reqs, steps=3, warmup=1, sample_layers=args.cpu_sample_layers, time_budget_s=60.0,
                        warm_decodes=args.warm_decodes, warm_max_iters=args.warm_max_iters)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return 0
        from paper_2504_14775_b200.modelspec import MODELS
        from oracle.cpu_path import run_cpu_path
        spec = MODELS[args.model]
        reqs = make_trace(args)
        r = run_cpu_path(spec, reqs, steps=args.steps, warmup=args.warmup, sample_layers=args.cpu_sample_layers,
                         time_budget_s=240.0, warm_decodes=args.warm_decodes, warm_max_iters=args.warm_max_iters)
        line = {"metric": "output_tokens_per_s", "value": r["value"], "unit": "tokens/s", "n_gpus": 0,
                "steps": r["steps"], "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"C2: {args.model} random-init, ShareGPT-like, Poisson {args.rate}/s, "
                                       f"{args.n_requests} requests, Token Throttling T=8", "parallelism": "cpu"},
                "cpu_baseline": {"value": r["value"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
                                 "sample": r["sample"]},
                "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "vs_baseline": None}
        print(json.dumps(line))
        return 0
    if world > 1:
        from paper_2504_14775_b200.pipeline import bench_pipeline
        return bench_pipeline(args)
    res, spec = run_ours(args)
    peaks = load_peaks()
    rl = roofline(res["profile"], peaks) if res["profile"] else None
    cpu = None
    if not args.no_cpu_baseline:
        c = cpu_baseline(args, spec)
        cpu = {"value": c["value"], "unit": "tokens/s", "cores": c["threads"], "kind": "port", "sample": c["sample"]}
    rep = res["report"]
    K = args.steps
    line = {
        "metric": "output_tokens_per_s", "value": round(res["value"], 2), "unit": "tokens/s", "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(res["wall_s"] * 1000 / K, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, seeded ShareGPT-like trace, PCG64 prompt tokens)",
        "config": {"workload": f"{'C2: ' if args.model == 'llama3-8b' and args.trace == 'sharegpt' else ''}"
                               f"{args.model} PP=1 on 1xB200, {args.trace} lengths, Poisson {args.rate}/s x "
                               f"{args.n_requests} requests, {args.scheduler} T=8 MaxP=2048 MinP=32 thr=0.05",
                   "model": args.model, "parallelism": "pp1", "page_size": 16, "kv_pages": res["num_pages"],
                   "tokens_per_step": round(res["tokens_per_step"], 1),
                   "decodes_per_step": round(res["decodes_per_step"], 1),
                   "l2": "inputs larger than L2 (16 GB of weights streamed per step)"},
        "e2e": {"value": round(res["e2e"], 2), "unit": "tokens/s",
                "h2d_bytes_per_step": int(res["h2d_bytes_per_step"]), "d2h_bytes_per_step": int(res["d2h_bytes_per_step"])},
        "gpu_launches": res["launches"],
        "roofline": rl,
        "cpu_baseline": cpu,
        "clocks": res["clocks"],
        "serving": {"p50_ttft_ms": rep.ttft_p50_ms, "p50_tpot_ms": rep.tpot_p50_ms,
                    "bubble_frac": res["bubble"], "finished": rep.finished_requests,
                    "token_stddev_per_iter": rep.token_stddev, "token_mean_per_iter": rep.token_mean,
                    "note": "latency stats over requests finished during the run (overloaded arrival rate)"},
        "profile": {k: {"launches": v["launches"], "ms": round(v["total_ms"], 3)} for k, v in (res["profile"] or {}).items()},
        "calibration": res.get("calibration"),
    }
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
