"""Generate the committed golden fixtures from the REFERENCE implementation.

Run in the build container only (the reference tree is not on the GPU box):

    python tests/golden/make_golden.py

It imports `tokensim` read-only from /root/reference/pkg/src and writes
small JSON(.gz) fixtures under tests/golden/. The fixtures pin:

* the four throttling equations on 10k seeded draws plus the reference's own
  hand examples (`pkg/tests/test_sched.py:41-106`, `test_acceptance.py:88-119`);
* planner outputs (`plan_throttled` / `plan_sarathi`) on random queues;
* KV accounting sequences (`kvcache.py:46-109`);
* workload synthesis (`workload.py:155-229`) for the bench configs;
* full engine timelines (`engine.py`) for the C1 trace at depth 1/2/4,
  the committed bursty fixture under the acceptance settings
  (`test_acceptance.py:73-82`), memory-pressure runs, the tick-simulator
  scenarios, and the 100 conservation runs of criterion 8 (as digests).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)

import tokensim as ts  # noqa: E402
from tokensim.engine import CommModel, Engine, PipelineConfig, StageCostModel  # noqa: E402
from tokensim.errors import UnschedulableError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    data = json.dumps(obj, separators=(",", ":"), sort_keys=True).encode()
    if name.endswith(".gz"):
        with gzip.GzipFile(path, "wb", mtime=0) as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)
    print(f"wrote {path} ({len(data)} bytes raw)")


def formulas():
    rng = np.random.Generator(np.random.PCG64(11))
    thresholds = (0.0, 0.05, 0.1, 0.25, 0.5)
    rows = []
    for _ in range(10_000):
        wp = int(rng.integers(0, 1_000_001))
        T = int(rng.integers(1, 65))
        min_p = int(rng.integers(1, 4097))
        max_p = min_p + int(rng.integers(0, 100_001))
        total = int(rng.integers(1, 100_001))
        free = int(rng.integers(0, total + 1))
        thresh = thresholds[int(rng.integers(0, len(thresholds)))]
        rd = int(rng.integers(0, 1_000_001))
        depth = int(rng.integers(1, 65))
        mode = ("combined", "wt_only", "ut_only")[int(rng.integers(0, 3))]
        cfg = ts.ThrottleConfig(T=T, max_p=max_p, min_p=min_p, kv_thresh=thresh, mode=mode)
        kv_free = free / total
        inputs = ts.SchedInputs(wp, rd, kv_free, depth)
        from tokensim.sched import _prefill_token_limit
        rows.append([wp, T, min_p, max_p, free, total, thresh, rd, depth, mode,
                     ts.throttle_prefill_wt(wp, cfg), ts.throttle_prefill_ut(kv_free, cfg),
                     ts.throttle_prefill_combined(wp, kv_free, cfg), ts.throttle_decode(rd, depth),
                     _prefill_token_limit(inputs, cfg)])
    # Dense sweep around exact-integer boundaries of Eq. 2/3 (the 1e-9 guard).
    for total in (20, 40, 64, 100, 1000, 4096):
        for free in range(total + 1):
            for thresh in (0.0, 0.05, 0.25):
                cfg = ts.ThrottleConfig(T=8, max_p=2048, min_p=32, kv_thresh=thresh)
                kv_free = free / total
                for wp in (1, 31, 33, 1000, 16384, 100000):
                    inputs = ts.SchedInputs(wp, 0, kv_free, 4)
                    from tokensim.sched import _prefill_token_limit
                    rows.append([wp, 8, 32, 2048, free, total, thresh, 0, 4, "combined",
                                 ts.throttle_prefill_wt(wp, cfg), ts.throttle_prefill_ut(kv_free, cfg),
                                 ts.throttle_prefill_combined(wp, kv_free, cfg), 0,
                                 _prefill_token_limit(inputs, cfg)])
    dump("formulas.json.gz", {"columns": ["wp", "T", "min_p", "max_p", "free", "total", "thresh", "rd",
                                          "depth", "mode", "wt", "ut", "combined", "decode", "limit"],
                              "rows": rows})


def plans():
    rng = np.random.Generator(np.random.PCG64(23))
    cases = []
    for i in range(3000):
        ps = int(rng.choice([1, 4, 16]))
        total = int(rng.integers(1, 400))
        free = int(rng.integers(0, total + 1))
        n_pf = int(rng.integers(0, 8))
        n_dec = int(rng.integers(0, 12))
        ids = rng.permutation(200)[: n_pf + n_dec].tolist()
        pq = [ts.PrefillCandidate(int(ids[k]), int(rng.integers(0, 600)), int(rng.integers(0, 300)))
              for k in range(n_pf)]
        dq = [ts.DecodeCandidate(int(ids[n_pf + k]), int(rng.integers(0, 500))) for k in range(n_dec)]
        wp = sum(max(c.remaining_tokens, 0) for c in pq) + int(rng.integers(0, 50))
        rd = n_dec + int(rng.integers(0, 20))
        depth = int(rng.choice([1, 2, 4, 8]))
        mode = ("combined", "wt_only", "ut_only")[i % 3]
        min_p = int(rng.choice([1, 8, 32]))
        cfg = ts.ThrottleConfig(T=int(rng.choice([1, 4, 8, 16])), max_p=int(rng.choice([min_p, 64, 2048])),
                                min_p=min_p, kv_thresh=float(rng.choice([0.0, 0.05, 0.3])), mode=mode)
        inputs = ts.SchedInputs(wp, rd, free / total, depth)
        view = ts.KvView(free, total, ps)
        budget = int(rng.choice([1, 16, 256, 2048]))
        pt = ts.plan_throttled(inputs, pq, dq, view, cfg)
        pS = ts.plan_sarathi(inputs, pq, dq, view, budget)
        cases.append({
            "inputs": [wp, rd, free, total, depth], "ps": ps,
            "cfg": [cfg.T, cfg.max_p, cfg.min_p, cfg.kv_thresh, cfg.mode], "budget": budget,
            "pq": [[c.id, c.remaining_tokens, c.stored_tokens] for c in pq],
            "dq": [[c.id, c.stored_tokens] for c in dq],
            "throttled": [pt.decode_ids, [list(x) for x in pt.prefill_chunks], pt.decode_context_tokens],
            "sarathi": [pS.decode_ids, [list(x) for x in pS.prefill_chunks], pS.decode_context_tokens],
        })
    dump("plans.json.gz", cases)


def kv_ops():
    rng = np.random.Generator(np.random.PCG64(31))
    seqs = []
    for _ in range(200):
        total = int(rng.integers(1, 64))
        ps = int(rng.choice([1, 3, 16]))
        kv = ts.KvCacheState(ts.KvConfig(total, ps))
        ops = []
        for _ in range(60):
            rid = int(rng.integers(0, 6))
            if rng.random() < 0.75:
                n = int(rng.integers(0, 40))
                ok = kv.allocate(rid, n)
                ops.append(["a", rid, n, ok, kv.free_pages, kv.stored_tokens(rid), kv.pages(rid)])
            else:
                try:
                    got = kv.release(rid)
                except KeyError:
                    got = None
                ops.append(["r", rid, got, kv.free_pages])
        seqs.append({"total": total, "ps": ps, "ops": ops})
    victims = []
    for _ in range(300):
        n = int(rng.integers(0, 6))
        cands = [(int(rng.integers(0, 20)), float(rng.integers(0, 5))) for _ in range(n)]
        victims.append([cands, ts.select_preemption_victim(cands)])
    dump("kv_ops.json.gz", {"sequences": seqs, "victims": victims})


def traces():
    out = {}
    specs = {
        "c1": (ts.ArrivalProcess.poisson(16.0, 0),
               ts.LengthDistribution.empirical([(i, 64) for i in range(128, 513)]), 64),
        "c2_rate32": (ts.ArrivalProcess.poisson(32.0, 0), ts.builtin_length_table("sharegpt-like"), 1000),
        "azure_rate4": (ts.ArrivalProcess.poisson(4.0, 3), ts.builtin_length_table("azure-like"), 200),
        "c5": (ts.ArrivalProcess.poisson(2.0, 0),
               ts.LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)]), 200),
        "lognormal": (ts.ArrivalProcess.poisson(40.0, 5),
                      ts.LengthDistribution.lognormal(60.0, 0.7, 15.0, 0.6, min_tokens=1, max_tokens=600), 300),
    }
    for name, (proc, dist, n) in specs.items():
        reqs = ts.synthesize_requests(proc, dist, n)
        out[name] = [[r.arrival_ms, r.input_tokens, r.output_tokens] for r in reqs]
    dump("traces.json.gz", out)


def timeline(raw) -> dict:
    return {
        "iterations": [[it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens] for it in raw.iterations],
        "requests": [[r.id, r.arrival_ms, r.first_token_ms, r.completion_ms, r.preemption_count] for r in raw.requests],
        "spans_sha": hashlib.sha256(json.dumps(raw.stage_spans).encode()).hexdigest(),
        "busy_sha": hashlib.sha256(json.dumps(raw.busy_intervals).encode()).hexdigest(),
        "makespan": raw.makespan_ms, "committed": raw.committed_tokens,
        "discarded": raw.discarded_tokens, "preemptions": raw.preemptions, "truncated": raw.truncated,
    }


def engine_runs():
    runs = []
    c1 = ts.synthesize_requests(ts.ArrivalProcess.poisson(16.0, 0),
                                ts.LengthDistribution.empirical([(i, 64) for i in range(128, 513)]), 64)
    for sched in ("throttle", "sarathi"):
        for depth in (1, 2, 4):
            raw = ts.run(c1, scheduler=sched, pipeline=PipelineConfig(depth=depth),
                         kv_config=ts.KvConfig(4096, 16), throttle=ts.ThrottleConfig())
            runs.append({"name": f"c1_{sched}_d{depth}", "trace": "c1", "scheduler": sched, "depth": depth,
                         "pages": 4096, "ps": 16, "T": 8, "thresh": 0.05, "budget": 2048,
                         "cost": [1.0, 0.01, 0.1], "comm": "default", "horizon": None, **timeline(raw)})
    bursty = ts.load_trace(os.path.join(REF_TESTS, "data", "bursty.jsonl"))
    b_trace = [[r.arrival_ms, r.input_tokens, r.output_tokens] for r in bursty]
    settings = [("throttle", 1024, 8, 0.05), ("sarathi", 1024, 8, 0.05), ("throttle", 192, 8, 0.0),
                ("throttle", 192, 8, 0.05), ("throttle", 1024, 1, 0.05), ("throttle", 1024, 4, 0.05),
                ("throttle", 1024, 16, 0.05)]  # sarathi at 192 pages livelocks (README:165-177)
    for sched, pages, T, thresh in settings:
        raw = ts.run(bursty, scheduler=sched,
                     pipeline=PipelineConfig(depth=4, cost=StageCostModel(), comm=CommModel.pcie()),
                     kv_config=ts.KvConfig(pages, 16), throttle=ts.ThrottleConfig(T=T, kv_thresh=thresh),
                     token_budget=2048)
        rep = ts.build_report(raw)
        runs.append({"name": f"bursty_{sched}_p{pages}_T{T}_th{thresh}", "trace": "bursty", "scheduler": sched,
                     "depth": 4, "pages": pages, "ps": 16, "T": T, "thresh": thresh, "budget": 2048,
                     "cost": [1.0, 0.01, 0.1], "comm": "pcie", "horizon": None,
                     "report": {"token_stddev": rep.token_stddev, "bubble_mean": rep.bubble_mean,
                                "ttft_mean_ms": rep.ttft_mean_ms, "tpot_mean_ms": rep.tpot_mean_ms},
                     **timeline(raw)})
    # a truncated (horizon) run
    raw = ts.run(bursty, scheduler="throttle", pipeline=PipelineConfig(depth=2),
                 kv_config=ts.KvConfig(1024, 16), horizon_ms=1500.0, record_events=True)
    runs.append({"name": "bursty_horizon", "trace": "bursty", "scheduler": "throttle", "depth": 2,
                 "pages": 1024, "ps": 16, "T": 8, "thresh": 0.05, "budget": 2048, "cost": [1.0, 0.01, 0.1],
                 "comm": "default", "horizon": 1500.0,
                 "events_sha": hashlib.sha256(json.dumps(raw.events).encode()).hexdigest(), **timeline(raw)})
    dump("engine_runs.json.gz", {"traces": {"bursty": b_trace}, "runs": runs})


def scenarios():
    """The tick-simulator scenarios of acceptance criterion 3 (seed PCG64(7)), engine outcome."""
    from oracle_sim import OracleLimit, random_scenario
    rng = np.random.Generator(np.random.PCG64(7))
    out = []
    tries = 0
    while len(out) < 60 and tries < 500:
        tries += 1
        scn = random_scenario(rng)
        try:
            tick = scn.tick()
        except OracleLimit:
            continue
        eng = scn.engine()
        stalled = []
        try:
            while eng.step():
                pass
        except UnschedulableError as exc:
            stalled = sorted(exc.request_ids)
        raw = eng.raw_data()
        out.append({
            "specs": [[r.id, r.arrival_ms, r.input_tokens, r.output_tokens] for r in scn.requests],
            "scheduler": scn.scheduler, "throttle": [scn.throttle.T, scn.throttle.max_p, scn.throttle.min_p,
                                                     scn.throttle.kv_thresh, scn.throttle.mode],
            "budget": scn.token_budget, "depth": scn.depth, "pages": scn.kv_config.total_pages,
            "ps": scn.kv_config.page_size, "c0": scn.c0, "c_tok": scn.c_tok, "c_ctx": scn.c_ctx,
            "latency": scn.latency, "stalled": stalled, "tick_stuck": list(tick.stuck),
            "spans": raw.stage_spans, **timeline(raw)})
    dump("scenarios.json.gz", out)


def conservation():
    """Criterion 8's 100 randomized runs (`test_acceptance.py:265-316`) as digests."""
    out = []
    for seed in range(100):
        n = 50 + (seed * 7) % 251
        depth = (1, 2, 4, 8)[seed % 4]
        sched = ("throttle", "sarathi")[seed % 2]
        pages = 64 if seed % 5 == 0 else 512
        reqs = ts.synthesize_requests(ts.ArrivalProcess.poisson(40.0, seed),
                                      ts.LengthDistribution.lognormal(60.0, 0.7, 15.0, 0.6, min_tokens=1, max_tokens=600), n)
        eng = Engine(reqs, scheduler=sched, pipeline=PipelineConfig(depth=depth, comm=CommModel.pcie()),
                     kv_config=ts.KvConfig(pages, 16), throttle=ts.ThrottleConfig())
        raw = eng.run()
        t = timeline(raw)
        out.append({"seed": seed, "n": n, "depth": depth, "scheduler": sched, "pages": pages,
                    "iters_sha": hashlib.sha256(json.dumps(t["iterations"]).encode()).hexdigest(),
                    "reqs_sha": hashlib.sha256(json.dumps(t["requests"]).encode()).hexdigest(),
                    "spans_sha": t["spans_sha"], "preemptions": raw.preemptions,
                    "committed": raw.committed_tokens, "discarded": raw.discarded_tokens})
    dump("conservation.json.gz", out)


def scale_runs():
    """C2-C5-scale timelines (digests): 1000-request ShareGPT-like traces at depth 1/2/4/8 for both
    schedulers, a 2048-page memory-pressure setting, and the C5 long-prompt trace at depth 8."""
    sg = ts.builtin_length_table("sharegpt-like")
    c5 = ts.LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)])
    cases = []
    for sched in ("throttle", "sarathi"):
        for depth in (1, 2, 4, 8):
            cases.append((f"c2_r32_{sched}_d{depth}", 32.0, "sharegpt", 1000, sched, depth, 16384))
        cases.append((f"c2_r64_{sched}_d4_p2048", 64.0, "sharegpt", 1000, sched, 4, 2048))
    cases.append(("c5_r2_throttle_d8", 2.0, "c5", 200, "throttle", 8, 16384))
    cases.append(("c5_r4_sarathi_d8_p4096", 4.0, "c5", 200, "sarathi", 8, 4096))
    out = []
    for name, rate, dist, n, sched, depth, pages in cases:
        reqs = ts.synthesize_requests(ts.ArrivalProcess.poisson(rate, 0), sg if dist == "sharegpt" else c5, n)
        tsha = hashlib.sha256(json.dumps([[r.arrival_ms, r.input_tokens, r.output_tokens]
                                          for r in reqs]).encode()).hexdigest()
        try:
            raw = ts.run(reqs, scheduler=sched, pipeline=PipelineConfig(depth=depth),
                         kv_config=ts.KvConfig(pages, 16), throttle=ts.ThrottleConfig(), token_budget=2048)
        except UnschedulableError as e:   # the reference's stall detection (`engine.py:271-276`)
            out.append({"name": name, "rate": rate, "dist": dist, "n": n, "scheduler": sched, "depth": depth,
                        "pages": pages, "trace_sha": tsha, "stuck": list(e.request_ids)})
            print(name, "stuck", len(e.request_ids))
            continue
        t = timeline(raw)
        rep = ts.build_report(raw)
        out.append({"name": name, "rate": rate, "dist": dist, "n": n, "scheduler": sched, "depth": depth,
                    "pages": pages,
                    "trace_sha": tsha,
                    "iters_sha": hashlib.sha256(json.dumps(t["iterations"]).encode()).hexdigest(),
                    "reqs_sha": hashlib.sha256(json.dumps(t["requests"]).encode()).hexdigest(),
                    "spans_sha": t["spans_sha"], "busy_sha": t["busy_sha"], "n_iters": len(t["iterations"]),
                    "makespan": raw.makespan_ms, "preemptions": raw.preemptions,
                    "committed": raw.committed_tokens, "discarded": raw.discarded_tokens,
                    "token_stddev": rep.token_stddev, "bubble_mean": rep.bubble_mean})
        print(name, len(t["iterations"]), raw.preemptions)
    dump("scale_runs.json.gz", out)


if __name__ == "__main__":
    if sys.argv[1:] == ["scale"]:
        scale_runs()
        sys.exit(0)
    formulas()
    plans()
    kv_ops()
    traces()
    engine_runs()
    scenarios()
    conservation()
    scale_runs()
