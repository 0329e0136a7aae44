"""Full engine timelines vs the reference (virtual clock, bit-exact).

Fixtures from tests/golden/make_golden.py: C1 trace at depth 1/2/4, the
reference's bursty fixture under its acceptance settings
(`pkg/tests/test_acceptance.py:73-82, 170-229`), tick-simulator scenarios
(`oracle_sim.py:397-469`) and the 100 conservation runs of criterion 8.
"""
import hashlib
import json

import pytest

from golden_io import load
from paper_2504_14775_b200 import (CommModel, Engine, KvConfig, PipelineConfig, RequestSpec, StageCostModel,
                                    ThrottleConfig, UnschedulableError, build_report, run)
from paper_2504_14775_b200.workload import ArrivalProcess, LengthDistribution, builtin_length_table, synthesize_requests

ENGINE = load("engine_runs.json.gz")
TRACES = load("traces.json.gz")
TRACES.update(ENGINE["traces"])


def _specs(rows):
    return [RequestSpec(i, a, b, c) for i, (a, b, c) in enumerate(rows)]


def _timeline(raw):
    return {
        "iterations": [[it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens] for it in raw.iterations],
        "requests": [[r.id, r.arrival_ms, r.first_token_ms, r.completion_ms, r.preemption_count] for r in raw.requests],
        "spans_sha": hashlib.sha256(json.dumps(raw.stage_spans).encode()).hexdigest(),
        "busy_sha": hashlib.sha256(json.dumps(raw.busy_intervals).encode()).hexdigest(),
        "makespan": raw.makespan_ms, "committed": raw.committed_tokens,
        "discarded": raw.discarded_tokens, "preemptions": raw.preemptions, "truncated": raw.truncated,
    }


@pytest.mark.parametrize("case", ENGINE["runs"], ids=[r["name"] for r in ENGINE["runs"]])
def test_engine_run_golden(case):
    comm = CommModel.pcie() if case["comm"] == "pcie" else CommModel()
    raw = run(_specs(TRACES[case["trace"]]), scheduler=case["scheduler"],
              pipeline=PipelineConfig(depth=case["depth"], cost=StageCostModel(*case["cost"]), comm=comm),
              kv_config=KvConfig(case["pages"], case["ps"]),
              throttle=ThrottleConfig(T=case["T"], kv_thresh=case["thresh"]),
              token_budget=case["budget"], horizon_ms=case["horizon"],
              record_events="events_sha" in case)
    got = _timeline(raw)
    for k, v in got.items():
        assert v == case[k], k
    if "events_sha" in case:
        assert hashlib.sha256(json.dumps(raw.events).encode()).hexdigest() == case["events_sha"]
    if "report" in case:
        rep = build_report(raw)
        for k, v in case["report"].items():
            assert getattr(rep, k) == v, k


def test_acceptance_pins():
    # The reference's pinned acceptance values (`test_acceptance.py:169-186`), recomputed here.
    by = {r["name"]: r for r in ENGINE["runs"]}
    assert by["bursty_throttle_p1024_T8_th0.05"]["report"]["token_stddev"] == pytest.approx(36.79826426303527, rel=1e-12)
    assert by["bursty_sarathi_p1024_T8_th0.05"]["report"]["token_stddev"] == pytest.approx(113.29596236956067, rel=1e-12)
    assert by["bursty_throttle_p192_T8_th0.0"]["preemptions"] == 142
    assert by["bursty_throttle_p192_T8_th0.05"]["preemptions"] == 3


SCEN = load("scenarios.json.gz")


@pytest.mark.parametrize("i", range(len(SCEN)))
def test_tick_scenarios(i):
    s = SCEN[i]
    reqs = [RequestSpec(a, b, c, d) for a, b, c, d in s["specs"]]
    T, max_p, min_p, th, mode = s["throttle"]
    eng = Engine(reqs, scheduler=s["scheduler"],
                 pipeline=PipelineConfig(depth=s["depth"], cost=StageCostModel(float(s["c0"]), float(s["c_tok"]), float(s["c_ctx"])),
                                         comm=CommModel(latency_ms=float(s["latency"]), bytes_per_token=0.0, bandwidth_bytes_per_ms=1.0)),
                 kv_config=KvConfig(s["pages"], s["ps"]),
                 throttle=ThrottleConfig(T=T, max_p=max_p, min_p=min_p, kv_thresh=th, mode=mode),
                 token_budget=s["budget"])
    stalled = []
    try:
        while eng.step():
            pass
    except UnschedulableError as exc:
        stalled = sorted(exc.request_ids)
    assert stalled == s["stalled"] == s["tick_stuck"]
    raw = eng.raw_data()
    assert [list(x) for x in raw.stage_spans] == s["spans"]
    got = _timeline(raw)
    for k in ("iterations", "requests", "committed", "discarded", "preemptions", "makespan"):
        assert got[k] == s[k], k


CONS = load("conservation.json.gz")


@pytest.mark.parametrize("case", CONS, ids=[f"seed{c['seed']}" for c in CONS])
def test_conservation_runs(case):
    seed = case["seed"]
    reqs = synthesize_requests(ArrivalProcess.poisson(40.0, seed),
                               LengthDistribution.lognormal(60.0, 0.7, 15.0, 0.6, min_tokens=1, max_tokens=600), case["n"])
    depth = case["depth"]
    eng = Engine(reqs, scheduler=case["scheduler"], pipeline=PipelineConfig(depth=depth, comm=CommModel.pcie()),
                 kv_config=KvConfig(case["pages"], 16), throttle=ThrottleConfig())
    while eng.step():
        # invariants of criterion 8 (`test_acceptance.py:288-300`)
        assert len(eng.in_flight) <= depth
        ids = [rid for b in eng.in_flight.values() for rid in b.plan.decode_ids + [r for r, _ in b.plan.prefill_chunks]]
        assert len(ids) == len(set(ids))
        assert eng.kv.free_pages + sum(eng.kv.pages(r) for r in eng.kv.holders) == eng.kv.config.total_pages
    raw = eng.raw_data()
    t = _timeline(raw)
    assert hashlib.sha256(json.dumps(t["iterations"]).encode()).hexdigest() == case["iters_sha"]
    assert hashlib.sha256(json.dumps(t["requests"]).encode()).hexdigest() == case["reqs_sha"]
    assert t["spans_sha"] == case["spans_sha"]
    assert (raw.preemptions, raw.committed_tokens, raw.discarded_tokens) == (case["preemptions"], case["committed"], case["discarded"])
    lifetimes = sum(r.input_tokens + r.output_tokens - 1 for r in raw.requests)
    assert raw.committed_tokens - raw.discarded_tokens == lifetimes


def test_unschedulable_upfront():
    with pytest.raises(UnschedulableError) as ei:
        Engine([RequestSpec(0, 0.0, 100, 10)], kv_config=KvConfig(2, 16))
    assert ei.value.request_ids == (0,)


SCALE = load("scale_runs.json.gz")


@pytest.mark.parametrize("case", SCALE, ids=[c["name"] for c in SCALE])
def test_scale_runs(case):
    """C2-C5-scale timelines (1000 ShareGPT-like requests at depth 1/2/4/8, both schedulers, a
    2048-page pressure run, the C5 long-prompt trace at depth 8) bit-exact with the reference."""
    sg = builtin_length_table("sharegpt-like")
    c5 = LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)])
    reqs = synthesize_requests(ArrivalProcess.poisson(case["rate"], 0), sg if case["dist"] == "sharegpt" else c5,
                               case["n"])
    tsha = hashlib.sha256(json.dumps([[r.arrival_ms, r.input_tokens, r.output_tokens] for r in reqs]).encode())
    assert tsha.hexdigest() == case["trace_sha"]
    kw = dict(scheduler=case["scheduler"], pipeline=PipelineConfig(depth=case["depth"]),
              kv_config=KvConfig(case["pages"], 16), throttle=ThrottleConfig(), token_budget=2048)
    if "stuck" in case:
        with pytest.raises(UnschedulableError) as ei:
            run(reqs, **kw)
        assert list(ei.value.request_ids) == case["stuck"]
        return
    raw = run(reqs, **kw)
    t = _timeline(raw)
    assert len(t["iterations"]) == case["n_iters"]
    assert hashlib.sha256(json.dumps(t["iterations"]).encode()).hexdigest() == case["iters_sha"]
    assert hashlib.sha256(json.dumps(t["requests"]).encode()).hexdigest() == case["reqs_sha"]
    assert (t["spans_sha"], t["busy_sha"]) == (case["spans_sha"], case["busy_sha"])
    assert (raw.makespan_ms, raw.preemptions, raw.committed_tokens, raw.discarded_tokens) == \
        (case["makespan"], case["preemptions"], case["committed"], case["discarded"])
    rep = build_report(raw)
    assert (rep.token_stddev, rep.bubble_mean) == (case["token_stddev"], case["bubble_mean"])


class _TimedFakeExecutor:
    """Executor stand-in for the measured-time replay: reports per-stage 'device' times."""

    def __init__(self, depth, times_fn):
        self.stages = [object()] * depth
        self.max_rows = None
        self.times_fn = times_fn
        self.plans = {}

    def launch(self, meta):
        self.plans[meta.seq] = meta

    def stage_times_ms(self, seq):
        return self.times_fn(self.plans[seq])

    def retire(self, seq):
        pass

    def on_finish(self, request_id, row):
        pass


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_measured_stage_times_reduce_to_cost_model(depth):
    """Replay with per-stage times equal to `stage_time` reproduces the cost-model timeline exactly."""
    from paper_2504_14775_b200.engine import stage_time
    reqs = _specs(TRACES[ENGINE["runs"][0]["trace"]])
    cost = StageCostModel(1.0, 0.01, 0.1)
    pipe = PipelineConfig(depth=depth, cost=cost)
    kv = KvConfig(2048, 16)
    ref = run(reqs, pipeline=pipe, kv_config=kv)

    eng = None

    def times(meta):
        plan = eng.in_flight[meta.seq].plan
        return [stage_time(plan, cost)] * depth

    eng = Engine(reqs, pipeline=pipe, kv_config=kv, executor=_TimedFakeExecutor(depth, times),
                 measured_stage_times=True)
    got = eng.run()
    assert _timeline(got) == _timeline(ref)


def test_measured_stage_times_per_stage():
    """Unequal per-stage times: each stage span lasts exactly its measured time, admission stays in order."""
    reqs = _specs(TRACES[ENGINE["runs"][0]["trace"]])[:20]
    per_stage = [0.7, 2.5, 1.1]
    eng = Engine(reqs, pipeline=PipelineConfig(depth=3), kv_config=KvConfig(2048, 16),
                 executor=_TimedFakeExecutor(3, lambda m: list(per_stage)), measured_stage_times=True)
    raw = eng.run()
    assert all(r.finished for r in raw.requests)
    for seq, stage, a, b in raw.stage_spans:
        assert b - a == pytest.approx(per_stage[stage])
    for ivs in raw.busy_intervals:
        assert all(ivs[i][1] <= ivs[i + 1][0] for i in range(len(ivs) - 1))
    with pytest.raises(Exception):
        Engine(reqs, pipeline=PipelineConfig(depth=2), executor=_TimedFakeExecutor(3, lambda m: per_stage),
               measured_stage_times=True)
