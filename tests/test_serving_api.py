"""Request intake (`submit`) and concurrency-bounded block-table rows, on CPU test doubles."""
import numpy as np
import pytest

from paper_2504_14775_b200 import (ConfigError, Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig,
                                    UnschedulableError, run)
from paper_2504_14775_b200.serving import ServingEngine
from paper_2504_14775_b200.stage import default_max_rows, pack_batch, prompt_source_with
from paper_2504_14775_b200.workload import ArrivalProcess, builtin_length_table, synthesize_requests


def _trace(n=60, rate=50.0):
    return synthesize_requests(ArrivalProcess.poisson(rate, 1), builtin_length_table("sharegpt-like"), n)


def _timeline(raw):
    return ([(it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens) for it in raw.iterations],
            [(r.id, r.first_token_ms, r.completion_ms) for r in raw.requests])


def test_engine_submit_equals_constructor_trace():
    reqs = _trace()
    want = _timeline(run(reqs, kv_config=KvConfig(4096, 16)))
    eng = Engine(reqs[:10], kv_config=KvConfig(4096, 16))
    for r in reqs[10:]:
        eng.submit(r)
    assert _timeline(eng.run()) == want


def test_engine_submit_validation():
    eng = Engine([RequestSpec(0, 5.0, 10, 2)], kv_config=KvConfig(64, 16))
    with pytest.raises(ConfigError):
        eng.submit(RequestSpec(0, 6.0, 10, 2))          # duplicate id
    with pytest.raises(UnschedulableError):
        eng.submit(RequestSpec(1, 6.0, 5000, 2))        # can never fit the cache
    while eng.step():
        pass
    with pytest.raises(ConfigError):
        eng.submit(RequestSpec(2, 1.0, 10, 2))          # arrives before the clock


class RowExec:
    """Executor double: checks that block-table rows are never shared by live requests."""

    def __init__(self, max_rows, requests=(), vocab=1000):
        self.max_rows = max_rows
        self.max_seq_len = 4096
        self.specs, self.prompts, self.outputs = {r.id: r for r in requests}, {}, {}
        self.src = prompt_source_with(self.prompts, self.specs, vocab)
        self.q = {}
        self.row_owner = {}
        self.peak = 0
        self.seen_prompts = {}

    def add_request(self, spec):
        self.specs[spec.id] = spec

    def register_prompt(self, rid, toks):
        self.prompts[rid] = np.asarray(toks, np.int32)

    def launch(self, meta):
        for rid, row in zip(meta.ids, meta.rows):
            assert 0 <= row < self.max_rows
            assert self.row_owner.setdefault(row, rid) == rid, (row, rid)
        for rid, row in meta.new_prompts:
            self.seen_prompts[rid] = self.src(rid).copy()
        self.peak = max(self.peak, len(self.row_owner))
        self.q[meta.seq] = pack_batch(meta, 32, self.src)

    def retire(self, seq):
        pb = self.q.pop(seq)
        for rid in pb.emit_ids:
            self.outputs.setdefault(rid, []).append(0)

    def on_finish(self, rid, row):
        assert self.row_owner.pop(row) == rid

    def stage0_idle(self):
        return True

    def wait(self, seq):
        pass

    def mark_epoch(self):
        pass

    def synchronize(self):
        pass

    def stage_busy_intervals(self):
        return [[]]


@pytest.mark.parametrize("lookahead", [False, True])
def test_rows_bounded_by_concurrency(lookahead):
    """More requests than rows: admission waits for a free row (FCFS), every request completes and
    no row is ever shared by two live requests."""
    reqs = [RequestSpec(i, 0.0, 20 + i % 7, 3 + i % 4) for i in range(40)]
    ex = RowExec(max_rows=6, requests=reqs)
    eng = ServingEngine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(512, 16),
                        throttle=ThrottleConfig(T=2, min_p=4, max_p=256), executor=ex, lookahead=lookahead,
                        time_scale=1e6)
    raw = eng.run()
    assert all(r.completion_ms is not None for r in raw.requests)
    assert ex.peak <= 6
    for r in reqs:
        assert len(ex.outputs[r.id]) == r.output_tokens


def test_serving_submit_with_prompt_ids():
    ex = RowExec(max_rows=8)
    eng = ServingEngine([], pipeline=PipelineConfig(depth=2), kv_config=KvConfig(256, 16), executor=ex,
                        lookahead=True, time_scale=1e6)
    rng = np.random.default_rng(0)
    prompts = {}
    for i in range(10):
        prompts[i] = rng.integers(0, 1000, 17 + i)
        eng.submit(RequestSpec(i, 0.0, 17 + i, 2), prompts[i])
    with pytest.raises(ConfigError):
        eng.submit(RequestSpec(99, 0.0, 5, 2), [1, 2, 3])        # wrong prompt length
    raw = eng.run()
    assert all(r.completion_ms is not None for r in raw.requests)
    for i in range(10):
        assert np.array_equal(ex.seen_prompts[i], prompts[i])
        assert eng.outputs(i) == [0, 0]


def test_default_max_rows():
    assert default_max_rows([RequestSpec(i, 0.0, 5, 5) for i in range(10)], 4096) == 10
    assert default_max_rows([RequestSpec(i, 0.0, 5, 5) for i in range(10_000)], 4096) == 4096
