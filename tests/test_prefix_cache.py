"""Prefix caching (opt-in; the paper's feature, `PAPER.md:325`, absent from the reference): page
sharing and refcounts in `PrefixCachingKvCache`, and the engine mapping cached prompt pages before
planning. GPU logits parity of a prefix-cached run is in tests/test_engine_gpu.py."""

import numpy as np
import pytest

from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig
from paper_2504_14775_b200.kvcache import PrefixCachingKvCache, prompt_page_hashes


def test_page_hashes_chain_prefixes():
    a = np.arange(64, dtype=np.int32)
    b = a.copy()
    b[40] = 999
    ha, hb = prompt_page_hashes(a, 16), prompt_page_hashes(b, 16)
    assert len(ha) == 4 and ha[:2] == hb[:2] and ha[2] != hb[2] and ha[3] != hb[3]
    assert prompt_page_hashes(a[:47], 16) == ha[:2]     # only full pages


def test_refcounts_cached_pages_and_reclaim():
    kv = PrefixCachingKvCache(KvConfig(8, 16))
    h = prompt_page_hashes(np.arange(80, dtype=np.int32), 16)   # 5 full pages
    kv.bind_row(1, 0)
    assert kv.allocate(1, 70)                  # 5 pages
    kv.register(1, h, 70)                      # pages 0-3 are full prompt pages
    assert kv.free_pages == 3
    kv.bind_row(2, 1)
    assert kv.match(2, h, 3) == 48             # shares 3 pages, no new page used
    assert kv.free_pages == 3 and kv.pages(2) == 3 and kv.stored_tokens(2) == 48
    assert kv.page_ids(2) == kv.page_ids(1)[:3]
    d = kv.take_deltas()
    assert d[-3:].tolist() == [[1, 0, kv.page_ids(1)[0]], [1, 1, kv.page_ids(1)[1]], [1, 2, kv.page_ids(1)[2]]]
    assert kv.release(1) == 5                  # 2 pages still held by request 2
    assert kv.free_pages == 5                  # 3 free + its 4th page (cached) + its 5th (free stack)
    assert len(kv._cached) == 1
    kv.bind_row(3, 2)
    assert kv.match(3, h, 4) == 64             # the cached 4th page comes back from the cache
    assert kv.free_pages == 4
    kv.release(2)
    kv.release(3)
    assert kv.free_pages == 8                  # everything free or cached
    kv.bind_row(4, 3)
    assert kv.allocate(4, 128)                 # all 8 pages: cached ones are reclaimed (hashes dropped)
    assert kv.free_pages == 0 and not kv._cached and not kv._by_hash
    kv.bind_row(5, 4)
    assert kv.match(5, h, 4) == 0


class _FakeExecutor:
    """Prompt source + executor protocol without a GPU."""

    def __init__(self, prompts):
        self.prompts = prompts
        self.max_rows = None
        self.metas = []

    def prompt_source(self, rid):
        return self.prompts[rid]

    def launch(self, meta):
        self.metas.append(meta)

    def retire(self, seq):
        pass

    def on_finish(self, rid, row):
        pass


def _shared_prefix_trace(n=12, prefix=96, seed=0):
    rng = np.random.default_rng(seed)
    system = rng.integers(0, 32000, prefix).astype(np.int32)
    reqs, prompts = [], {}
    for i in range(n):
        tail = rng.integers(0, 32000, int(rng.integers(5, 60))).astype(np.int32)
        prompts[i] = np.concatenate([system, tail])
        reqs.append(RequestSpec(i, 5.0 * i, len(prompts[i]), 6))
    return reqs, prompts


@pytest.mark.parametrize("depth", [1, 2])
def test_engine_prefix_caching_skips_cached_prompt_pages(depth):
    reqs, prompts = _shared_prefix_trace()
    kvc = KvConfig(256, 16)
    base = Engine(reqs, pipeline=PipelineConfig(depth=depth), kv_config=kvc, executor=_FakeExecutor(prompts)).run()
    ex = _FakeExecutor(prompts)
    eng = Engine(reqs, pipeline=PipelineConfig(depth=depth), kv_config=kvc, executor=ex, prefix_caching=True)
    raw = eng.run()
    assert all(r.finished for r in raw.requests)
    pf_base = sum(it.prefill_tokens for it in base.iterations)
    pf = sum(it.prefill_tokens for it in raw.iterations)
    assert eng.kv.hit_tokens > 0 and pf == pf_base - eng.kv.hit_tokens
    assert pf_base - pf >= (len(reqs) - 2) * 96        # the shared 6-page system prompt, mostly reused
    # a cache-hit request's first prefill chunk starts after its cached (page-aligned) tokens
    first = {}
    for m in ex.metas:
        for rid, start, n_new in zip(m.ids, m.starts, m.n_new):
            if n_new > 1 or start < reqs[rid].input_tokens:
                first.setdefault(rid, start)
    assert all(s % 16 == 0 for s in first.values())
    assert sum(1 for s in first.values() if s >= 96) >= len(reqs) - 2
    assert eng.kv.free_pages == kvc.total_pages        # all released (cached pages count as free)
    # decode work is unchanged: same output tokens for every request
    assert sum(it.decode_tokens for it in raw.iterations) == sum(it.decode_tokens for it in base.iterations)


def test_prefix_caching_off_is_reference_behaviour():
    reqs, prompts = _shared_prefix_trace()
    kvc = KvConfig(256, 16)
    a = Engine(reqs, kv_config=kvc).run()
    b = Engine(reqs, kv_config=kvc, executor=_FakeExecutor(prompts)).run()
    assert [(i.schedule_time_ms, i.prefill_tokens, i.decode_tokens) for i in a.iterations] == \
        [(i.schedule_time_ms, i.prefill_tokens, i.decode_tokens) for i in b.iterations]


def test_prefix_caching_under_preemption():
    """KV pressure: preempted requests re-match their cached prompt pages; accounting stays exact."""
    reqs, prompts = _shared_prefix_trace(n=24, prefix=64, seed=3)
    reqs = [RequestSpec(r.id, r.arrival_ms * 0.05, r.input_tokens, 40) for r in reqs]
    kvc = KvConfig(40, 16)
    eng = Engine(reqs, pipeline=PipelineConfig(depth=2), kv_config=kvc, executor=_FakeExecutor(prompts),
                 throttle=ThrottleConfig(T=2), prefix_caching=True)
    raw = eng.run()
    assert all(r.finished for r in raw.requests)
    assert eng.kv.free_pages == kvc.total_pages and not eng.kv._ref
