"""KV accounting, physical pages and workload synthesis vs the reference's golden outputs."""
import numpy as np
import pytest

from golden_io import load
from paper_2504_14775_b200 import kvcache as K
from paper_2504_14775_b200 import workload as W
from paper_2504_14775_b200.errors import ConfigError, TraceError


def test_kv_sequences_golden():
    g = load("kv_ops.json.gz")
    for seq in g["sequences"]:
        for cls in (K.KvCacheState, K.PagedKvCache):
            kv = cls(K.KvConfig(seq["total"], seq["ps"]))
            if cls is K.PagedKvCache:
                for rid in range(6):
                    kv.bind_row(rid, rid)
            for op in seq["ops"]:
                if op[0] == "a":
                    _, rid, n, ok, free, stored, pages = op
                    assert kv.allocate(rid, n) == ok
                    assert (kv.free_pages, kv.stored_tokens(rid), kv.pages(rid)) == (free, stored, pages)
                else:
                    _, rid, got, free = op
                    if got is None:
                        with pytest.raises(KeyError):
                            kv.release(rid)
                    else:
                        assert kv.release(rid) == got
                    assert kv.free_pages == free
                if cls is K.PagedKvCache:
                    # physical ids are a partition of the pool
                    owned = [p for r in range(6) for p in kv.page_ids(r)]
                    assert len(owned) == len(set(owned)) == seq["total"] - kv.free_pages
                    assert all(len(kv.page_ids(r)) == kv.pages(r) for r in range(6))
    for cands, victim in g["victims"]:
        assert K.select_preemption_victim([tuple(c) for c in cands]) == victim


def test_pages_needed_examples():
    assert K.pages_needed(0, 1, 16) == 1
    assert K.pages_needed(15, 1, 16) == 0
    assert K.pages_needed(16, 1, 16) == 1
    assert K.pages_needed(0, 0, 16) == 0
    assert K.pages_needed(5, 40, 16) == 2  # ceil(45/16) - ceil(5/16)
    with pytest.raises(ConfigError):
        K.pages_needed(0, 1, 0)
    with pytest.raises(ConfigError):
        K.pages_needed(-1, 1, 16)


def test_block_table_deltas_deterministic():
    kv = K.PagedKvCache(K.KvConfig(8, 4))
    kv.bind_row(7, 0)
    kv.bind_row(9, 1)
    assert kv.allocate(7, 5)        # 2 pages
    assert kv.allocate(9, 4)        # 1 page
    d = kv.take_deltas()
    assert d.tolist() == [[0, 0, 0], [0, 1, 1], [1, 0, 2]]
    assert kv.take_deltas().shape == (0, 3)
    kv.release(7)
    assert kv.allocate(9, 5)        # reuses freed ids LIFO
    assert kv.page_ids(9) == [2, 0, 1]


def test_traces_golden():
    g = load("traces.json.gz")
    specs = {
        "c1": (W.ArrivalProcess.poisson(16.0, 0), W.LengthDistribution.empirical([(i, 64) for i in range(128, 513)]), 64),
        "c2_rate32": (W.ArrivalProcess.poisson(32.0, 0), W.builtin_length_table("sharegpt-like"), 1000),
        "azure_rate4": (W.ArrivalProcess.poisson(4.0, 3), W.builtin_length_table("azure-like"), 200),
        "c5": (W.ArrivalProcess.poisson(2.0, 0),
               W.LengthDistribution.empirical([(p, o) for p in range(4096, 8193, 128) for o in (100, 200, 300, 400, 500)]), 200),
        "lognormal": (W.ArrivalProcess.poisson(40.0, 5),
                      W.LengthDistribution.lognormal(60.0, 0.7, 15.0, 0.6, min_tokens=1, max_tokens=600), 300),
    }
    for name, (proc, dist, n) in specs.items():
        got = [[r.arrival_ms, r.input_tokens, r.output_tokens] for r in W.synthesize_requests(proc, dist, n)]
        assert got == g[name], name


def test_trace_roundtrip_and_errors(tmp_path):
    reqs = W.synthesize_requests(W.ArrivalProcess.poisson(8.0, 1), W.builtin_length_table("sharegpt-like"), 50)
    p = tmp_path / "t.jsonl"
    W.save_trace(reqs, str(p))
    assert W.load_trace(str(p)) == reqs
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"arrival_ms": 1, "input_tokens": 1.5, "output_tokens": 2}\n')
    with pytest.raises(TraceError):
        W.load_trace(str(bad))
    bad.write_text('{"arrival_ms": 1, "input_tokens": 0, "output_tokens": 2}\n')
    with pytest.raises(TraceError):
        W.load_trace(str(bad))


def test_prompt_tokens_seeded():
    a = W.prompt_token_ids(3, 100, 32000)
    b = W.prompt_token_ids(3, 100, 32000)
    assert a.dtype == np.int32 and (a == b).all() and a.max() < 32000 and a.min() >= 0
    assert not (W.prompt_token_ids(4, 100, 32000) == a).all()
