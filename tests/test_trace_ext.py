"""Trace-format extension: token seeds, resampled replay, Azure-style CSV."""
import gzip
import json
import os

import numpy as np
import pytest

from paper_2504_14775_b200 import (
    RequestSpec,
    TraceError,
    load_azure_trace,
    load_trace,
    prompt_token_ids,
    resample_arrivals,
    save_trace,
)
from paper_2504_14775_b200.stage import default_prompt_source

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "trace_resample.json.gz")


def _cases():
    with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", range(3))
def test_resample_matches_reference_build_workload(tmp_path, case):
    """Reference `cli.build_workload` with source=trace + resample_rate_per_s (`cli.py:71-79`)."""
    c = _cases()[case]
    path = tmp_path / "t.jsonl"
    path.write_text(c["trace"], encoding="utf-8")
    out = resample_arrivals(load_trace(str(path)), c["resample_rate_per_s"], c["seed"])
    assert [[s.id, s.arrival_ms, s.input_tokens, s.output_tokens] for s in out] == c["rows"]


def test_plain_trace_keeps_reference_bytes(tmp_path):
    """Traces without token seeds round-trip byte for byte in the reference's format."""
    c = _cases()[0]
    src = tmp_path / "a.jsonl"
    src.write_text(c["trace"], encoding="utf-8")
    dst = tmp_path / "b.jsonl"
    save_trace(load_trace(str(src)), str(dst))
    assert dst.read_bytes() == src.read_bytes()
    assert b"token_seed" not in dst.read_bytes()


def test_token_seed_round_trip_and_prompt_ids(tmp_path):
    specs = [RequestSpec(0, 0.0, 5, 3), RequestSpec(1, 1.5, 7, 2, token_seed=42)]
    p = tmp_path / "s.jsonl"
    save_trace(specs, str(p))
    lines = p.read_text().splitlines()
    assert "token_seed" not in lines[0] and json.loads(lines[1])["token_seed"] == 42
    back = load_trace(str(p))
    assert back == specs
    # default seed 1000 + id; an explicit seed replaces it
    a = prompt_token_ids(1, 7, 32000)
    b = prompt_token_ids(1, 7, 32000, token_seed=42)
    assert np.array_equal(a, np.random.Generator(np.random.PCG64(1001)).integers(0, 32000, 7).astype(np.int32))
    assert np.array_equal(b, np.random.Generator(np.random.PCG64(42)).integers(0, 32000, 7).astype(np.int32))
    assert not np.array_equal(a, b)
    # the GPU path's prompt source follows the trace's seed
    src = default_prompt_source({s.id: s for s in back}, 32000)
    assert np.array_equal(src(1), b) and np.array_equal(src(0), prompt_token_ids(0, 5, 32000))
    # resampling keeps ids, lengths and seeds
    assert [s.token_seed for s in resample_arrivals(back, 3.0, 1)] == [None, 42]


def test_token_seed_must_be_int(tmp_path):
    p = tmp_path / "bad.jsonl"
    p.write_text('{"arrival_ms": 0, "input_tokens": 3, "output_tokens": 2, "token_seed": "x"}\n')
    with pytest.raises(TraceError, match="token_seed"):
        load_trace(str(p))


def test_azure_csv_replay(tmp_path):
    p = tmp_path / "azure.csv"
    p.write_text("TIMESTAMP,ContextTokens,GeneratedTokens\n"
                 "2023-11-16 18:15:46.6805900,374,44\n"
                 "2023-11-16 18:15:46.2000000,396,0\n"
                 "2023-11-16 18:15:50.1234567,879,12\n")
    specs = load_azure_trace(str(p))
    assert [(s.id, s.input_tokens, s.output_tokens) for s in specs] == [(1, 396, 1), (0, 374, 44), (2, 879, 12)]
    assert [s.arrival_ms for s in specs] == pytest.approx([0.0, 480.59, 3923.4567], abs=1e-6)
    # numeric seconds, clamps, and it feeds the same trace writer
    q = tmp_path / "sec.csv"
    q.write_text("timestamp,contexttokens,generatedtokens\n10.5,9000,3\n10.0,5,5\n")
    specs = load_azure_trace(str(q), max_tokens=8192)
    assert [(s.arrival_ms, s.input_tokens) for s in specs] == [(0.0, 5), (500.0, 8192)]
    out = tmp_path / "t.jsonl"
    save_trace(specs, str(out))
    assert load_trace(str(out)) == [RequestSpec(0, 0.0, 5, 5), RequestSpec(1, 500.0, 8192, 3)]


def test_azure_csv_errors(tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("TIMESTAMP,ContextTokens\n1.0,3\n")
    with pytest.raises(TraceError, match="missing column"):
        load_azure_trace(str(p))
    p.write_text("TIMESTAMP,ContextTokens,GeneratedTokens\nyesterday,3,4\n")
    with pytest.raises(TraceError, match="TIMESTAMP"):
        load_azure_trace(str(p))
    p.write_text("TIMESTAMP,ContextTokens,GeneratedTokens\n1.0,-3,4\n")
    with pytest.raises(TraceError, match="negative"):
        load_azure_trace(str(p))
