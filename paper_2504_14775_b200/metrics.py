"""Serving metrics over per-request and per-iteration records.

Definitions follow `pkg/src/tokensim/metrics.py` so simulated and measured
runs report the same quantities: TTFT = first - arrival, TPOT =
(done - first) / (out - 1) (None below two output tokens), means over
finished requests, population stddev of per-iteration tokens, and absent
metrics as None (`metrics.py:1-6, 24-172`). `requests.csv` /
`iterations.csv` use the reference columns and `str()` cell formatting so a
virtual-clock run is byte-comparable with the reference (`metrics.py:205-307`).

Added for the B200 runs (BASELINE metric): p50 TTFT/TPOT and output-only
tokens/s (the reference `throughput` counts input+output tokens).
"""

from __future__ import annotations

import csv
import io
import json
import math
import os
from dataclasses import dataclass
from typing import Sequence

from .errors import ConfigError


@dataclass(frozen=True)
class RequestRecord:
    id: int
    arrival_ms: float
    first_token_ms: float | None
    completion_ms: float | None
    input_tokens: int
    output_tokens: int
    preemption_count: int = 0

    @property
    def finished(self) -> bool:
        return self.completion_ms is not None

    @property
    def ttft_ms(self) -> float | None:
        return None if self.first_token_ms is None else self.first_token_ms - self.arrival_ms

    @property
    def tpot_ms(self) -> float | None:
        if self.completion_ms is None or self.first_token_ms is None or self.output_tokens < 2:
            return None
        return (self.completion_ms - self.first_token_ms) / (self.output_tokens - 1)

    @property
    def e2el_ms(self) -> float | None:
        return None if self.completion_ms is None else self.completion_ms - self.arrival_ms


@dataclass(frozen=True)
class IterationRecord:
    batch_seq: int
    schedule_time_ms: float
    prefill_tokens: int
    decode_tokens: int

    @property
    def total_tokens(self) -> int:
        return self.prefill_tokens + self.decode_tokens


def _mean(xs: list[float]) -> float | None:
    return sum(xs) / len(xs) if xs else None


def _median(xs: list[float]) -> float | None:
    if not xs:
        return None
    s = sorted(xs)
    m = len(s) // 2
    return s[m] if len(s) % 2 else (s[m - 1] + s[m]) / 2.0


def ttft(records: Sequence[RequestRecord]) -> float | None:
    return _mean([r.ttft_ms for r in records if r.finished and r.ttft_ms is not None])


def tpot(records: Sequence[RequestRecord]) -> float | None:
    return _mean([r.tpot_ms for r in records if r.tpot_ms is not None])


def e2el(records: Sequence[RequestRecord]) -> float | None:
    return _mean([r.e2el_ms for r in records if r.e2el_ms is not None])


def ttft_p50(records: Sequence[RequestRecord]) -> float | None:
    return _median([r.ttft_ms for r in records if r.finished and r.ttft_ms is not None])


def tpot_p50(records: Sequence[RequestRecord]) -> float | None:
    return _median([r.tpot_ms for r in records if r.tpot_ms is not None])


def throughput(records: Sequence[RequestRecord], window_ms: float | None = None) -> float | None:
    """Finished input+output tokens per second (reference definition)."""
    done = [r for r in records if r.finished]
    if not done:
        return None
    if window_ms is None:
        window_ms = max(r.completion_ms for r in done) - min(r.arrival_ms for r in records)
    if window_ms <= 0:
        return None
    return sum(r.input_tokens + r.output_tokens for r in done) / (window_ms / 1000.0)


def output_throughput(records: Sequence[RequestRecord], window_ms: float | None = None) -> float | None:
    """Finished OUTPUT tokens per second, first arrival to last completion (BASELINE metric)."""
    done = [r for r in records if r.finished]
    if not done:
        return None
    if window_ms is None:
        window_ms = max(r.completion_ms for r in done) - min(r.arrival_ms for r in records)
    if window_ms <= 0:
        return None
    return sum(r.output_tokens for r in done) / (window_ms / 1000.0)


def slo_attainment(records: Sequence[RequestRecord], ttft_limit_ms: float,
                   tpot_limit_ms: float) -> float | None:
    if ttft_limit_ms <= 0 or tpot_limit_ms <= 0:
        raise ConfigError("SLO limits must be > 0")
    done = [r for r in records if r.finished]
    if not done:
        return None
    ok = sum(1 for r in done if r.ttft_ms is not None and r.ttft_ms <= ttft_limit_ms
             and (r.tpot_ms is None or r.tpot_ms <= tpot_limit_ms))
    return ok / len(done)


def token_fluctuation(iterations: Sequence[IterationRecord]) -> tuple[float, float] | None:
    if not iterations:
        return None
    xs = [it.total_tokens for it in iterations]
    mu = sum(xs) / len(xs)
    return mu, math.sqrt(sum((x - mu) ** 2 for x in xs) / len(xs))


def ideal_balance_reference(iterations: Sequence[IterationRecord]) -> float | None:
    return sum(it.total_tokens for it in iterations) / len(iterations) if iterations else None


@dataclass(frozen=True)
class Report:
    ttft_mean_ms: float | None
    tpot_mean_ms: float | None
    e2el_mean_ms: float | None
    throughput_tokens_per_s: float | None
    slo_attainment: float | None
    slo_ttft_ms: float
    slo_tpot_ms: float
    token_mean: float | None
    token_stddev: float | None
    ideal_balance_level: float | None
    bubble_fractions: tuple[float, ...]
    bubble_mean: float | None
    makespan_ms: float
    finished_requests: int
    unfinished_requests: int
    preemptions: int
    committed_tokens: int
    discarded_tokens: int
    truncated: bool
    requests: tuple[RequestRecord, ...]
    iterations: tuple[IterationRecord, ...]
    ttft_p50_ms: float | None = None
    tpot_p50_ms: float | None = None
    output_tokens_per_s: float | None = None


def build_report(raw, slo_ttft_ms: float = 3000.0, slo_tpot_ms: float = 150.0) -> Report:
    recs = raw.requests
    fl = token_fluctuation(raw.iterations)
    bub = tuple(raw.bubble_fractions())
    return Report(
        ttft_mean_ms=ttft(recs), tpot_mean_ms=tpot(recs), e2el_mean_ms=e2el(recs),
        throughput_tokens_per_s=throughput(recs),
        slo_attainment=slo_attainment(recs, slo_ttft_ms, slo_tpot_ms),
        slo_ttft_ms=slo_ttft_ms, slo_tpot_ms=slo_tpot_ms,
        token_mean=None if fl is None else fl[0], token_stddev=None if fl is None else fl[1],
        ideal_balance_level=ideal_balance_reference(raw.iterations),
        bubble_fractions=bub, bubble_mean=_mean(list(bub)), makespan_ms=raw.makespan_ms,
        finished_requests=sum(1 for r in recs if r.finished),
        unfinished_requests=sum(1 for r in recs if not r.finished),
        preemptions=raw.preemptions, committed_tokens=raw.committed_tokens,
        discarded_tokens=raw.discarded_tokens, truncated=raw.truncated,
        requests=tuple(recs), iterations=tuple(raw.iterations),
        ttft_p50_ms=ttft_p50(recs), tpot_p50_ms=tpot_p50(recs),
        output_tokens_per_s=output_throughput(recs),
    )


REQUEST_COLUMNS = ("id", "arrival_ms", "first_token_ms", "completion_ms", "input_tokens",
                   "output_tokens", "preemption_count")
ITERATION_COLUMNS = ("batch_seq", "schedule_time_ms", "prefill_tokens", "decode_tokens", "total_tokens")

_REFERENCE_JSON_KEYS = ("ttft_mean_ms", "tpot_mean_ms", "e2el_mean_ms", "throughput_tokens_per_s",
                        "slo_attainment", "slo_ttft_ms", "slo_tpot_ms", "token_mean", "token_stddev",
                        "ideal_balance_level", "bubble_fractions", "bubble_mean", "makespan_ms",
                        "finished_requests", "unfinished_requests", "preemptions",
                        "committed_tokens", "discarded_tokens", "truncated")


def _fmt(v) -> str:
    return "" if v is None else str(v)


def requests_csv(recs: Sequence[RequestRecord]) -> str:
    return _csv(REQUEST_COLUMNS, [[_fmt(getattr(r, c)) for c in REQUEST_COLUMNS] for r in recs])


def iterations_csv(its: Sequence[IterationRecord]) -> str:
    return _csv(ITERATION_COLUMNS, [[_fmt(it.batch_seq), _fmt(it.schedule_time_ms), _fmt(it.prefill_tokens),
                                     _fmt(it.decode_tokens), _fmt(it.total_tokens)] for it in its])


def _csv(header, rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(header)
    w.writerows(rows)
    return buf.getvalue()


def report_to_json(report: Report, extended: bool = False) -> str:
    doc = {k: getattr(report, k) for k in _REFERENCE_JSON_KEYS}
    doc["bubble_fractions"] = list(report.bubble_fractions)
    if extended:
        doc.update(ttft_p50_ms=report.ttft_p50_ms, tpot_p50_ms=report.tpot_p50_ms,
                   output_tokens_per_s=report.output_tokens_per_s)
    return json.dumps(doc, indent=2, sort_keys=True) + "\n"


def write_atomic(path: str, text: str) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w", encoding="utf-8", newline="") as fh:
        fh.write(text)
    os.replace(tmp, path)


def write_report(report: Report, outdir: str, extended: bool = False) -> list[str]:
    os.makedirs(outdir, exist_ok=True)
    out = []
    for name, text in (("report.json", report_to_json(report, extended)),
                       ("requests.csv", requests_csv(report.requests)),
                       ("iterations.csv", iterations_csv(report.iterations))):
        p = os.path.join(outdir, name)
        write_atomic(p, text)
        out.append(p)
    return out
