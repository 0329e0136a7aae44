"""Per-iteration engine: schedule -> KV apply -> launch -> stage execution -> commit.

Drop-in for `pkg/src/tokensim/engine.py` (same constructor, `step`, `run`,
`raw_data`, public `in_flight`, `kv`, `clock`; same `RawRunData`). Two
things differ by design:

1. **O(active) scheduling.** The reference rescans every request for #WP
   and #RD and re-sorts both queues at every schedule point
   (`engine.py:399-400, 411-419`; 12.7 s of 17.0 s at 2k requests, SURVEY
   §0.6). Here #WP/#RD are counters updated at the five transitions that
   change them (arrival, launch, commit, finish, preempt) and the queues
   are kept FCFS-sorted by insertion, so a schedule step touches only the
   requests it plans.
2. **Real execution.** An optional `executor` receives each launched
   micro-batch with its device metadata (block-table deltas, per-sequence
   row/start/length, which rows emit a token) and runs it on the GPU stages;
   `_commit` retires it. `Engine` keeps the reference's virtual clock
   (cost model) so its decisions are bit-exact with the reference while the
   GPU does the real work; `ServingEngine` (serving.py) drives the same state
   machine from measured time instead.

Semantics preserved (each cited at its use below): events at
one timestamp drain in push order, then exactly one schedule attempt; #RD
counts in-flight decodes; #WP subtracts in-flight chunks; LIFO victims drawn
from the decode-ready queue including this plan's decodes; self-preemption;
decode context recomputed after allocation; commit decodes before chunks.
"""

from __future__ import annotations

import heapq
from bisect import bisect_left, insort
from dataclasses import dataclass, field

from .errors import ConfigError, UnschedulableError
from .kvcache import KvCacheState, KvConfig, PagedKvCache, PrefixCachingKvCache, pages_needed, prompt_page_hashes
from .metrics import IterationRecord, RequestRecord
from .sched import MicroBatchPlan, ThrottleConfig, fill_prefill, prefill_token_limit, throttle_decode
from .workload import RequestSpec

SCHEDULERS = ("throttle", "sarathi")

ARRIVAL = "arrival"
SCHEDULE_POINT = "schedule_point"
STAGE_COMPLETE = "stage_complete"
TRANSFER_COMPLETE = "transfer_complete"
_EV_ARRIVAL, _EV_STAGE, _EV_XFER = 0, 1, 2


@dataclass(frozen=True)
class StageCostModel:
    """Virtual-clock stage latency: c0 + c_tok*tokens + c_ctx*decode_ctx/1024 (`engine.py:45-57`)."""

    c0: float = 1.0
    c_tok: float = 0.01
    c_ctx: float = 0.1

    def __post_init__(self) -> None:
        if min(self.c0, self.c_tok, self.c_ctx) < 0:
            raise ConfigError("stage cost coefficients must be >= 0")
        if self.c0 + self.c_tok <= 0:
            raise ConfigError("need c0 + c_tok > 0 so nonempty batches take time")


@dataclass(frozen=True)
class CommModel:
    """Virtual-clock activation hand-off: latency + tokens*bytes/bandwidth (`engine.py:60-82`)."""

    latency_ms: float = 0.1
    bytes_per_token: float = 16384.0
    bandwidth_bytes_per_ms: float = 20.79e6

    def __post_init__(self) -> None:
        if self.bandwidth_bytes_per_ms <= 0:
            raise ConfigError(f"bandwidth must be > 0, got {self.bandwidth_bytes_per_ms}")
        if self.latency_ms < 0 or self.bytes_per_token < 0:
            raise ConfigError("comm latency and payload must be >= 0")

    @classmethod
    def pcie(cls, latency_ms: float = 0.1, bytes_per_token: float = 16384.0) -> "CommModel":
        return cls(latency_ms, bytes_per_token, 20.79e6)

    @classmethod
    def network(cls, latency_ms: float = 0.1, bytes_per_token: float = 16384.0) -> "CommModel":
        return cls(latency_ms, bytes_per_token, 73.28e9 / 8.0 / 1000.0)


@dataclass(frozen=True)
class PipelineConfig:
    depth: int = 4
    cost: StageCostModel = StageCostModel()
    comm: CommModel = CommModel()

    def __post_init__(self) -> None:
        if self.depth < 1:
            raise ConfigError(f"pipeline.depth must be >= 1, got {self.depth}")


def stage_time(plan: MicroBatchPlan, cost: StageCostModel) -> float:
    if plan.is_empty():
        return 0.0
    return cost.c0 + cost.c_tok * plan.total_tokens + cost.c_ctx * plan.decode_context_tokens / 1024.0


def transfer_time(plan: MicroBatchPlan, comm: CommModel) -> float:
    return comm.latency_ms + plan.total_tokens * comm.bytes_per_token / comm.bandwidth_bytes_per_ms


def bubble_accounting(busy_intervals: list[list[tuple[float, float]]], makespan_ms: float) -> list[float]:
    """Idle fraction of [0, makespan] per stage; intervals must be ordered and disjoint (`engine.py:108-125`)."""
    out = []
    for ivs in busy_intervals:
        busy = 0.0
        last = None
        for a, b in ivs:
            if b < a or (last is not None and a < last):
                raise ValueError("stage busy intervals overlap or are out of order")
            busy += b - a
            last = b
        out.append(0.0 if makespan_ms <= 0 else (makespan_ms - busy) / makespan_ms)
    return out


class _Req:
    __slots__ = ("spec", "key", "target", "done", "inflight", "generated", "preemptions",
                 "incarnation", "arrived", "decoding", "in_flight", "first_ms", "finish_ms", "row")

    def __init__(self, spec: RequestSpec):
        self.spec = spec
        self.key = (spec.arrival_ms, spec.id)
        self.target = spec.input_tokens
        self.done = 0
        self.inflight = 0
        self.generated = 0
        self.preemptions = 0
        self.incarnation = 0
        self.arrived = False
        self.decoding = False
        self.in_flight = False
        self.first_ms = None
        self.finish_ms = None
        self.row = -1

    @property
    def finished(self) -> bool:
        return self.finish_ms is not None


@dataclass
class SeqMeta:
    """One sequence of a launched micro-batch, in plan order (decodes, then chunks)."""

    request_id: int
    row: int          # block-table / token-history row
    start: int        # tokens already in the KV cache before this batch
    n_new: int        # tokens this batch appends (1 for a decode)
    emits: bool       # this batch samples the sequence's next token


@dataclass
class BatchMeta:
    """Everything a stage worker needs for one micro-batch (the paper's pre-broadcast metadata).

    Columnar (one list per field, plan order) so packing is vectorised; `seqs`
    materialises per-sequence `SeqMeta` views when a caller wants them.
    """

    seq: int
    ids: list[int]
    rows: list[int]
    starts: list[int]
    n_new: list[int]
    emits: list[bool]
    page_deltas: object                   # int32 [n, 3] (row, page_index, page_id)
    new_prompts: list[tuple[int, int]] = field(default_factory=list)  # (request_id, row)

    @classmethod
    def from_seqs(cls, seq: int, seqs: list[SeqMeta], page_deltas, new_prompts=()) -> "BatchMeta":
        return cls(seq, [s.request_id for s in seqs], [s.row for s in seqs], [s.start for s in seqs],
                   [s.n_new for s in seqs], [bool(s.emits) for s in seqs], page_deltas, list(new_prompts))

    @property
    def seqs(self) -> list[SeqMeta]:
        return [SeqMeta(*t) for t in zip(self.ids, self.rows, self.starts, self.n_new, self.emits)]

    @property
    def n_tokens(self) -> int:
        return sum(self.n_new)

    @property
    def n_emit(self) -> int:
        return sum(self.emits)


@dataclass
class _Batch:
    seq: int
    plan: MicroBatchPlan
    stage_ms: float
    transfer_ms: float
    meta: BatchMeta | None = None
    stage_list: list[float] | None = None   # per-stage measured device ms (measured-time replay)


@dataclass
class RawRunData:
    requests: list[RequestRecord]
    iterations: list[IterationRecord]
    busy_intervals: list[list[tuple[float, float]]]
    stage_spans: list[tuple[int, int, float, float]]
    makespan_ms: float
    committed_tokens: int
    discarded_tokens: int
    preemptions: int
    truncated: bool
    events: list[dict] | None = None

    def bubble_fractions(self) -> list[float]:
        return bubble_accounting(self.busy_intervals, self.makespan_ms)


class EngineCore:
    """Request state machine shared by the virtual-clock and wall-clock drivers."""

    def __init__(self, requests: list[RequestSpec], scheduler: str = "throttle",
                 pipeline: PipelineConfig | None = None, kv_config: KvConfig | None = None,
                 throttle: ThrottleConfig | None = None, token_budget: int = 2048,
                 executor=None, max_rows: int | None = None, prefix_caching: bool = False):
        if scheduler not in SCHEDULERS:
            raise ConfigError(f"scheduler must be one of {SCHEDULERS}, got {scheduler!r}")
        self._scheduler = scheduler
        self._pipeline = pipeline if pipeline is not None else PipelineConfig()
        kv_config = kv_config if kv_config is not None else KvConfig(total_pages=4096, page_size=16)
        self._throttle = throttle if throttle is not None else ThrottleConfig()
        if token_budget < 1:
            raise ConfigError(f"token_budget must be >= 1, got {token_budget}")
        self._token_budget = token_budget
        ids: set[int] = set()
        prev = None
        for spec in requests:
            if spec.id in ids:
                raise ConfigError(f"duplicate request id {spec.id}")
            ids.add(spec.id)
            if prev is not None and spec.arrival_ms < prev:
                raise ConfigError("workload must be sorted by arrival time")
            prev = spec.arrival_ms
            need = pages_needed(0, spec.input_tokens + spec.output_tokens - 1, kv_config.page_size)
            if need > kv_config.total_pages:
                raise UnschedulableError(
                    f"request {spec.id} needs {need} KV pages over its lifetime "
                    f"but the cache has only {kv_config.total_pages}", (spec.id,))
        self._reqs: dict[int, _Req] = {s.id: _Req(s) for s in requests}
        self._order = [s.id for s in requests]
        self.executor = executor
        if prefix_caching and (executor is None or not hasattr(executor, "prompt_source")):
            raise ConfigError("prefix caching needs a GPU executor with prompt tokens")
        # Prefix caching (opt-in; the reference has none): full prompt pages shared by requests
        # with equal token prefixes, see `_match_prefixes` and `PrefixCachingKvCache`.
        self._prefix = prefix_caching
        self._hashes: dict[int, list[int]] = {}
        self.kv: KvCacheState = (PrefixCachingKvCache(kv_config) if prefix_caching else
                                 PagedKvCache(kv_config) if executor is not None else KvCacheState(kv_config))
        self._rows_free: list[int] = []
        self._rows_next = 0
        if max_rows is None:
            max_rows = getattr(executor, "max_rows", None) or max(1, min(len(requests) or kv_config.total_pages,
                                                                         kv_config.total_pages))
        self._max_rows = max_rows
        self.clock = 0.0
        self.makespan_ms = 0.0
        self.committed_tokens = 0
        self.discarded_tokens = 0
        self.preemptions = 0
        self.truncated = False
        depth = self._pipeline.depth
        self.in_flight: dict[int, _Batch] = {}
        self._waiting: list[tuple[float, int]] = []   # FCFS keys, kept sorted
        self._ready: list[tuple[float, int]] = []     # decode-ready FCFS keys, kept sorted
        self._wp = 0
        self._rd = 0
        self._free_at = [0.0] * depth
        self._busy: list[list[tuple[float, float]]] = [[] for _ in range(depth)]
        self._spans: list[tuple[int, int, float, float]] = []
        self._iters: list[IterationRecord] = []
        self._events: list[dict] | None = None
        self._seq = 0
        self._pending_prompts: list[tuple[int, int]] = []
        self._ctx_log: dict[int, int] = {}   # seq -> decode context tokens (cost-model calibration)

    # -- request intake ----------------------------------------------------------

    def _validate_new(self, spec: RequestSpec) -> None:
        if spec.id in self._reqs:
            raise ConfigError(f"duplicate request id {spec.id}")
        kvc = self.kv.config
        need = pages_needed(0, spec.input_tokens + spec.output_tokens - 1, kvc.page_size)
        if need > kvc.total_pages:
            raise UnschedulableError(
                f"request {spec.id} needs {need} KV pages over its lifetime "
                f"but the cache has only {kvc.total_pages}", (spec.id,))
        lim = getattr(self.executor, "max_seq_len", None)
        if lim is not None and spec.input_tokens + spec.output_tokens + 1 > lim:
            raise ConfigError(f"request {spec.id}: {spec.input_tokens}+{spec.output_tokens} tokens exceed "
                              f"the executor's max_seq_len={lim}")

    def _add_request(self, spec: RequestSpec, prompt_ids=None) -> _Req:
        """Register a request (front-end submit, `PAPER.md:252`); its prompt tokens, if given, are
        what the first stage embeds (else the seeded synthetic prompt of the trace format)."""
        self._validate_new(spec)
        if prompt_ids is not None:
            import numpy as _np
            ids = _np.asarray(prompt_ids, dtype=_np.int32).reshape(-1)
            if ids.size != spec.input_tokens:
                raise ConfigError(f"request {spec.id}: {ids.size} prompt ids for input_tokens={spec.input_tokens}")
            if self.executor is None or not hasattr(self.executor, "register_prompt"):
                raise ConfigError("prompt ids need a GPU executor")
            self.executor.register_prompt(spec.id, ids)
        if self.executor is not None and hasattr(self.executor, "add_request"):
            self.executor.add_request(spec)
        r = _Req(spec)
        self._reqs[spec.id] = r
        self._order.append(spec.id)
        return r

    # -- logging ---------------------------------------------------------------

    def _log(self, t: float, kind: str, stage, batch, plan: MicroBatchPlan | None) -> None:
        if self._events is not None:
            self._events.append({"time_ms": t, "kind": kind, "stage": stage, "batch": batch,
                                 "prefill_tokens": 0 if plan is None else plan.prefill_tokens,
                                 "decode_tokens": 0 if plan is None else plan.decode_tokens})

    # -- transitions that move #WP / #RD -------------------------------------------

    def _arrive(self, rid: int) -> None:
        r = self._reqs[rid]
        r.arrived = True
        self._wp += r.target - r.done - r.inflight
        insort(self._waiting, r.key)

    def _finish(self, r: _Req, t: float) -> None:
        r.finish_ms = t
        if r.decoding:
            self._rd -= 1
        r.decoding = False
        self.kv.release(r.spec.id)
        if r.row >= 0:
            if isinstance(self.kv, PagedKvCache):
                self.kv.unbind_row(r.spec.id)
            if self.executor is not None:
                self.executor.on_finish(r.spec.id, r.row)
            self._rows_free.append(r.row)
            r.row = -1

    def _enter_decode(self, r: _Req) -> None:
        r.decoding = True
        self._rd += 1

    def _preempt(self, rid: int) -> None:
        """Evict and queue for recompute (`engine.py:371-384`)."""
        r = self._reqs[rid]
        self.kv.release(rid)
        self.preemptions += 1
        r.preemptions += 1
        self.discarded_tokens += r.incarnation
        r.incarnation = 0
        # The rebuilt cache is the prompt plus every generated token but the newest.
        r.target = r.spec.input_tokens + max(r.generated - 1, 0)
        r.done = 0
        if r.decoding:
            self._rd -= 1
        r.decoding = False
        self._wp += r.target
        _remove_key(self._ready, r.key)
        insort(self._waiting, r.key)

    def _commit(self, t: float, batch: _Batch, retire: bool = True) -> None:
        """Last-stage commit (`engine.py:334-364`): decodes first, then prefill chunks.

        `retire=False` commits the request state only (the asynchronous serving
        loop retires the device work later and re-stamps the times, see serving.py).
        """
        plan = batch.plan
        del self.in_flight[batch.seq]
        if self.executor is not None and retire:
            self.executor.retire(batch.seq)
        self.committed_tokens += plan.total_tokens
        back: list = []
        reqs = self._reqs
        for rid in plan.decode_ids:
            r = reqs[rid]
            r.in_flight = False
            r.generated += 1
            r.incarnation += 1
            if r.generated >= r.spec.output_tokens:
                self._finish(r, t)
            else:
                back.append(r.key)
        if back:
            # re-queue in one merge (timsort on two sorted runs) instead of an insort per decode
            self._ready.extend(back)
            self._ready.sort()
        for rid, n in plan.prefill_chunks:
            r = self._reqs[rid]
            r.in_flight = False
            r.inflight = 0
            r.done += n
            r.incarnation += n
            if self._prefix:
                self.kv.register(rid, self._page_hashes(rid), min(r.done, r.spec.input_tokens))
            if r.done >= r.target:
                self._enter_decode(r)
                if r.generated == 0:
                    r.generated = 1      # the final prompt chunk yields the first token
                    r.first_ms = t
                    if r.generated >= r.spec.output_tokens:
                        self._finish(r, t)
                        continue
                insort(self._ready, r.key)
            else:
                insort(self._waiting, r.key)

    # -- scheduling ----------------------------------------------------------------

    def _plan(self) -> MicroBatchPlan:
        """Snapshot + planner call; O(planned) thanks to the counters (`engine.py:410-445`)."""
        kv = self.kv
        ps = kv.config.page_size
        free = kv.free_pages
        reqs = self._reqs
        if self._scheduler == "throttle":
            n_dec = throttle_decode(self._rd, self._pipeline.depth)
            chosen = [k[1] for k in self._ready[:n_dec]]
            limit = prefill_token_limit(self._wp, free / kv.config.total_pages, self._throttle)
        else:
            chosen = [k[1] for k in self._ready]
            limit = min(max(0, self._token_budget - len(chosen)), self._wp)
        toks = kv._tokens
        stored = [toks[rid] for rid in chosen]   # decode-ready requests always hold KV
        reserved = sum(1 for s in stored if s % ps == 0)

        paged = self.executor is not None
        rows_left = len(self._rows_free) + self._max_rows - self._rows_next

        def cands():
            nonlocal rows_left
            for _, rid in self._waiting:
                r = reqs[rid]
                if paged and r.row < 0:
                    # a new request needs a block-table row; rows are bounded by concurrency, so
                    # when none is free the FCFS fill stops here, as it does at a KV truncation
                    if rows_left <= 0:
                        return
                    rows_left -= 1
                yield rid, r.target - r.done, kv.stored_tokens(rid)

        chunks = fill_prefill(cands(), limit, free - reserved, ps)
        return MicroBatchPlan(chosen, chunks, sum(stored) + len(stored))

    def _bind_row(self, rid: int) -> None:
        r = self._reqs[rid]
        if r.row >= 0:
            return
        if self._rows_free:
            r.row = self._rows_free.pop()
        else:
            if self._rows_next >= self._max_rows:   # planning admits only as many new rows as are free
                raise AssertionError(f"out of block-table rows (max_rows={self._max_rows})")
            r.row = self._rows_next
            self._rows_next += 1
        self.kv.bind_row(rid, r.row)
        self._pending_prompts.append((rid, r.row))

    def _apply_kv(self, plan: MicroBatchPlan) -> bool:
        """Allocate the plan's pages, evicting LIFO decodes on failure (`engine.py:447-480`)."""
        kv = self.kv
        paged = isinstance(kv, PagedKvCache)
        mutated = False
        # Fast path: a decode needs a page only when its stored length is a page multiple;
        # if every such page is free, sequential allocate(rid, 1) would succeed for all of
        # them with no eviction, so apply them in bulk (same state, same delta order).
        if plan.decode_ids and kv.bulk_append_one(plan.decode_ids):
            plan.decode_context_tokens = kv.last_bulk_context
            for rid, n in plan.prefill_chunks:
                if paged:
                    self._bind_row(rid)
                if not kv.allocate(rid, n):
                    raise AssertionError("prefill pages were reserved at planning time")
            return False
        kept: list[int] = []
        dropped: set[int] = set()
        for rid in plan.decode_ids:
            if rid in dropped:
                continue
            ok = True
            while not kv.allocate(rid, 1):
                # Victims come from the decode-ready queue, which still holds this
                # plan's decodes (`engine.py:460-461`); the latest arrival loses.
                victim = self._ready[-1][1]
                self._preempt(victim)
                mutated = True
                dropped.add(victim)
                if victim == rid:
                    ok = False
                    break
                if victim in kept:
                    kept.remove(victim)
            if ok:
                kept.append(rid)
        if len(kept) != len(plan.decode_ids):
            plan.decode_ids = kept
        plan.decode_context_tokens = sum(kv.stored_tokens(rid) for rid in kept)
        for rid, n in plan.prefill_chunks:
            if paged:
                self._bind_row(rid)
            if not kv.allocate(rid, n):
                raise AssertionError("prefill pages were reserved at planning time")
        return mutated

    def _page_hashes(self, rid: int) -> list[int]:
        h = self._hashes.get(rid)
        if h is None:
            h = prompt_page_hashes(self.executor.prompt_source(rid), self.kv.config.page_size)
            self._hashes[rid] = h
        return h

    def _match_prefixes(self) -> None:
        """Prefix caching: before planning, requests at the head of the FCFS queue that hold no KV
        map the registered pages of their prompt prefix (at least one prompt token is always left
        to compute, it yields the first token); their prefill starts after the cached tokens, so
        #WP drops by them. Only the head that the next prefill budget can reach is examined."""
        kv = self.kv
        ps = kv.config.page_size
        budget = self._throttle.max_p if self._scheduler == "throttle" else self._token_budget
        seen = 0
        for _, rid in list(self._waiting):
            r = self._reqs[rid]
            if r.done == 0 and not r.in_flight and kv.stored_tokens(rid) == 0:
                hashes = self._page_hashes(rid)
                limit = min(len(hashes), (r.target - 1) // ps)
                if limit > 0:
                    if r.row < 0:
                        if not self._rows_free and self._rows_next >= self._max_rows:
                            break
                        self._bind_row(rid)
                    got = kv.match(rid, hashes, limit)
                    if got:
                        r.done = got      # cached, not computed: no incarnation (discard) credit
                        self._wp -= got
            seen += r.target - r.done
            if seen >= budget:
                break

    def _try_plan(self) -> MicroBatchPlan | None:
        """Plan + allocate; re-plan after an eviction that emptied the plan (`engine.py:391-408`)."""
        while True:
            if not self._waiting and not self._ready:
                return None
            if self._prefix:
                self._match_prefixes()
            plan = self._plan()
            mutated = self._apply_kv(plan)
            if not plan.is_empty():
                return plan
            if not mutated:
                return None

    def _make_batch(self, t: float, plan: MicroBatchPlan) -> _Batch:
        """Launch bookkeeping (`engine.py:482-516`) plus the device metadata."""
        seq = self._seq
        self._seq += 1
        batch = _Batch(seq, plan, stage_time(plan, self._pipeline.cost),
                       transfer_time(plan, self._pipeline.comm))
        reqs = self._reqs
        dec = plan.decode_ids
        dec_reqs = [reqs[rid] for rid in dec]
        for r in dec_reqs:
            r.in_flight = True
        for rid, n in plan.prefill_chunks:
            r = reqs[rid]
            r.in_flight = True
            r.inflight = n
            self._wp -= n
        if self.executor is not None:
            toks = self.kv._tokens
            chunks = plan.prefill_chunks
            ch_reqs = [reqs[rid] for rid, _ in chunks]
            batch.meta = BatchMeta(
                seq,
                dec + [rid for rid, _ in chunks],
                [r.row for r in dec_reqs] + [r.row for r in ch_reqs],
                # stored_tokens already counts the token a decode appends now
                [toks[rid] - 1 for rid in dec] + [r.done for r in ch_reqs],
                [1] * len(dec) + [n for _, n in chunks],
                [True] * len(dec) + [r.done + n >= r.target and r.generated == 0 for r, (_, n) in zip(ch_reqs, chunks)],
                self.kv.take_deltas(), self._pending_prompts)
            self._pending_prompts = []
        _remove_prefix_ids(self._ready, dec, reqs)
        _remove_prefix_ids(self._waiting, [rid for rid, _ in plan.prefill_chunks], reqs)
        self.in_flight[seq] = batch
        self._iters.append(IterationRecord(seq, t, plan.prefill_tokens, plan.decode_tokens))
        self._ctx_log[seq] = plan.decode_context_tokens
        return batch

    # -- results -------------------------------------------------------------------

    def _records(self) -> list[RequestRecord]:
        recs = [RequestRecord(r.spec.id, r.spec.arrival_ms, r.first_ms, r.finish_ms,
                              r.spec.input_tokens, r.spec.output_tokens, r.preemptions)
                for r in self._reqs.values()]
        recs.sort(key=lambda x: x.id)
        return recs

    def raw_data(self) -> RawRunData:
        if self.truncated:
            lim = self.makespan_ms
            self._busy = [[(a, min(b, lim)) for a, b in ivs if a < lim] for ivs in self._busy]
            self._spans = [(q, s, a, min(b, lim)) for q, s, a, b in self._spans if a < lim]
        return RawRunData(self._records(), list(self._iters), [list(v) for v in self._busy],
                          list(self._spans), self.makespan_ms, self.committed_tokens,
                          self.discarded_tokens, self.preemptions, self.truncated,
                          None if self._events is None else list(self._events))


def _remove_key(keys: list, key) -> None:
    i = bisect_left(keys, key)
    if i < len(keys) and keys[i] == key:
        del keys[i]
    else:  # pragma: no cover - state corruption
        raise AssertionError(f"key {key} not queued")


def _remove_prefix_ids(keys: list, ids: list[int], reqs: dict) -> None:
    """Drop launched ids; they are almost always a prefix of the FCFS queue."""
    if not ids:
        return
    n = len(ids)
    if n <= len(keys) and [k[1] for k in keys[:n]] == ids:
        del keys[:n]
        return
    for rid in ids:
        _remove_key(keys, reqs[rid].key)


class Engine(EngineCore):
    """Virtual-clock engine: the reference's discrete-event timeline, optionally driving GPUs.

    Time advances by `StageCostModel`/`CommModel`, so every decision is
    bit-exact with `tokensim.Engine` on the same trace; with an executor each
    launched micro-batch also runs on the device stages (launch at
    `_launch`, retire at the last-stage commit).
    """

    def __init__(self, requests: list[RequestSpec], scheduler: str = "throttle",
                 pipeline: PipelineConfig | None = None, kv_config: KvConfig | None = None,
                 throttle: ThrottleConfig | None = None, token_budget: int = 2048,
                 horizon_ms: float | None = None, record_events: bool = False,
                 executor=None, max_rows: int | None = None, measured_stage_times: bool = False,
                 prefix_caching: bool = False):
        super().__init__(requests, scheduler, pipeline, kv_config, throttle, token_budget,
                         executor, max_rows, prefix_caching)
        if horizon_ms is not None and horizon_ms < 0:
            raise ConfigError(f"horizon_ms must be >= 0, got {horizon_ms}")
        if measured_stage_times:
            n = len(getattr(executor, "stages", ()))
            if executor is None or not hasattr(executor, "stage_times_ms") or n != self._pipeline.depth:
                raise ConfigError("measured_stage_times needs an executor holding pipeline.depth stages "
                                  "with stage_times_ms(seq)")
        # Measured-time replay: each stage's duration is that stage's measured device time for this
        # micro-batch (all stages executed for real, one at a time on one GPU, CUDA-event timed)
        # instead of `stage_time`'s cost model; the event loop (in-order admission, transfers,
        # commit order, the schedule gate) is unchanged.
        self._measured = measured_stage_times
        self._horizon = horizon_ms
        self._events = [] if record_events else None
        depth = self._pipeline.depth
        self._expect = [0] * depth
        self._arrived_at: list[dict[int, float]] = [dict() for _ in range(depth)]
        self._heap: list[tuple[float, int, int, int, int]] = []
        self._eseq = 0
        self._unfinished = len(self._reqs)
        for rid in self._order:
            self._push(self._reqs[rid].spec.arrival_ms, _EV_ARRIVAL, rid, 0)

    def submit(self, spec: RequestSpec, prompt_ids=None) -> None:
        """Add a request at `spec.arrival_ms` (>= the engine clock) with optional real prompt ids."""
        if spec.arrival_ms < self.clock:
            raise ConfigError(f"request {spec.id} arrives at {spec.arrival_ms} ms, before the clock {self.clock}")
        self._add_request(spec, prompt_ids)
        self._unfinished += 1
        self._push(spec.arrival_ms, _EV_ARRIVAL, spec.id, 0)

    def _push(self, t: float, kind: int, a: int, b: int) -> None:
        heapq.heappush(self._heap, (t, self._eseq, kind, a, b))
        self._eseq += 1

    def step(self) -> bool:
        """Drain every event at the next timestamp, then schedule at most once (`engine.py:265-289`)."""
        heap = self._heap
        if not heap:
            stuck = tuple(sorted(rid for rid, r in self._reqs.items() if not r.finished))
            if stuck:
                raise UnschedulableError(f"no forward progress possible; stuck requests: {list(stuck)}", stuck)
            return False
        t = heap[0][0]
        if self._horizon is not None and t > self._horizon:
            self.truncated = True
            self.makespan_ms = self._horizon
            return False
        self.clock = t
        if t > self.makespan_ms:
            self.makespan_ms = t
        while heap and heap[0][0] == t:
            _, _, kind, a, b = heapq.heappop(heap)
            if kind == _EV_ARRIVAL:
                self._arrive(a)
                self._log(t, ARRIVAL, None, None, None)
            elif kind == _EV_STAGE:
                batch = self.in_flight[b]
                self._log(t, STAGE_COMPLETE, a, b, batch.plan)
                if a == self._pipeline.depth - 1:
                    self._commit(t, batch)
                else:
                    self._push(t + batch.transfer_ms, _EV_XFER, a + 1, b)
            else:
                self._log(t, TRANSFER_COMPLETE, a, b, self.in_flight[b].plan)
                self._arrived_at[a][b] = t
                self._admit(a)
        self._schedule(t)
        return True

    def run(self) -> RawRunData:
        while self.step():
            pass
        return self.raw_data()

    def _admit(self, stage: int) -> None:
        """In-order stage entry: start = max(arrival, stage free) (`engine.py:317-330`)."""
        pend = self._arrived_at[stage]
        while self._expect[stage] in pend:
            seq = self._expect[stage]
            start = max(pend.pop(seq), self._free_at[stage])
            b = self.in_flight[seq]
            end = start + (b.stage_list[stage] if b.stage_list is not None else b.stage_ms)
            self._busy[stage].append((start, end))
            self._spans.append((seq, stage, start, end))
            self._free_at[stage] = end
            self._expect[stage] += 1
            self._push(end, _EV_STAGE, stage, seq)

    def _schedule(self, t: float) -> None:
        if len(self.in_flight) >= self._pipeline.depth or self._free_at[0] > t:
            return
        plan = self._try_plan()
        if plan is None:
            return
        batch = self._make_batch(t, plan)
        self._log(t, SCHEDULE_POINT, 0, batch.seq, plan)
        if self.executor is not None:
            self.executor.launch(batch.meta)
            if self._measured:
                batch.stage_list = self.executor.stage_times_ms(batch.seq)
        end = t + (batch.stage_list[0] if batch.stage_list is not None else batch.stage_ms)
        self._busy[0].append((t, end))
        self._spans.append((batch.seq, 0, t, end))
        self._free_at[0] = end
        self._expect[0] += 1
        self._push(end, _EV_STAGE, 0, batch.seq)


def run(requests: list[RequestSpec], scheduler: str = "throttle", pipeline: PipelineConfig | None = None,
        kv_config: KvConfig | None = None, throttle: ThrottleConfig | None = None,
        token_budget: int = 2048, horizon_ms: float | None = None, record_events: bool = False,
        executor=None) -> RawRunData:
    return Engine(requests, scheduler, pipeline, kv_config, throttle, token_budget, horizon_ms,
                  record_events, executor).run()
