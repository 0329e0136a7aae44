"""Wall-clock serving loop: the same request state machine as `Engine`, driven by real time.

Arrivals are released when the wall clock passes their `arrival_ms`; a
micro-batch commits when its device work has finished (its sampled tokens are
on the host), and the commit time is the request's TTFT / completion stamp.
Scheduling keeps the reference gate (`engine.py:391-398`): fewer than `depth`
batches in flight and stage 0 free, at most one launch per scheduling point.

Per-stage busy intervals come from CUDA events on the stage streams, so
`bubble_accounting` (`engine.py:108-125`) reports the measured pipeline
bubble on the same definition the reference simulates.

Every schedule point can be logged (`record_decisions=True`) as
(#WP, #RD, free pages, FCFS queues, plan) for decision-replay parity against
the reference planner.
"""

from __future__ import annotations

import time
from bisect import bisect_left
from collections import deque

from .engine import EngineCore, PipelineConfig, RawRunData
from .errors import UnschedulableError
from .kvcache import KvConfig
from .metrics import IterationRecord
from .sched import ThrottleConfig


class ServingEngine(EngineCore):
    def __init__(self, requests, scheduler: str = "throttle", pipeline: PipelineConfig | None = None,
                 kv_config: KvConfig | None = None, throttle: ThrottleConfig | None = None,
                 token_budget: int = 2048, executor=None, max_rows: int | None = None,
                 time_scale: float = 1.0, record_decisions: bool = False, lookahead: bool = False,
                 prefix_caching: bool = False):
        if executor is None:
            raise ValueError("ServingEngine needs a GPU executor")
        super().__init__(requests, scheduler, pipeline, kv_config, throttle, token_budget, executor, max_rows,
                         prefix_caching)
        self._arrivals = sorted(requests, key=lambda s: (s.arrival_ms, s.id))
        self._arrival_keys = [(s.arrival_ms, s.id) for s in self._arrivals]
        self._next_arrival = 0
        self._time_scale = time_scale
        self._t0 = None
        self._unfinished = len(requests)
        self.decisions: list[tuple] | None = [] if record_decisions else None
        self.commit_log: list[tuple[int, float, int]] = []   # (seq, commit wall ms, sampled tokens)
        self.launch_log: list[tuple[int, float]] = []        # (seq, launch wall ms)
        self._lookahead = lookahead
        self._pending: deque = deque()      # lookahead: launched batches the device has not retired
        self._uncommitted: deque = deque()  # lookahead: launched batches whose commit is not applied yet

    def now_ms(self) -> float:
        if self._t0 is None:
            return 0.0
        return (time.perf_counter() - self._t0) * 1000.0 * self._time_scale

    def submit(self, spec, prompt_ids=None) -> None:
        """Front-end request intake (`PAPER.md:252`): the request arrives at `spec.arrival_ms` on the
        serving clock (ms since `run` started; pass `now_ms()` for "now"), optionally with its real
        prompt token ids. Safe to call before `run` or from `on_commit` callbacks during it."""
        self._add_request(spec, prompt_ids)
        self._unfinished += 1
        key = (spec.arrival_ms, spec.id)
        i = len(self._arrivals)
        if self._arrival_keys and key < self._arrival_keys[-1]:
            i = max(bisect_left(self._arrival_keys, key), self._next_arrival)
        self._arrivals.insert(i, spec)
        self._arrival_keys.insert(i, key)

    def outputs(self, request_id: int) -> list[int]:
        """Sampled token ids of a request so far (retired micro-batches only)."""
        return list(getattr(self.executor, "outputs", {}).get(request_id, []))

    def _release_arrivals(self, t: float) -> None:
        arr = self._arrivals
        while self._next_arrival < len(arr) and arr[self._next_arrival].arrival_ms <= t:
            self._arrive(arr[self._next_arrival].id)
            self._next_arrival += 1

    def _decision_snapshot(self):
        kv = self.kv
        return (self._wp, self._rd, kv.free_pages, [k[1] for k in self._waiting], [k[1] for k in self._ready],
                {rid: (self._reqs[rid].target - self._reqs[rid].done, kv.stored_tokens(rid))
                 for _, rid in self._waiting},
                {rid: kv.stored_tokens(rid) for _, rid in self._ready})

    def _launch_now(self, t: float) -> bool:
        if len(self.in_flight) >= self._pipeline.depth or not self.executor.stage0_idle():
            return False
        snap = self._decision_snapshot() if self.decisions is not None else None
        plan = self._try_plan()
        if plan is None:
            return False
        batch = self._make_batch(t, plan)
        if snap is not None:
            self.decisions.append((batch.seq, snap, list(plan.decode_ids), list(plan.prefill_chunks)))
        self.executor.launch(batch.meta)
        self.launch_log.append((batch.seq, t))
        return True

    def run(self, max_commits: int | None = None, on_commit=None) -> RawRunData:
        """Serve until every request finished (or `max_commits` micro-batches committed)."""
        if self._lookahead:
            return self._run_lookahead(max_commits, on_commit)
        ex = self.executor
        self._t0 = time.perf_counter()
        ex.mark_epoch()
        commits = 0
        while self._unfinished > 0:
            t = self.now_ms()
            self._release_arrivals(t)
            if self._launch_now(t):
                continue
            if self.in_flight:
                seq = min(self.in_flight)
                ex.wait(seq)
                t = self.now_ms()
                self.clock = t
                self.makespan_ms = max(self.makespan_ms, t)
                batch = self.in_flight[seq]
                n_out = batch.meta.n_emit
                self._commit(t, batch)
                self.commit_log.append((seq, t, n_out))
                commits += 1
                if on_commit is not None:
                    on_commit(seq, t, n_out)
                if max_commits is not None and commits >= max_commits:
                    break
                continue
            if self._next_arrival < len(self._arrivals):
                wait = (self._arrivals[self._next_arrival].arrival_ms - t) / 1000.0 / self._time_scale
                if wait > 0:
                    time.sleep(min(wait, 0.05))
                continue
            stuck = tuple(sorted(rid for rid, r in self._reqs.items() if not r.finished))
            raise UnschedulableError(f"no forward progress possible; stuck requests: {list(stuck)}", stuck)
        ex.synchronize()
        self._busy = ex.stage_busy_intervals()
        return self.raw_data()

    # -- asynchronous scheduling -------------------------------------------------------
    #
    # Scheduling never reads token values (termination is by output count,
    # `engine.py:343`), and a batch's device work depends on earlier batches only through
    # device memory written in stream order (sampled ids -> token history, KV pages). In the
    # reference at depth D, batch b is planned right after batch b-D commits, with batches
    # b-D+1..b-1 still in flight (`engine.py:391-398`). So right after launching batch b-1 the
    # host can apply batch b-D's commit to the request state (FIFO of D launched batches),
    # plan batch b and enqueue it: the plan sees exactly the state the reference would, and the
    # device orders b's forward after b-D's sampled tokens (executor `lag` = D). At D = 1 this
    # is "commit i right after launching it, plan i+1". Times are stamped when the device
    # actually finishes a batch; with lookahead off the loop waits for each commit instead.

    def _state_commit(self, t: float) -> None:
        """Apply the oldest uncommitted batch's commit to the request state (provisional times)."""
        entry = self._uncommitted.popleft()
        batch = entry["batch"]
        ids = batch.meta.ids if batch.meta is not None else \
            batch.plan.decode_ids + [r for r, _ in batch.plan.prefill_chunks]
        reqs = self._reqs
        no_first = [rid for rid in ids if reqs[rid].first_ms is None]
        no_finish = [rid for rid in ids if reqs[rid].finish_ms is None]
        self._commit(t, batch, retire=False)
        entry["firsts"] = [rid for rid in no_first if reqs[rid].first_ms is not None]
        entry["done"] = [rid for rid in no_finish if reqs[rid].finish_ms is not None]
        entry["committed"] = True

    def _launch_ahead(self, t: float) -> bool:
        depth = self._pipeline.depth
        if len(self._pending) > depth:
            return False
        if self._uncommitted and len(self._uncommitted) >= depth:
            self._state_commit(t)
        snap = self._decision_snapshot() if self.decisions is not None else None
        plan = self._try_plan()
        if plan is None:
            return False
        batch = self._make_batch(t, plan)
        if snap is not None:
            self.decisions.append((batch.seq, snap, list(plan.decode_ids), list(plan.prefill_chunks)))
        self.executor.launch(batch.meta)
        self.launch_log.append((batch.seq, t))
        entry = {"batch": batch, "committed": False, "firsts": [], "done": []}
        self._pending.append(entry)
        self._uncommitted.append(entry)
        if depth == 1:
            self._state_commit(t)     # nothing else can be in flight: plan the next batch now
        return True

    def _run_lookahead(self, max_commits, on_commit) -> RawRunData:
        ex = self.executor
        self._t0 = time.perf_counter()
        ex.mark_epoch()
        commits = 0
        while self._unfinished > 0 or self._pending:
            t = self.now_ms()
            self._release_arrivals(t)
            if self._unfinished > 0 and self._launch_ahead(t):
                continue
            if self._pending:
                entry = self._pending[0]
                batch = entry["batch"]
                ex.wait(batch.seq)
                ex.retire(batch.seq)
                t = self.now_ms()
                self.clock = t
                self.makespan_ms = max(self.makespan_ms, t)
                if not entry["committed"]:       # nothing newer was planned: commit on completion
                    self._state_commit(t)
                self._pending.popleft()
                for rid in entry["firsts"]:
                    self._reqs[rid].first_ms = t
                for rid in entry["done"]:
                    self._reqs[rid].finish_ms = t
                n_out = batch.meta.n_emit
                self.commit_log.append((batch.seq, t, n_out))
                commits += 1
                if on_commit is not None:
                    on_commit(batch.seq, t, n_out)
                if max_commits is not None and commits >= max_commits:
                    break
                continue
            if self._next_arrival < len(self._arrivals):
                wait = (self._arrivals[self._next_arrival].arrival_ms - t) / 1000.0 / self._time_scale
                if wait > 0:
                    time.sleep(min(wait, 0.05))
                continue
            stuck = tuple(sorted(rid for rid, r in self._reqs.items() if not r.finished))
            raise UnschedulableError(f"no forward progress possible; stuck requests: {list(stuck)}", stuck)
        ex.synchronize()
        self._busy = ex.stage_busy_intervals()
        return self.raw_data()

    def _finish(self, r, t):  # count completions for the loop condition
        super()._finish(r, t)
        self._unfinished -= 1

