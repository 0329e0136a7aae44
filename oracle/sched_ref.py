"""Plain restatement of the reference scheduler + KV accounting + event loop (TEST INFRASTRUCTURE).

Written for obviousness, not speed: every schedule point rescans all requests
and re-sorts both queues exactly as the reference does, so it is an
independent check on the product engine's incremental counters. Pinned
against the golden fixtures the reference itself produced
(tests/test_oracle_golden.py).

Citations are to /root/reference/pkg/src/tokensim/.
"""

from __future__ import annotations

import heapq
import math

EPS = 1e-9  # sched.py:30


def cdiv(a: int, b: int) -> int:                      # sched.py:38-39, kvcache.py:17-18
    return -(-a // b)


def pages_needed(cur: int, new: int, ps: int) -> int:  # kvcache.py:21-27
    return cdiv(cur + new, ps) - cdiv(cur, ps)


def prefill_wt(wp, T, min_p, max_p):                  # sched.py:136-141  (Eq. 1)
    if wp <= 0:
        return 0
    return min(min(max(cdiv(wp, T), min_p), max_p), wp)


def prefill_ut(kv_free, min_p, max_p):                # sched.py:144-146  (Eq. 2)
    return math.ceil(max(max_p * kv_free, float(min_p)) - EPS)


def prefill_combined(wp, kv_free, T, min_p, max_p, th):  # sched.py:149-157 (Eq. 3 + suspend)
    if wp <= 0 or kv_free <= th:
        return 0
    head = (kv_free - th) / (1.0 - th)
    return min(math.ceil(max(min(wp / T, max_p * head), float(min_p)) - EPS), wp)


def decode_count(rd, depth):                          # sched.py:160-168  (Eq. 4)
    return 0 if rd == 0 else cdiv(rd, depth)


def prefill_limit(wp, kv_free, cfg):                  # sched.py:171-181
    T, max_p, min_p, th, mode = cfg
    if wp <= 0 or kv_free <= th:
        return 0
    if mode == "combined":
        return prefill_combined(wp, kv_free, T, min_p, max_p, th)
    if mode == "wt_only":
        return prefill_wt(wp, T, min_p, max_p)
    return min(prefill_ut(kv_free, min_p, max_p), wp)


def fill(queue, limit, avail, ps):                    # sched.py:184-215
    """queue: [(id, remaining, stored)] FCFS."""
    out = []
    budget = limit
    avail = max(avail, 0)
    for rid, rem, stored in queue:
        if budget <= 0:
            break
        if rem <= 0:
            continue
        want = min(rem, budget)
        fit = (ps - stored % ps) % ps + avail * ps
        take = min(want, fit)
        if take <= 0:
            break
        avail -= pages_needed(stored, take, ps)
        budget -= take
        out.append((rid, take))
        if take < want:
            break
    return out


def plan(scheduler, wp, rd, free, total, ps, depth, pq, dq, cfg, budget):
    """sched.py:218-257. pq=[(id, remaining, stored)], dq=[(id, stored)] FCFS."""
    if scheduler == "throttle":
        chosen = dq[: decode_count(rd, depth)]
        limit = prefill_limit(wp, free / total, cfg)
    else:
        chosen = list(dq)
        limit = min(max(0, budget - len(chosen)), wp)
    reserve = sum(pages_needed(s, 1, ps) for _, s in chosen)
    chunks = fill(pq, limit, free - reserve, ps)
    return [r for r, _ in chosen], chunks, sum(s + 1 for _, s in chosen)


class Kv:                                             # kvcache.py:46-95
    def __init__(self, total, ps):
        self.total, self.ps, self.free = total, ps, total
        self.tok, self.pg = {}, {}

    def alloc(self, rid, n):
        if n == 0:
            return True
        need = pages_needed(self.tok.get(rid, 0), n, self.ps)
        if need > self.free:
            return False
        self.free -= need
        self.tok[rid] = self.tok.get(rid, 0) + n
        self.pg[rid] = self.pg.get(rid, 0) + need
        return True

    def release(self, rid):
        n = self.pg.pop(rid)
        del self.tok[rid]
        self.free += n
        return n


class RefEngine:
    """engine.py:175-558 restated. `forward(plan_tuple)` is called at each launch (CPU model hook)."""

    def __init__(self, reqs, scheduler="throttle", depth=4, total_pages=4096, ps=16,
                 cfg=(8, 2048, 32, 0.05, "combined"), budget=2048, cost=(1.0, 0.01, 0.1),
                 comm=(0.1, 16384.0, 20.79e6), forward=None):
        self.reqs = {r[0]: dict(id=r[0], arr=r[1], inp=r[2], out=r[3], target=r[2], done=0, infl=0, gen=0,
                                pre=0, inc=0, arrived=False, dec=False, first=None, fin=None) for r in reqs}
        self.sched, self.depth, self.cfg, self.budget = scheduler, depth, cfg, budget
        self.cost, self.comm = cost, comm
        self.kv = Kv(total_pages, ps)
        self.forward = forward
        self.heap, self.eseq = [], 0
        self.waiting, self.ready = [], []
        self.free_at = [0.0] * depth
        self.nxt = [0] * depth
        self.pend = [dict() for _ in range(depth)]
        self.inflight = {}
        self.iters, self.spans = [], []
        self.seq = 0
        self.makespan = 0.0
        self.committed = self.discarded = self.preemptions = 0
        for r in reqs:
            self.push(r[1], "arr", r[0], 0)

    def push(self, t, kind, a, b):
        heapq.heappush(self.heap, (t, self.eseq, kind, a, b))
        self.eseq += 1

    def key(self, rid):
        return (self.reqs[rid]["arr"], rid)

    def stage_ms(self, d, p, ctx):                    # engine.py:96-100
        if d + p == 0:
            return 0.0
        c0, ct, cc = self.cost
        return c0 + ct * (d + p) + cc * ctx / 1024.0

    def run(self, max_iters=None, stop=None):
        while self.heap and not (stop is not None and stop()):
            t = self.heap[0][0]
            self.makespan = max(self.makespan, t)
            while self.heap and self.heap[0][0] == t:
                _, _, kind, a, b = heapq.heappop(self.heap)
                if kind == "arr":
                    self.reqs[a]["arrived"] = True
                    self.waiting.append(a)
                elif kind == "stage":
                    if a == self.depth - 1:
                        self.commit(t, self.inflight.pop(b))
                    else:
                        self.push(t + self.inflight[b]["xfer_ms"], "xfer", a + 1, b)
                else:
                    self.pend[a][b] = t
                    while self.nxt[a] in self.pend[a]:
                        s = self.nxt[a]
                        st = max(self.pend[a].pop(s), self.free_at[a])
                        en = st + self.inflight[s]["ms"]
                        self.spans.append((s, a, st, en))
                        self.free_at[a] = en
                        self.nxt[a] += 1
                        self.push(en, "stage", a, s)
            self.schedule(t)
            if max_iters is not None and len(self.iters) >= max_iters:
                break
        return self

    def schedule(self, t):
        while len(self.inflight) < self.depth and self.free_at[0] <= t and (self.waiting or self.ready):
            self.waiting.sort(key=self.key)
            self.ready.sort(key=self.key)
            wp = rd = 0
            for r in self.reqs.values():
                if r["arrived"] and r["fin"] is None:
                    if r["dec"]:
                        rd += 1
                    else:
                        wp += r["target"] - r["done"] - r["infl"]
            pq = [(rid, self.reqs[rid]["target"] - self.reqs[rid]["done"], self.kv.tok.get(rid, 0)) for rid in self.waiting]
            dq = [(rid, self.kv.tok.get(rid, 0)) for rid in self.ready]
            dec, chunks, _ = plan(self.sched, wp, rd, self.kv.free, self.kv.total, self.kv.ps, self.depth,
                                  pq, dq, self.cfg, self.budget)
            mutated = False
            kept, dropped = [], set()
            for rid in dec:                            # engine.py:456-473
                if rid in dropped:
                    continue
                while not self.kv.alloc(rid, 1):
                    victim = max(self.ready, key=self.key)
                    self.preempt(victim)
                    mutated = True
                    dropped.add(victim)
                    if victim == rid:
                        break
                    if victim in kept:
                        kept.remove(victim)
                else:
                    kept.append(rid)
            ctx = sum(self.kv.tok[r] for r in kept)
            for rid, n in chunks:
                assert self.kv.alloc(rid, n)
            if not kept and not chunks:
                if mutated:
                    continue
                return
            self.launch(t, kept, chunks, ctx)
            return

    def preempt(self, rid):                           # engine.py:371-384
        r = self.reqs[rid]
        self.kv.release(rid)
        self.preemptions += 1
        r["pre"] += 1
        self.discarded += r["inc"]
        r["inc"] = 0
        r["target"] = r["inp"] + max(r["gen"] - 1, 0)
        r["done"] = 0
        r["dec"] = False
        self.ready.remove(rid)
        self.waiting.append(rid)

    def launch(self, t, dec, chunks, ctx):            # engine.py:482-516
        s = self.seq
        self.seq += 1
        p = sum(n for _, n in chunks)
        ms = self.stage_ms(len(dec), p, ctx)
        lat, bpt, bw = self.comm                       # engine.py:103-105
        self.inflight[s] = dict(dec=dec, chunks=chunks, ms=ms, tokens=len(dec) + p,
                                xfer_ms=lat + (len(dec) + p) * bpt / bw)
        for rid, n in chunks:
            self.reqs[rid]["infl"] = n
        taken = set(dec) | {r for r, _ in chunks}
        self.waiting = [r for r in self.waiting if r not in taken]
        self.ready = [r for r in self.ready if r not in taken]
        self.iters.append((s, t, p, len(dec)))
        self.spans.append((s, 0, t, t + ms))
        self.free_at[0] = t + ms
        self.nxt[0] += 1
        self.push(t + ms, "stage", 0, s)
        if self.forward is not None:
            self.forward(s, dec, chunks, {rid: self.kv.tok[rid] for rid in dec}, self.reqs)

    def commit(self, t, b):                           # engine.py:334-369
        self.committed += b["tokens"]
        for rid in b["dec"]:
            r = self.reqs[rid]
            r["gen"] += 1
            r["inc"] += 1
            if r["gen"] >= r["out"]:
                self.finish(r, t)
            else:
                self.ready.append(rid)
        for rid, n in b["chunks"]:
            r = self.reqs[rid]
            r["infl"] = 0
            r["done"] += n
            r["inc"] += n
            if r["done"] >= r["target"]:
                r["dec"] = True
                if r["gen"] == 0:
                    r["gen"] = 1
                    r["first"] = t
                    if r["gen"] >= r["out"]:
                        self.finish(r, t)
                        continue
                self.ready.append(rid)
            else:
                self.waiting.append(rid)

    def finish(self, r, t):
        r["fin"] = t
        r["dec"] = False
        self.kv.release(r["id"])
