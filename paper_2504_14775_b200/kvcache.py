"""Paged KV-cache manager: page accounting plus physical page ids.

`KvCacheState` keeps the reference's accounting contract bit for bit
(`pkg/src/tokensim/kvcache.py:46-95`): per-request stored-token and page
counts, all-or-nothing `allocate`, `release` raising `KeyError` for unknown
ids, `idle_rate = free / total` as a float. `select_preemption_victim`
is the LIFO rule of `kvcache.py:98-109`.

The reference stops at counts. `PagedKvCache` adds what a GPU needs
(north-star item 1): each request owns an ordered list of physical page ids
drawn from a deterministic LIFO free stack, and every allocation appends
(row, page_index, page_id) triples to a delta log that the executor ships
to the device-resident block table once per micro-batch. Device-side slot
mapping (`slot = table[row, pos // ps] * ps + pos % ps`) is computed inside
the CUDA metadata kernel, never on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .errors import ConfigError


def pages_needed(current_tokens: int, new_tokens: int, page_size: int) -> int:
    """Extra pages to grow a request from current to current+new tokens (`kvcache.py:21-27`)."""
    if page_size < 1:
        raise ConfigError(f"page_size must be >= 1, got {page_size}")
    if current_tokens < 0 or new_tokens < 0:
        raise ConfigError("token counts must be >= 0")
    return -(-(current_tokens + new_tokens) // page_size) + (-current_tokens // page_size)


@dataclass(frozen=True)
class KvConfig:
    total_pages: int
    page_size: int

    def __post_init__(self) -> None:
        if self.total_pages < 1:
            raise ConfigError(f"kv.total_pages must be >= 1, got {self.total_pages}")
        if self.page_size < 1:
            raise ConfigError(f"kv.page_size must be >= 1, got {self.page_size}")

    @property
    def total_tokens(self) -> int:
        return self.total_pages * self.page_size


class KvCacheState:
    """Page pool with per-request token/page counts (reference-compatible)."""

    def __init__(self, config: KvConfig):
        self.config = config
        self.free_pages = config.total_pages
        self._tokens: dict[int, int] = {}
        self._pages: dict[int, int] = {}

    def stored_tokens(self, request_id: int) -> int:
        return self._tokens.get(request_id, 0)

    def pages(self, request_id: int) -> int:
        return self._pages.get(request_id, 0)

    @property
    def allocated_pages(self) -> int:
        return self.config.total_pages - self.free_pages

    @property
    def holders(self) -> tuple[int, ...]:
        return tuple(self._pages)

    def idle_rate(self) -> float:
        return self.free_pages / self.config.total_pages

    def allocate(self, request_id: int, new_tokens: int) -> bool:
        if new_tokens < 0:
            raise ConfigError(f"new_tokens must be >= 0, got {new_tokens}")
        if new_tokens == 0:
            return True
        have = self._tokens.get(request_id, 0)
        ps = self.config.page_size
        need = -(-(have + new_tokens) // ps) - (-(-have // ps))
        if need > self.free_pages:
            return False
        self.free_pages -= need
        self._tokens[request_id] = have + new_tokens
        self._pages[request_id] = self._pages.get(request_id, 0) + need
        if need:
            self._grant(request_id, need)
        return True

    def release(self, request_id: int) -> int:
        if request_id not in self._pages:
            raise KeyError(f"request {request_id} holds no pages")
        n = self._pages.pop(request_id)
        del self._tokens[request_id]
        self.free_pages += n
        self._revoke(request_id)
        return n

    def bulk_append_one(self, request_ids) -> bool:
        """Append one token to each request iff that needs no more pages than are free.

        Equivalent to calling `allocate(rid, 1)` in order when every call would
        succeed (each needs 0 or 1 page, so that holds exactly when the total fits);
        returns False and changes nothing otherwise. Sets `last_bulk_context` to
        the sum of the new stored lengths (the plan's decode context).
        """
        ps = self.config.page_size
        toks = self._tokens
        crossing = [rid for rid in request_ids if toks[rid] % ps == 0]
        if len(crossing) > self.free_pages:
            return False
        ctx = 0
        for rid in request_ids:
            v = toks[rid] + 1
            toks[rid] = v
            ctx += v
        pages = self._pages
        for rid in crossing:
            pages[rid] += 1
            self._grant(rid, 1)
        self.free_pages -= len(crossing)
        self.last_bulk_context = ctx
        return True

    # hooks for the physical layer
    def _grant(self, request_id: int, n_pages: int) -> None:
        pass

    def _revoke(self, request_id: int) -> None:
        pass


class PagedKvCache(KvCacheState):
    """KvCacheState plus physical page ids and a block-table delta log.

    Page ids come off a LIFO free stack initialised to ``0..total-1`` (page 0
    on top), so the same schedule always yields the same physical layout.
    Each request is bound to a block-table row by the caller (`bind_row`)
    before its first allocation.
    """

    def __init__(self, config: KvConfig):
        super().__init__(config)
        self._stack: list[int] = list(range(config.total_pages - 1, -1, -1))
        self._owned: dict[int, list[int]] = {}
        self._row: dict[int, int] = {}
        self._delta_row: list[int] = []
        self._delta_idx: list[int] = []
        self._delta_page: list[int] = []

    def bind_row(self, request_id: int, row: int) -> None:
        self._row[request_id] = row

    def unbind_row(self, request_id: int) -> None:
        self._row.pop(request_id, None)

    def row_of(self, request_id: int) -> int:
        return self._row[request_id]

    def page_ids(self, request_id: int) -> list[int]:
        return list(self._owned.get(request_id, ()))

    def _grant(self, request_id: int, n_pages: int) -> None:
        owned = self._owned.setdefault(request_id, [])
        row = self._row.get(request_id, -1)
        if row < 0:
            raise ConfigError(f"request {request_id} has no block-table row")
        base = len(owned)
        for k in range(n_pages):
            pid = self._stack.pop()
            owned.append(pid)
            self._delta_row.append(row)
            self._delta_idx.append(base + k)
            self._delta_page.append(pid)

    def _revoke(self, request_id: int) -> None:
        owned = self._owned.pop(request_id, [])
        # Return in reverse so a release followed by the same allocation pattern
        # hands back the same ids.
        self._stack.extend(reversed(owned))

    def take_deltas(self) -> np.ndarray:
        """Pending (row, page_index, page_id) triples as an int32 [n, 3] array; clears the log."""
        out = np.empty((len(self._delta_row), 3), dtype=np.int32)
        if len(self._delta_row):
            out[:, 0] = self._delta_row
            out[:, 1] = self._delta_idx
            out[:, 2] = self._delta_page
        self._delta_row.clear()
        self._delta_idx.clear()
        self._delta_page.clear()
        return out


def select_preemption_victim(candidates: Iterable[tuple[int, float]]) -> int | None:
    """Latest arrival loses; ties go to the larger id (`kvcache.py:98-109`)."""
    best = None
    for rid, arrival in candidates:
        if best is None or (arrival, rid) > best:
            best = (arrival, rid)
    return None if best is None else best[1]


def prompt_page_hashes(tokens, page_size: int) -> list[int]:
    """Chained hashes of the full pages of a prompt: h_i = H(h_{i-1}, tokens of page i). Equal
    hashes mean equal token prefixes (up to 64-bit collisions), so page i's KV can be shared."""
    import hashlib

    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
    out, prev = [], b""
    for i in range(len(t) // page_size):
        d = hashlib.blake2b(prev + t[i * page_size:(i + 1) * page_size].tobytes(), digest_size=8).digest()
        out.append(int.from_bytes(d, "little"))
        prev = d
    return out


class PrefixCachingKvCache(PagedKvCache):
    """PagedKvCache whose full prompt pages are shared between requests with the same token prefix
    (the paper's prefix caching, `PAPER.md:325`; absent from the reference's cost model).

    * Every physical page has a reference count. A prompt page whose KV is complete is registered
      under its chained prefix hash (`register`); a later request whose prompt starts with the
      same pages maps them into its block-table row (`match`) instead of recomputing them.
    * A page whose last holder releases it stays cached while its hash is registered: it counts
      as free for the scheduler (Token Throttling sees the same free/total ratio as without
      sharing) and is reclaimed least-recently-released first when the free stack runs dry.
    * Counts keep the reference's meaning per request: `stored_tokens` / `pages` include shared
      pages; `free_pages` counts each physical page once.
    """

    def __init__(self, config: KvConfig):
        super().__init__(config)
        from collections import OrderedDict

        self._ref: dict[int, int] = {}
        self._by_hash: dict[int, int] = {}
        self._hash_of: dict[int, int] = {}
        self._cached: "OrderedDict[int, None]" = OrderedDict()   # ref 0, hash registered: reclaimable
        self.hit_tokens = 0

    def _take_page(self) -> int:
        if self._stack:
            return self._stack.pop()
        pid, _ = self._cached.popitem(last=False)      # least recently released cached page
        del self._by_hash[self._hash_of.pop(pid)]
        return pid

    def _grant(self, request_id: int, n_pages: int) -> None:
        owned = self._owned.setdefault(request_id, [])
        row = self._row.get(request_id, -1)
        if row < 0:
            raise ConfigError(f"request {request_id} has no block-table row")
        base = len(owned)
        for k in range(n_pages):
            pid = self._take_page()
            self._ref[pid] = 1
            owned.append(pid)
            self._delta_row.append(row)
            self._delta_idx.append(base + k)
            self._delta_page.append(pid)

    def _revoke(self, request_id: int) -> None:
        owned = self._owned.pop(request_id, [])
        freed = []
        for pid in owned:
            r = self._ref[pid] - 1
            if r:
                self._ref[pid] = r
                continue
            del self._ref[pid]
            if pid in self._hash_of:
                self._cached[pid] = None
            else:
                freed.append(pid)
        self._stack.extend(reversed(freed))

    def release(self, request_id: int) -> int:
        """Release every page the request maps; `free_pages` grows by the pages no one else holds."""
        if request_id not in self._pages:
            raise KeyError(f"request {request_id} holds no pages")
        before = len(self._stack) + len(self._cached)
        n = self._pages.pop(request_id)
        del self._tokens[request_id]
        self._revoke(request_id)
        self.free_pages += len(self._stack) + len(self._cached) - before
        return n

    def match(self, request_id: int, hashes: list[int], max_pages: int) -> int:
        """Map the longest registered prefix (<= max_pages pages) of `hashes` into this request's
        row, which must hold no KV yet. Returns the tokens now cached (pages x page_size)."""
        if self._tokens.get(request_id, 0):
            raise ConfigError(f"request {request_id} already holds KV")
        row = self._row.get(request_id, -1)
        if row < 0:
            raise ConfigError(f"request {request_id} has no block-table row")
        pids = []
        for h in hashes[:max_pages]:
            pid = self._by_hash.get(h)
            if pid is None:
                break
            pids.append(pid)
        if not pids:
            return 0
        owned = self._owned.setdefault(request_id, [])
        for k, pid in enumerate(pids):
            if pid in self._cached:
                del self._cached[pid]
                self.free_pages -= 1
                self._ref[pid] = 1
            else:
                self._ref[pid] += 1
            owned.append(pid)
            self._delta_row.append(row)
            self._delta_idx.append(k)
            self._delta_page.append(pid)
        n_tok = len(pids) * self.config.page_size
        self._tokens[request_id] = n_tok
        self._pages[request_id] = len(pids)
        self.hit_tokens += n_tok
        return n_tok

    def register(self, request_id: int, hashes: list[int], n_tokens: int) -> None:
        """The request's first `n_tokens` prompt tokens have their KV written: publish the full
        pages among them under their prefix hashes (first writer wins)."""
        owned = self._owned.get(request_id, ())
        for i in range(min(n_tokens // self.config.page_size, len(hashes), len(owned))):
            h, pid = hashes[i], owned[i]
            if h in self._by_hash or pid in self._hash_of:
                continue
            self._by_hash[h] = pid
            self._hash_of[pid] = h
