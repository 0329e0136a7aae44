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
