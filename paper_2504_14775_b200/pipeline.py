"""Pipeline-parallel runtime: one process per GPU, stage s holds layers stage_layers(L, PP, s).

Real counterpart of the reference's simulated pipeline (`engine.py:85-93,
296-330`): the reference charges `transfer_time()` per hop and admits batches
to each stage in sequence order; here rank s runs stage s on its own GPU and
the hops are real messages:

* metadata  : rank 0 (driver + stage 0) -> every rank, on a CPU (gloo) group,
              sent ahead of the activations (the paper's dual-phase design,
              `PAPER.md:262`): header [seq, n_seqs, n_tokens, n_emit, n_work,
              n_prefill_work, n_deltas, n_prompts, n_ints] + the packed int32 buffer.
* activations: rank s -> s+1, `[n_tokens, d]` bf16 residual stream (NCCL
              send/recv over NVLink on a dedicated comm stream).
* tokens    : last rank -> rank 0, `[n_emit]` int32 sampled ids, written into
              stage 0's token history as the next decode inputs.

Every rank processes micro-batches strictly in `seq` order (in-order stage
admission, `engine.py:317-330`), so the point-to-point message order is
identical on both ends of every link and no size handshake is needed: the
receiver learns `n_tokens`/`n_emit` from the metadata that arrived first.

The activation transport is pluggable: `NcclTransport` (product, device
buffers) and `HostTransport` (tests: host staging over the gloo group, which
lets a 2-process pipeline share one GPU or run on CPU test doubles).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np

from .modelspec import ModelSpec, stage_layers
from .stage import (PackedBatch, StageWorker, default_max_rows, default_max_seq_len, pack_batch,
                    prompt_source_with)

HEADER = 10
STOP = -1
FLAG_PROFILE = 1   # header flag: capture this batch with the native profiler on every rank


def header_of(pb: PackedBatch) -> np.ndarray:
    return np.array([pb.seq, pb.n_seqs, pb.n_tokens, pb.n_emit, pb.n_work, pb.n_prefill_work, pb.n_deltas,
                     pb.n_prompts, pb.flags, pb.data.size], dtype=np.int32)


def batch_from(header: np.ndarray, data: np.ndarray) -> PackedBatch:
    seq, n_seqs, n_tokens, n_emit, n_work, n_pf, n_deltas, n_prompts, flags, _ = (int(x) for x in header)
    return PackedBatch(seq, n_seqs, n_tokens, n_emit, n_work, n_pf, n_deltas, n_prompts, data, [], [], flags)


# ------------------------------------------------------------------ transports


class MetaChannel:
    """Driver -> workers metadata on a CPU process group (async sends from rank 0)."""

    def __init__(self, group, world: int):
        self.group = group
        self.world = world
        self._pending = []

    def publish(self, pb: PackedBatch | None) -> None:
        import torch
        import torch.distributed as dist

        h = header_of(pb) if pb is not None else np.full(HEADER, STOP, dtype=np.int32)
        ht = torch.from_numpy(h.copy())
        dt = torch.from_numpy(pb.data.copy()) if pb is not None else None
        self._pending = [(w, t) for w, t in self._pending if not w.is_completed()]
        for r in range(1, self.world):
            self._pending.append((dist.isend(ht, dst=r, group=self.group), ht))
            if dt is not None and dt.numel():
                self._pending.append((dist.isend(dt, dst=r, group=self.group), dt))

    def receive(self) -> PackedBatch | None:
        import torch
        import torch.distributed as dist

        ht = torch.empty(HEADER, dtype=torch.int32)
        dist.recv(ht, src=0, group=self.group)
        h = ht.numpy().copy()
        if h[0] == STOP:
            return None
        dt = torch.empty(int(h[-1]), dtype=torch.int32)
        if dt.numel():
            dist.recv(dt, src=0, group=self.group)
        return batch_from(h, dt.numpy())

    def flush(self) -> None:
        for w, _ in self._pending:
            w.wait()
        self._pending = []


class NcclTransport:
    """Device-to-device P2P over NVLink, one NCCL communicator per directed link.

    `links[(src, dst)]` is a two-rank NCCL group. Separate communicators matter: NCCL runs
    each communicator's operations in order on its own stream, so on a single shared
    communicator rank 0's send of batch i+1's activations would queue behind its receive of
    batch i's sampled ids, which completes only after batch i has left the last stage --
    serialising the pipeline. With one communicator per link (and a distinct one for the
    token return path, even at PP=2) every hop progresses independently.
    """

    def __init__(self, rank: int, links: dict):
        self.rank = rank
        self.links = links

    def send(self, tensor, dst: int, stream) -> None:
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(stream) if stream is not None else _null():
            dist.send(tensor, dst=dst, group=self.links[(self.rank, dst)])

    def recv(self, tensor, src: int, stream) -> None:
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(stream) if stream is not None else _null():
            dist.recv(tensor, src=src, group=self.links[(src, self.rank)])


def make_links(world: int, backend: str = "nccl") -> dict:
    """Two-rank groups for stage s -> s+1 and for last -> 0 (collective: every rank calls it;
    `backend="gloo"` gives the CPU tests the same routing)."""
    import torch.distributed as dist

    links = {}
    for s in range(world - 1):
        links[(s, s + 1)] = dist.new_group([s, s + 1], backend=backend)
    if world > 1:
        links[(world - 1, 0)] = dist.new_group([0, world - 1], backend=backend)
    return links


class HostTransport:
    """Test transport: stage through host memory over a gloo group (sync, in order)."""

    def __init__(self, group):
        self.group = group

    def send(self, tensor, dst: int, stream) -> None:
        import torch.distributed as dist

        if stream is not None:
            stream.synchronize()
        dist.send(tensor.detach().to("cpu"), dst=dst, group=self.group)

    def recv(self, tensor, src: int, stream) -> None:
        import torch
        import torch.distributed as dist

        buf = torch.empty(tensor.shape, dtype=tensor.dtype)
        dist.recv(buf, src=src, group=self.group)
        with torch.cuda.stream(stream) if tensor.is_cuda else _null():
            tensor.copy_(buf, non_blocking=False)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ------------------------------------------------------------------ driver side (rank 0)


@dataclass
class _Flight:
    pb: PackedBatch
    fwd_done: object      # CUDA event: stage-0 forward finished (stage 0 free again)
    done: object          # CUDA event: sampled tokens committed to the history and copied to the host
    host: object


class _PinnedSlots:
    """Pinned host staging for the metadata of the last `n` micro-batches (H2D copies stay async):
    slot k is rewritten only after the copy that last read it (event) has run."""

    def __init__(self, n: int, n_ints: int, pinned: bool):
        import torch

        self.pinned = pinned
        self.host = [torch.empty(n_ints, dtype=torch.int32, pin_memory=pinned) for _ in range(n)]
        self.read = [None] * n

    def stage(self, k: int, data: np.ndarray):
        import torch

        if self.read[k] is not None:
            self.read[k].synchronize()
        if data.size > self.host[k].numel():
            self.host[k] = torch.empty(2 * data.size, dtype=torch.int32, pin_memory=self.pinned)
        self.host[k][: data.size].numpy()[:] = data
        return self.host[k][: data.size]


class PipelineExecutor:
    """Executor protocol (see executor.py) for rank 0 of a PP=world pipeline.

    Rank 0 holds stage 0 and the token history; it publishes each launched micro-batch's
    metadata, runs stage 0 on the compute stream, sends the activations to rank 1 on the send
    stream and receives the sampled ids from the last rank on the recv stream, where they are
    also committed into the token history and copied to the host. Nothing on the compute stream
    waits for a batch's own round trip: batch b's forward waits only for
      * the sampled ids of batch b - `lag` (the newest batch whose commit the scheduler had
        applied when it planned b: `lag` = depth, see ServingEngine lookahead), and
      * the send / token receive of batch b - ring (ring slot k = b % ring is reused).
    so stage 0 runs batch b+1 while b is on later stages (inter-batch overlap, `PAPER.md:258-263`).
    """

    def __init__(self, spec: ModelSpec, requests, *, world: int, meta: MetaChannel, transport, num_pages: int,
                 page_size: int = 16, max_tokens: int = 4096, max_emit: int | None = None, seed: int = 0,
                 device="cuda", stage_factory=None, ring: int = 8, max_rows: int | None = None,
                 max_seq_len: int | None = None, lag: int | None = None):
        import torch

        self.spec = spec
        self.world = world
        self.meta = meta
        self.transport = transport
        self.device = torch.device(device)
        self.specs = {r.id: r for r in requests}
        max_rows = max_rows if max_rows is not None else default_max_rows(requests, num_pages)
        max_seq_len = max_seq_len if max_seq_len is not None else default_max_seq_len(requests)
        self.max_emit = max_emit if max_emit is not None else max(1, min(max_rows, max_tokens))
        factory = stage_factory or StageWorker
        self.stage = factory(spec, stage_layers(spec.n_layers, world, 0), is_first=True, is_last=(world == 1),
                             num_pages=num_pages, page_size=page_size, max_rows=max_rows, max_seq_len=max_seq_len,
                             max_tokens=max_tokens, max_emit=self.max_emit, seed=seed, device=self.device)
        self.q_tile = self.stage.q_tile
        self.prompts: dict[int, np.ndarray] = {}
        self.prompt_source = prompt_source_with(self.prompts, self.specs, spec.vocab)
        on_gpu = self.device.type == "cuda"
        self.on_gpu = on_gpu
        self.compute = torch.cuda.Stream(device=self.device) if on_gpu else None
        # separate streams: activations out to rank 1 must not queue behind the token
        # receive from the last rank (different peers, independent progress)
        self.send_stream = torch.cuda.Stream(device=self.device) if on_gpu else None
        self.recv_stream = torch.cuda.Stream(device=self.device) if on_gpu else None
        ring = max(ring, world + 2)    # depth batches in flight + one queued + one being packed
        self.ring = ring
        self.lag = lag if lag is not None else world
        n_ints = 16 * max_tokens + 8 * max_rows + 4 * max_seq_len
        self.hidden = [torch.empty((max_tokens, spec.d_model), dtype=torch.bfloat16, device=self.device)
                       for _ in range(ring)]
        self.sampled = [torch.empty(self.max_emit, dtype=torch.int32, device=self.device) for _ in range(ring)]
        self.sampled_host = [torch.empty(self.max_emit, dtype=torch.int32, pin_memory=on_gpu) for _ in range(ring)]
        self.meta_dev = [torch.empty(n_ints, dtype=torch.int32, device=self.device) for _ in range(ring)]
        self.staging = _PinnedSlots(ring, n_ints, on_gpu)
        self._slot_free = [None] * ring      # event: slot k's send + token commit of its last batch done
        self._tok_done: dict[int, object] = {}
        self._inflight: dict[int, _Flight] = {}
        self._done: dict[int, object] = {}   # seq -> tokens-committed event (device windows)
        self._last_fwd = None
        self.outputs: dict[int, list[int]] = {}
        self.timings: list = []
        self._epoch = None
        self.launches = 0
        self.publish_flags = 0
        self.h2d_bytes: dict[int, int] = {}
        if on_gpu:
            torch.cuda.synchronize(self.device)

    def _event(self):
        import torch
        return torch.cuda.Event(enable_timing=True) if self.on_gpu else _HostEvent()

    def _record(self, ev, stream):
        ev.record(stream) if stream is not None else ev.record()
        return ev

    def register_prompt(self, request_id: int, tokens) -> None:
        self.prompts[request_id] = np.asarray(tokens, dtype=np.int32)

    def add_request(self, spec) -> None:
        self.specs[spec.id] = spec

    def launch(self, meta) -> None:
        import torch

        pb = pack_batch(meta, self.q_tile, self.prompt_source)
        pb.flags = self.publish_flags
        seq, k = pb.seq, pb.seq % self.ring
        self.meta.publish(pb)                         # metadata ahead of activations
        md = self.meta_dev[k]
        if pb.data.size > md.numel():
            self.meta_dev[k] = md = torch.empty(2 * pb.data.size, dtype=torch.int32, device=self.device)
        staged = self.staging.stage(k, pb.data)
        self.h2d_bytes[seq] = int(pb.data.nbytes)
        a, b = self._event(), self._event()
        with _on(self.compute):
            if self.on_gpu:
                if self._slot_free[k] is not None:        # batch seq - ring released slot k
                    self.compute.wait_event(self._slot_free[k])
                dep = self._tok_done.pop(seq - self.lag, None)
                if dep is not None:                       # decode inputs sampled by batch seq - lag
                    self.compute.wait_event(dep)
            md[: pb.data.size].copy_(staged, non_blocking=True)
            self.staging.read[k] = self._record(self._event(), self.compute)
            self._record(a, self.compute)
            self.stage.forward(pb, md, hidden=self.hidden[k], sampled=self.sampled[k], stream=self.compute)
            self._record(b, self.compute)
        host = self.sampled_host[k]
        if self.world > 1:
            if self.on_gpu:
                self.send_stream.wait_event(b)
            self.transport.send(self.hidden[k][: pb.n_tokens], 1, self.send_stream)
            sent = self._record(self._event(), self.send_stream)
            with _on(self.recv_stream):
                if self.on_gpu:
                    self.recv_stream.wait_event(sent)     # slot k free only after both
                if pb.n_emit:
                    self.transport.recv(self.sampled[k][: pb.n_emit], self.world - 1, self.recv_stream)
                    self.stage.commit_tokens(pb, md, self.sampled[k], stream=self.recv_stream)
                    host[: pb.n_emit].copy_(self.sampled[k][: pb.n_emit], non_blocking=True)
                done = self._record(self._event(), self.recv_stream)
        else:
            with _on(self.compute):
                if pb.n_emit:
                    host[: pb.n_emit].copy_(self.sampled[k][: pb.n_emit], non_blocking=True)
                done = self._record(self._event(), self.compute)
        self._slot_free[k] = done
        self._tok_done[seq] = done
        self._done[seq] = done
        self._inflight[seq] = _Flight(pb, b, done, host)
        self._last_fwd = b
        self.timings.append((seq, [(a, b)]))
        self.launches += 1

    def stage0_idle(self) -> bool:
        return self._last_fwd is None or self._last_fwd.query()

    def wait(self, seq: int) -> None:
        self._inflight[seq].done.synchronize()

    def retire(self, seq: int) -> list[int]:
        f = self._inflight.pop(seq)
        f.done.synchronize()
        if self.on_gpu:
            from . import native
            native.check_meta_errors()
        toks = f.host[: f.pb.n_emit].tolist()
        for rid, tok in zip(f.pb.emit_ids, toks):
            self.outputs.setdefault(rid, []).append(tok)
        return toks

    def on_finish(self, request_id: int, row: int) -> None:
        self.prompts.pop(request_id, None)

    def mark_epoch(self) -> None:
        self._epoch = self._record(self._event(), self.compute)
        self.timings.clear()

    def synchronize(self) -> None:
        if self.compute is not None:
            self.compute.synchronize()
            self.send_stream.synchronize()
            self.recv_stream.synchronize()

    def stage_busy_intervals(self) -> list[list[tuple[float, float]]]:
        self.synchronize()
        if self._epoch is None:
            return [[]]
        return [[(self._epoch.elapsed_time(a), self._epoch.elapsed_time(b)) for _, ((a, b),) in self.timings]]

    def batch_device_ms(self) -> dict[int, float]:
        self.synchronize()
        return {seq: a.elapsed_time(b) for seq, ((a, b),) in self.timings}

    def device_window_ms(self, first: int, last: int) -> float:
        """Device time from stage 0 starting batch `first` to batch `last`'s sampled tokens being
        committed (they return from the last stage): the pipeline's whole span on this GPU."""
        self.synchronize()
        start = next(a for s, ((a, _),) in self.timings if s == first)
        return start.elapsed_time(self._done[last])

    def stage_busy_ms(self, first: int, last: int) -> float:
        self.synchronize()
        return sum(a.elapsed_time(b) for s, ((a, b),) in self.timings if first <= s <= last)

    def h2d_bytes_total_for(self, seqs) -> int:
        return sum(self.h2d_bytes.get(s, 0) for s in seqs)

    def shutdown(self) -> None:
        self.meta.publish(None)
        self.meta.flush()


# ------------------------------------------------------------------ worker side (ranks >= 1)


def worker_loop(spec: ModelSpec, requests, *, rank: int, world: int, meta: MetaChannel, transport, num_pages: int,
                page_size: int = 16, max_tokens: int = 4096, max_emit: int | None = None, seed: int = 0,
                device="cuda", stage_factory=None, ring: int = 8, max_rows: int | None = None,
                max_seq_len: int | None = None, stage=None) -> dict:
    """Run stage `rank` until the driver publishes STOP; returns per-batch CUDA-event spans.

    The host loop never waits on the device except to reuse a pinned metadata slot (ring
    batches back): metadata is received on the CPU group, staged in pinned memory and copied
    asynchronously; the activation receive (recv stream) and the send (send stream) are ordered
    against the forward by events.
    """
    import torch

    dev = torch.device(device)
    max_rows = max_rows if max_rows is not None else default_max_rows(requests, num_pages)
    max_seq_len = max_seq_len if max_seq_len is not None else default_max_seq_len(requests)
    max_emit = max_emit if max_emit is not None else max(1, min(max_rows, max_tokens))
    if stage is None:
        factory = stage_factory or StageWorker
        stage = factory(spec, stage_layers(spec.n_layers, world, rank), is_first=False, is_last=(rank == world - 1),
                        num_pages=num_pages, page_size=page_size, max_rows=max_rows, max_seq_len=max_seq_len,
                        max_tokens=max_tokens, max_emit=max_emit, seed=seed, device=dev)
    on_gpu = dev.type == "cuda"
    ring = max(ring, world + 2)
    compute = torch.cuda.Stream(device=dev) if on_gpu else None
    recv_s = torch.cuda.Stream(device=dev) if on_gpu else None
    send_s = torch.cuda.Stream(device=dev) if on_gpu else None
    n_ints = 16 * max_tokens + 8 * max_rows + 4 * max_seq_len
    hidden = [torch.empty((max_tokens, spec.d_model), dtype=torch.bfloat16, device=dev) for _ in range(ring)]
    sampled = [torch.empty(max_emit, dtype=torch.int32, device=dev) for _ in range(ring)]
    meta_dev = [torch.empty(n_ints, dtype=torch.int32, device=dev) for _ in range(ring)]
    staging = _PinnedSlots(ring, n_ints, on_gpu)
    sent = [None] * ring
    mk = (lambda: torch.cuda.Event(enable_timing=True)) if on_gpu else _HostEvent
    if on_gpu:
        torch.cuda.synchronize(dev)
    epoch = mk()
    epoch.record(compute) if on_gpu else epoch.record()
    spans = {}
    n = 0
    profiling, profile = False, None
    from . import native as _native
    while True:
        pb = meta.receive()
        if pb is None:
            break
        if on_gpu and bool(pb.flags & FLAG_PROFILE) != profiling:
            if profiling:                   # the profiled window ended with the previous batch
                torch.cuda.synchronize(dev)
                profile = _native.profile_end()
            else:
                _native.profile_begin()
            profiling = not profiling
        k = pb.seq % ring
        md = meta_dev[k]
        if pb.data.size > md.numel():
            meta_dev[k] = md = torch.empty(2 * pb.data.size, dtype=torch.int32, device=dev)
        staged = staging.stage(k, pb.data)
        with _on(recv_s):
            if on_gpu and sent[k] is not None:
                recv_s.wait_event(sent[k])        # slot k's previous send has drained
            transport.recv(hidden[k][: pb.n_tokens], rank - 1, recv_s)
            got = mk()
            got.record(recv_s) if on_gpu else got.record()
        a, b = mk(), mk()
        with _on(compute):
            if on_gpu:
                compute.wait_event(got)
            md[: pb.data.size].copy_(staged, non_blocking=True)
            rd = mk()
            rd.record(compute) if on_gpu else rd.record()
            staging.read[k] = rd
            a.record(compute) if on_gpu else a.record()
            stage.forward(pb, md, hidden=hidden[k], sampled=sampled[k], stream=compute)
            b.record(compute) if on_gpu else b.record()
        with _on(send_s):
            if on_gpu:
                send_s.wait_event(b)
            if rank == world - 1:
                if pb.n_emit:
                    transport.send(sampled[k][: pb.n_emit], 0, send_s)
            else:
                transport.send(hidden[k][: pb.n_tokens], rank + 1, send_s)
            ev = mk()
            ev.record(send_s) if on_gpu else ev.record()
            sent[k] = ev
        spans[pb.seq] = (a, b)
        n += 1
        if on_gpu:
            from . import native
            native.check_meta_errors()    # host-mapped flag: no sync (reports a violation a batch late)
    if on_gpu:
        torch.cuda.synchronize(dev)
        from . import native
        native.check_meta_errors()
        if profiling:
            profile = native.profile_end()
    return {"batches": n, "profile": profile, "busy": [(epoch.elapsed_time(a), epoch.elapsed_time(b)) for a, b in spans.values()],
            "spans": {seq: (epoch.elapsed_time(a), epoch.elapsed_time(b)) for seq, (a, b) in spans.items()}}


class _on:
    """`torch.cuda.stream(s)` that tolerates s=None (CPU test doubles)."""

    def __init__(self, stream):
        self.stream = stream
        self.ctx = None

    def __enter__(self):
        if self.stream is not None:
            import torch
            self.ctx = torch.cuda.stream(self.stream)
            self.ctx.__enter__()
        return self

    def __exit__(self, *a):
        if self.ctx is not None:
            return self.ctx.__exit__(*a)
        return False


class _HostEvent:
    """Wall-clock stand-in for a CUDA event (CPU test doubles only)."""

    def __init__(self):
        self.t = None

    def record(self, *_):
        self.t = time.perf_counter()

    def query(self):
        return True

    def synchronize(self):
        pass

    def elapsed_time(self, other):
        return (other.t - self.t) * 1000.0
