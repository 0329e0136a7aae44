"""Executors: run the engine's launched micro-batches on GPU stage workers.

`LocalExecutor` keeps every stage of the pipeline in this process on one
device (PP=1, or several stages chained back to back on one GPU for tests);
the multi-GPU pipeline lives in `pipeline.py`. Both implement the executor
protocol the engine calls:

    launch(meta: BatchMeta)        -> enqueue the micro-batch (async, returns at once)
    retire(seq: int)               -> wait for that batch's sampled tokens (last-stage commit)
    on_finish(request_id, row)     -> request finished; its row may be reused

Per-iteration host->device traffic is ONE int32 metadata copy from a pinned
ring buffer (`stage.pack_batch`); device->host is the sampled token ids.
"""

from __future__ import annotations

import numpy as np

from . import native
from .modelspec import ModelSpec, stage_layers
from .stage import (PackedBatch, StageWorker, default_max_rows, default_max_seq_len, pack_batch,
                    pad_decode_batch, prompt_source_with)

# decode-only micro-batches run as captured CUDA graphs at these padded batch sizes
GRAPH_BUCKETS = (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 160, 192, 256)


class _PinnedRing:
    """Pinned host staging + device metadata buffers reused round-robin, guarded by events."""

    def __init__(self, slots: int, n_ints: int, device):
        import torch

        self.host = [torch.empty(n_ints, dtype=torch.int32, pin_memory=True) for _ in range(slots)]
        self.dev = [torch.empty(n_ints, dtype=torch.int32, device=device) for _ in range(slots)]
        self.events = [None] * slots
        self.i = 0

    def upload(self, data: np.ndarray, stream):
        import torch

        k = self.i
        self.i = (self.i + 1) % len(self.host)
        if self.events[k] is not None:
            self.events[k].synchronize()
        n = data.size
        if n > self.host[k].numel():
            self.host[k] = torch.empty(2 * n, dtype=torch.int32, pin_memory=True)
            self.dev[k] = torch.empty(2 * n, dtype=torch.int32, device=self.dev[k].device)
        self.host[k][:n].numpy()[:] = data
        with torch.cuda.stream(stream):
            self.dev[k][:n].copy_(self.host[k][:n], non_blocking=True)
        return k, self.dev[k]

    def fence(self, k: int, event) -> None:
        self.events[k] = event


class LocalExecutor:
    """All pipeline stages of `spec` on one GPU, executed in launch order on one stream."""

    def __init__(self, spec: ModelSpec, requests, *, num_pages: int, page_size: int = 16, n_stages: int = 1,
                 max_rows: int | None = None, max_tokens: int = 4096, max_emit: int | None = None,
                 seed: int = 0, device="cuda", record_logits: bool = False, record_ids=None,
                 ring_slots: int = 8, max_seq_len: int | None = None, cuda_graphs: bool = False,
                 graph_max_batch: int = 256):
        import torch

        self.spec = spec
        self.device = torch.device(device)
        self.specs = {r.id: r for r in requests}
        max_rows = max_rows if max_rows is not None else default_max_rows(requests, num_pages)
        max_seq_len = max_seq_len if max_seq_len is not None else default_max_seq_len(requests)
        self.max_rows, self.max_seq_len = max_rows, max_seq_len
        max_emit = max_emit if max_emit is not None else max(1, min(max_rows, max_tokens))
        self.max_tokens = max_tokens
        self.stages = [StageWorker(spec, stage_layers(spec.n_layers, n_stages, s), is_first=(s == 0),
                                   is_last=(s == n_stages - 1), num_pages=num_pages, page_size=page_size,
                                   max_rows=max_rows, max_seq_len=max_seq_len, max_tokens=max_tokens,
                                   max_emit=max(max_emit, graph_max_batch if cuda_graphs else 0), seed=seed,
                                   device=self.device, scratch=cuda_graphs) for s in range(n_stages)]
        self.q_tile = self.stages[0].q_tile
        self.prompts: dict[int, np.ndarray] = {}
        self.prompt_source = prompt_source_with(self.prompts, self.specs, spec.vocab)
        self.stream = torch.cuda.Stream(device=self.device)
        n_ints = 16 * max_tokens + 8 * max_rows + 4 * max_seq_len
        self.ring = _PinnedRing(ring_slots, n_ints, self.device)
        self.hidden = torch.empty((max_tokens, spec.d_model), dtype=torch.bfloat16, device=self.device)
        # CUDA graphs (decode-only batches): (bucket, decode KV-split class) -> captured per-stage graphs
        # over fixed metadata / sampled buffers; see _enqueue_graph
        self.cuda_graphs = cuda_graphs
        self.graph_buckets = tuple(b for b in GRAPH_BUCKETS if b <= min(graph_max_batch, max_tokens))
        self._graphs: dict = {}
        self.graph_replays = 0
        self.graph_kernel_launches = 0   # kernels run inside graph replays (the native launch counter misses them)
        self.sampled_dev = [torch.empty(max_emit, dtype=torch.int32, device=self.device) for _ in range(ring_slots)]
        self.sampled_host = [torch.empty(max_emit, dtype=torch.int32, pin_memory=True) for _ in range(ring_slots)]
        self.record_logits = record_logits
        self.record_ids = None if record_ids is None else set(record_ids)
        self.logits_dev = (torch.empty((self.stages[-1].max_emit, spec.vocab), dtype=torch.bfloat16, device=self.device)
                           if record_logits else None)
        self._inflight: dict[int, tuple] = {}
        self._done: dict[int, object] = {}                # seq -> batch-finished event (device windows)
        self.outputs: dict[int, list[int]] = {}          # request id -> sampled tokens, in order
        self.logits: list[tuple[int, int, np.ndarray]] = []  # (request id, position, fp32 logits)
        self.timings: list = []                           # (seq, [(start, end) event per stage])
        self.launches = 0
        self._epoch = None
        self.h2d_bytes: dict[int, int] = {}              # seq -> metadata bytes copied host->device
        # Weights, block tables and token history were initialised on torch's current stream;
        # the executor stream is non-blocking, so order it after that work once.
        torch.cuda.synchronize(self.device)

    # -- executor protocol ----------------------------------------------------------

    def launch(self, meta) -> None:
        import torch

        pb = pack_batch(meta, self.q_tile, self.prompt_source)
        self._enqueue(pb)

    def _enqueue(self, pb: PackedBatch) -> None:
        import torch

        if pb.n_tokens > self.max_tokens:
            raise ValueError(f"micro-batch of {pb.n_tokens} tokens exceeds max_tokens={self.max_tokens}")
        if self.cuda_graphs and pb.n_prefill_work == 0 and pb.n_prompts == 0 and not native.profiling():
            bucket = next((b for b in self.graph_buckets if b >= pb.n_seqs), None)
            if bucket is not None and pb.n_deltas <= bucket and pb.n_emit == pb.n_seqs:
                return self._enqueue_graph(pb, bucket)
        st = self.stream
        k, meta_dev = self.ring.upload(pb.data, st)
        self.h2d_bytes[pb.seq] = int(pb.data.nbytes)
        sampled = self.sampled_dev[k]
        evs = []
        with torch.cuda.stream(st):
            for w in self.stages:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                w.forward(pb, meta_dev, hidden=self.hidden, sampled=sampled,
                          logits=self.logits_dev if w.is_last else None, stream=st)
                if w.is_last and len(self.stages) > 1 and pb.n_emit:
                    self.stages[0].commit_tokens(pb, meta_dev, sampled, stream=st)
                b.record(st)
                evs.append((a, b))
            host = self.sampled_host[k]
            if pb.n_emit:
                host[:pb.n_emit].copy_(sampled[:pb.n_emit], non_blocking=True)
            logits_host = None
            if self.record_logits and pb.n_emit:
                logits_host = self.logits_dev[:pb.n_emit].to("cpu", non_blocking=True)
            done = torch.cuda.Event(enable_timing=True)
            done.record(st)
        self.ring.fence(k, done)
        self._inflight[pb.seq] = (pb, done, host, logits_host)
        self._done[pb.seq] = done
        self.timings.append((pb.seq, evs))
        self.launches += 1

    def _split_class(self, pb: PackedBatch) -> int:
        """The decode attention's KV-split request for this batch (attention.cu launch_attn: the
        longest decode's pages / (3 stages x 8 warps), at most 4): part of the graph key, since the
        split baked into a graph is chosen from the capture batch's host metadata."""
        info = pb.data[:5 * pb.n_seqs].reshape(pb.n_seqs, 5)
        pages = int(((info[:, 1] + 1 + self.stages[0].page_size - 1) // self.stages[0].page_size).max())
        return min(4, max(1, -(-pages // 24)))

    def _enqueue_graph(self, pb: PackedBatch, bucket: int) -> None:
        """Decode-only batch through a captured CUDA graph of the stage forwards at a padded batch
        size. The first batch of a (bucket, split class) runs eagerly on the graph's fixed buffers
        (warming every kernel) and is then captured; later batches copy their padded metadata into
        the fixed buffer and replay. Timing events bracket each stage's graph as in the eager path."""
        import torch

        st = self.stream
        w0 = self.stages[0]
        padded = pad_decode_batch(pb, bucket, w0.scratch_row, w0.scratch_page)
        key = (bucket, self._split_class(pb))
        k, meta_dev = self.ring.upload(padded.data, st)
        self.h2d_bytes[pb.seq] = int(padded.data.nbytes)
        n = padded.data.size
        ent = self._graphs.get(key)
        fresh = ent is None
        if fresh:
            ent = {"meta": torch.empty(n, dtype=torch.int32, device=self.device),
                   "sampled": torch.empty(bucket, dtype=torch.int32, device=self.device), "graphs": None}
            self._graphs[key] = ent
        gmeta, gsampled = ent["meta"], ent["sampled"]

        def stage_calls(s, w):
            w.forward(padded, gmeta, hidden=self.hidden, sampled=gsampled,
                      logits=self.logits_dev if w.is_last else None, stream=st)
            if w.is_last and len(self.stages) > 1:
                self.stages[0].commit_tokens(padded, gmeta, gsampled, stream=st)

        evs = []
        with torch.cuda.stream(st):
            gmeta.copy_(meta_dev[:n], non_blocking=True)
            for s, w in enumerate(self.stages):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                if fresh:
                    stage_calls(s, w)
                else:
                    ent["graphs"][s].replay()
                    self.graph_kernel_launches += ent["kernels"][s]
                b.record(st)
                evs.append((a, b))
            host = self.sampled_host[k]
            host[:pb.n_emit].copy_(gsampled[:pb.n_emit], non_blocking=True)
            logits_host = None
            if self.record_logits:
                logits_host = self.logits_dev[:pb.n_emit].to("cpu", non_blocking=True)
            done = torch.cuda.Event(enable_timing=True)
            done.record(st)
        if fresh:
            graphs, kernels = [], []
            for s, w in enumerate(self.stages):
                g = torch.cuda.CUDAGraph()
                l0 = native.launch_count()
                with torch.cuda.graph(g, stream=st, capture_error_mode="thread_local"):
                    stage_calls(s, w)
                kernels.append(native.launch_count() - l0)
                graphs.append(g)
            ent["graphs"], ent["kernels"] = graphs, kernels
        else:
            self.graph_replays += 1
        self.ring.fence(k, done)
        self._inflight[pb.seq] = (pb, done, host, logits_host)
        self._done[pb.seq] = done
        self.timings.append((pb.seq, evs))
        self.launches += 1

    def retire(self, seq: int) -> list[int]:
        pb, done, host, logits_host = self._inflight.pop(seq)
        done.synchronize()
        native.check_meta_errors()
        toks = host[:pb.n_emit].tolist()
        for rid, tok in zip(pb.emit_ids, toks):
            self.outputs.setdefault(rid, []).append(tok)
        if logits_host is not None:
            lg = logits_host.float().numpy()
            for i, (rid, pos) in enumerate(zip(pb.emit_ids, pb.emit_pos)):
                if self.record_ids is None or rid in self.record_ids:
                    self.logits.append((rid, pos, lg[i].copy()))
        return toks

    def on_finish(self, request_id: int, row: int) -> None:
        self.prompts.pop(request_id, None)

    def register_prompt(self, request_id: int, tokens) -> None:
        self.prompts[request_id] = np.asarray(tokens, dtype=np.int32)

    def add_request(self, spec) -> None:
        self.specs[spec.id] = spec

    # -- wall-clock driver hooks ------------------------------------------------------

    def stage0_idle(self) -> bool:
        return True   # one stream: the engine's depth gate is the only limit

    def wait(self, seq: int) -> None:
        self._inflight[seq][1].synchronize()

    def mark_epoch(self) -> None:
        import torch

        self._epoch = torch.cuda.Event(enable_timing=True)
        self._epoch.record(self.stream)
        self.timings.clear()

    def synchronize(self) -> None:
        self.stream.synchronize()

    def stage_times_ms(self, seq: int) -> list[float]:
        """Device ms of each stage's forward for batch `seq` (waits for it; measured-time replay)."""
        self._inflight[seq][1].synchronize()
        for s, evs in reversed(self.timings):
            if s == seq:
                return [a.elapsed_time(b) for a, b in evs]
        raise KeyError(seq)

    def batch_device_ms(self) -> dict[int, float]:
        """seq -> device ms of the whole micro-batch (all stages), from CUDA events on the launch stream."""
        self.synchronize()
        return {seq: evs[0][0].elapsed_time(evs[-1][1]) for seq, evs in self.timings}

    def device_window_ms(self, first: int, last: int) -> float:
        """Device time from batch `first` starting to batch `last` finishing (gaps included)."""
        self.synchronize()
        start = next(evs[0][0] for s, evs in self.timings if s == first)
        return start.elapsed_time(self._done[last])

    def stage_busy_ms(self, first: int, last: int) -> float:
        self.synchronize()
        return sum(evs[0][0].elapsed_time(evs[-1][1]) for s, evs in self.timings if first <= s <= last)

    def h2d_bytes_total_for(self, seqs) -> int:
        return sum(self.h2d_bytes.get(s, 0) for s in seqs)

    def stage_busy_intervals(self) -> list[list[tuple[float, float]]]:
        """Per-stage (start, end) ms since `mark_epoch`, measured by CUDA events."""
        self.synchronize()
        out = [[] for _ in self.stages]
        if self._epoch is None:
            return out
        for _, evs in self.timings:
            for s, (a, b) in enumerate(evs):
                out[s].append((self._epoch.elapsed_time(a), self._epoch.elapsed_time(b)))
        return out
