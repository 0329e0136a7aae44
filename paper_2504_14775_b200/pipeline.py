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
from .stage import PackedBatch, StageWorker, default_prompt_source, pack_batch

HEADER = 9
STOP = -1


def header_of(pb: PackedBatch) -> np.ndarray:
    return np.array([pb.seq, pb.n_seqs, pb.n_tokens, pb.n_emit, pb.n_work, pb.n_prefill_work, pb.n_deltas,
                     pb.n_prompts, pb.data.size], dtype=np.int32)


def batch_from(header: np.ndarray, data: np.ndarray) -> PackedBatch:
    seq, n_seqs, n_tokens, n_emit, n_work, n_pf, n_deltas, n_prompts, _ = (int(x) for x in header)
    return PackedBatch(seq, n_seqs, n_tokens, n_emit, n_work, n_pf, n_deltas, n_prompts, data, [], [])


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
    done: object          # CUDA event: sampled tokens on the host
    host: object


class PipelineExecutor:
    """Executor protocol (see executor.py) for rank 0 of a PP=world pipeline.

    Rank 0 holds stage 0 and the token history; it publishes each launched
    micro-batch's metadata, runs stage 0, sends the activations to rank 1 and
    posts the receive of the sampled ids from the last rank.
    """

    def __init__(self, spec: ModelSpec, requests, *, world: int, meta: MetaChannel, transport, num_pages: int,
                 page_size: int = 16, max_tokens: int = 4096, max_emit: int | None = None, seed: int = 0,
                 device="cuda", stage_factory=None, ring: int = 8):
        import torch

        self.spec = spec
        self.world = world
        self.meta = meta
        self.transport = transport
        self.device = torch.device(device)
        self.specs = {r.id: r for r in requests}
        max_rows = max(1, len(requests))
        max_seq_len = max(r.input_tokens + r.output_tokens for r in requests) + 1 if requests else 16
        self.max_emit = max_emit if max_emit is not None else max(1, min(max_rows, max_tokens))
        factory = stage_factory or StageWorker
        self.stage = factory(spec, stage_layers(spec.n_layers, world, 0), is_first=True, is_last=(world == 1),
                             num_pages=num_pages, page_size=page_size, max_rows=max_rows, max_seq_len=max_seq_len,
                             max_tokens=max_tokens, max_emit=self.max_emit, seed=seed, device=self.device)
        self.q_tile = self.stage.q_tile
        self.prompt_source = default_prompt_source(self.specs, spec.vocab)
        on_gpu = self.device.type == "cuda"
        self.compute = torch.cuda.Stream(device=self.device) if on_gpu else None
        # separate streams: activations out to rank 1 must not queue behind the token
        # receive from the last rank (different peers, independent progress)
        self.send_stream = torch.cuda.Stream(device=self.device) if on_gpu else None
        self.recv_stream = torch.cuda.Stream(device=self.device) if on_gpu else None
        self.ring = ring
        self.hidden = [torch.empty((max_tokens, spec.d_model), dtype=torch.bfloat16, device=self.device)
                       for _ in range(ring)]
        self.sampled = [torch.empty(self.max_emit, dtype=torch.int32, device=self.device) for _ in range(ring)]
        self.sampled_host = [torch.empty(self.max_emit, dtype=torch.int32, pin_memory=on_gpu) for _ in range(ring)]
        self.meta_dev = [torch.empty(16 * max_tokens + 8 * max_rows + 4 * max_seq_len, dtype=torch.int32,
                                     device=self.device) for _ in range(ring)]
        self._inflight: dict[int, _Flight] = {}
        self._last_fwd = None
        self.outputs: dict[int, list[int]] = {}
        self.timings: list = []
        self._epoch = None
        self.launches = 0
        self.h2d_bytes: dict[int, int] = {}
        if on_gpu:
            torch.cuda.synchronize(self.device)

    def _event(self):
        import torch
        return torch.cuda.Event(enable_timing=True) if self.device.type == "cuda" else _HostEvent()

    def launch(self, meta) -> None:
        import torch

        pb = pack_batch(meta, self.q_tile, self.prompt_source)
        k = pb.seq % self.ring
        self.meta.publish(pb)                         # metadata ahead of activations
        md = self.meta_dev[k]
        if pb.data.size > md.numel():
            self.meta_dev[k] = md = torch.empty(2 * pb.data.size, dtype=torch.int32, device=self.device)
        src = torch.from_numpy(pb.data)
        self.h2d_bytes[pb.seq] = int(pb.data.nbytes)
        a, b = self._event(), self._event()
        with _on(self.compute):
            md[: pb.data.size].copy_(src.pin_memory() if self.device.type == "cuda" else src, non_blocking=True)
            a.record(self.compute) if self.compute is not None else a.record()
            self.stage.forward(pb, md, hidden=self.hidden[k], sampled=self.sampled[k], stream=self.compute)
            b.record(self.compute) if self.compute is not None else b.record()
        host = self.sampled_host[k]
        if self.world > 1:
            if self.send_stream is not None:
                self.send_stream.wait_event(b)
            self.transport.send(self.hidden[k][: pb.n_tokens], 1, self.send_stream)
            if pb.n_emit:
                self.transport.recv(self.sampled[k][: pb.n_emit], self.world - 1, self.recv_stream)
                with _on(self.compute):
                    if self.compute is not None:
                        self.compute.wait_stream(self.recv_stream)
                    self.stage.commit_tokens(pb, md, self.sampled[k], stream=self.compute)
            # the next use of hidden[k] (batch seq+ring) must follow this send
            if self.compute is not None:
                self.compute.wait_stream(self.send_stream)
        with _on(self.compute):
            if pb.n_emit:
                host[: pb.n_emit].copy_(self.sampled[k][: pb.n_emit], non_blocking=True)
            done = self._event()
            done.record(self.compute) if self.compute is not None else done.record()
        self._inflight[pb.seq] = _Flight(pb, b, done, host)
        self._last_fwd = b
        self.timings.append((pb.seq, [(a, b)]))
        self.launches += 1

    def stage0_idle(self) -> bool:
        return self._last_fwd is None or self._last_fwd.query()

    def wait(self, seq: int) -> None:
        self._inflight[seq].done.synchronize()

    def retire(self, seq: int) -> list[int]:
        f = self._inflight.pop(seq)
        f.done.synchronize()
        toks = f.host[: f.pb.n_emit].tolist()
        for rid, tok in zip(f.pb.emit_ids, toks):
            self.outputs.setdefault(rid, []).append(tok)
        return toks

    def on_finish(self, request_id: int, row: int) -> None:
        pass

    def mark_epoch(self) -> None:
        self._epoch = self._event()
        self._epoch.record(self.compute) if self.compute is not None else self._epoch.record()
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

    def h2d_bytes_total_for(self, seqs) -> int:
        return sum(self.h2d_bytes.get(s, 0) for s in seqs)

    def shutdown(self) -> None:
        self.meta.publish(None)
        self.meta.flush()


# ------------------------------------------------------------------ worker side (ranks >= 1)


def worker_loop(spec: ModelSpec, requests, *, rank: int, world: int, meta: MetaChannel, transport, num_pages: int,
                page_size: int = 16, max_tokens: int = 4096, max_emit: int | None = None, seed: int = 0,
                device="cuda", stage_factory=None, ring: int = 8) -> dict:
    """Run stage `rank` until the driver publishes STOP; returns busy intervals (ms since start)."""
    import torch

    dev = torch.device(device)
    max_rows = max(1, len(requests))
    max_seq_len = max(r.input_tokens + r.output_tokens for r in requests) + 1 if requests else 16
    max_emit = max_emit if max_emit is not None else max(1, min(max_rows, max_tokens))
    factory = stage_factory or StageWorker
    stage = factory(spec, stage_layers(spec.n_layers, world, rank), is_first=False, is_last=(rank == world - 1),
                    num_pages=num_pages, page_size=page_size, max_rows=max_rows, max_seq_len=max_seq_len,
                    max_tokens=max_tokens, max_emit=max_emit, seed=seed, device=dev)
    on_gpu = dev.type == "cuda"
    compute = torch.cuda.Stream(device=dev) if on_gpu else None
    recv_s = torch.cuda.Stream(device=dev) if on_gpu else None
    send_s = torch.cuda.Stream(device=dev) if on_gpu else None
    hidden = [torch.empty((max_tokens, spec.d_model), dtype=torch.bfloat16, device=dev) for _ in range(ring)]
    sampled = [torch.empty(max_emit, dtype=torch.int32, device=dev) for _ in range(ring)]
    meta_dev = torch.empty(16 * max_tokens + 8 * max_rows + 4 * max_seq_len, dtype=torch.int32, device=dev)
    if on_gpu:
        torch.cuda.synchronize(dev)
    epoch = torch.cuda.Event(enable_timing=True) if on_gpu else _HostEvent()
    epoch.record(compute) if on_gpu else epoch.record()
    spans = []
    n = 0
    while True:
        pb = meta.receive()
        if pb is None:
            break
        k = pb.seq % ring
        if pb.data.size > meta_dev.numel():
            meta_dev = torch.empty(2 * pb.data.size, dtype=torch.int32, device=dev)
        with _on(compute):
            meta_dev[: pb.data.size].copy_(torch.from_numpy(pb.data), non_blocking=False)
        if on_gpu:
            recv_s.wait_stream(send_s)        # slot k's previous send has drained
        transport.recv(hidden[k][: pb.n_tokens], rank - 1, recv_s)
        a = torch.cuda.Event(enable_timing=True) if on_gpu else _HostEvent()
        b = torch.cuda.Event(enable_timing=True) if on_gpu else _HostEvent()
        with _on(compute):
            if on_gpu:
                compute.wait_stream(recv_s)
                a.record(compute)
            else:
                a.record()
            stage.forward(pb, meta_dev, hidden=hidden[k], sampled=sampled[k], stream=compute)
            b.record(compute) if on_gpu else b.record()
        if on_gpu:
            send_s.wait_event(b)
        if rank == world - 1:
            if pb.n_emit:
                transport.send(sampled[k][: pb.n_emit], 0, send_s)
        else:
            transport.send(hidden[k][: pb.n_tokens], rank + 1, send_s)
        spans.append((a, b))
        n += 1
    if on_gpu:
        torch.cuda.synchronize(dev)
    return {"batches": n, "busy": [(epoch.elapsed_time(a), epoch.elapsed_time(b)) for a, b in spans]}


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


# ------------------------------------------------------------------ bench entry (torchrun, N > 1)


def _bubble(busy) -> float:
    """Idle fraction of one stage between its first start and last end (CUDA-event busy intervals;
    the reference's per-stage bubble definition, `engine.py:108-125`, over the measured run)."""
    if not busy:
        return 0.0
    t0 = min(a for a, _ in busy)
    t1 = max(b for _, b in busy)
    return 1.0 - sum(b - a for a, b in busy) / max(t1 - t0, 1e-9)


def bench_pipeline(args) -> int:
    """`bench.py --gpus N` under torchrun: PP=N over the same model and trace (strong scaling)."""
    import json
    import statistics

    import torch
    import torch.distributed as dist

    from . import KvConfig, PipelineConfig, ThrottleConfig, build_report
    from .modelspec import MODELS
    from .serving import ServingEngine
    from .workload import ArrivalProcess, builtin_length_table, synthesize_requests

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev_id = local % torch.cuda.device_count()
    torch.cuda.set_device(dev_id)
    # GLLM_PP_TRANSPORT=host: activations staged through host memory over gloo (lets all ranks
    # share one GPU for testing); default: NCCL send/recv between the ranks' GPUs.
    host_transport = os.environ.get("GLLM_PP_TRANSPORT", "nccl") == "host"
    if host_transport:
        dist.init_process_group("gloo")
        gloo = dist.group.WORLD
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev_id))
        gloo = dist.new_group(backend="gloo")
    spec = MODELS[args.model]
    reqs = synthesize_requests(ArrivalProcess.poisson(args.rate, 0), builtin_length_table("sharegpt-like"),
                               args.n_requests)
    page_size = 16
    max_tokens = (2048 + args.n_requests + 255) // 256 * 256
    layers = len(stage_layers(spec.n_layers, world, 0))
    need_pages = sum(-(-(r.input_tokens + r.output_tokens) // page_size) for r in reqs)
    free, _ = torch.cuda.mem_get_info()
    free //= max(1, sum(1 for r in range(world) if r % torch.cuda.device_count() == dev_id))  # shared GPU
    w_bytes = layers * spec.params_per_layer * 2 + 2 * spec.vocab * spec.d_model * 2
    page_bytes = layers * spec.kv_bytes_per_token_layer * page_size
    fit = int((free - w_bytes - max_tokens * (10 * spec.d_model + 6 * spec.d_ff) * 2 * 4 - (10 << 30)) // page_bytes)
    num_pages = torch.tensor([max(1024, min(need_pages, fit))], dtype=torch.int64)
    dist.all_reduce(num_pages, op=dist.ReduceOp.MIN, group=gloo)   # one shared page table: same pool size
    num_pages = int(num_pages.item())
    meta = MetaChannel(gloo, world)
    transport = HostTransport(gloo) if host_transport else NcclTransport(rank, make_links(world))
    from . import native
    launches0 = native.launch_count()
    dist.barrier(group=gloo)
    if rank != 0:
        out = worker_loop(spec, reqs, rank=rank, world=world, meta=meta, transport=transport, num_pages=num_pages,
                          page_size=page_size, max_tokens=max_tokens, max_emit=args.n_requests,
                          device=f"cuda:{dev_id}")
        # per-batch launches of this stage (the timed window is only known to rank 0)
        stats = torch.tensor([0.0, (native.launch_count() - launches0) / max(out["batches"], 1), 0.0],
                             dtype=torch.float64)
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=gloo)
        bub = torch.zeros(world, dtype=torch.float64)
        bub[rank] = _bubble(out["busy"])
        dist.all_reduce(bub, op=dist.ReduceOp.SUM, group=gloo)
        dist.destroy_process_group()
        return 0
    ex = PipelineExecutor(spec, reqs, world=world, meta=meta, transport=transport, num_pages=num_pages,
                          page_size=page_size, max_tokens=max_tokens, max_emit=args.n_requests,
                          device=f"cuda:{dev_id}")
    eng = ServingEngine(reqs, scheduler=args.scheduler, pipeline=PipelineConfig(depth=world),
                        kv_config=KvConfig(num_pages, page_size), throttle=ThrottleConfig(), executor=ex)
    st = {"phase": "warm", "n": 0, "timed": []}
    W, K = args.warmup, args.steps

    class _Stop(Exception):
        pass

    def hook(seq, t, n_out):
        if st["phase"] == "warm":
            st["n"] += 1
            if eng._rd >= args.warm_decodes or st["n"] >= args.warm_max_iters:
                st["phase"], st["c"] = "warmup", 0
        elif st["phase"] == "warmup":
            st["c"] += 1
            if st["c"] >= W:
                st["phase"], st["t0"] = "timed", time.perf_counter()
        else:
            st["timed"].append((seq, t, n_out))
            if len(st["timed"]) >= K:
                st["t1"] = time.perf_counter()
                raise _Stop

    from bench import ClockSampler
    clocks = ClockSampler(dev_id)
    clocks.start()
    try:
        eng.run(on_commit=hook)
    except _Stop:
        pass
    clk = clocks.stop()
    ex.shutdown()
    # rank 0's driver clock spans every stage of every timed batch (a batch commits only after
    # the last rank's tokens arrive), so it is the max over ranks of the pipeline's time.
    stats = torch.tensor([st["t1"] - st["t0"], (native.launch_count() - launches0) / max(ex.launches, 1), 0.0],
                         dtype=torch.float64)
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=gloo)
    bub = torch.zeros(world, dtype=torch.float64)
    bub[0] = _bubble(ex.stage_busy_intervals()[0])
    dist.all_reduce(bub, op=dist.ReduceOp.SUM, group=gloo)
    wall = stats[0:1]
    out_tok = sum(n for _, _, n in st["timed"])
    raw = eng.raw_data()
    rep = build_report(raw)
    line = {"metric": "output_tokens_per_s", "value": round(out_tok / wall.item(), 2), "unit": "tokens/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(wall.item() * 1000 / K, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, seeded ShareGPT-like trace)",
            "config": {"workload": f"{args.model} PP={world}, ShareGPT-like Poisson {args.rate}/s x {args.n_requests}",
                       "model": args.model, "parallelism": f"pp{world}"},
            "e2e": {"value": round(out_tok / wall.item(), 2), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(ex.h2d_bytes_total_for([s for s, _, _ in st["timed"]]) / max(K, 1)),
                    "d2h_bytes_per_step": int(4 * out_tok / max(K, 1))},
            "gpu_launches": int(round(stats[1].item() * K)),  # sum over stages of launches per batch x K
            "clocks": clk,
            "transport": "host-staged gloo (test)" if host_transport else "nccl p2p",
            "serving": {"p50_ttft_ms": rep.ttft_p50_ms, "p50_tpot_ms": rep.tpot_p50_ms,
                        "bubble_frac_per_stage": [round(float(b), 4) for b in bub.tolist()],
                        "decodes_per_step": statistics.mean(eng._iters[s].decode_tokens for s, _, _ in st["timed"])}}
    print(json.dumps(line))
    dist.destroy_process_group()
    return 0
