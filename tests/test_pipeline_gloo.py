"""Multi-process pipeline runtime on CPU (gloo, world 2 and 3) with a deterministic stage test double.

Exercises everything of pipeline.py except the kernels: metadata published by
the driver ahead of activations, in-order activation hand-off rank s -> s+1,
sampled ids back to rank 0 and into the token history, the wall-clock engine
with depth = world, and decision replay of every schedule point against the
oracle planner (`oracle/sched_ref.py`).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_14775_b200 import KvConfig, PipelineConfig, RequestSpec, ThrottleConfig
from paper_2504_14775_b200.modelspec import MODELS

VOCAB = 32000
SPEC = MODELS["tiny"]


class FakeStage:
    """StageWorker interface; hidden[t] = (token % 251, pos % 251, layers seen)."""

    def __init__(self, spec, layers, *, is_first, is_last, num_pages, page_size, max_rows, max_seq_len, max_tokens,
                 max_emit, seed, device):
        self.spec = spec
        self.layers = list(layers)
        self.is_first, self.is_last = is_first, is_last
        self.q_tile = 32
        self.page_size = page_size
        self.token_hist = np.zeros((max_rows, max_seq_len), np.int64) if is_first else None
        self.table = np.full((max_rows, -(-max_seq_len // page_size)), -1, np.int64)

    def _parse(self, pb, meta_dev):
        d = meta_dev[: pb.data.size].numpy()
        info = d[: 5 * pb.n_seqs].reshape(-1, 5)
        o = 5 * pb.n_seqs + 2 * pb.n_work
        deltas = d[o: o + 3 * pb.n_deltas].reshape(-1, 3)
        o += 3 * pb.n_deltas
        hdr = d[o: o + 3 * pb.n_prompts].reshape(-1, 3)
        toks = d[o + 3 * pb.n_prompts:]
        return info, deltas, hdr, toks

    def forward(self, pb, meta_dev, hidden=None, sampled=None, logits=None, stream=None):
        info, deltas, hdr, toks = self._parse(pb, meta_dev)
        for row, idx, page in deltas:
            self.table[row, idx] = page
        for seq_row, (row, start, n, off, emit) in enumerate(info):
            for p in range(start, start + n):      # every token's page must be mapped on every stage
                assert self.table[row, p // self.page_size] >= 0
        if self.is_first:
            for row, ln, off in hdr:
                self.token_hist[row, :ln] = toks[off: off + ln]
            for row, start, n, off, emit in info:
                for t in range(n):
                    hidden[off + t, 0] = float(self.token_hist[row, start + t] % 251)
                    hidden[off + t, 1] = float((start + t) % 251)
                    hidden[off + t, 2] = 0.0
        for row, start, n, off, emit in info:
            hidden[off: off + n, 2] += float(len(self.layers))
        if self.is_last:
            for row, start, n, off, emit in info:
                if emit >= 0:
                    h = hidden[off + n - 1]
                    sampled[emit] = int((int(h[0]) * 31 + int(h[1]) + int(h[2])) % VOCAB)
            if self.is_first:
                self.commit_tokens(pb, meta_dev, sampled)

    def commit_tokens(self, pb, meta_dev, sampled, stream=None):
        info, _, _, _ = self._parse(pb, meta_dev)
        for row, start, n, off, emit in info:
            if emit >= 0:
                self.token_hist[row, start + n] = int(sampled[emit])


def _requests():
    rng = np.random.Generator(np.random.PCG64(5))
    return [RequestSpec(i, float(i) * 0.3, int(rng.integers(5, 60)), int(rng.integers(1, 8))) for i in range(12)]


def _prompts():
    rng = np.random.Generator(np.random.PCG64(99))
    return {r.id: rng.integers(0, VOCAB, r.input_tokens).astype(np.int32) for r in _requests()}


def _run(rank, world, port, q, transport="host", lookahead=False, submit=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_14775_b200.pipeline import (HostTransport, MetaChannel, NcclTransport, PipelineExecutor,
                                                make_links, worker_loop)
    from paper_2504_14775_b200.serving import ServingEngine
    reqs = _requests()
    g = dist.group.WORLD
    meta = MetaChannel(g, world)
    # "links": the product transport's per-link group routing (one two-rank group per hop and
    # one for the token return path), on gloo groups with CPU tensors
    tr = HostTransport(g) if transport == "host" else NcclTransport(rank, make_links(world, backend="gloo"))
    pages = 64
    try:
        rows = dict(max_rows=len(reqs), max_seq_len=128) if submit else {}
        if rank == 0:
            ex = PipelineExecutor(SPEC, [] if submit else reqs, world=world, meta=meta, transport=tr,
                                  num_pages=pages, page_size=4, max_tokens=512, device="cpu",
                                  stage_factory=FakeStage, **rows)
            eng = ServingEngine([] if submit else reqs, pipeline=PipelineConfig(depth=world),
                                kv_config=KvConfig(pages, 4), throttle=ThrottleConfig(T=2, min_p=4, max_p=64),
                                executor=ex, record_decisions=True, lookahead=lookahead)
            if submit:
                prompts = _prompts()
                for r in reqs:          # the front end hands requests (and their prompt ids) over
                    eng.submit(r, prompts[r.id])
            eng.run()
            ex.shutdown()
            raw = eng.raw_data()
            q.put(("ok", {r.id: ex.outputs.get(r.id, []) for r in reqs},
                   [(r.id, r.completion_ms is not None) for r in raw.requests], eng.decisions,
                   [(it.prefill_tokens, it.decode_tokens) for it in raw.iterations]))
        else:
            out = worker_loop(SPEC, [] if submit else reqs, rank=rank, world=world, meta=meta, transport=tr,
                              num_pages=pages, page_size=4, max_tokens=512, device="cpu", stage_factory=FakeStage,
                              **rows)
            q.put(("worker", rank, out["batches"]))
    except Exception as e:  # surface worker failures to the test
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,transport,lookahead,submit", [
    (2, "host", False, False), (3, "host", False, False), (2, "links", False, False), (3, "links", False, False),
    (2, "links", True, False), (3, "links", True, False), (2, "host", True, True)])
def test_pipeline_end_to_end_gloo(world, transport, lookahead, submit):
    """`lookahead`: batch b is planned right after batch b-1 launches, with batch b-depth's commit
    applied (the reference's state at that schedule point); `submit`: requests and their real
    prompt ids enter through `ServingEngine.submit` instead of the constructor's trace."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q, transport, lookahead, submit)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errors = [m for m in msgs if m[0] == "error"]
    assert not errors, errors[0][2]
    main = next(m for m in msgs if m[0] == "ok")
    _, outputs, finished, decisions, iters = main
    reqs = _requests()
    assert all(done for _, done in finished)
    n_batches = len(iters)
    assert all(m[2] == n_batches for m in msgs if m[0] == "worker")
    # tokens: each sampled id is the fake model applied to the previous token at its position,
    # after passing through every stage (all 4 layers) in order
    from paper_2504_14775_b200.workload import prompt_token_ids
    prompts = _prompts()
    for r in reqs:
        out = outputs[r.id]
        assert len(out) == r.output_tokens
        hist = list(prompts[r.id] if submit else prompt_token_ids(r.id, r.input_tokens, SPEC.vocab))
        for tok in out:
            p = len(hist) - 1
            assert tok == (hist[p] % 251 * 31 + p % 251 + SPEC.n_layers) % VOCAB
            hist.append(tok)
    # decision replay: every schedule point equals the oracle planner on the same snapshot
    from oracle.sched_ref import plan
    for seq, (wp, rd, free, waiting, ready, pq, dq), dec, chunks in decisions:
        pq_l = [(rid, pq[rid][0], pq[rid][1]) for rid in waiting]
        dq_l = [(rid, dq[rid]) for rid in ready]
        want_dec, want_chunks, _ = plan("throttle", wp, rd, free, 64, 4, world, pq_l, dq_l,
                                        (2, 64, 4, 0.05, "combined"), 2048)
        # the engine may drop decodes by preemption after planning; with 64 pages none happen here
        assert dec == want_dec and chunks == want_chunks, seq


def test_lookahead_serving_matches_planner_and_completes():
    """Asynchronous (lookahead) wall-clock loop on a CPU test double: every decision is the
    oracle planner on its snapshot, every request gets its tokens, times are monotone."""
    from oracle.sched_ref import plan
    from paper_2504_14775_b200.pipeline import HostTransport, MetaChannel, PipelineExecutor  # noqa: F401
    from paper_2504_14775_b200.serving import ServingEngine
    from paper_2504_14775_b200.stage import default_prompt_source, pack_batch

    reqs = _requests()

    class Exec:
        def __init__(self):
            self.src = default_prompt_source({r.id: r for r in reqs}, SPEC.vocab)
            self.q, self.outputs = {}, {}

        def launch(self, meta):
            self.q[meta.seq] = pack_batch(meta, 32, self.src)

        def retire(self, seq):
            pb = self.q.pop(seq)
            for rid in pb.emit_ids:
                self.outputs.setdefault(rid, []).append(0)

        def stage0_idle(self):
            return True

        def wait(self, seq):
            pass

        def on_finish(self, rid, row):
            pass

        def mark_epoch(self):
            pass

        def synchronize(self):
            pass

        def stage_busy_intervals(self):
            return [[]]

    ex = Exec()
    eng = ServingEngine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(64, 4),
                        throttle=ThrottleConfig(T=2, min_p=4, max_p=64), executor=ex, record_decisions=True,
                        lookahead=True, time_scale=50.0)
    raw = eng.run()
    for r in raw.requests:
        assert r.completion_ms is not None and r.first_token_ms is not None
        assert r.arrival_ms <= r.first_token_ms <= r.completion_ms
        assert len(ex.outputs[r.id]) == r.output_tokens
    for seq, (wp, rd, free, waiting, ready, pq, dq), dec, chunks in eng.decisions:
        want = plan("throttle", wp, rd, free, 64, 4, 1, [(rid, pq[rid][0], pq[rid][1]) for rid in waiting],
                    [(rid, dq[rid]) for rid in ready], (2, 64, 4, 0.05, "combined"), 2048)
        assert (dec, chunks) == want[:2], seq
