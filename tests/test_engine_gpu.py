"""End-to-end on the B200: the engine drives real stage workers.

* Schedules: with the virtual clock the GPU-backed engine must reproduce the
  reference timeline bit for bit (golden C1 runs, generated from `tokensim`).
* Logits: under teacher forcing (the oracle consumes the exact token sequence
  the GPU produced), every sampled step's bf16 logits are within 2e-2
  relative L2 of the fp32 CPU oracle (`oracle/model_ref.py`).
* Tokens: every request gets exactly output_tokens sampled tokens, and each
  equals the oracle's argmax wherever the oracle's top-2 margin is clear.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import load  # noqa: E402
from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig  # noqa: E402
from paper_2504_14775_b200.workload import prompt_token_ids  # noqa: E402

pytestmark = pytest.mark.gpu

ENGINE = load("engine_runs.json.gz")
TRACES = load("traces.json.gz")


def _c1():
    return [RequestSpec(i, a, b, c) for i, (a, b, c) in enumerate(TRACES["c1"])]


@pytest.mark.parametrize("depth,n_stages", [(2, 2), (1, 1)])
def test_tiny_engine_schedule_and_logits(cuda_ok, depth, n_stages):
    from oracle.model_ref import from_stage_workers
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    spec = MODELS["tiny"]
    reqs = _c1()
    watch = [0, 5, 17, 40]
    ex = LocalExecutor(spec, reqs, num_pages=4096, page_size=16, n_stages=n_stages, max_tokens=2560,
                       record_logits=True, record_ids=watch, seed=1)
    eng = Engine(reqs, scheduler="throttle", pipeline=PipelineConfig(depth=depth), kv_config=KvConfig(4096, 16),
                 throttle=ThrottleConfig(), executor=ex)
    raw = eng.run()
    gold = {r["name"]: r for r in ENGINE["runs"]}[f"c1_throttle_d{depth}"]
    assert [[it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens] for it in raw.iterations] \
        == gold["iterations"]
    assert [[r.id, r.arrival_ms, r.first_token_ms, r.completion_ms, r.preemption_count] for r in raw.requests] \
        == gold["requests"]
    for r in reqs:
        assert len(ex.outputs[r.id]) == r.output_tokens

    oracle = from_stage_workers(ex.stages)
    by_req = {}
    for rid, pos, lg in ex.logits:
        by_req.setdefault(rid, []).append((pos, lg))
    worst, agree, clear = 0.0, 0, 0
    for rid in watch:
        spec_r = reqs[rid]
        seq = np.concatenate([prompt_token_ids(rid, spec_r.input_tokens, spec.vocab),
                              np.asarray(ex.outputs[rid][:-1], dtype=np.int32)])
        ref = oracle.logits(seq).numpy()               # [len, vocab], row p predicts token p+1
        for pos, lg in by_req[rid]:
            want = ref[pos - 1]
            rel = np.linalg.norm(lg - want) / np.linalg.norm(want)
            worst = max(worst, rel)
            top2 = np.sort(want)[-2:]
            if top2[1] - top2[0] > 0.05:
                clear += 1
                agree += int(np.argmax(lg) == np.argmax(want))
    assert worst < 2e-2, worst
    assert clear > 0 and agree == clear, (agree, clear)


def test_preemption_on_gpu(cuda_ok):
    """Memory pressure: evictions + recompute on real KV pages keep schedules exact and outputs complete."""
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    trace = ENGINE["traces"]["bursty"]
    reqs = [RequestSpec(i, a, b, c) for i, (a, b, c) in enumerate(trace)]
    gold = {r["name"]: r for r in ENGINE["runs"]}["bursty_throttle_p192_T8_th0.0"]
    ex = LocalExecutor(MODELS["tiny"], reqs, num_pages=192, page_size=16, n_stages=2, max_tokens=2560, seed=3)
    from paper_2504_14775_b200 import CommModel, StageCostModel
    eng = Engine(reqs, scheduler="throttle",
                 pipeline=PipelineConfig(depth=4, cost=StageCostModel(), comm=CommModel.pcie()),
                 kv_config=KvConfig(192, 16), throttle=ThrottleConfig(T=8, kv_thresh=0.0), executor=ex)
    raw = eng.run()
    assert raw.preemptions == gold["preemptions"] == 142
    assert [[it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens] for it in raw.iterations] \
        == gold["iterations"]
    for r in reqs:
        # a recompute never re-samples a token that was already generated
        assert len(ex.outputs[r.id]) == r.output_tokens


def test_fused_norm_matches_separate_rmsnorm(cuda_ok):
    """Fused RMSNorm (norm weights folded into w_qkv / w_gate_up, row scales in the GEMM epilogues,
    statistics accumulated by the O / down epilogues) and separate RMSNorm kernels both stay within
    2e-2 of the fp32 oracle of the same (unfolded) model, with non-unit norm weights, across
    prefill + decode micro-batches of the tiny model (2 stages on one GPU)."""
    import torch
    from oracle.model_ref import from_stage_workers
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.stage import StageWorker

    spec = MODELS["tiny"]
    reqs = [RequestSpec(0, 0.0, 40, 6), RequestSpec(1, 0.5, 75, 5), RequestSpec(2, 2.0, 17, 7)]
    oracle, worst = None, {}
    for fused in (False, True):
        ex = LocalExecutor(spec, reqs, num_pages=64, page_size=16, n_stages=2, max_tokens=256, record_logits=True,
                           seed=7)
        g = torch.Generator(device="cpu").manual_seed(11)
        for i, st in enumerate(ex.stages):
            new = StageWorker(spec, st.layer_ids, is_first=st.is_first, is_last=st.is_last, num_pages=64,
                              page_size=16, max_rows=st.max_rows, max_seq_len=st.max_seq_len, max_tokens=256,
                              max_emit=st.max_emit, seed=7, device=st.device, fused_norm=False)
            for w in new.layers:
                for nrm in ("attn_norm", "mlp_norm"):
                    w[nrm].copy_((0.5 + torch.rand(w[nrm].shape, generator=g)).to(w[nrm].device).bfloat16())
            ex.stages[i] = new
        if oracle is None:
            oracle = from_stage_workers(ex.stages)      # the unfolded model, non-unit norms
        if fused:
            for st in ex.stages:
                st.refold_norms()
        eng = Engine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(64, 16),
                     throttle=ThrottleConfig(T=2, min_p=8), executor=ex)
        eng.run()
        torch.cuda.synchronize()
        w_max = 0.0
        for rid, pos, lg in ex.logits:
            r = reqs[rid]
            seq = np.concatenate([prompt_token_ids(rid, r.input_tokens, spec.vocab),
                                  np.asarray(ex.outputs[rid], dtype=np.int32)])[:pos]
            want = oracle.logits(seq).numpy()[pos - 1]
            w_max = max(w_max, float(np.linalg.norm(lg - want) / np.linalg.norm(want)))
        worst[fused] = w_max
    assert worst[False] < 2e-2 and worst[True] < 2e-2, worst


def test_pdl_bit_identical(cuda_ok):
    """Programmatic dependent launch lets kernels start before their predecessor finishes; every
    kernel must wait (griddepcontrol.wait) before touching shared memory. A missed wait is a race:
    the served tokens and logits must be bit-identical with PDL on and off."""
    import json
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for pdl in ("1", "0"):
        env = dict(os.environ, GLLM_PDL=pdl)
        r = subprocess.run([sys.executable, os.path.join(here, "pdl_equivalence_run.py")], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["launches"] > 10
    assert outs[0]["tokens"] == outs[1]["tokens"]
    assert outs[0]["logits_sha256"] == outs[1]["logits_sha256"]


@pytest.mark.parametrize("lookahead", [True, False])
def test_wall_clock_serving_decision_replay(cuda_ok, lookahead):
    """SURVEY §8(c)(i) on the GPU: the wall-clock serving loop (host planning overlapped with the
    device when `lookahead`) drives real stage kernels; every logged schedule point, replayed
    through the oracle planner on its snapshot, gives the same plan, and every request completes."""
    from oracle.sched_ref import plan
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.serving import ServingEngine

    spec = MODELS["llama3-8b"].with_layers(2)
    reqs = [RequestSpec(i, 2.0 * i, 40 + (37 * i) % 300, 3 + (11 * i) % 17) for i in range(24)]
    pages, ps = 1024, 16
    ex = LocalExecutor(spec, reqs, num_pages=pages, page_size=ps, max_tokens=1024, max_emit=32, seed=5)
    thr = ThrottleConfig(T=4, max_p=512, min_p=32)
    eng = ServingEngine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(pages, ps), throttle=thr,
                        executor=ex, record_decisions=True, lookahead=lookahead)
    raw = eng.run()
    for r in raw.requests:
        assert r.completion_ms is not None and r.arrival_ms <= r.first_token_ms <= r.completion_ms
        assert len(ex.outputs[r.id]) == r.output_tokens
    assert raw.preemptions == 0
    assert len(eng.decisions) > 0
    for seq, (wp, rd, free, waiting, ready, pq, dq), dec, chunks in eng.decisions:
        want = plan("throttle", wp, rd, free, pages, ps, 1, [(rid, pq[rid][0], pq[rid][1]) for rid in waiting],
                    [(rid, dq[rid]) for rid in ready], (thr.T, thr.max_p, thr.min_p, thr.kv_thresh, "combined"), 2048)
        assert (dec, chunks) == want[:2], seq


def test_metadata_bounds_checks(cuda_ok):
    """Out-of-range rows / page ids / positions in a micro-batch's metadata are never written through
    (no block-table or KV write lands outside the stage's tables) and raise at retire."""
    import ctypes as C

    from paper_2504_14775_b200 import native
    from paper_2504_14775_b200.errors import NativeError
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.stage import PackedBatch, StageWorker

    spec = MODELS["tiny"]
    w = StageWorker(spec, range(spec.n_layers), is_first=True, is_last=True, num_pages=8, page_size=16, max_rows=4,
                    max_seq_len=64, max_tokens=64, max_emit=8)
    native.check_meta_errors()
    dev = "cuda"

    def prep(info, deltas, prompts=()):
        hdr, toks = [], []
        off = 0
        for row, t in prompts:
            hdr.append((row, len(t), off))
            toks += list(t)
            off += len(t)
        data = np.array(sum(info, []) + sum([list(d) for d in deltas], []) + sum([list(h) for h in hdr], []) + toks,
                        np.int32)
        pb = PackedBatch(0, len(info), sum(i[2] for i in info), 0, 0, 0, len(deltas), len(hdr), data, [], [])
        md = torch.from_numpy(data).to(dev)
        T = max(pb.n_tokens, 1)
        tp, ts, ti, er = (torch.full((T,), -7, dtype=torch.int32, device=dev) for _ in range(4))
        native.call("gllm_prepare_batch", C.byref(w.cstage), C.byref(w.cbatch(pb, md)), tp.data_ptr(),
                    ts.data_ptr(), ti.data_ptr(), er.data_ptr(), native.stream_handle())
        torch.cuda.synchronize()
        return ts.cpu().tolist()

    table0 = w.block_table.clone()
    # valid batch: row 1 gets pages 3, 2; tokens 0..19 map to slots on them
    slots = prep([[1, 0, 20, 0, -1]], [(1, 0, 3), (1, 1, 2)], [(1, list(range(20)))])
    assert slots == [3 * 16 + p for p in range(16)] + [2 * 16 + p for p in range(4)]
    assert native.load().gllm_meta_errors(0) == 0
    before = w.block_table.clone()
    # bad delta (row 9 of 4, page 99 of 8), bad prompt row, bad seq row, position past max_seq_len
    prep([[1, 0, 2, 0, -1]], [(9, 0, 1), (1, 2, 99), (1, 40, 1)], [(7, [1, 2])])
    assert torch.equal(w.block_table, before)             # nothing written through
    flags = native.load().gllm_meta_errors(0)
    assert flags & 1 and flags & 2 and not flags & 4, flags
    with pytest.raises(NativeError):
        native.check_meta_errors()
    # a token whose page was never mapped (row 2 is empty) -> slot -1, flagged
    slots = prep([[2, 0, 3, 0, -1]], [])
    assert slots == [-1, -1, -1] and native.load().gllm_meta_errors(1) & 8
    slots = prep([[5, 0, 1, 0, -1], [0, 60, 10, 1, -1]], [])
    assert slots == [-1] * 11 and native.load().gllm_meta_errors(1) & 4
    del table0


@pytest.mark.parametrize("n_stages", [1, 2])
def test_cuda_graph_decode_batches(cuda_ok, n_stages):
    """Decode-only micro-batches replayed from captured CUDA graphs (padded batch buckets): the
    virtual-clock schedule is unchanged, every request completes, and the sampled-step logits stay
    within 2e-2 of the fp32 oracle with tokens equal to its argmax wherever the margin is clear."""
    from oracle.model_ref import from_stage_workers
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    spec = MODELS["tiny"]
    reqs = _c1()
    watch = [0, 5, 17, 40]
    ex = LocalExecutor(spec, reqs, num_pages=4096, page_size=16, n_stages=n_stages, max_tokens=2560,
                       record_logits=True, record_ids=watch, seed=1, cuda_graphs=True)
    eng = Engine(reqs, scheduler="throttle", pipeline=PipelineConfig(depth=1), kv_config=KvConfig(4096, 16),
                 throttle=ThrottleConfig(), executor=ex)
    raw = eng.run()
    gold = {r["name"]: r for r in ENGINE["runs"]}["c1_throttle_d1"]
    assert [[it.batch_seq, it.schedule_time_ms, it.prefill_tokens, it.decode_tokens] for it in raw.iterations] \
        == gold["iterations"]
    assert ex.graph_replays > 20 and len(ex._graphs) >= 2, (ex.graph_replays, list(ex._graphs))
    for r in reqs:
        assert len(ex.outputs[r.id]) == r.output_tokens
    oracle = from_stage_workers(ex.stages)
    by_req = {}
    for rid, pos, lg in ex.logits:
        by_req.setdefault(rid, []).append((pos, lg))
    worst, agree, clear = 0.0, 0, 0
    for rid in watch:
        spec_r = reqs[rid]
        seq = np.concatenate([prompt_token_ids(rid, spec_r.input_tokens, spec.vocab),
                              np.asarray(ex.outputs[rid][:-1], dtype=np.int32)])
        ref = oracle.logits(seq).numpy()
        for pos, lg in by_req[rid]:
            want = ref[pos - 1]
            worst = max(worst, np.linalg.norm(lg - want) / np.linalg.norm(want))
            top2 = np.sort(want)[-2:]
            if top2[1] - top2[0] > 0.05:
                clear += 1
                agree += int(np.argmax(lg) == np.argmax(want))
    print(f"cuda graphs, {n_stages} stage(s): {ex.graph_replays} replays over {len(ex._graphs)} graphs, "
          f"worst logits rel err {worst:.3e}")
    assert worst < 2e-2, worst
    assert clear > 0 and agree == clear, (agree, clear)


def test_prefix_caching_logits(cuda_ok):
    """Requests sharing a 6-page system prompt: later requests map the cached pages instead of
    recomputing them; their sampled-step logits still match the fp32 oracle run on the FULL
    prompt (so the shared KV pages hold exactly the prefix's keys and values)."""
    from oracle.model_ref import from_stage_workers
    from paper_2504_14775_b200.executor import LocalExecutor
    from paper_2504_14775_b200.modelspec import MODELS

    spec = MODELS["tiny"]
    rng = np.random.default_rng(5)
    system = rng.integers(0, spec.vocab, 96).astype(np.int32)
    reqs, prompts = [], {}
    for i in range(10):
        tail = rng.integers(0, spec.vocab, int(rng.integers(3, 50))).astype(np.int32)
        prompts[i] = np.concatenate([system, tail])
        reqs.append(RequestSpec(i, 4.0 * i, len(prompts[i]), 5))
    ex = LocalExecutor(spec, reqs, num_pages=512, page_size=16, max_tokens=1024, record_logits=True, seed=2)
    for i, p in prompts.items():
        ex.register_prompt(i, p)
    eng = Engine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(512, 16), executor=ex,
                 throttle=ThrottleConfig(T=2, min_p=8), prefix_caching=True)
    eng.run()
    assert eng.kv.hit_tokens >= 8 * 96, eng.kv.hit_tokens
    oracle = from_stage_workers(ex.stages)
    worst = 0.0
    for rid, pos, lg in ex.logits:
        seq = np.concatenate([prompts[rid], np.asarray(ex.outputs[rid], dtype=np.int32)])[:pos]
        want = oracle.logits(seq).numpy()[pos - 1]
        worst = max(worst, float(np.linalg.norm(lg - want) / np.linalg.norm(want)))
    for r in reqs:
        assert len(ex.outputs[r.id]) == r.output_tokens
    print(f"prefix caching: {eng.kv.hit_tokens} cached prompt tokens reused, worst logits rel err {worst:.3e}")
    assert worst < 2e-2, worst


def test_graft_entry_smoke(cuda_ok):
    """The driver's round-end smoke: one tiny engine run on cuda:0 checked against the fp32 oracle."""
    import importlib
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    importlib.import_module("__graft_entry__").smoke()
