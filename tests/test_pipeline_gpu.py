"""PP=2 pipeline runtime with REAL stage workers: two processes sharing cuda:0.

NCCL cannot put two ranks on one GPU, so activations go through the host
(HostTransport over gloo); everything else is the production path: metadata
published ahead of activations, stage 0 on rank 0, stage 1 (+LM head, argmax)
on rank 1, sampled ids returned to rank 0's token history. Tokens are checked
against the fp32 oracle under teacher forcing.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _reqs():
    from paper_2504_14775_b200 import RequestSpec
    rng = np.random.Generator(np.random.PCG64(9))
    return [RequestSpec(i, float(i) * 2.0, int(rng.integers(20, 200)), int(rng.integers(2, 10))) for i in range(10)]


def _run(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2504_14775_b200 import KvConfig, PipelineConfig, ThrottleConfig
    from paper_2504_14775_b200.modelspec import MODELS
    from paper_2504_14775_b200.pipeline import HostTransport, MetaChannel, PipelineExecutor, worker_loop
    from paper_2504_14775_b200.serving import ServingEngine
    spec = MODELS["tiny"]
    reqs = _reqs()
    g = dist.group.WORLD
    meta, tr = MetaChannel(g, world), HostTransport(g)
    try:
        if rank == 0:
            ex = PipelineExecutor(spec, reqs, world=world, meta=meta, transport=tr, num_pages=256, page_size=16,
                                  max_tokens=1024, seed=4)
            eng = ServingEngine(reqs, pipeline=PipelineConfig(depth=world), kv_config=KvConfig(256, 16),
                                throttle=ThrottleConfig(T=4, min_p=16), executor=ex)
            eng.run()
            ex.shutdown()
            q.put(("ok", {r.id: ex.outputs.get(r.id, []) for r in reqs}))
        else:
            out = worker_loop(spec, reqs, rank=rank, world=world, meta=meta, transport=tr, num_pages=256,
                              page_size=16, max_tokens=1024, seed=4)
            q.put(("worker", out["batches"]))
    except Exception:
        import traceback
        q.put(("error", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_pp2_real_stages_share_one_gpu(cuda_ok):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    err = [m for m in msgs if m[0] == "error"]
    assert not err, err[0][1]
    outputs = next(m for m in msgs if m[0] == "ok")[1]

    from oracle.model_ref import RefDecoder
    from paper_2504_14775_b200.modelspec import MODELS, init_embed, init_layer
    from paper_2504_14775_b200.workload import prompt_token_ids
    spec = MODELS["tiny"]
    dev = torch.device("cuda")
    oracle = RefDecoder(spec, [init_layer(spec, l, 4, dev) for l in range(spec.n_layers)], None,
                        init_embed(spec, 4, dev, "embed"), init_embed(spec, 4, dev, "final_norm"),
                        init_embed(spec, 4, dev, "lm_head"))
    clear = agree = 0
    for r in _reqs():
        out = outputs[r.id]
        assert len(out) == r.output_tokens
        seq = np.concatenate([prompt_token_ids(r.id, r.input_tokens, spec.vocab), np.asarray(out[:-1], np.int32)])
        ref = oracle.logits(seq).numpy()
        for i, tok in enumerate(out):
            row = ref[r.input_tokens - 1 + i]
            top2 = np.sort(row)[-2:]
            if top2[1] - top2[0] > 0.05:
                clear += 1
                agree += int(np.argmax(row) == tok)
    assert clear > 0 and agree == clear, (agree, clear)
