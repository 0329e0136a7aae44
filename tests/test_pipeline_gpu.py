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


def _run(rank, world, port, q, lookahead=False):
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
                                throttle=ThrottleConfig(T=4, min_p=16), executor=ex, lookahead=lookahead)
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


@pytest.mark.parametrize("lookahead", [False, True])
def test_pp2_real_stages_share_one_gpu(cuda_ok, lookahead):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run, args=(r, 2, port, q, lookahead)) for r in range(2)]
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


# One command per BASELINE pipeline config (README / DESIGN "Multi-GPU"): bench.py under torchrun,
# every rank on cuda:0 with host-staged activations (NCCL cannot put two ranks on one GPU).
# Layers are truncated (--layers) so 8 stage processes fit one GPU; the shapes (d, heads, d_ff,
# vocab, bias, RoPE scaling), trace, scheduler and depth are the config's own.
PP_CONFIGS = {
    "c3_pp2": ["--model", "qwen2.5-14b", "--gpus", "2", "--layers", "8"],
    "c3_pp4": ["--model", "qwen2.5-14b", "--gpus", "4", "--layers", "8"],
    "c4_pp4_throttle": ["--model", "qwen2.5-32b", "--gpus", "4", "--layers", "8", "--scheduler", "throttle"],
    "c4_pp4_sarathi": ["--model", "qwen2.5-32b", "--gpus", "4", "--layers", "8", "--scheduler", "sarathi"],
    # 4-8k prompts: warm in until the first prompts finished and decodes run (the timed window must
    # hold output tokens)
    "c5_pp8": ["--model", "llama3.1-70b", "--gpus", "8", "--layers", "8", "--trace", "c5", "--rate", "4",
               "--warm-max-iters", "60", "--warm-decodes", "8"],
}


@pytest.mark.parametrize("name", list(PP_CONFIGS))
def test_bench_pipeline_configs_one_gpu(cuda_ok, name):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = PP_CONFIGS[name]
    n = args[args.index("--gpus") + 1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py",
           "--n-requests", "48", "--steps", "4", "--warmup", "3", "--warm-max-iters", "6", "--profile-steps", "3",
           "--no-cpu-baseline", *args]   # the config's own flags last: they override the defaults
    env = dict(os.environ, GLLM_PP_TRANSPORT="host")
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    rank0 = "\n".join(ln for ln in r.stderr.splitlines() if "[rank0]" in ln or "Error" in ln)
    assert r.returncode == 0, r.stdout[-2000:] + rank0[-6000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    print(f"\n{name}: {line['value']:.1f} tok/s device window, e2e {line['e2e']['value']:.1f}, "
          f"bubble {line['serving']['bubble_frac_per_stage']}, dominant {line['roofline']['kernel']}")
    assert line["n_gpus"] == int(n) and line["config"]["parallelism"] == f"pp{n}"
    assert line["steps"] == 4 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert len(line["serving"]["bubble_frac_per_stage"]) == int(n)
    assert all(0.0 <= b <= 1.0 for b in line["serving"]["bubble_frac_per_stage"])
    # the profiled window covers every stage: the last stage's LM head and the first's embedding
    assert "gemm_lm_head" in line["roofline"]["classes"] and "embed" in line["roofline"]["classes"]
    assert line["gpu_launches"] > 0
