"""Find the first micro-batch/stage that produces non-finite activations (tiny model, 2 stages)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from golden_io import load  # noqa: E402
from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig  # noqa: E402
from paper_2504_14775_b200 import stage as stage_mod  # noqa: E402
from paper_2504_14775_b200.executor import LocalExecutor  # noqa: E402
from paper_2504_14775_b200.modelspec import MODELS  # noqa: E402

stages = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rows = load("traces.json.gz")["c1"]
reqs = [RequestSpec(i, a, b, c) for i, (a, b, c) in enumerate(rows)]
ex = LocalExecutor(MODELS["tiny"], reqs, num_pages=4096, page_size=16, n_stages=stages, max_tokens=2560, seed=1)
orig = stage_mod.StageWorker.forward


def fwd(self, pb, meta_dev, hidden=None, sampled=None, logits=None, stream=None):
    orig(self, pb, meta_dev, hidden, sampled, logits, stream)
    torch.cuda.synchronize()
    h = hidden[: pb.n_tokens].float()
    bad = ~torch.isfinite(h).all(-1)
    ws = self.workspace
    if bad.any() or (self.is_last and pb.n_emit and (sampled[: pb.n_emit] >= self.spec.vocab).any()):
        idx = bad.nonzero().flatten().tolist()
        info = pb.data[: 5 * pb.n_seqs].reshape(-1, 5).tolist()
        print("NONFINITE seq", pb.seq, "stage_first", self.is_first, "tokens", pb.n_tokens, "bad rows", idx[:10], len(idx))
        print("seq_info", info[:30])
        sp = self.spec
        T = self.max_tokens
        a256 = lambda x: (x + 255) // 256 * 256
        off_h = a256(T * sp.d_model * 2)
        off_qkv = off_h + a256(T * sp.d_model * 2)
        off_attn = off_qkv + a256(T * sp.qkv_width * 2)
        n = pb.n_tokens
        qkv = ws[off_qkv: off_qkv + n * sp.qkv_width * 2].view(torch.bfloat16).view(n, -1).float()
        att = ws[off_attn: off_attn + n * sp.n_heads * 128 * 2].view(torch.bfloat16).view(n, -1).float()
        print("qkv finite", torch.isfinite(qkv).all().item(), "attn finite", torch.isfinite(att).all().item())
        print("attn head0[:8]", att[0, :8].tolist(), "head1[:8]", att[0, 128:136].tolist())
        L = self.k_cache.shape[0]
        row = info[0][0]
        pages = self.block_table[row, :20].tolist()
        print("pages", pages)
        kc = self.k_cache[L - 1, pages].float()
        print("k_cache finite", torch.isfinite(kc).all().item(), "v finite", torch.isfinite(self.v_cache[L - 1, pages].float()).all().item())
        nf = (~torch.isfinite(kc)).nonzero()[:5].tolist()
        print("nonfinite k at", nf)
        raise SystemExit(1)


stage_mod.StageWorker.forward = fwd
eng = Engine(reqs, pipeline=PipelineConfig(depth=2), kv_config=KvConfig(4096, 16), throttle=ThrottleConfig(), executor=ex)
n = 0
while eng.step():
    n += 1
print("ok", n, ex.launches)
