import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from golden_io import load  # noqa: E402
from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, RequestSpec, ThrottleConfig, native  # noqa: E402
from paper_2504_14775_b200 import stage as stage_mod  # noqa: E402
from paper_2504_14775_b200.executor import LocalExecutor  # noqa: E402
from paper_2504_14775_b200.modelspec import MODELS  # noqa: E402

rows = load("traces.json.gz")["c1"][:4]
reqs = [RequestSpec(i, a, b, c) for i, (a, b, c) in enumerate(rows)]
ex = LocalExecutor(MODELS["tiny"], reqs, num_pages=4096, page_size=16, n_stages=2, max_tokens=2560, seed=1)
orig = stage_mod.StageWorker.forward
count = [0]


def fwd(self, pb, meta_dev, hidden=None, sampled=None, logits=None, stream=None):
    if self.is_first and count[0] < 3:
        count[0] += 1
        torch.cuda.synchronize()
        print("pb", pb.n_seqs, pb.n_tokens, pb.n_emit, pb.n_work, pb.n_deltas, pb.n_prompts, pb.data[:40].tolist())
        print("meta_dev", meta_dev[:40].tolist())
        T = pb.n_tokens
        tp = torch.full((T,), -7, dtype=torch.int32, device="cuda")
        ts = torch.full((T,), -7, dtype=torch.int32, device="cuda")
        ti = torch.full((T,), -7, dtype=torch.int32, device="cuda")
        er = torch.full((max(pb.n_emit, 1),), -7, dtype=torch.int32, device="cuda")
        b = self.cbatch(pb, meta_dev, hidden, sampled, logits)
        native.call("gllm_prepare_batch", C.byref(self.cstage), C.byref(b), tp.data_ptr(), ts.data_ptr(), ti.data_ptr(),
                    er.data_ptr(), native.stream_handle(stream))
        torch.cuda.synchronize()
        print("tok_pos", tp[:8].tolist(), tp[-4:].tolist())
        print("tok_slot", ts[:8].tolist())
        print("tok_id", ti[:8].tolist(), ti[-4:].tolist())
        print("hist row0", self.token_hist[0, :8].tolist())
        print("table row0", self.block_table[0, :8].tolist())
    return orig(self, pb, meta_dev, hidden, sampled, logits, stream)


stage_mod.StageWorker.forward = fwd
eng = Engine(reqs, pipeline=PipelineConfig(depth=2), kv_config=KvConfig(4096, 16), throttle=ThrottleConfig(), executor=ex)
for _ in range(6):
    eng.step()
torch.cuda.synchronize()
print("done")
