import sys, os, torch
sys.path.insert(0, '/root/repo')
from paper_2504_14775_b200 import native
seqs = eval(sys.argv[1]); n_heads = int(sys.argv[2]); n_kv = 8; ps = 16; hd = 128
ctx = [s + n for s, n in seqs]
pages_per = [-(-c // ps) for c in ctx]; num_pages = sum(pages_per) + 8; mpr = max(pages_per) + 1
perm = torch.randperm(num_pages); table = torch.zeros(len(seqs), mpr, dtype=torch.int32); k = 0
for i, p in enumerate(pages_per): table[i, :p] = perm[k:k + p]; k += p
table = table.cuda(); kc = torch.randn(num_pages, n_kv, ps, hd, device="cuda").bfloat16(); vc = torch.randn_like(kc)
T = sum(n for _, n in seqs); qkv = torch.randn(T, (n_heads + 2 * n_kv) * hd, device="cuda").bfloat16(); out = torch.empty(T, n_heads * hd, device="cuda").bfloat16()
qt = native.load().gllm_attention_q_tile(n_heads, n_kv); info, work, off = [], [], 0
for i, (s, n) in enumerate(seqs):
    info.append([i, s, n, off, -1]); work += [[i, q0] for q0 in range(0, n, qt)]; off += n
info = torch.tensor(info, dtype=torch.int32, device="cuda"); work_t = torch.tensor(work, dtype=torch.int32, device="cuda")
native.call("gllm_attn_mixed_paged", qkv.data_ptr(), info.data_ptr(), work_t.data_ptr(), len(work), len(work), table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(), native.stream_handle())
torch.cuda.synchronize(); print("ok", sys.argv[1], out.float().abs().mean().item(), flush=True)
