"""Per-kernel parity on the B200 through the C-ABI (fp32 torch references of the same op)."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib(cuda_ok):
    from paper_2504_14775_b200 import native
    return native


def _rel(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


GEMM_SHAPES = [
    (1, 512, 256), (7, 256, 256), (64, 1536, 256), (128, 512, 4096), (130, 4096, 4096),
    (300, 6144, 4096), (1000, 4096, 14336), (33, 28672, 4096), (2048, 4096, 4096),
    (2009, 6144, 4096),
    (2009, 4096, 14336),  # auto: swap-AB units of 512 weights x 224 tokens (gemm_swab.cu), bias + residual
]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_tcgen05(lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    ref = A.float() @ B.float().T
    for bn in (0, 64, 128, 256):
        if N % (bn or 64):
            continue
        for splits in (0, 1, 3):
            C_ = torch.full((M, N), float("nan"), device="cuda").bfloat16()
            lib.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C_.data_ptr(), N, M, N, K, None, None, 0,
                     bn, splits, ws.data_ptr(), ws.numel(), lib.stream_handle())
            torch.cuda.synchronize()
            assert torch.isfinite(C_.float()).all(), (bn, splits)
            assert _rel(C_, ref) < 8e-3, (bn, splits, _rel(C_, ref))
    C_ = torch.empty((M, N), device="cuda").bfloat16()
    lib.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C_.data_ptr(), N, M, N, K, bias.data_ptr(),
             res.data_ptr(), N, 0, 0, ws.data_ptr(), ws.numel(), lib.stream_handle())
    torch.cuda.synchronize()
    assert _rel(C_, ref + bias.float() + res.float()) < 8e-3


@pytest.mark.parametrize("M,N,K", [(4, 5120, 5120), (1, 32000, 256), (16, 4096, 14336), (32, 6144, 4096), (31, 5120, 5120),
                                   (7, 256, 768), (48, 5120, 5120), (64, 4096, 14336), (33, 6144, 4096),
                                   (100, 7168, 5120), (128, 5120, 5120), (65, 4096, 4096)])
def test_gemm_skinny_stream_k(lib, M, N, K):
    """Decode-sized GEMMs (swap-AB stream-K: tiles shared by CTAs fixed up by the last arriver) vs
    fp32, with bias + residual, after a split-K GEMM has used the same workspace (its partials
    must not clobber the tile counters), and bit-stable across runs."""
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    A2 = torch.randn(100, K, device="cuda", generator=g).bfloat16()
    junk = torch.empty(100, N, device="cuda").bfloat16()
    ref = A.float() @ B.float().T + bias.float() + res.float()
    outs = []
    for _ in range(2):
        lib.call("gllm_gemm_bf16", A2.data_ptr(), K, B.data_ptr(), K, junk.data_ptr(), N, 100, N, K, None, None, 0,
                 0, 3, ws.data_ptr(), ws.numel(), lib.stream_handle())            # split-K on the same workspace
        C_ = torch.full((M, N), float("nan"), device="cuda").bfloat16()
        lib.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C_.data_ptr(), N, M, N, K, bias.data_ptr(),
                 res.data_ptr(), N, 0, 0, ws.data_ptr(), ws.numel(), lib.stream_handle())
        outs.append(C_)
    torch.cuda.synchronize()
    assert _rel(outs[0], ref) < 8e-3, _rel(outs[0], ref)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,N,K", [(64, 5120, 5120), (33, 4096, 4096), (100, 4096, 14336), (128, 5120, 13824),
                                   (64, 8192, 8192), (48, 6144, 4096)])
def test_gemm_one_row_tile(lib, M, N, K):
    """One row tile (33-128 tokens, the medium decode batches): the auto plan (whole-K narrow tiles or
    split-K + reduce) with bias + residual against fp32, bit-stable across runs, and the forced
    whole-K plan."""
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    outs = []
    for splits in (0, 0, 1):
        C_ = torch.full((M, N), float("nan"), device="cuda").bfloat16()
        lib.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C_.data_ptr(), N, M, N, K, bias.data_ptr(),
                 res.data_ptr(), N, 0, splits, ws.data_ptr(), ws.numel(), lib.stream_handle())
        outs.append(C_)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T + bias.float() + res.float()
    assert torch.isfinite(outs[0].float()).all()
    assert _rel(outs[0], ref) < 8e-3 and _rel(outs[2], ref) < 8e-3
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,N,K", [(2048, 4096, 14336), (33, 28672, 4096), (1000, 4096, 4096), (3, 6144, 4096),
                                   (2009, 6144, 4096), (1500, 8192, 8192),
                                   # swap-AB units: token widths 224 / 224 / 192 / 160, ragged last tiles
                                   (2009, 4096, 4096), (1800, 4096, 14336), (1536, 4096, 4096), (1024, 5120, 5120),
                                   (512, 5120, 5120), (512, 5120, 13824), (480, 4096, 14336)])
def test_gemm_deterministic(lib, M, N, K):
    """Auto tiling (incl. split-K partial sums) is bit-stable across runs and agrees with whole-tile
    (force_splits=1) tiling to fp32 rounding."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    outs = []
    for splits in (0, 0, 0, 1):
        C_ = torch.full((M, N), float("nan"), device="cuda").bfloat16()
        lib.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C_.data_ptr(), N, M, N, K, None, res.data_ptr(),
                 N, 0, splits, ws.data_ptr(), ws.numel(), lib.stream_handle())
        outs.append(C_)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    ref = A.float() @ B.float().T + res.float()
    assert _rel(outs[0], ref) < 8e-3 and _rel(outs[3], ref) < 8e-3


@pytest.mark.parametrize("M,d_ff,K", [(1, 768, 256), (37, 14336, 4096), (300, 768, 256), (2048, 14336, 4096),
                                      (2009, 14336, 4096)])   # swap-AB SwiGLU epilogue when GLLM_GEMM_SWAB_SWIGLU=1
def test_gemm_swiglu_fused(lib, M, d_ff, K):
    from paper_2504_14775_b200.modelspec import interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(M + d_ff)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(2 * d_ff, K, device="cuda", generator=g) * 0.05).bfloat16()
    Wi = interleave_gate_up(W, d_ff).contiguous()
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    gu = (A.float() @ W.float().T).bfloat16().float()
    ref = torch.nn.functional.silu(gu[:, :d_ff]).bfloat16().float() * gu[:, d_ff:]
    for bn, splits in ((0, 0), (128, 1), (256, 1), (128, 3)):
        if splits > 1 and M * 2 * d_ff * 4 * splits > ws.numel():
            continue
        act = torch.full((M, d_ff), float("nan"), device="cuda").bfloat16()
        lib.call("gllm_gemm_swiglu_bf16", A.data_ptr(), K, Wi.data_ptr(), K, act.data_ptr(), d_ff, M, d_ff, K, bn,
                 splits, ws.data_ptr(), ws.numel(), lib.stream_handle())
        torch.cuda.synchronize()
        assert torch.isfinite(act.float()).all(), (bn, splits)
        assert _rel(act, ref) < 1e-2, (bn, splits, _rel(act, ref))


@pytest.mark.parametrize("M,name,splits", [(5, "llama3-8b", 0), (300, "llama3-8b", 0), (2009, "llama3-8b", 1),
                                           (77, "qwen2.5-14b", 1), (64, "qwen2.5-14b", 0), (130, "tiny", 1),
                                           # swap-AB RoPE + KV-write epilogue (+ bias) when GLLM_GEMM_SWAB_QKV=1
                                           (2009, "llama3-8b", 0), (1024, "qwen2.5-14b", 0), (1500, "llama3.1-70b", 0)])
def test_gemm_qkv_rope_fused_matches_unfused(lib, M, name, splits):
    """Fused QKV+RoPE+KV-write epilogue == GEMM(+bias) -> rope_kv_write (bit-identical when both use the same
    tile width; the auto-tuned tilings may differ, giving <= 1 bf16 ulp from fp32 accumulation order)."""
    from paper_2504_14775_b200.modelspec import MODELS, rope_table
    spec = MODELS[name]
    H, KV, d, ps = spec.n_heads, spec.n_kv_heads, spec.d_model, 16
    Q = spec.qkv_width
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    W = (torch.randn(Q, d, device="cuda", generator=g) * 0.03).bfloat16()
    bias = torch.randn(Q, device="cuda", generator=g).bfloat16() if spec.qkv_bias else None
    rope = torch.from_numpy(rope_table(spec, 4096)).cuda()
    pos = torch.randint(0, 4000, (M,), dtype=torch.int32, device="cuda")
    slot = torch.randperm(512 * ps, device="cuda")[:M].to(torch.int32)
    ws = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
    st = lib.stream_handle()
    # unfused reference path
    ref = torch.empty(M, Q, device="cuda").bfloat16()
    lib.call("gllm_gemm_bf16", A.data_ptr(), d, W.data_ptr(), d, ref.data_ptr(), Q, M, Q, d,
             None if bias is None else bias.data_ptr(), None, 0, 0, 1 if splits == 1 else 0, ws.data_ptr(),
             ws.numel(), st)
    kr = torch.zeros(512, KV, ps, 128, device="cuda").bfloat16()
    vr = torch.zeros_like(kr)
    lib.call("gllm_rope_kv_write", ref.data_ptr(), M, H, KV, 128, pos.data_ptr(), slot.data_ptr(), rope.data_ptr(),
             kr.data_ptr(), vr.data_ptr(), ps, st)
    # fused
    out = torch.zeros(M, Q, device="cuda").bfloat16()
    kf = torch.zeros_like(kr)
    vf = torch.zeros_like(kr)
    lib.call("gllm_gemm_qkv_rope_bf16", A.data_ptr(), d, W.data_ptr(), d, None if bias is None else bias.data_ptr(),
             out.data_ptr(), M, d, H, KV, pos.data_ptr(), slot.data_ptr(), rope.data_ptr(), kf.data_ptr(), vf.data_ptr(),
             ps, 0, splits, ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    assert _rel(out[:, : H * 128], ref[:, : H * 128]) < 4e-3
    assert _rel(kf, kr) < 4e-3 and _rel(vf, vr) < 4e-3
    # and against an fp32 torch reference of the whole fused op (GEMM + bias -> RoPE on q/k -> paged K/V)
    x = A.float() @ W.float().T + (bias.float() if bias is not None else 0.0)
    cs = rope[pos.long()]
    c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]

    def rot(t):
        return torch.cat([t[..., :64] * c - t[..., 64:] * s, t[..., 64:] * c + t[..., :64] * s], -1)
    pg, off = (slot // ps).long(), (slot % ps).long()
    q32 = rot(x[:, : H * 128].view(M, H, 128))
    k32 = rot(x[:, H * 128:(H + KV) * 128].view(M, KV, 128))
    v32 = x[:, (H + KV) * 128:].view(M, KV, 128)
    errs = (_rel(out[:, : H * 128].view(M, H, 128), q32), _rel(kf[pg, :, off], k32), _rel(vf[pg, :, off], v32))
    print(f"fused qkv+rope M={M} {name}: rel err vs fp32 q/k/v = {errs[0]:.2e} / {errs[1]:.2e} / {errs[2]:.2e}")
    assert max(errs) < 8e-3, errs
    if splits == 1 and M >= 2000:   # same 256-wide tiles on both paths: bit-identical
        assert torch.equal(out[:, : H * 128], ref[:, : H * 128]) and torch.equal(kf, kr) and torch.equal(vf, vr)


def test_rmsnorm_and_silu(lib):
    x = torch.randn(37, 4096, device="cuda").bfloat16()
    w = (torch.rand(4096, device="cuda") + 0.5).bfloat16()
    out = torch.empty_like(x)
    lib.call("gllm_rmsnorm", x.data_ptr(), 4096, None, w.data_ptr(), out.data_ptr(), 37, 4096, 1e-5, lib.stream_handle())
    idx = torch.tensor([5, 0, 36], dtype=torch.int32, device="cuda")
    out2 = torch.empty(3, 4096, device="cuda").bfloat16()
    lib.call("gllm_rmsnorm", x.data_ptr(), 4096, idx.data_ptr(), w.data_ptr(), out2.data_ptr(), 3, 4096, 1e-5,
             lib.stream_handle())
    torch.cuda.synchronize()
    xf = x.float()
    ref = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert _rel(out, ref) < 5e-3
    assert torch.equal(out2, out[[5, 0, 36]])
    gu = torch.randn(19, 2 * 768, device="cuda").bfloat16()
    act = torch.empty(19, 768, device="cuda").bfloat16()
    lib.call("gllm_silu_mul", gu.data_ptr(), 768, act.data_ptr(), 19, lib.stream_handle())
    torch.cuda.synchronize()
    g, u = gu.float()[:, :768], gu.float()[:, 768:]
    assert _rel(act, torch.nn.functional.silu(g) * u) < 5e-3


def test_argmax(lib):
    for V in (32000, 128256, 152064):
        x = torch.randn(9, V, device="cuda").bfloat16()
        x[3, 777] = 50.0
        x[4, :] = 1.0       # ties -> lowest index
        out = torch.empty(9, dtype=torch.int32, device="cuda")
        lib.call("gllm_argmax", x.data_ptr(), 9, V, out.data_ptr(), lib.stream_handle())
        torch.cuda.synchronize()
        ref = x.float().argmax(-1)
        assert out.tolist() == ref.tolist()
        assert out[3].item() == 777 and out[4].item() == 0


def _paged_setup(n_kv, hd, ps, ctx_lens, num_pages, seed=0):
    """Random paged K/V; returns caches, block table and the dense per-seq K/V."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    perm = torch.randperm(num_pages, generator=g).tolist()
    mpr = max(-(-c // ps) for c in ctx_lens) + 1
    table = torch.zeros(len(ctx_lens), mpr, dtype=torch.int32)
    kc = torch.randn(num_pages, n_kv, ps, hd, generator=g).bfloat16()
    vc = torch.randn(num_pages, n_kv, ps, hd, generator=g).bfloat16()
    dense = []
    for i, c in enumerate(ctx_lens):
        pages = [perm.pop() for _ in range(-(-c // ps))]
        table[i, : len(pages)] = torch.tensor(pages)
        idx = torch.tensor([pages[p // ps] for p in range(c)])
        off = torch.tensor([p % ps for p in range(c)])
        dense.append((kc[idx, :, off], vc[idx, :, off]))  # [c, n_kv, hd]
        # stale slots past the context in the last page hold garbage (NaN here): must never leak
        if c % ps:
            kc[pages[-1], :, c % ps:] = float("nan")
            vc[pages[-1], :, c % ps:] = float("nan")
    return kc.cuda(), vc.cuda(), table.cuda(), mpr, dense


LONG_SEQS = [(37, 1), (1500, 517), (0, 300), (2000, 129), (4, 1), (900, 2)]


@pytest.mark.parametrize("n_heads,n_kv,ps,seqs,n_split", [(32, 8, 16, None, 1), (40, 8, 16, None, 1),
                                                          (64, 8, 16, None, 1), (2, 1, 16, None, 1),
                                                          (32, 8, 16, LONG_SEQS, 1), (40, 8, 8, LONG_SEQS, 1),
                                                          (64, 8, 16, LONG_SEQS, 1), (32, 8, 16, LONG_SEQS, 3),
                                                          (40, 8, 8, LONG_SEQS, 2), (64, 8, 16, LONG_SEQS, 8),
                                                          (32, 8, 16, None, 4)])
def test_attention_mixed(lib, n_heads, n_kv, ps, seqs, n_split):
    hd = 128
    # (start, n_new): decodes, a first chunk, a later chunk, a long decode
    seqs = seqs or [(37, 1), (0, 45), (100, 70), (511, 1), (15, 1), (3, 200)]
    ctx = [s + n for s, n in seqs]
    kc, vc, table, mpr, dense = _paged_setup(n_kv, hd, ps, ctx, num_pages=sum(-(-c // ps) for c in ctx) + 64)
    T = sum(n for _, n in seqs)
    qkv = torch.randn(T, (n_heads + 2 * n_kv) * hd, device="cuda").bfloat16()
    q_tile = lib.load().gllm_attention_q_tile(n_heads, n_kv)
    info, work, off = [], [], 0
    for i, (s, n) in enumerate(seqs):
        info.append([i, s, n, off, -1])
        if n > 1:
            work += [[i, q0] for q0 in range(0, n, q_tile)]
        off += n
    n_pf = len(work)
    work += [[i, 0] for i, (s, n) in enumerate(seqs) if n == 1]   # contract: prefill tiles first
    info_t = torch.tensor(info, dtype=torch.int32, device="cuda")
    work_t = torch.tensor(work, dtype=torch.int32, device="cuda")
    out = torch.zeros(T, n_heads * hd, device="cuda").bfloat16()
    if n_split == 1:
        lib.call("gllm_attn_mixed_paged", qkv.data_ptr(), info_t.data_ptr(), work_t.data_ptr(), len(work), n_pf,
                 table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(),
                 lib.stream_handle())
    else:
        ws = torch.empty(lib.load().gllm_attn_split_workspace_bytes(n_pf, n_split, n_kv), dtype=torch.uint8,
                         device="cuda")
        lib.call("gllm_attn_mixed_paged_split", qkv.data_ptr(), info_t.data_ptr(), work_t.data_ptr(), len(work), n_pf,
                 table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(),
                 n_split, ws.data_ptr(), ws.numel(), lib.stream_handle())
    torch.cuda.synchronize()
    g = n_heads // n_kv
    for i, (s, n) in enumerate(seqs):
        o = info[i][3]
        q = qkv[o:o + n, : n_heads * hd].float().view(n, n_heads, hd)
        k, v = dense[i]
        k = k.float().repeat_interleave(g, dim=1)
        v = v.float().repeat_interleave(g, dim=1)
        att = torch.einsum("thd,shd->hts", q.cpu(), k) / hd ** 0.5
        qpos = torch.arange(s, s + n)[:, None]
        kpos = torch.arange(s + n)[None, :]
        att = att.masked_fill(kpos > qpos, float("-inf")).softmax(-1)
        ref = torch.einsum("hts,shd->thd", att, v).reshape(n, -1)
        assert _rel(out[o:o + n].cpu(), ref) < 1e-2, (i, s, n)


def test_rope_kv_write(lib):
    from paper_2504_14775_b200.modelspec import MODELS, rope_table
    spec = MODELS["llama3-8b"]
    H, KV, hd, ps = spec.n_heads, spec.n_kv_heads, spec.head_dim, 16
    T = 23
    rope = torch.from_numpy(rope_table(spec, 4096)).cuda()
    qkv = torch.randn(T, (H + 2 * KV) * hd, device="cuda").bfloat16()
    orig = qkv.clone()
    pos = torch.randint(0, 4000, (T,), dtype=torch.int32, device="cuda")
    slot = torch.randperm(64 * ps, device="cuda")[:T].to(torch.int32)
    kc = torch.zeros(64, KV, ps, hd, device="cuda").bfloat16()
    vc = torch.zeros_like(kc)
    lib.call("gllm_rope_kv_write", qkv.data_ptr(), T, H, KV, hd, pos.data_ptr(), slot.data_ptr(), rope.data_ptr(),
             kc.data_ptr(), vc.data_ptr(), ps, lib.stream_handle())
    torch.cuda.synchronize()
    cs = rope[pos.long()]
    c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]

    def rot(x):
        x1, x2 = x[..., :64], x[..., 64:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)
    of = orig.float()
    q_ref = rot(of[:, : H * hd].view(T, H, hd))
    k_ref = rot(of[:, H * hd:(H + KV) * hd].view(T, KV, hd))
    v_ref = of[:, (H + KV) * hd:].view(T, KV, hd)
    assert _rel(qkv[:, : H * hd].view(T, H, hd), q_ref) < 5e-3
    pg, off = (slot // ps).long(), (slot % ps).long()
    assert _rel(kc[pg, :, off], k_ref) < 5e-3
    assert torch.equal(vc[pg, :, off], v_ref.bfloat16())


DECODE_SETS = {
    "mixed_ctx": (0, 1, 15, 16, 17, 300, 1023, 2047),
    "two_long": (2999, 700),          # few sequences: cluster KV split of up to 4 ranks
    "one_very_long": (8191,),
    "short_and_long": (5, 1500, 40),  # ranks with empty page ranges
    # 48 decodes x 8 kv heads = 384 items: one wave of three 4-warp CTAs per SM (2-stage page ring)
    "medium_batch": tuple((37 * i) % 900 for i in range(48)),
}


@pytest.mark.parametrize("n_heads,n_kv,ctxs,auto", [(32, 8, "mixed_ctx", False), (64, 8, "mixed_ctx", False),
                                                    (40, 8, "mixed_ctx", False), (32, 8, "mixed_ctx", True),
                                                    (64, 8, "two_long", True), (40, 8, "two_long", True),
                                                    (32, 8, "one_very_long", True), (40, 8, "short_and_long", True),
                                                    (32, 8, "two_long", False), (40, 8, "medium_batch", False),
                                                    (64, 8, "medium_batch", True)])
def test_attention_decode_only_launch(lib, n_heads, n_kv, ctxs, auto):
    """All-decode micro-batch: the decode-only instantiation (no prefill resources) must agree too;
    `auto` passes the host metadata, so few long sequences take the cluster KV split."""
    hd, ps = 128, 16
    seqs = [(c, 1) for c in DECODE_SETS[ctxs]]
    ctx = [s + 1 for s, _ in seqs]
    kc, vc, table, mpr, dense = _paged_setup(n_kv, hd, ps, ctx, num_pages=sum(-(-c // ps) for c in ctx) + 64, seed=3)
    T = len(seqs)
    qkv = torch.randn(T, (n_heads + 2 * n_kv) * hd, device="cuda").bfloat16()
    info_h = torch.tensor([[i, s, 1, i, -1] for i, (s, _) in enumerate(seqs)], dtype=torch.int32)
    work_h = torch.tensor([[i, 0] for i in range(T)], dtype=torch.int32)
    info, work = info_h.cuda(), work_h.cuda()
    out = torch.zeros(T, n_heads * hd, device="cuda").bfloat16()
    if auto:
        lib.call("gllm_attn_mixed_paged_auto", qkv.data_ptr(), info.data_ptr(), work.data_ptr(), T, 0, table.data_ptr(),
                 mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(),
                 info_h.data_ptr(), work_h.data_ptr(), None, 0, lib.stream_handle())
    else:
        lib.call("gllm_attn_mixed_paged", qkv.data_ptr(), info.data_ptr(), work.data_ptr(), T, 0, table.data_ptr(), mpr,
                 kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(), lib.stream_handle())
    torch.cuda.synchronize()
    g = n_heads // n_kv
    for i, (s, _) in enumerate(seqs):
        q = qkv[i, : n_heads * hd].float().view(n_heads, hd)
        k, v = dense[i]
        k = k.float().repeat_interleave(g, dim=1)
        v = v.float().repeat_interleave(g, dim=1)
        att = (torch.einsum("hd,shd->hs", q.cpu(), k) / hd ** 0.5).softmax(-1)
        ref = torch.einsum("hs,shd->hd", att, v).reshape(-1)
        assert _rel(out[i].cpu(), ref) < 1e-2, (i, s)


def _attn_ref_gpu(qkv, n_heads, n_kv, hd, s, n, o, k, v):
    """fp32 causal attention of one sequence's n new queries over its s+n keys (GPU, per head)."""
    g = n_heads // n_kv
    q = qkv[o:o + n, : n_heads * hd].float().view(n, n_heads, hd)
    k = k.cuda().float()
    v = v.cuda().float()
    qpos = torch.arange(s, s + n, device="cuda")[:, None]
    kpos = torch.arange(s + n, device="cuda")[None, :]
    out = torch.empty(n, n_heads, hd, device="cuda")
    for h in range(n_heads):
        att = (q[:, h] @ k[:, h // g].T) / hd ** 0.5
        att = att.masked_fill(kpos > qpos, float("-inf")).softmax(-1)
        out[:, h] = att @ v[:, h // g]
    return out.reshape(n, -1)


C5_SEQS = [(4096, 2048), (6016, 2048), (8064, 128), (8191, 1), (8000, 1), (7000, 1), (2, 1)]
DECODE_8K = [(8191, 1)] * 8 + [(8100, 1)] * 8


@pytest.mark.parametrize("n_heads,n_kv,seqs,n_split", [(64, 8, "c5", 1), (40, 8, "c5", 1), (64, 8, "c5", 4),
                                                       (64, 8, "dec8k", 1), (40, 8, "dec8k", 1)])
def test_attention_long_context(lib, n_heads, n_kv, seqs, n_split):
    """C5 shapes: 2048-token prefill chunks after 4096-6016 cached tokens, a tail chunk at 8064,
    and decode batches at ~8k context (G=8 Llama-3.1-70B, G=5 Qwen2.5); fp32 GPU reference."""
    hd, ps = 128, 16
    seqs = C5_SEQS if seqs == "c5" else DECODE_8K
    ctx = [s + n for s, n in seqs]
    kc, vc, table, mpr, dense = _paged_setup(n_kv, hd, ps, ctx, num_pages=sum(-(-c // ps) for c in ctx) + 64, seed=7)
    T = sum(n for _, n in seqs)
    qkv = torch.randn(T, (n_heads + 2 * n_kv) * hd, device="cuda").bfloat16()
    q_tile = lib.load().gllm_attention_q_tile(n_heads, n_kv)
    info, work, off = [], [], 0
    for i, (s, n) in enumerate(seqs):
        info.append([i, s, n, off, -1])
        if n > 1:
            work += [[i, q0] for q0 in range(0, n, q_tile)]
        off += n
    n_pf = len(work)
    work += [[i, 0] for i, (s, n) in enumerate(seqs) if n == 1]
    info_h = torch.tensor(info, dtype=torch.int32)
    work_h = torch.tensor(work, dtype=torch.int32)
    info_t, work_t = info_h.cuda(), work_h.cuda()
    out = torch.zeros(T, n_heads * hd, device="cuda").bfloat16()
    if n_split == 1:
        lib.call("gllm_attn_mixed_paged_auto", qkv.data_ptr(), info_t.data_ptr(), work_t.data_ptr(), len(work), n_pf,
                 table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps,
                 out.data_ptr(), info_h.data_ptr(), work_h.data_ptr(), None, 0, lib.stream_handle())
    else:
        ws = torch.empty(lib.load().gllm_attn_split_workspace_bytes(n_pf, n_split, n_kv), dtype=torch.uint8,
                         device="cuda")
        lib.call("gllm_attn_mixed_paged_split", qkv.data_ptr(), info_t.data_ptr(), work_t.data_ptr(), len(work), n_pf,
                 table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd, ps, out.data_ptr(),
                 n_split, ws.data_ptr(), ws.numel(), lib.stream_handle())
    torch.cuda.synchronize()
    worst = 0.0
    for i, (s, n) in enumerate(seqs):
        o = info[i][3]
        ref = _attn_ref_gpu(qkv, n_heads, n_kv, hd, s, n, o, *dense[i])
        e = _rel(out[o:o + n], ref)
        worst = max(worst, e)
        assert e < 1e-2, (i, s, n, e)
    print(f"\nattention H={n_heads} KV={n_kv} {len(seqs)} seqs split={n_split}: worst rel err {worst:.3e}")
