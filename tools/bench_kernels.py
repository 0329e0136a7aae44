"""Kernel microbenchmarks at the bench's shapes (CUDA events, warm, L2 flushed between reps).

    python tools/bench_kernels.py [--only attn|gemm]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_14775_b200 import native  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists("MEASURED_PEAKS.json") else {"hbm_gbs": 6554.2, "bf16_tflops": 1644.5}
FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def attn_case(name, seqs, n_heads=32, n_kv=8, ps=16, force_mixed=False, split=1, auto=False):
    hd = 128
    ctx = [s + n for s, n in seqs]
    pages_per = [-(-c // ps) for c in ctx]
    num_pages = sum(pages_per) + 8
    mpr = max(pages_per) + 1
    perm = torch.randperm(num_pages)
    table = torch.zeros(len(seqs), mpr, dtype=torch.int32)
    k = 0
    for i, p in enumerate(pages_per):
        table[i, :p] = perm[k:k + p]
        k += p
    table = table.cuda()
    kc = torch.randn(num_pages, n_kv, ps, hd, device="cuda").bfloat16()
    vc = torch.randn_like(kc)
    T = sum(n for _, n in seqs)
    qkv = torch.randn(T, (n_heads + 2 * n_kv) * hd, device="cuda").bfloat16()
    out = torch.empty(T, n_heads * hd, device="cuda").bfloat16()
    qt = native.load().gllm_attention_q_tile(n_heads, n_kv)
    info, work, off = [], [], 0
    for i, (s, n) in enumerate(seqs):
        info.append([i, s, n, off, -1])
        work += [[i, q0] for q0 in range(0, n, qt)] if n > 1 else []
        off += n
    work = work + [[i, 0] for i, (s, n) in enumerate(seqs) if n == 1]   # prefill tiles first (as the packer)
    info_h = torch.tensor(info, dtype=torch.int32)
    work_h = torch.tensor(work, dtype=torch.int32)
    info, work_t = info_h.cuda(), work_h.cuda()
    st = native.stream_handle()
    n_pf = max(int(force_mixed), sum(1 for i, _ in work if seqs[i][1] > 1))
    if auto:   # splits chosen from the host metadata, as the stage forward does
        fn = lambda: native.call("gllm_attn_mixed_paged_auto", qkv.data_ptr(), info.data_ptr(), work_t.data_ptr(),
                                 len(work), n_pf, table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(),
                                 n_heads, n_kv, hd, ps, out.data_ptr(), info_h.data_ptr(), work_h.data_ptr(), None, 0,
                                 st)
    elif split > 1:
        ws = torch.empty(native.load().gllm_attn_split_workspace_bytes(n_pf, split, n_kv), dtype=torch.uint8, device="cuda")
        fn = lambda: native.call("gllm_attn_mixed_paged_split", qkv.data_ptr(), info.data_ptr(), work_t.data_ptr(), len(work),
                                 n_pf, table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd,
                                 ps, out.data_ptr(), split, ws.data_ptr(), ws.numel(), st)
    else:
        fn = lambda: native.call("gllm_attn_mixed_paged", qkv.data_ptr(), info.data_ptr(), work_t.data_ptr(), len(work),
                                 n_pf, table.data_ptr(), mpr, kc.shape[0], kc.data_ptr(), vc.data_ptr(), n_heads, n_kv, hd,
                                 ps, out.data_ptr(), st)
    ms = timeit(fn)
    kv_bytes = sum(ctx) * n_kv * hd * 2 * 2 + T * n_heads * hd * 2 * 2
    flops = sum(4 * n_heads * hd * (n * s + n * (n + 1) / 2) for s, n in seqs)
    print(json.dumps({"kernel": "attention", "case": name, "ms": round(ms, 4), "GB/s": round(kv_bytes / ms / 1e6, 1),
                      "hbm_frac": round(kv_bytes / ms / 1e6 / PEAK["hbm_gbs"], 3), "TFLOP/s": round(flops / ms / 1e9, 1)}))


def gemm_case(M, N, K, bn=0, splits=0, swiglu=False, wscale=1.0):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * wscale).bfloat16()
    C = torch.empty(M, N, device="cuda").bfloat16()
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    st = native.stream_handle()
    if swiglu:
        fn = lambda: native.call("gllm_gemm_swiglu_bf16", A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N // 2, M,
                                 N // 2, K, bn, splits, ws.data_ptr(), ws.numel(), st)
    else:
        fn = lambda: native.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None,
                                 None, 0, bn, splits, ws.data_ptr(), ws.numel(), st)
    ms = timeit(fn)
    fl = 2 * M * N * K
    by = 2 * (M * K + N * K + M * N)
    ref = timeit(lambda: torch.matmul(A, B.T))
    print(json.dumps({"kernel": "gemm", "M": M, "N": N, "K": K, "bn": bn, "splits": splits, "ms": round(ms, 4),
                      "TFLOP/s": round(fl / ms / 1e9, 1), "GB/s": round(by / ms / 1e6, 1),
                      "cublas_ms": round(ref, 4), "cublas_TFLOP/s": round(fl / ref / 1e9, 1)}))


def qkv_rope_case(M, model="llama3-8b", ps=16):
    """Fused QKV GEMM + RoPE + paged KV write (the stage's QKV launch) vs the plain GEMM of the same shape."""
    from paper_2504_14775_b200.modelspec import MODELS, rope_table
    spec = MODELS[model]
    H, KV, d = spec.n_heads, spec.n_kv_heads, spec.d_model
    Q = spec.qkv_width
    A = torch.randn(M, d, device="cuda").bfloat16()
    W = (torch.randn(Q, d, device="cuda") * 0.02).bfloat16()
    bias = torch.randn(Q, device="cuda").bfloat16() if spec.qkv_bias else None
    rope = torch.from_numpy(rope_table(spec, 8192)).cuda()
    pos = torch.randint(0, 8000, (M,), dtype=torch.int32, device="cuda")
    n_pages = (M + ps - 1) // ps + 64
    slot = torch.randperm(n_pages * ps, device="cuda")[:M].to(torch.int32)
    kc = torch.zeros(n_pages, KV, ps, 128, device="cuda").bfloat16()
    vc = torch.zeros_like(kc)
    out = torch.empty(M, Q, device="cuda").bfloat16()
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    st = native.stream_handle()
    fused = lambda: native.call("gllm_gemm_qkv_rope_bf16", A.data_ptr(), d, W.data_ptr(), d,
                                None if bias is None else bias.data_ptr(), out.data_ptr(), M, d, H, KV, pos.data_ptr(),
                                slot.data_ptr(), rope.data_ptr(), kc.data_ptr(), vc.data_ptr(), ps, 0, 0,
                                ws.data_ptr(), ws.numel(), st)
    plain = lambda: native.call("gllm_gemm_bf16", A.data_ptr(), d, W.data_ptr(), d, out.data_ptr(), Q, M, Q, d,
                                None, None, 0, 0, 0, ws.data_ptr(), ws.numel(), st)
    tf, tp = timeit(fused), timeit(plain)
    fl = 2 * M * Q * d
    print(json.dumps({"kernel": "qkv_rope", "model": model, "M": M, "fused_ms": round(tf, 4), "plain_ms": round(tp, 4),
                      "fused_TFLOP/s": round(fl / tf / 1e9, 1), "plain_TFLOP/s": round(fl / tp / 1e9, 1)}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--case", default="")
    ap.add_argument("--wscale", type=float, default=1.0, help="weight std (0.02 = the stages' init)")
    ap.add_argument("--gemm", default="", help="M,N,K[,bn,splits] single GEMM case (bn/splits 0 = auto)")
    ap.add_argument("--swiglu", action="store_true")
    ap.add_argument("--qkv-rope", default="", help="M[,model]: fused QKV + RoPE + KV write vs plain GEMM")
    a = ap.parse_args()
    if a.qkv_rope:
        v = a.qkv_rope.split(",")
        qkv_rope_case(int(v[0]), *(v[1:2] or ["llama3-8b"]))
        raise SystemExit(0)
    if a.gemm:
        v = [int(x) for x in a.gemm.split(",")] + [0, 0]
        gemm_case(v[0], v[1], v[2], bn=v[3], splits=v[4], swiglu=a.swiglu, wscale=a.wscale)
        raise SystemExit(0)
    if a.case:
        _orig = attn_case
        attn_case = lambda name, *x, **k: _orig(name, *x, **k) if name == a.case else None
    torch.manual_seed(0)
    if a.only in ("", "attn"):
        attn_case("decode800_ctx500", [(500, 1)] * 800)
        attn_case("decode64_ctx2000", [(2000, 1)] * 64)
        attn_case("decode8_ctx8000", [(8000, 1)] * 8)
        attn_case("decode800_ctx500_mixedkernel", [(500, 1)] * 800, force_mixed=True)
        attn_case("bench_like_mix", [(500, 1)] * 800 + [(0, 300)] * 4 + [(150, 300)] * 1 + [(0, 50)] * 2)
        attn_case("prefill_4x300_from0", [(0, 300)] * 4)
        attn_case("prefill_chunk512_after1500", [(1500, 512)])
        attn_case("mixed_bench", [(500, 1)] * 800 + [(0, 300)] * 3 + [(200, 300)] * 1)
        attn_case("prefill_2048_from0_8b", [(0, 2048)])
        attn_case("prefill_2048_after4096_70b", [(4096, 2048)], n_heads=64)
        attn_case("prefill_640_after6000_70b", [(6000, 640)], n_heads=64)
        attn_case("prefill_640_after6000_70b_split2", [(6000, 640)], n_heads=64, split=2)
        attn_case("prefill_640_after6000_70b_split4", [(6000, 640)], n_heads=64, split=4)
        attn_case("prefill_2x256_after7000_70b_split8", [(7000, 256)] * 2, n_heads=64, split=8)
        attn_case("prefill_2x256_after7000_70b", [(7000, 256)] * 2, n_heads=64)
        attn_case("prefill_4x512_after2000_qwen", [(2000, 512)] * 4, n_heads=40)
        attn_case("decode256_qwen", [(600, 1)] * 256, n_heads=40)
        attn_case("decode128_70b", [(4000, 1)] * 128, n_heads=64)
        for auto in (False, True):
            sfx = "_auto" if auto else ""
            attn_case("decode4_ctx512_qwen" + sfx, [(512, 1)] * 4, n_heads=40, auto=auto)
            attn_case("decode1_ctx2048_8b" + sfx, [(2048, 1)], auto=auto)
            attn_case("decode2_ctx3000_70b" + sfx, [(3000, 1)] * 2, n_heads=64, auto=auto)
            attn_case("decode8_ctx8000" + sfx, [(8000, 1)] * 8, auto=auto)
            attn_case("decode16_ctx1000" + sfx, [(1000, 1)] * 16, auto=auto)
        for b in (24, 32, 48, 64):
            for c in (512, 2000):
                attn_case(f"decode{b}_ctx{c}_qwen", [(c, 1)] * b, n_heads=40)
    if a.only in ("", "gemm"):
        for M in (1, 16, 64, 128, 256, 512, 1024, 2048, 2944):
            for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
                gemm_case(M, N, K)
        gemm_case(1000, 128256, 4096)
