"""Every projection GEMM the five configs issue (C1 tiny excluded), ours vs cuBLAS (torch.matmul), over
the serving M range: decode batches, medium mixed batches and full 2k-token micro-batches.

    python tools/gemm_sweep.py [--m 4,16,64,128,256,512,1024,2009] [--out gpurun_out/gemm_sweep.csv]

Gate-up runs through the fused SwiGLU entry point (its output is N/2 wide); cuBLAS does the plain
[M, K] x [K, N] product. Weights are N(0, 0.02^2) like the stages' init, activations N(0, 1). L2 is
flushed between reps (tools/bench_kernels.timeit).
"""
import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402

import bench_kernels as bk  # noqa: E402
from paper_2504_14775_b200 import native  # noqa: E402
from paper_2504_14775_b200.modelspec import MODELS  # noqa: E402

CONFIGS = [("C2", "llama3-8b"), ("C3", "qwen2.5-14b"), ("C4", "qwen2.5-32b"), ("C5", "llama3.1-70b")]


def shapes(spec):
    hd = spec.head_dim
    qkv = (spec.n_heads + 2 * spec.n_kv_heads) * hd
    return [("qkv", qkv, spec.d_model, False), ("o", spec.d_model, spec.n_heads * hd, False),
            ("gate_up", 2 * spec.d_ff, spec.d_model, True), ("down", spec.d_model, spec.d_ff, False),
            ("lm_head", spec.vocab, spec.d_model, False)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="4,16,64,128,256,512,1024,2009")
    ap.add_argument("--out", default="gpurun_out/gemm_sweep.csv")
    a = ap.parse_args()
    ms_list = [int(x) for x in a.m.split(",")]
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = native.stream_handle()
    rows = []
    for cfg, model in CONFIGS:
        spec = MODELS[model]
        for name, N, K, swiglu in shapes(spec):
            B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
            for M in ms_list:
                if name == "lm_head" and M > 1024:
                    continue
                A = torch.randn(M, K, device="cuda").bfloat16()
                if swiglu:
                    C = torch.empty(M, N // 2, device="cuda").bfloat16()
                    fn = lambda: native.call("gllm_gemm_swiglu_bf16", A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(),
                                             N // 2, M, N // 2, K, 0, 0, ws.data_ptr(), ws.numel(), st)
                else:
                    C = torch.empty(M, N, device="cuda").bfloat16()
                    fn = lambda: native.call("gllm_gemm_bf16", A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N,
                                             K, None, None, 0, 0, 0, ws.data_ptr(), ws.numel(), st)
                ours = bk.timeit(fn)
                ref = bk.timeit(lambda: torch.matmul(A, B.T))
                fl = 2 * M * N * K
                row = {"config": cfg, "model": model, "gemm": name, "M": M, "N": N, "K": K,
                       "ours_us": round(ours * 1e3, 2), "cublas_us": round(ref * 1e3, 2),
                       "ours_TFLOPs": round(fl / ours / 1e9, 1), "cublas_TFLOPs": round(fl / ref / 1e9, 1),
                       "ours_GBs": round(2 * N * K / ours / 1e6, 1), "speedup_vs_cublas": round(ref / ours, 3)}
                rows.append(row)
                print(",".join(str(v) for v in row.values()), flush=True)
                del A, C
            del B
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    worse = [r for r in rows if r["speedup_vs_cublas"] < 0.95]
    print(f"{len(rows)} shapes; ours >= 0.95x cuBLAS on {len(rows) - len(worse)}; slower: "
          + "; ".join(f"{r['config']} {r['gemm']} M={r['M']} {r['speedup_vs_cublas']}x" for r in worse))


if __name__ == "__main__":
    main()
