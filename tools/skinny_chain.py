"""In-stream cost of decode-sized GEMMs: a chain of back-to-back skinny GEMMs over distinct
weights (so nothing hits L2), launched as the stage launches them (PDL on), timed with CUDA
events around the whole chain. Sweeping K separates the fixed per-launch cost from streaming.

    python tools/skinny_chain.py [--m 4] [--n 5120] [--ks 1280,2560,5120,10240] [--chain 24]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_14775_b200 import native  # noqa: E402


def chain_ms(M, N, K, chain, reps=10, bn=0, splits=0):
    lib = native.load()
    A = torch.randn(M, K, device="cuda").bfloat16()
    Ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(chain)]
    C = torch.empty(M, N, device="cuda").bfloat16()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    st = native.stream_handle()

    def run():
        for W in Ws:
            native.call("gllm_gemm_bf16", A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, M, N, K, None, None, 0,
                        bn, splits, ws.data_ptr(), ws.numel(), st)

    native.call("gllm_gemm_workspace_reset", ws.data_ptr(), st)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / chain)
    ts.sort()
    del lib
    return ts[len(ts) // 2]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=5120)
    ap.add_argument("--ks", default="1280,2560,5120,10240")
    ap.add_argument("--chain", type=int, default=24)
    ap.add_argument("--bn", type=int, default=0, help="force the 128-row tile width (0 = auto)")
    ap.add_argument("--splits", type=int, default=0, help="force split-K (0 = auto, 1 = whole K)")
    a = ap.parse_args()
    hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6554.2
    for K in (int(k) for k in a.ks.split(",")):
        ms = chain_ms(a.m, a.n, K, a.chain, bn=a.bn, splits=a.splits)
        by = 2 * a.n * K
        print(json.dumps({"M": a.m, "N": a.n, "K": K, "bn": a.bn, "splits": a.splits, "us_per_gemm": round(ms * 1e3, 2),
                          "floor_us": round(by / hbm / 1e3, 2), "GB/s": round(by / ms / 1e6, 1)}))
