"""Phase timeline of a chain of skinny (decode) GEMMs, from the %globaltimer stamps of the
GLLM_TRACE debug build:

    python -m paper_2504_14775_b200.build --define GLLM_TRACE --out old_lib/libgllm_trace.so
    GLLM_LIB=old_lib/libgllm_trace.so python tools/skinny_trace.py [--m 4 --n 5120 --k 5120]

Per launch (µs, relative to the previous launch's last CTA exit): CTA start, setup done,
PDL wait released (producer), first MMA, first non-prefetched stage, last accumulator ready,
epilogue done, exit — min / median / max over the CTAs.
"""
import argparse
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_14775_b200 import native  # noqa: E402

L, CTAS, EV = 64, 160, 12
NAMES = ["start", "setup", "pdl_rel", "mma0", "stage8", "acc_last", "epi_done", "exit", "tmem_ld", "fenced", "counted", "summed"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=5120)
    ap.add_argument("--k", type=int, default=5120)
    ap.add_argument("--chain", type=int, default=12)
    ap.add_argument("--detail", type=int, default=0, help="print the N slowest CTAs of the last launch")
    a = ap.parse_args()
    lib = native.load()
    M, N, K = a.m, a.n, a.k
    A = torch.randn(M, K, device="cuda").bfloat16()
    Ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(a.chain)]
    C = torch.empty(M, N, device="cuda").bfloat16()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    st = native.stream_handle()
    native.call("gllm_gemm_workspace_reset", ws.data_ptr(), st)
    for _ in range(2):
        for W in Ws:
            native.call("gllm_gemm_bf16", A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, M, N, K, None, None, 0,
                        0, 0, ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    buf = np.zeros((L, CTAS, EV), dtype=np.uint64)
    fn = lib.gllm_debug_trace_read
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    work = (N // 128) * (K // 64)
    per = max(-(-work // 148), min(4, K // 64))
    grid = -(-work // per)
    print(f"M={M} N={N} K={K} grid={grid} per={per} K-blocks/CTA; floor {2 * N * K / 6554e3:.2f} us")
    tags = list(range(a.chain + 1, 2 * a.chain))
    print("launch " + " ".join(f"{n:>20s}" for n in NAMES[:8]))
    for tg in tags:
        prev_exit = int(buf[(tg - 1) % L, :grid, 7].max())
        cur = buf[tg % L, :grid, :].astype(np.int64) - prev_exit
        cols = []
        for e in range(8):
            v = cur[:, e]
            v = v[buf[tg % L, :grid, e] > 0]
            cols.append(f"{v.min() / 1e3:6.2f}/{np.median(v) / 1e3:6.2f}/{v.max() / 1e3:6.2f}" if len(v) else "-")
        print(f"{tg:6d} " + " ".join(f"{c:>20s}" for c in cols))
    gaps = [(int(buf[tg % L, :grid, 7].max()) - int(buf[(tg - 1) % L, :grid, 7].max())) / 1e3 for tg in tags]
    print(f"exit-to-exit per launch: median {statistics.median(gaps):.2f} us")
    if a.detail:
        tg = tags[-1]
        prev_exit = int(buf[(tg - 1) % L, :grid, 7].max())
        cur = buf[tg % L, :grid, :].astype(np.int64) - prev_exit
        kbs = K // 64
        for b in np.argsort(-cur[:, 7])[:a.detail]:
            g0, g1 = b * per, min(b * per + per, work)
            segs = [(t, max(g0, t * kbs) - t * kbs, min(g1, t * kbs + kbs) - t * kbs) for t in range(g0 // kbs, (g1 - 1) // kbs + 1)]
            print(f"cta {b:4d} segs(tile,kb0,kb1)={segs} " + " ".join(f"{n}={cur[b, e] / 1e3:.2f}" for e, n in enumerate(NAMES) if buf[tg % L, b, e] > 0))


if __name__ == "__main__":
    main()
