"""Phase timeline of the prefill attention kernel from the clock64 stamps of the GLLM_TRACE build:

    python -m paper_2504_14775_b200.build --define GLLM_TRACE --out old_lib/libgllm_trace.so
    GLLM_LIB=old_lib/libgllm_trace.so python tools/attn_trace.py [--case 70b|8b]

Per key block of the first wave's CTAs (cycles, median over CTAs and interior blocks):
softmax of tile t from S ready to P published (and its load + max + rescale part), the wait of
tile t for its next S (= the tensor core's P.V_t + S_t latency plus queueing behind the other
tile), and the MMA warp's period per block.
"""
import argparse
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402

import bench_kernels as bk  # noqa: E402
from paper_2504_14775_b200 import native  # noqa: E402

CTAS, BLK, EV = 148, 64, 12
CASES = {"70b": ([(4096, 2048)], 64), "8b": ([(0, 2048)], 32), "qwen": ([(2000, 512)] * 4, 40),
         # decode role (one query token per sequence)
         "dec32x512": ([(512, 1)] * 32, 40), "dec48x512": ([(512, 1)] * 48, 40), "dec8x8000": ([(8000, 1)] * 8, 32),
         "dec800x500": ([(500, 1)] * 800, 32)}
DEC_CTAS, DEC_W, DEC_IT = 296, 8, 32


def decode_report(lib, name):
    buf = np.zeros((DEC_CTAS, DEC_W, DEC_IT, 3), dtype=np.uint32)
    fn = lib.gllm_debug_dec_trace_read
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    wait, comp, first, end = [], [], [], []
    for c in range(DEC_CTAS):
        for w in range(DEC_W):
            ev = buf[c, w]
            n = int(np.count_nonzero(ev[:, 2]))
            if n == 0:
                continue
            first.append(int(ev[0, 1]))
            end.append(int(ev[n - 1, 2]))
            for i in range(n):
                wait.append(int(ev[i, 1]) - int(ev[i, 0]))
                comp.append(int(ev[i, 2]) - int(ev[i, 1]))
    print(f"case {name}: warps traced {len(first)}")
    print(f"  first page ready {med(first):.0f} cyc after CTA start; warp done {med(end):.0f} cyc (max {max(end)})")
    print(f"  per page: wait for data {med(wait):.0f} cyc (p90 {np.percentile(wait, 90):.0f}), "
          f"compute {med(comp):.0f} cyc (p90 {np.percentile(comp, 90):.0f})")


def med(xs):
    return statistics.median(xs) if xs else float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="70b", choices=sorted(CASES))
    ap.add_argument("--dump", type=int, default=-1, help="print the raw stamps of this CTA")
    a = ap.parse_args()
    seqs, heads = CASES[a.case]
    bk.attn_case(a.case, seqs, n_heads=heads)
    lib = native.load()
    if a.case.startswith("dec"):
        decode_report(lib, a.case)
        return
    buf = np.zeros((CTAS, BLK, EV), dtype=np.uint32)
    fn = lib.gllm_debug_attn_trace_read
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    sm_d = {0: [], 1: []}
    sm_max = {0: [], 1: []}
    wait = {0: [], 1: []}
    mma_p = []
    overlap = []
    w_v, w_p0, w_p1, iss = [], [], [], []
    for c in range(CTAS):
        nb = int(np.count_nonzero(buf[c, :, 7]))
        if nb < 6:
            continue
        for l in range(1, nb - 2):
            for t in (0, 1):
                s0, s1, s2 = (int(x) for x in buf[c, l, 3 * t:3 * t + 3])
                nxt = int(buf[c, l + 1, 3 * t])
                if s0 and s2 and nxt:
                    sm_d[t].append(s2 - s0)
                    sm_max[t].append(s1 - s0)
                    wait[t].append(nxt - s2)
            mma_p.append(int(buf[c, l + 1, 7]) - int(buf[c, l, 7]))
            e = [int(x) for x in buf[c, l]]
            w_v.append(e[9] - e[8])       # MMA warp waiting for V_l (TMA)
            w_p0.append(e[10] - e[9])     # ... for tile 0's P (incl. its first-half P.V issue)
            w_p1.append(e[11] - e[10])    # ... for tile 1's P (incl. tile 0's P.V / S issue)
            # softmax of both tiles running at once: overlap of [s0, s2] intervals
            a0, a2 = int(buf[c, l, 0]), int(buf[c, l, 2])
            b0, b2 = int(buf[c, l, 3]), int(buf[c, l, 5])
            overlap.append(max(0, min(a2, b2) - max(a0, b0)))
    if a.dump >= 0:
        names = ["sm0_S", "sm0_max", "sm0_P", "sm1_S", "sm1_max", "sm1_P", "mma_S0iss", "mma_end", "mma_l", "mma_V",
                 "mma_P0", "mma_P1"]
        base = int(buf[a.dump, 0, 8])
        for l in range(min(12, BLK)):
            ev = sorted((int(buf[a.dump, l, e]) - base, names[e]) for e in range(EV) if buf[a.dump, l, e])
            print(f"blk {l:2d}: " + " ".join(f"{n}={t}" for t, n in ev))
    print(f"case {a.case}: CTAs traced {sum(1 for c in range(CTAS) if buf[c, 0, 7])}")
    for t in (0, 1):
        print(f"tile {t}: softmax {med(sm_d[t]):.0f} cyc (load+max+rescale {med(sm_max[t]):.0f}), "
              f"wait for next S {med(wait[t]):.0f} cyc")
    print(f"MMA warp period per block {med(mma_p):.0f} cyc; softmax overlap of the two tiles {med(overlap):.0f} cyc")
    print(f"MMA warp: wait V {med(w_v):.0f}, V->P0 full {med(w_p0):.0f}, P0->P1 full {med(w_p1):.0f} cyc")
    print("ideal tensor time per block (2 tiles x (S + P.V), 128x128x128 each at 8192 FLOP/clk): 2048 cyc")


if __name__ == "__main__":
    main()
