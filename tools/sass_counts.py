"""Per-kernel SASS instruction counts of the built libgllm.so (evidence that the hot kernels run on
tcgen05 / TMEM / TMA, not mma.sync or plain loads).

    python tools/sass_counts.py > profiles/r2/sass_counts.txt

Columns: UTCHMMA / UTCHMMA.2CTA = tcgen05.mma (cta_group::1 / ::2); UTMALDG = TMA tensor loads;
UBLKCP = cp.async.bulk; LDTM / STTM = tcgen05.ld / st (TMEM <-> registers); HMMA = mma.sync
(legacy tensor core path, used by the decode attention); FFMA2 / FADD2 / FMUL2 = packed fp32;
MUFU.EX2 = exp2; SYNCS = mbarrier ops.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_14775_b200", "libgllm.so")

COLS = [("UTCHMMA", r"UTCHMMA(?!\.2CTA)"), ("UTCHMMA.2CTA", r"UTCHMMA\.2CTA"),
        ("UTMALDG", r"UTMALDG"), ("UBLKCP", r"UBLKCP"), ("LDTM", r"\bLDTM"), ("STTM", r"\bSTTM"),
        ("HMMA", r"\bHMMA"), ("FFMA2", r"\bFFMA2"), ("FADD2", r"\bFADD2"), ("FMUL2", r"\bFMUL2"),
        ("MUFU.EX2", r"MUFU\.EX2"), ("SYNCS", r"\bSYNCS"), ("LDG", r"\bLDG"), ("STG", r"\bSTG")]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
        return out.stdout.splitlines()
    except Exception:
        return list(names)


def main() -> int:
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs: list[tuple[str, Counter, int]] = []
    cur, cnt, n = None, Counter(), 0
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                funcs.append((cur, cnt, n))
            cur, cnt, n = m.group(1), Counter(), 0
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
            n += 1
            for col, pat in COLS:
                if re.search(pat, line):
                    cnt[col] += 1
    if cur:
        funcs.append((cur, cnt, n))
    names = demangle([f[0] for f in funcs])
    print("# cuobjdump -sass paper_2504_14775_b200/libgllm.so (sm_100a): instruction counts per kernel")
    print("# columns: see the docstring of tools/sass_counts.py")
    hdr = ["kernel", "instrs"] + [c for c, _ in COLS]
    print("\t".join(hdr))
    for (raw, c, n), name in zip(funcs, names):
        short = re.sub(r"\(anonymous namespace\)::", "", name)
        short = re.sub(r"\(.*", "", short).replace("gllm::", "")
        print("\t".join([short, str(n)] + [str(c[col]) for col, _ in COLS]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
