"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel (shares, not absolutes)."""
import csv
import re
import sys
from collections import defaultdict


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()
        name = re.sub(r"<.*", lambda m: "<" + m.group(0)[1:].split(">")[0] + ">", name)
        val = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "nsecond"
        us = val / 1000.0 if unit.startswith("n") else val if unit.startswith("u") else val * 1000.0
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:60]:60s} {n:8d} {us:12.1f} {us / total:7.1%}")
    lines.append(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {total:12.1f}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
