"""Golden fixture for trace replay with resampled arrivals, from the REFERENCE.

Run in the build container only (the reference tree is not on the GPU box):

    python tests/golden/make_trace_golden.py

A reference-synthesised trace is saved with the reference `save_trace`, then
materialised by the reference `cli.build_workload` with `source = "trace"` and
`resample_rate_per_s` set (`cli.py:71-79`). The fixture keeps the trace bytes
and the resulting (id, arrival_ms, input, output) rows.
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
from types import SimpleNamespace

sys.path.insert(0, "/root/reference/pkg/src")

import tokensim as ts  # noqa: E402
from tokensim import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    cases = []
    for seed, rate, resample, n in ((0, 16.0, 4.0, 50), (7, 2.0, 64.0, 120), (3, 1000.0, 0.5, 30)):
        specs = ts.synthesize_requests(ts.ArrivalProcess.poisson(rate, seed),
                                       ts.builtin_length_table("azure-like"), n)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "t.jsonl")
            ts.save_trace(specs, path)
            text = open(path, encoding="utf-8").read()
            cfg = SimpleNamespace(source="trace", trace_path=path, resample_rate_per_s=resample, seed=seed + 11)
            out = cli.build_workload(cfg)
        cases.append({"trace": text, "resample_rate_per_s": resample, "seed": seed + 11,
                      "rows": [[s.id, s.arrival_ms, s.input_tokens, s.output_tokens] for s in out]})
    with gzip.open(os.path.join(HERE, "trace_resample.json.gz"), "wt", encoding="utf-8") as fh:
        json.dump(cases, fh)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
