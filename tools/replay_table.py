"""Markdown table of tools/pp_replay.py rows (one JSON object per line).

    python tools/replay_table.py profiles/r2/pp_replay_c4.jsonl [more.jsonl ...]
"""
import json
import sys


def main(paths):
    rows = []
    for p in paths:
        with open(p) as fh:
            rows += [json.loads(ln) for ln in fh if ln.strip()]
    print("| model | PP | scheduler | rate/s | requests | finished | output tok/s | p50 TTFT ms | p50 TPOT ms "
          "| mean TPOT ms | bubble mean | token stddev | preemptions | trace hash |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['model']} | {r['pp']} | {r['scheduler']} | {r['rate_per_s']:g} | {r['n_requests']} | "
              f"{r['finished']} | {r['output_tok_s']:.0f} | {r['p50_ttft_ms']:.0f} | {r['p50_tpot_ms']:.1f} | "
              f"{r['mean_tpot_ms']:.1f} | {r['bubble_mean']:.3f} | {r['token_stddev']:.0f} | {r['preemptions']} | "
              f"{r['trace_hash']} |")


if __name__ == "__main__":
    main(sys.argv[1:])
