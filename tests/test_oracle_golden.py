"""Pin the CPU oracle (oracle/sched_ref.py) against the reference's own golden outputs."""
import pytest

from golden_io import load
from oracle import sched_ref as R


def test_oracle_formulas():
    g = load("formulas.json.gz")
    for wp, T, min_p, max_p, free, total, th, rd, depth, mode, wt, ut, comb, dec, lim in g["rows"]:
        kv_free = free / total
        assert R.prefill_wt(wp, T, min_p, max_p) == wt
        assert R.prefill_ut(kv_free, min_p, max_p) == ut
        assert R.prefill_combined(wp, kv_free, T, min_p, max_p, th) == comb
        assert R.decode_count(rd, depth) == dec
        assert R.prefill_limit(wp, kv_free, (T, max_p, min_p, th, mode)) == lim


def test_oracle_plans():
    for c in load("plans.json.gz"):
        wp, rd, free, total, depth = c["inputs"]
        T, max_p, min_p, th, mode = c["cfg"]
        for sched, key in (("throttle", "throttled"), ("sarathi", "sarathi")):
            dec, chunks, ctx = R.plan(sched, wp, rd, free, total, c["ps"], depth, [tuple(x) for x in c["pq"]],
                                      [tuple(x) for x in c["dq"]], (T, max_p, min_p, th, mode), c["budget"])
            assert [dec, [list(x) for x in chunks], ctx] == c[key]


ENGINE = load("engine_runs.json.gz")
TRACES = load("traces.json.gz")
TRACES.update(ENGINE["traces"])


@pytest.mark.parametrize("case", [r for r in ENGINE["runs"] if r["horizon"] is None], ids=lambda r: r["name"])
def test_oracle_engine_runs(case):
    rows = TRACES[case["trace"]]
    reqs = [(i, a, b, c) for i, (a, b, c) in enumerate(rows)]
    comm = (0.1, 16384.0, 20.79e6)
    eng = R.RefEngine(reqs, case["scheduler"], case["depth"], case["pages"], case["ps"],
                      (case["T"], 2048, 32, case["thresh"], "combined"), case["budget"], tuple(case["cost"]), comm).run()
    assert [list(x) for x in eng.iters] == case["iterations"]
    got = [[rid, r["arr"], r["first"], r["fin"], r["pre"]] for rid, r in sorted(eng.reqs.items())]
    assert got == case["requests"]
    assert (eng.committed, eng.discarded, eng.preemptions) == (case["committed"], case["discarded"], case["preemptions"])
