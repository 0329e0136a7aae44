"""Token Throttling equations and planners vs the reference's golden outputs (bit-exact)."""
import pytest

from golden_io import load
from paper_2504_14775_b200 import sched as S
from paper_2504_14775_b200.errors import ConfigError


def test_reference_hand_examples():
    # `pkg/tests/test_acceptance.py:88-99`
    base = S.ThrottleConfig()
    assert S.throttle_prefill_wt(16384, base) == 2048
    assert S.throttle_prefill_wt(0, base) == 0
    assert S.throttle_prefill_wt(100, base) == 32
    assert S.throttle_prefill_ut(1.0, base) == 2048
    assert S.throttle_prefill_ut(0.0, base) == 32
    assert S.throttle_prefill_ut(0.5, base) == 1024
    assert S.throttle_prefill_combined(100000, 0.525, base) == 1024
    assert S.throttle_prefill_combined(16384, 0.05, base) == 0
    assert S.throttle_prefill_combined(16384, 1.0, base) == 2048
    assert S.throttle_decode(12, 4) == 3
    assert S.throttle_decode(0, 4) == 0
    assert S.throttle_decode(10, 4) == 3


def test_formulas_golden():
    g = load("formulas.json.gz")
    n = 0
    for wp, T, min_p, max_p, free, total, th, rd, depth, mode, wt, ut, comb, dec, lim in g["rows"]:
        cfg = S.ThrottleConfig(T=T, max_p=max_p, min_p=min_p, kv_thresh=th, mode=mode)
        kv_free = free / total
        assert S.throttle_prefill_wt(wp, cfg) == wt
        assert S.throttle_prefill_ut(kv_free, cfg) == ut
        assert S.throttle_prefill_combined(wp, kv_free, cfg) == comb
        assert S.throttle_decode(rd, depth) == dec
        assert S.prefill_token_limit(wp, kv_free, cfg) == lim
        n += 1
    assert n > 10_000


def test_plans_golden():
    for case in load("plans.json.gz"):
        wp, rd, free, total, depth = case["inputs"]
        T, max_p, min_p, th, mode = case["cfg"]
        cfg = S.ThrottleConfig(T=T, max_p=max_p, min_p=min_p, kv_thresh=th, mode=mode)
        inputs = S.SchedInputs(wp, rd, free / total, depth)
        view = S.KvView(free, total, case["ps"])
        pq = [S.PrefillCandidate(*c) for c in case["pq"]]
        dq = [S.DecodeCandidate(*c) for c in case["dq"]]
        pt = S.plan_throttled(inputs, pq, dq, view, cfg)
        ps = S.plan_sarathi(inputs, pq, dq, view, case["budget"])
        for plan, (dec, chunks, ctx) in ((pt, case["throttled"]), (ps, case["sarathi"])):
            assert plan.decode_ids == dec
            assert [list(c) for c in plan.prefill_chunks] == chunks
            assert plan.decode_context_tokens == ctx


@pytest.mark.parametrize("kw", [dict(T=0), dict(min_p=0), dict(min_p=10, max_p=5), dict(kv_thresh=1.0),
                                dict(kv_thresh=-0.1), dict(mode="bogus")])
def test_config_validation(kw):
    with pytest.raises(ConfigError):
        S.ThrottleConfig(**kw)


def test_inputs_validation():
    with pytest.raises(ConfigError):
        S.SchedInputs(-1, 0, 0.5, 1)
    with pytest.raises(ConfigError):
        S.SchedInputs(0, 0, 1.5, 1)
    with pytest.raises(ConfigError):
        S.SchedInputs(0, 0, 0.5, 0)
    with pytest.raises(ConfigError):
        S.throttle_decode(-1, 2)
    with pytest.raises(ConfigError):
        S.plan_sarathi(S.SchedInputs(0, 0, 1.0, 1), [], [], S.KvView(1, 1, 16), 0)


def test_plan_is_pure_and_page_truncated():
    # `pkg/tests/test_sched.py` style: slack of a partly used page is free.
    pq = [S.PrefillCandidate(1, 100, 10), S.PrefillCandidate(2, 50, 0)]
    plan = S.plan_throttled(S.SchedInputs(150, 0, 0.5, 1), pq, [], S.KvView(1, 10, 16), S.ThrottleConfig(T=1, min_p=1))
    assert plan.prefill_chunks == [(1, 22)]   # 6 slack + 16 from the one free page, then stop
    assert pq[0].remaining_tokens == 100
