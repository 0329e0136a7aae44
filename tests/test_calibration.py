"""Cost-model calibration: recovers known coefficients; fitted model drives the engine."""
import numpy as np
import pytest

from paper_2504_14775_b200 import Engine, KvConfig, PipelineConfig, ThrottleConfig
from paper_2504_14775_b200.calibration import fit_stage_cost
from paper_2504_14775_b200.engine import stage_time
from paper_2504_14775_b200.sched import MicroBatchPlan
from paper_2504_14775_b200.workload import ArrivalProcess, builtin_length_table, synthesize_requests


def test_recovers_linear_model():
    rng = np.random.Generator(np.random.PCG64(3))
    tok = rng.integers(1, 3000, 200)
    ctx = rng.integers(0, 400_000, 200)
    y = 1.7 + 0.012 * tok + 0.08 * ctx / 1024 + rng.normal(0, 0.01, 200)
    m, diag = fit_stage_cost(tok, ctx, y)
    assert m.c0 == pytest.approx(1.7, abs=0.02)
    assert m.c_tok == pytest.approx(0.012, rel=0.01)
    assert m.c_ctx == pytest.approx(0.08, rel=0.02)
    assert diag["r2"] > 0.999


def test_nonnegative_and_usable_by_engine():
    tok = np.array([10, 20, 30, 40])
    ctx = np.array([0, 0, 0, 0])
    y = np.array([5.0, 4.0, 3.0, 2.0])        # decreasing: unconstrained slope would be negative
    m, _ = fit_stage_cost(tok, ctx, y)
    assert m.c_tok >= 0 and m.c0 > 0 and m.c_ctx >= 0
    plan = MicroBatchPlan([1, 2], [(3, 10)], 100)
    assert stage_time(plan, m) == pytest.approx(m.c0 + m.c_tok * 12 + m.c_ctx * 100 / 1024)
    reqs = synthesize_requests(ArrivalProcess.poisson(20.0, 1), builtin_length_table("sharegpt-like"), 30)
    raw = Engine(reqs, pipeline=PipelineConfig(depth=2, cost=m), kv_config=KvConfig(4096, 16),
                 throttle=ThrottleConfig()).run()
    assert all(r.completion_ms is not None for r in raw.requests)
