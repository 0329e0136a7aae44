"""Host-side cost of one engine iteration (plan + KV + metadata pack + commit) with an instant fake device."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_14775_b200 import KvConfig, PipelineConfig, ThrottleConfig  # noqa: E402
from paper_2504_14775_b200.serving import ServingEngine  # noqa: E402
from paper_2504_14775_b200.stage import default_prompt_source, pack_batch  # noqa: E402
from paper_2504_14775_b200.workload import ArrivalProcess, builtin_length_table, synthesize_requests  # noqa: E402


class FakeExec:
    def __init__(self, reqs):
        self.src = default_prompt_source({r.id: r for r in reqs}, 128256)
        self.q = {}

    def launch(self, meta):
        self.q[meta.seq] = pack_batch(meta, 32, self.src)

    def retire(self, seq):
        return [0] * self.q.pop(seq).n_emit

    def stage0_idle(self):
        return True

    def wait(self, seq):
        pass

    def on_finish(self, rid, row):
        pass

    def mark_epoch(self):
        pass

    def synchronize(self):
        pass

    def stage_busy_intervals(self):
        return [[]]


reqs = synthesize_requests(ArrivalProcess.poisson(2000.0, 0), builtin_length_table("sharegpt-like"), 2000)
eng = ServingEngine(reqs, pipeline=PipelineConfig(depth=1), kv_config=KvConfig(64359, 16), throttle=ThrottleConfig(),
                    executor=FakeExec(reqs), time_scale=1000.0)
n = [0]


class Stop(Exception):
    pass


def hook(seq, t, n_out):
    n[0] += 1
    if n[0] == 300:
        raise Stop


PROF = "--profile" in sys.argv
t0 = time.perf_counter()
pr = cProfile.Profile()
if PROF:
    pr.enable()
try:
    eng.run(on_commit=hook)
except Stop:
    pass
pr.disable()
dt = time.perf_counter() - t0
print(f"{n[0]} iterations, {dt / n[0] * 1e3:.3f} ms/iter (profiler {'on' if PROF else 'off'}), decodes now {eng._rd}")
if PROF:
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
