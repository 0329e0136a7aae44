"""The reference's OWN test files run against this package (drop-in check).

`tokensim` is aliased to `paper_2504_14775_b200` by tests/refalias/tokensim_alias.py and
pytest runs `pkg/tests/test_{sched,kvcache,engine,metrics,workload}.py` unmodified (194
tests; `oracle_sim.compare_with_engine` inside test_engine.py drives our Engine).
`test_acceptance.py` / `test_cli.py` / `test_config.py` need `tokensim.cli` / `.config`,
the reference's CLI, which is out of scope. Skipped where the reference tree
is absent (the GPU box).
"""
import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
FILES = ("test_sched.py", "test_kvcache.py", "test_engine.py", "test_metrics.py", "test_workload.py")


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
def test_reference_suite_passes_against_package():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([os.path.join(HERE, "refalias"), REF_TESTS]))
    cmd = [sys.executable, "-m", "pytest", "-p", "tokensim_alias", "-p", "no:cacheprovider", "-q",
           "-m", "not slow", *[os.path.join(REF_TESTS, f) for f in FILES]]
    r = subprocess.run(cmd, cwd="/tmp", env=env, capture_output=True, text=True, timeout=900)
    tail = r.stdout[-2000:]
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert " passed" in tail and "failed" not in tail, tail
    n = int(tail.strip().splitlines()[-1].split(" passed")[0].split()[-1])
    assert n >= 194, tail
