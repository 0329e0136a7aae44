"""pytest plugin: make `import tokensim[.x]` resolve to this package (drop-in check).

Loaded with `-p tokensim_alias` when running the REFERENCE's own test files
(`/root/reference/pkg/tests/test_{sched,kvcache,engine,metrics,workload}.py`)
against `paper_2504_14775_b200`; see tests/test_reference_suite.py.
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_pkg = importlib.import_module("paper_2504_14775_b200")
sys.modules["tokensim"] = _pkg
for _name in ("engine", "sched", "kvcache", "workload", "errors", "metrics"):
    sys.modules[f"tokensim.{_name}"] = importlib.import_module(f"paper_2504_14775_b200.{_name}")
