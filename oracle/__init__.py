"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline. The product path (paper_2504_14775_b200) never imports it.

* sched_ref.py  — plain restatement of the reference scheduler, KV accounting
                  and event loop (pkg/src/tokensim/{sched,kvcache,engine}.py),
                  pinned against tests/golden/ (generated from the reference).
* model_ref.py  — fp32 CPU Llama/Qwen2 decoder with full (unpaged) causal
                  attention recomputed over the whole prefix; the logits
                  oracle. The reference has no model, so logits parity is
                  pinned only by this oracle ("parity unpinned by the
                  reference").
"""
