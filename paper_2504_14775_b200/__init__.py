"""B200-native per-iteration path of gLLM (arXiv 2504.14775): Token Throttling + paged GPU stages.

The public names mirror the reference simulator's API
(`pkg/src/tokensim/__init__.py:3-109`), so code written against `tokensim`
switches by changing the import. GPU-side pieces (stage workers, kernels,
pipeline runtime) live in `stage`, `native` and `serving` and load the CUDA
extension lazily; nothing here falls back to a CPU implementation.
"""

from .engine import (
    CommModel,
    Engine,
    PipelineConfig,
    RawRunData,
    StageCostModel,
    bubble_accounting,
    run,
    stage_time,
    transfer_time,
)
from .errors import ConfigError, NativeError, SimError, TraceError, UnschedulableError
from .kvcache import KvCacheState, KvConfig, PagedKvCache, pages_needed, select_preemption_victim
from .metrics import (
    IterationRecord,
    Report,
    RequestRecord,
    build_report,
    e2el,
    ideal_balance_reference,
    output_throughput,
    slo_attainment,
    throughput,
    token_fluctuation,
    tpot,
    tpot_p50,
    ttft,
    ttft_p50,
    write_report,
)
from .sched import (
    DecodeCandidate,
    KvView,
    MicroBatchPlan,
    PrefillCandidate,
    SchedInputs,
    ThrottleConfig,
    plan_sarathi,
    plan_throttled,
    throttle_decode,
    throttle_prefill_combined,
    throttle_prefill_ut,
    throttle_prefill_wt,
)
from .workload import (
    ArrivalProcess,
    LengthDistribution,
    RequestSpec,
    builtin_length_table,
    generate_arrivals,
    load_azure_trace,
    load_trace,
    prompt_token_ids,
    resample_arrivals,
    sample_lengths,
    save_trace,
    synthesize_requests,
)

__version__ = "0.1.0"
