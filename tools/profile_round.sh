#!/bin/bash
# Round profile capture on one B200 (run under gpurun): launch list of bench.py's timed region,
# full ncu captures of the dominant kernels at the bench's shapes. Outputs land in gpurun_out/.
set -x
TAG=${1:-r1b}
# 1. every launch of the NVTX-tagged timed region of bench.py (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" \
  --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
# 2. full captures: gate-up GEMM + SwiGLU epilogue (2-CTA) at the bench's M, decode attention at the
#    bench's decode population, prefill attention on a long-prompt chunk (C5 shape)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 \
  -o gpurun_out/${TAG}_gemm_gateup python tools/bench_kernels.py --gemm 2009,28672,4096 --swiglu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 3 -c 1 \
  -o gpurun_out/${TAG}_attn_decode python tools/bench_kernels.py --only attn --case decode800_ctx500 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 3 -c 1 \
  -o gpurun_out/${TAG}_attn_prefill python tools/bench_kernels.py --only attn --case prefill_2048_after4096_70b > /dev/null 2>&1
ls -la gpurun_out/
