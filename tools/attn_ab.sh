# A/B of prefill-attention builds on the C2-C5 prefill shapes (microbench, L2 flushed between reps).
#   bash tools/attn_ab.sh lib1.so lib2.so ...
for lib in "$@"; do
  for c in prefill_2048_after4096_70b prefill_2048_from0_8b prefill_4x512_after2000_qwen prefill_640_after6000_70b prefill_chunk512_after1500 mixed_bench; do
    echo -n "$(basename $lib) "; GLLM_LIB=$lib timeout 120 python tools/bench_kernels.py --only attn --case $c
  done
done
