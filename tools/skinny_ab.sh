# A/B of decode-sized GEMMs: skinny swap-AB stream-K kernel (default) vs 128-row tiles + split-K
for SK in 1 0; do
  echo "== GLLM_GEMM_SKINNY=$SK"
  for shape in 4,7168,5120 4,5120,5120 4,5120,13824 4,152064,5120 16,6144,4096 16,4096,14336 32,28672,4096 1,4096,4096; do
    GLLM_GEMM_SKINNY=$SK timeout 60 python tools/bench_kernels.py --gemm $shape
  done
  GLLM_GEMM_SKINNY=$SK timeout 60 python tools/bench_kernels.py --gemm 4,27648,5120 --swiglu
done
