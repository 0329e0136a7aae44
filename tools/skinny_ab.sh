# A/B of decode-sized GEMMs: skinny swap-AB stream-K kernel (default) vs 128-row tiles + split-K
for SK in 1 0; do
  echo "== GLLM_GEMM_SKINNY=$SK"
  for shape in 4,7168,5120 4,5120,5120 4,5120,13824 16,4096,14336 32,4096,4096 32,28672,4096; do
    GLLM_GEMM_SKINNY=$SK timeout 60 python tools/bench_kernels.py --gemm $shape
  done
  GLLM_GEMM_SKINNY=$SK timeout 60 python tools/bench_kernels.py --gemm 32,28672,4096 --swiglu
done
