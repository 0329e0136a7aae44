# A/B of the GEMM tilings at the bench's shapes: GLLM_GEMM_CG=1 (1-CTA) vs default (2-CTA for M > 128)
for CG in 2 1; do
  echo "== GLLM_GEMM_CG=$CG"
  for shape in 2009,6144,4096 2009,4096,4096 2009,28672,4096 2009,4096,14336 2944,28672,4096 1000,128256,4096 646,10240,8192 646,8192,8192 646,57344,8192 646,8192,28672 300,6144,4096; do
    GLLM_GEMM_CG=$CG timeout 60 python tools/bench_kernels.py --gemm $shape
  done
done
