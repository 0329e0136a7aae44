# Forced (BN, split-K) and 1-CTA / 2-CTA configurations on the GEMM shapes where the auto tiling
# trails cuBLAS most (profiles/r2/gemm_vs_cublas_sweep.csv, 129 <= M <= 1024). One JSON line each.
for shape in 256,10240,8192 512,10240,8192 512,5120,5120 512,5120,13824 512,5120,27648 256,5120,5120 1024,5120,27648; do
  timeout 40 python tools/bench_kernels.py --gemm $shape --wscale 0.02 | sed 's/^/auto /'
  for bn in 128 256; do for sp in 1 2 3 4 6; do
    for cg in 2 1; do GLLM_GEMM_CG=$cg timeout 40 python tools/bench_kernels.py --gemm $shape,$bn,$sp --wscale 0.02 | sed "s/^/cg$cg /"; done
  done; done
done
