# GEMM tiling across the serving M range (decode -> saturated prefill) at Llama-3-8B / Qwen / 70B shapes
for shape in 800,4096,4096 800,6144,4096 800,28672,4096 646,8192,8192 646,10240,8192 646,8192,28672 1030,4096,14336 2009,6144,4096 2009,4096,4096 2009,28672,4096 2009,4096,14336 2944,28672,4096; do
  timeout 60 python tools/bench_kernels.py --gemm $shape
done
