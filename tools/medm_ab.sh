# medium-M GEMMs (decode batches of 33..~1000 tokens): split-K choice
for shape in 213,5120,27648 213,55296,5120 213,7168,5120 213,5120,5120 128,4096,14336 64,4096,4096 300,6144,4096 500,4096,14336 800,4096,4096; do
  timeout 60 python tools/bench_kernels.py --gemm $shape
done
