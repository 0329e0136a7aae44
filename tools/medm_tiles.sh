# Medium-M (decode-heavy batches, M ~ 200-500) GEMM tilings: auto vs forced (BN, splits)
for shape in 214,7168,5120 214,5120,5120 214,5120,27648 214,55296,5120 420,7168,5120 420,5120,5120; do
  for t in 0,0 128,1 256,1 64,1 128,2; do
    timeout 60 python tools/bench_kernels.py --gemm $shape,$t
  done
done
