# Medium-M (one 128-row tile) GEMM tilings: forced (BN, split-K) grid at decode shapes, to see how
# the weight-stream rate scales with the number of CTAs streaming (split-K adds a reduce launch).
for shape in 64,5120,5120 64,4096,4096 64,7168,5120 64,5120,13824 128,5120,5120; do
  for cfg in 0,0 64,1 64,2 64,3 128,1 128,2 128,3 128,4 256,4 256,8; do
    timeout 60 python tools/bench_kernels.py --gemm $shape,$cfg --wscale 0.02
  done
done
