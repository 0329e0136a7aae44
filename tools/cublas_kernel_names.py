"""cuBLAS (torch.matmul) on the M ~ 2k projections, for reading its kernel choice off an ncu launch list:

    ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic \
        --clock-control none --csv --log-file gpurun_out/cublas_names.csv python tools/cublas_kernel_names.py

(profiles/r2/cublas_kernel_names.txt: nvjet 2-CTA kernels with 256 x 224 / 192 x 224 CTA tiles, one tile per CTA.)
"""
import torch

SHAPES = [(2009, 4096, 4096), (2009, 6144, 4096), (2009, 4096, 14336), (2009, 8192, 8192), (2009, 28672, 4096)]

for M, N, K in SHAPES:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        c = a @ b.T
    torch.cuda.synchronize()
