"""cuBLAS (torch.matmul bf16) on the c3 verify GEMM shapes, for `ncu` to name the
kernels cuBLAS picks (tile / cluster configuration). Not a measurement."""
import torch
M = 2080
for N, K in [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        torch.matmul(a, w.T)
torch.cuda.synchronize()
