"""Phase trace of single tcgen05 GEMM launches on the c2 shapes (HSD_GEMM_TRACE):
per CTA 0 / last CTA: start, weights prefetched (pre-PDL), PDL released, first
stage landed (MMA), last stage landed, epilogue start, epilogue end, CTA end (us)."""
import os, sys
os.environ["HSD_GEMM_TRACE"] = "1"
sys.path.insert(0, '.')
import torch
from paper_2602_21224_b200 import hsd
for name, M, N, K in [("o", 65, 4096, 4096), ("qkv", 65, 12288, 4096), ("down", 65, 4096, 11008)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.01 for _ in range(6)]
    C = torch.zeros(M, N, device="cuda")
    for i in range(6):
        hsd.debug_gemm(A, Ws[i], C, accumulate=True, use_tc=True)
    torch.cuda.synchronize()
    print(name, flush=True)
