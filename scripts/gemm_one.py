"""One c3 verify-GEMM shape through the library and through cuBLAS (for ncu).
python scripts/gemm_one.py M N K"""
import sys
sys.path.insert(0, '.')
import torch
from paper_2602_21224_b200 import hsd
M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
W = (torch.randn(N, K, device="cuda") * 0.01).to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda")
for _ in range(2):
    hsd.debug_gemm(A, W, C, use_tc=True)
    torch.matmul(A, W.t())
torch.cuda.synchronize()
