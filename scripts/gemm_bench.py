"""Time the library's tcgen05 GEMM on the c2 decode shapes (CUDA events)."""
import os, sys, json
sys.path.insert(0, '.')
import torch
from paper_2602_21224_b200 import hsd
torch.manual_seed(0)
shapes = [("qkv", 65, 12288, 4096), ("o", 65, 4096, 4096), ("gu", 65, 22016, 4096), ("down", 65, 4096, 11008),
          ("head", 65, 32000, 4096), ("draft_qkv", 7, 12288, 4096), ("chain_gu", 1, 22016, 4096)]
res = {}
for name, M, N, K in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.01
    C = torch.zeros(M, N, device="cuda")
    for _ in range(3):
        hsd.debug_gemm(A, W, C, accumulate=True, use_tc=True)
    torch.cuda.synchronize()
    # flush L2 between reps by rotating through 8 weight copies (> 126 MB total for big shapes)
    Ws = [W.clone() for _ in range(max(1, int(400e6 // W.numel() // 2)))]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 40
    e0.record()
    for i in range(reps):
        hsd.debug_gemm(A, Ws[i % len(Ws)], C, accumulate=True, use_tc=True)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    byt = N * K * 2 + M * K * 2 + M * N * 8
    res[name] = (round(us, 2), round(byt / us / 1e3, 1))
    print(f"{name:10s} M={M:4d} N={N:6d} K={K:6d}  {us:8.2f} us  {byt/us/1e3:8.1f} GB/s", flush=True)
print(json.dumps(res))
