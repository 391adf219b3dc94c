"""The library's tcgen05 GEMMs against cuBLAS (torch.matmul, bf16) on the verify
shapes of a config (default c3: M = 32 x 65 rows), back to back, CUDA events.
python scripts/gemm_vs_cublas.py [c3|c4|c5]"""
import sys
sys.path.insert(0, '.')
import torch
from paper_2602_21224_b200 import hsd
from synth import get_config

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
T = 1 + cfg.budget_B + cfg.resample_budget_Br             # tree slots per request
M = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else cfg.batch * T
H, F = cfg.hidden, cfg.ffn
qkv = (cfg.q_heads + 2 * cfg.kv_heads) * cfg.head_dim
shapes = [("qkv", M, qkv, H, False), ("o", M, H, cfg.q_heads * cfg.head_dim, True), ("gu", M, 2 * F, H, "swiglu"),
          ("down", M, H, F, True)]
torch.manual_seed(0)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


if "--head" in sys.argv:   # the verify lm_head (fp32 logits store) as a fifth shape
    shapes.append(("head", M, cfg.vocab, H, False))
tot_h = tot_c = 0.0
for name, m, n, k, mode in shapes:
    A = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    W = (torch.randn(n, k, device="cuda") * 0.01).to(torch.bfloat16)
    C = torch.zeros(m, n, device="cuda")
    if mode == "swiglu":
        Hb = torch.empty(m, n // 2, device="cuda", dtype=torch.bfloat16)
        us_h = timeit(lambda: hsd.debug_gemm(A, W, Hb, use_tc="swiglu"))
    else:
        us_h = timeit(lambda: hsd.debug_gemm(A, W, C, accumulate=bool(mode), use_tc=True))
    Wt = W.t()
    us_c = timeit(lambda: torch.matmul(A, Wt))
    fl = 2.0 * m * n * k
    tot_h += us_h; tot_c += us_c
    print(f"{name:5s} M={m:5d} N={n:6d} K={k:6d}  hsd {us_h:8.1f} us {fl/us_h/1e6:7.1f} TF/s   "
          f"cublas {us_c:8.1f} us {fl/us_c/1e6:7.1f} TF/s   ratio {us_c/us_h:5.2f}", flush=True)
print(f"layer total: hsd {tot_h:.1f} us, cublas {tot_c:.1f} us, ratio {tot_c/tot_h:.2f}")
