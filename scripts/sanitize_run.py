"""Small workloads for compute-sanitizer (scripts/sanitize.sh): prefill + speculative
steps through the C ABI, eager (no CUDA graph) so every launch is checked.

  python scripts/sanitize_run.py fp32   c1, fp32-verify (SIMT GEMM / attention, K-TREE, walk, compaction)
  python scripts/sanitize_run.py bf16   GQA 8/2 hd 128, 600-token prompt: tcgen05 GEMMs (stream-K and
                                        data-parallel), tcgen05 tree attention with key splits + the 2-CTA
                                        cluster merge, K-TREE with the bf16 table, stochastic walk
  python scripts/sanitize_run.py pair   c3 widths (GQA 32/8, hd 128), 1 layer, 2048-token prompt: the
                                        CTA-pair GEMM with its fused QKV (RoPE / paged KV) epilogue,
                                        TMA reduce-add residual epilogue and SwiGLU epilogue in the prefill
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth import get_config, prompts  # noqa: E402
from paper_2602_21224_b200 import hsd  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fp32"
if mode == "fp32":
    cfg = get_config("c1")
    ctx = hsd.init_model(cfg, device=0, stream=None, precision=hsd.FP32_VERIFY, seed=0,
                         max_ctx=cfg.prompt_len + 8 * (cfg.steps_N + 1) + 8)
elif mode == "pair":
    cfg = get_config("c3").replace(layers=1, vocab=4096, hot_tokens=0, batch=1, prompt_len=2048, accept="greedy")
    ctx = hsd.init_model(cfg, device=0, stream=None, precision=hsd.BF16, seed=0, tcgen05=True, max_batch=1,
                         max_ctx=cfg.prompt_len + 8 * (cfg.steps_N + 1) + 8)
else:
    cfg = get_config("c1").replace(hidden=512, q_heads=8, kv_heads=2, head_dim=128, ffn=1024, vocab=1024, layers=2,
                                   steps_N=5, branch_k=3, budget_B=16, prompt_len=600, accept="stochastic")
    ctx = hsd.init_model(cfg, device=0, stream=None, precision=hsd.BF16, seed=0, tcgen05=True,
                         max_ctx=cfg.prompt_len + 8 * (cfg.steps_N + 1) + 8)
ctx.prefill(np.array(prompts(cfg)))
n = 0
for _ in range(4):                     # staged calls: build / verify / accept
    ctx.build_tree()
    ctx.verify_tree()
    ctx.accept_and_compact()
    n += 1
ctx.sync()
print(f"sanitize_run {mode}: {n} steps ok")
ctx.destroy()
