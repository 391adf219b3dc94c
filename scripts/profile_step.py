"""One profiled stage of a speculative step, for ncu --profile-from-start off.

usage: python scripts/profile_step.py CFG [--batch B] [--stage verify|build|step|prefill]

Sets the config up like bench.py (bf16, tcgen05, RESAMPLE|FUSION), prefills,
runs 3 warm steps, then opens a CUDA profiler range around exactly one staged
call: verify_tree (S2: L target layers over the tree), build_tree (S0 + S1:
draft chain, one-pass head, K-TREE) or a whole step. So `ncu -k regex:X -c n`
captures the first n launches of X inside that stage -- e.g. the four GEMMs of
verify layer 0 -- with no launch-skip arithmetic.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import get_config, prompts, vocab_permutation
from paper_2602_21224_b200 import hsd

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--stage", default="verify", choices=["verify", "build", "step", "prefill"])
a = ap.parse_args()
cfg = get_config(a.config)
if a.batch:
    cfg = cfg.replace(batch=a.batch)
N = cfg.steps_N
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=cfg.batch,
                     max_ctx=cfg.prompt_len + 16 * (N + 1) + 64 * (N + 1),
                     vocab_perm=vocab_permutation(cfg.vocab, 0) if cfg.hot_tokens else None,
                     tcgen05=True, flags=hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION)
if a.stage == "prefill":   # one request's prefill (target forward + first token + draft prefill)
    pr1 = prompts(cfg, batch=1)
    ctx.prefill(pr1)
    ctx.sync()
    torch.cuda.profiler.start()
    ctx.prefill(pr1)
    ctx.sync()
    torch.cuda.profiler.stop()
    sys.exit(0)
ctx.prefill(prompts(cfg, batch=cfg.batch))
for _ in range(3):
    ctx.step()
ctx.sync()
if a.stage == "step":
    torch.cuda.profiler.start()
    ctx.step()
    ctx.sync()
    torch.cuda.profiler.stop()
else:
    if a.stage == "build":
        torch.cuda.profiler.start()
    ctx.build_tree()
    ctx.sync()
    if a.stage == "build":
        torch.cuda.profiler.stop()
    else:
        torch.cuda.profiler.start()
        ctx.verify_tree()
        ctx.sync()
        torch.cuda.profiler.stop()
print("profiled", a.config, a.stage, "batch", cfg.batch)
