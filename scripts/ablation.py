"""ablation toggles and the one-pass head, measured on B200.

Ablations (c2 shapes, planted continuation R24 so that acceptance is real and
controlled; the verify / walk / compaction kernels run unmodified):
  full            re-sampling (Alg. 2) + verification fusion        (the method)
  resample-off    no Alg. 2 re-sampled tree                          (P:355-375 off)
  fusion-off      re-sampling WITHOUT fusion: the Alg. 2 tree is verified by a dedicated
                  extra target pass in the same step (Fig. 12's "+resampling")
  token-info-off  zero token-info table: Alg. 1 degenerates to a beam tree over the draft
                  logits alone (Fig. 5a; Table 4 "w/o token info")
  first-token-off the root pair enters the draft without its token embedding (Table 4
                  "w/o first token", R26)
  token-ar-draft  NEXT-2: the draft chain feeds back its own top-1 token each step
                  (EAGLE-style token-level AR, R27) -- lm_head GEMV + argmax + fc per step
Reported per variant: tau (emitted / step / request), ms / step, tokens / s, and the per-depth
conditional acceptance P(m >= d | m >= d-1) measured from the emitted counts -- with re-sampling
off it should reproduce the planted rates a_d (a check of the planted mechanism itself).

One-pass head (NEXT-2): the draft's N lm_head rows as ONE [b*N, n] x [n, V] GEMM
against N separate [b, n] x [n, V] GEMMs (what an iterative token-level draft pays), timed with
CUDA events on the library's tcgen05 GEMM.

usage: python scripts/ablation.py [--config c2] [--steps 30] [--warmup 5] [--out FILE.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
from synth import get_config, prompts, vocab_permutation
from paper_2602_21224_b200 import hsd

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--out", default="")
ap.add_argument("--batch", type=int, default=0, help="requests per step (more samples of the planted acceptance)")
ap.add_argument("--seeds", default="0,1,2", help="weight seeds; tau / acceptance pooled over the seeds' runs that "
                                                "stayed on the planted continuation")
a = ap.parse_args()
cfg = get_config(a.config)
if a.batch:
    cfg = cfg.replace(batch=a.batch)
N, b = cfg.steps_N, cfg.batch
rates = bench.PLANT_RATES[:N] + [bench.PLANT_RATES[-1]] * max(0, N - len(bench.PLANT_RATES))
VARIANTS = [("full", hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION),
            ("resample-off", hsd.FLAG_FUSION),
            ("fusion-off", hsd.FLAG_RESAMPLE),
            ("token-info-off", hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_ZERO_TABLE),
            ("first-token-off", hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_NO_FIRST_TOKEN),
            ("token-ar-draft", hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_TOKEN_AR)]
stream = torch.cuda.Stream()
pr = prompts(cfg, batch=b)
need_ctx = cfg.prompt_len + (a.steps + a.warmup + 12) * (N + 1) * 2 + 16
rows = []
seeds = [int(x) for x in a.seeds.split(",")]
for name, flags in VARIANTS:
    all_m, ms_l, tps_l, att, on = [], [], [], [], 0
    for seed in seeds:
        ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=seed, max_batch=b,
                             max_ctx=need_ctx + 64 * (N + 1), tcgen05=True, flags=flags | hsd.FLAG_PLANTED,
                             plant_rates=rates,
                             vocab_perm=vocab_permutation(cfg.vocab, 0) if cfg.hot_tokens else None)
        with torch.cuda.stream(stream):
            tau, tps, ms, info, counts = bench.planted_leg(ctx, pr, cfg, b, N, a.steps, a.warmup, stream,
                                                           return_counts=True, attempts=8)
        ms_l.append(ms)
        att.append(info["attempts"])
        if info["on_continuation"]:   # acceptance statistics only from runs that stayed on the continuation
            on += 1
            all_m.append(counts.reshape(-1))
            tps_l.append(tps)
        ctx.destroy()
        del ctx
        torch.cuda.empty_cache()
    em = np.concatenate(all_m) if all_m else np.zeros(0)
    m = em - 1
    cond = []
    for d in range(1, N + 1):
        base = int((m >= d - 1).sum())
        cond.append(round(float((m >= d).sum()) / base, 3) if base else None)
    ms_mean = float(np.mean(ms_l))
    tau = float(em.mean()) if em.size else None
    rows.append({"variant": name, "tau": round(tau, 3) if tau else None, "ms_per_step": round(ms_mean, 3),
                 "tokens_per_s": round(tau * b / (ms_mean / 1e3), 1) if tau else None,
                 "cond_accept_by_depth": cond, "samples": int(em.size), "seeds_on_continuation": f"{on}/{len(seeds)}",
                 "attempts": att})
    print(json.dumps(rows[-1]), flush=True)

# NEXT-2: one-pass head vs N iterative head GEMMs (weights [V, n] bf16 streamed each time)
W = (torch.randn(cfg.vocab, cfg.hidden, device="cuda") * 0.01).to(torch.bfloat16)
head = {}
for label, M, reps in [("one-pass [b*N rows]", b * N, 1), ("iterative (N x [b rows])", b, N)]:
    A = torch.randn(M, cfg.hidden, device="cuda").to(torch.bfloat16)
    C = torch.zeros(M, cfg.vocab, device="cuda")
    for _ in range(3):
        hsd.debug_gemm(A, W, C, use_tc=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record()
    for _ in range(it):
        for _ in range(reps):
            hsd.debug_gemm(A, W, C, use_tc=True)
    e1.record()
    torch.cuda.synchronize()
    head[label] = round(e0.elapsed_time(e1) * 1e3 / it, 2)
print(json.dumps({"head_us": head, "rows": b * N, "vocab": cfg.vocab, "hidden": cfg.hidden}), flush=True)
if a.out:
    json.dump({"config": a.config, "batch": b, "planted_rates": rates, "steps": a.steps, "ablation": rows, "head_us": head},
              open(a.out, "w"), indent=1)
