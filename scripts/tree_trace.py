"""Phase trace of one fresh K-TREE launch (HSD_TREE_TRACE): thread 0 of request 0's
leader CTA stamps %globaltimer per Alg. 1 round (sweep / warp merge / cluster barrier /
merge + TopkByJointProb), then prune, fusion, linearisation."""
import os, sys; sys.path.insert(0, '.')
os.environ["HSD_TREE_TRACE"] = "1"
import numpy as np, torch
from synth import get_config, prompts, vocab_permutation
from paper_2602_21224_b200 import hsd
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = cfg.replace(batch=batch)
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=batch,
                     max_ctx=cfg.prompt_len + 100, tcgen05=True,
                     vocab_perm=vocab_permutation(cfg.vocab, 0) if cfg.hot_tokens else None,
                     flags=int(os.environ.get("TT_FLAGS", hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION)))
ctx.prefill(prompts(cfg, batch=batch))
for _ in range(3): ctx.step()
ctx.build_tree()
t = ctx.tensor("tree_trace").cpu().numpy().astype(np.int64)
t0 = t[0]
us = lambda i: (t[i] - t0) / 1e3
print(f"pdl_wait done {us(1):8.2f} us")
prev = t[1]
for i in range(cfg.steps_N):
    a, b, c, d = (t[2 + 4 * i] - prev) / 1e3, (t[3 + 4 * i] - t[2 + 4 * i]) / 1e3, (t[4 + 4 * i] - t[3 + 4 * i]) / 1e3, (t[5 + 4 * i] - t[4 + 4 * i]) / 1e3
    print(f"round {i}: sweep {a:7.2f}  warp-merge {b:7.2f}  leader+cluster.sync {c:7.2f}  merge+frontier {d:7.2f}   (end {us(5 + 4 * i):8.2f})")
    prev = t[5 + 4 * i]
for i, nm in [(40, "build done"), (41, "prune"), (42, "fusion"), (43, "prune B+Br"), (44, "linearised+written")]:
    print(f"{nm:20s} {us(i):8.2f} us")
