"""Time hsd_prefill (the e2e leg's first part) on a config: wall time of ctx.prefill."""
import sys, time
sys.path.insert(0, '.')
import torch
from synth import get_config, prompts, vocab_permutation
from paper_2602_21224_b200 import hsd
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=cfg.batch,
                     max_ctx=cfg.prompt_len + 200, tcgen05=True,
                     vocab_perm=vocab_permutation(cfg.vocab, 0) if cfg.hot_tokens else None)
pr = prompts(cfg, batch=cfg.batch)
ctx.prefill(pr)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); ctx.prefill(pr); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
print(f"{cfg.name} prefill of {cfg.batch} x {cfg.prompt_len} tokens: {min(ts)*1e3:.2f} ms (min of 3)")
