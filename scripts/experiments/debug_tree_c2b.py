import sys; sys.path.insert(0, '.')
import numpy as np, torch
from synth import get_config, prompts
from paper_2602_21224_b200 import hsd
from oracle import tree as T
from tests.test_gpu_fullsize import GpuTableRows
from tests.gpu_lockstep import gpu_tree, gpu_pending
cfg = get_config("c2")
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=1,
                     max_ctx=cfg.prompt_len + 100, tcgen05=True)
ctx.prefill(prompts(cfg))
for s in range(2): ctx.step()
ctx.sync()
table = GpuTableRows(ctx, cfg, None)
for it in range(3):
    pend = gpu_pending(ctx, 0)
    root = int(ctx.tensor("root_tok").cpu()[0])
    ctx.build_tree(); ctx.sync()
    L = ctx.tensor("draft_logits").cpu().numpy().astype(np.float64)[0]
    n, tok, par, depth, lj = gpu_tree(ctx, 0)
    fresh = T.prune(T.build_subtree(L, root, cfg.branch_k, cfg.steps_N, table), cfg.budget_B)
    lin_f = T.linearize(fresh)
    fused = T.prune(T.fuse(fresh, pend), cfg.budget_B + cfg.resample_budget_Br) if len(pend) > 1 else fresh
    lin = T.linearize(fused)
    print("iter", it, "root", root, "pending", [(x['tok'], x['par'], round(x['lj'],3)) for x in pend])
    print("  gpu n", n, "oracle fused n", lin["T"], "oracle fresh n", lin_f["T"])
    gp = set(); po = set()
    def paths(tk, pr):
        out = []
        for i in range(len(tk)):
            out.append(() if pr[i] < 0 else out[pr[i]] + (int(tk[i]),))
        return out
    G = paths(tok, par); O = paths(lin["tok"], lin["par"])
    print("  only gpu:", sorted(set(G) - set(O))[:6])
    print("  only oracle:", sorted(set(O) - set(G))[:6])
    ctx.verify_tree(); ctx.accept_and_compact(); ctx.sync()
    print("  acc_n", int(ctx.tensor("acc_n").cpu()[0]), "bonus", int(ctx.tensor("bonus").cpu()[0]))
