import sys; sys.path.insert(0, '.')
import numpy as np, torch
from synth import get_config, prompts
from paper_2602_21224_b200 import hsd
from oracle import tree as T
from tests.test_gpu_fullsize import GpuTableRows
from tests.gpu_lockstep import gpu_tree
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=cfg.batch,
                     max_ctx=cfg.prompt_len + 100, tcgen05=True)
ctx.prefill(prompts(cfg))
root = int(ctx.tensor("root_tok").cpu()[0])
ctx.build_tree(); ctx.sync()
L = ctx.tensor("draft_logits").cpu().numpy().astype(np.float64)[0]
table = GpuTableRows(ctx, cfg, None)
v = L[0] + table.row(root)
order = np.argsort(-v)[:8]
print("root", root, "oracle top8 step1:", [(int(i), round(float(v[i]), 4)) for i in order])
print("lse", float(np.log(np.sum(np.exp(v - v.max()))) + v.max()))
n, tok, par, depth, lj = gpu_tree(ctx, 0)
print("gpu depth-1 nodes:", [(int(tok[i]), round(float(lj[i]), 4)) for i in range(n) if depth[i] == 1])
mg = []
fresh = T.build_subtree(L, root, cfg.branch_k, cfg.steps_N, table, mg)
print("oracle depth-1:", [(n_['tok'], round(n_['lj'], 4)) for n_ in fresh if n_['depth'] == 1])
lin = T.linearize(T.prune(fresh, cfg.budget_B))
print("gpu n", n, "oracle n", lin["T"])
for i in range(min(n, lin["T"])):
    if tok[i] != lin["tok"][i] or par[i] != lin["par"][i]:
        print("first diff slot", i, "gpu", tok[i], par[i], depth[i], lj[i], "oracle", lin["tok"][i], lin["par"][i], lin["depth"][i], lin["lj"][i])
        break
print("gpu lj by depth", [round(float(x), 3) for x in lj[:12]])
print("orc lj by depth", [round(float(x), 3) for x in lin["lj"][:12]])
