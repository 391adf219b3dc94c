import os, sys; sys.path.insert(0, '.')
os.environ["HSD_ATTN_TRACE"] = "1"
import numpy as np, torch
from synth import get_config, prompts, vocab_permutation
from paper_2602_21224_b200 import hsd
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
stream = torch.cuda.Stream()
ctx = hsd.init_model(cfg, device=0, stream=stream.cuda_stream, precision=hsd.BF16, seed=0, max_batch=batch,
                     max_ctx=cfg.prompt_len + 100, tcgen05=True,
                     vocab_perm=vocab_permutation(cfg.vocab, 0) if cfg.hot_tokens else None)
ctx.prefill(prompts(cfg, batch=batch))
for _ in range(3): ctx.step()
ctx.build_tree()
if len(sys.argv) > 3:   # HSD_ATTN_EXP timing experiment on the traced verify pass only
    os.environ["HSD_ATTN_EXP"] = sys.argv[3]
ctx.verify_tree()   # the trace holds the last attention launch (verify layer 31)
os.environ.pop("HSD_ATTN_EXP", None)
t_all = ctx.tensor("attn_trace").cpu().numpy().astype(np.int64)
t = t_all[:128]
t1 = t_all[128:]   # CTA x = 1 (the pair follower in CTA-pair mode, else split 1)
t0 = t[0]
names = {0: "start", 1: "barriers+tmem", 2: "pdl_wait", 3: "Q landed (mma)", 4: "last PV done", 5: "end"}
for i in [0, 1, 2, 3]:
    print(f"{names[i]:16s} {(t[i]-t0)/1e3:8.2f} us")
n = int(t[7])
print("chunks", n)
for j in range(min(n, 12)):  # pv(j-1) is only stamped when the chunk rescales O
    print(f" chunk {j}: S ready {(t[8+4*j]-t0)/1e3:7.2f}  max done {(t[9+4*j]-t0)/1e3:7.2f}  pv(j-1) done {(t[10+4*j]-t0)/1e3 if j>0 else float('nan'):7.2f}  P written {(t[11+4*j]-t0)/1e3:7.2f}")
for i, nm in [(56, "epi: l exchanged"), (57, "epi: O staged"), (58, "epi: rows written"), (59, "warp0 at end"), (60, "warp1 at end"), (61, "thr64 at end"), (62, "thr96 at end")]:
    print(f"{nm:16s} {(t[i]-t0)/1e3:8.2f} us")
print("MMA warp: S_{j+1} issued / P_j V_j issued (us)")
for j in range(min(n, 16)):
    print(f" j {j:2d}: S{j+1} issued {(t[64+2*j]-t0)/1e3:7.2f}  PV{j} issued {(t[65+2*j]-t0)/1e3:7.2f}"
          f"  | K{j} load issued {(t[96+j]-t0)/1e3:7.2f}  K{j} landed {(t[112+j]-t0)/1e3:7.2f}")
for i in [4, 5]:
    print(f"{names[i]:16s} {(t[i]-t0)/1e3:8.2f} us")

if t1[0] != 0:
    print("CTA x=1 (pair follower / split 1), same origin")
    for j in range(min(int(t1[7]), 10)):
        print(f" chunk {j}: S ready {(t1[8+4*j]-t0)/1e3:7.2f}  max done {(t1[9+4*j]-t0)/1e3:7.2f}  P written {(t1[11+4*j]-t0)/1e3:7.2f}"
              f"  | K{j} load issued {(t1[96+j]-t0)/1e3:7.2f}")

if os.environ.get("TC2_TRACE"):
    print("two-tile kernel: per chunk  S_A ready / P_A written / S_B ready / P_B written; MMA warp: V_j landed, K_j+1 landed")
    for j in range(min(int(t[7]), 12)):
        f = lambda i: (t[i] - t0) / 1e3
        print(f" chunk {j:2d}: A {f(8+4*j):7.2f} {f(9+4*j):7.2f}   B {f(10+4*j):7.2f} {f(11+4*j):7.2f}   "
              f"| V{j} {f(64+2*j):7.2f} K{j+1} {f(65+2*j):7.2f}")
