import sys, itertools
sys.path.insert(0, '.')
import numpy as np
from synth import get_config
from tests.test_gpu_parity import run_lockstep
from paper_2602_21224_b200 import hsd
for hd, qh, kvh, pl in [(64, 8, 2, 32), (64, 4, 4, 32), (64, 8, 2, 100), (128, 8, 2, 32), (64, 2, 2, 32), (128, 4, 4, 32)]:
    cfg = get_config("c1").replace(hidden=512, q_heads=qh, kv_heads=kvh, head_dim=hd, ffn=1024, vocab=1024,
                                   layers=2, steps_N=5, branch_k=3, budget_B=16, prompt_len=pl)
    try:
        ls, accs = run_lockstep(cfg, hsd.BF16, steps=4, tcgen05=True, planted=True)
        print(hd, qh, kvh, pl, "OK", ls.max_err)
    except AssertionError as e:
        print(hd, qh, kvh, pl, "FAIL", str(e)[:80])
