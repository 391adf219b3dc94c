"""GPU sampling uniform / Gumbel-max parity (reading R13).

The stochastic walk's residual draw and the prefill's first token are Gumbel-max
samples over the whole vocabulary. At V = 128256 a draw reads 128256 uniforms,
so any uniform the GPU rounds differently from the oracle (e.g. a 24-bit k + 0.5
rounding to 2^24 in fp32, which made u = 1 and the Gumbel score infinite) shows
up in a fraction of draws. Here 10^4 (seed, slot) draws on the walk's own device
code (hsd_debug_gumbel) must pick the oracle's token wherever the oracle's top-2
score margin is above the fp32 rounding of the score (1e-5 absolute); draws
under that margin are counted and must stay rare.
"""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

from oracle.accept import gumbel_argmax
from oracle.philox import gumbel_uniforms

pytestmark = pytest.mark.gpu
hsd = pytest.importorskip("paper_2602_21224_b200.hsd")

V = 128256
ROWS = 8
SEEDS = list(range(10))
SLOTS = 1000
REQ, STEP, TEMP = 7, 3, 1.0
MARGIN = 1e-5


def _oracle_draw(lg, seed, slot):
    return gumbel_argmax(lg, TEMP, gumbel_uniforms(seed, REQ, STEP, slot, V))


def test_gumbel_argmax_identical_to_oracle_v128256():
    rng = np.random.default_rng(42)
    # flat-ish logits (std 2): the Gumbel noise decides most draws, so every uniform matters
    logits = (rng.standard_normal((ROWS, V)) * 2.0).astype(np.float32)
    d_logits = torch.from_numpy(logits).cuda()
    rows = np.arange(SLOTS, dtype=np.int32) % ROWS
    slots = np.arange(SLOTS, dtype=np.int32)
    d_rows, d_slots = torch.from_numpy(rows).cuda(), torch.from_numpy(slots).cuda()
    gpu = {}
    for seed in SEEDS:
        gpu[seed] = hsd.debug_gumbel(d_logits, d_rows, d_slots, TEMP, seed, REQ, STEP).cpu().numpy()
    torch.cuda.synchronize()
    lg64 = logits.astype(np.float64)
    jobs = [(seed, int(s)) for seed in SEEDS for s in slots]
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        res = list(ex.map(lambda j: _oracle_draw(lg64[rows[j[1]]], j[0], j[1]), jobs))
    mism, flagged = [], 0
    for (seed, s), (tok, margin) in zip(jobs, res):
        if margin < MARGIN:
            flagged += 1
            continue
        if int(gpu[seed][s]) != tok:
            mism.append((seed, s, int(gpu[seed][s]), tok, margin))
    assert not mism, f"{len(mism)} of {len(jobs)} Gumbel draws differ: {mism[:5]}"
    assert flagged <= len(jobs) // 1000, flagged
