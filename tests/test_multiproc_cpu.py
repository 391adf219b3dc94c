"""Multi-process (gloo, world size 2, CPU) tests of the batch-sharded path's
host logic: request partitioning, max-over-ranks timing / summed tokens, and
that sharding never changes a result (random streams use GLOBAL request ids)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import get_config, prompts, shard_requests


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg_name, batch, bpg, strong = case
    lo, hi, gb, kind, par = bench.plan_shard(cfg_name, batch, world, rank, batch_per_gpu=bpg, strong=strong)
    ms = 10.0 + rank            # rank 1 is the slow one
    emitted = float(hi - lo) * 3
    ms_max, em_sum = bench.reduce_over_ranks(ms, emitted)
    out[rank] = (lo, hi, gb, kind, ms_max, em_sum)
    dist.destroy_process_group()


# (config, config batch, --batch-per-gpu, --strong)
CASES = [("c3", 32, None, False),   # weak: 32 requests per GPU, global batch 64
         ("c3", 32, 5, False),      # weak with --batch-per-gpu 5
         ("c2", 1, None, False),    # batch-1 config: one request per GPU, distinct requests
         ("c4", 64, None, False),   # strong: the fixed global batch of 64 split 32 / 32
         ("c5", 5, None, True)]     # strong, uneven: 3 / 2


@pytest.mark.parametrize("case", CASES)
def test_gloo_world2_shard_and_reduce(case):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    assert all(r[4] == 11.0 for r in res)                      # max over ranks
    gb = res[0][2]
    assert all(r[2] == gb for r in res)
    covered = sorted(i for lo, hi, *_ in res for i in range(lo, hi))
    assert covered == list(range(gb))                          # a partition of the global batch
    assert all(r[5] == 3.0 * gb for r in res)                  # tokens summed over ranks
    cfg_name, batch, bpg, strong = case
    if strong or cfg_name in ("c4",):
        assert all(r[3] == "strong" for r in res) and gb == batch
    else:
        assert all(r[3] == "weak" for r in res) and gb == world * (bpg or batch)


def test_shard_requests_balanced():
    for n in range(1, 70):
        for w in (1, 2, 4, 8):
            spans = [shard_requests(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_sharding_invariance_of_the_stochastic_method():
    """The oracle on requests [0,4) in one engine == the same requests split
    over two 'ranks' with req_offset: the Philox streams are keyed by global id."""
    from oracle.model import Model
    from oracle.table import TokenInfoTable
    from oracle.engine import Engine
    cfg = get_config("c1").replace(accept="stochastic", vocab=64, hidden=32, q_heads=2, kv_heads=1,
                                   head_dim=16, ffn=64, layers=1, prompt_len=8, max_new=10)
    m = Model(cfg, seed=2)
    pr = prompts(cfg, batch=4, length=8)
    whole = Engine(m, TokenInfoTable(m), cfg, seed=5).decode(pr, 10)
    parts = []
    for lo, hi in (shard_requests(4, 2, 0), shard_requests(4, 2, 1)):
        parts += Engine(m, TokenInfoTable(m), cfg, seed=5, req_offset=lo).decode(pr[lo:hi], 10)
    assert whole == parts


def _shard_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_21224_b200 import hsd
    nid = hsd.shard_nccl_id()
    cfg = get_config("c1")
    c, _ = hsd.make_config(cfg, shard_mode=hsd.SHARD_NCCL, vocab_shards=world, shard_rank=rank, nccl_id=nid)
    out[rank] = (bytes(c.nccl_id), c.shard_rank, c.vocab_shards, c.shard_mode)
    dist.destroy_process_group()


def test_gloo_world2_vocab_shard_bootstrap():
    """Vocab-sharded lm_head bootstrap: shard 0's NCCL unique id
    reaches every rank intact through the process group, and each rank's config
    names its own shard of the same G-shard group."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ids = [out[r][0] for r in range(world)]
    assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])
    assert [out[r][1] for r in range(world)] == [0, 1]
    assert all(out[r][2] == world and out[r][3] == 1 for r in range(world))


# ---- R29: stochastic acceptance over a vocab-sharded head, merged across ranks
KG = 16   # Gumbel candidates per shard record (HSD_SHARD_KG)


def _records(L, lo, hi, T, U, tree_tok):
    """One shard's per-row record over its columns [lo, hi): (max and sum exp of
    l/T, its top-KG Gumbel scores l/T + G with token ids, the logits of the tree
    tokens it owns) -- DESIGN.md R29."""
    z = L[:, lo:hi] / T
    m = z.max(axis=1)
    s = np.exp(z - m[:, None]).sum(axis=1)
    g = z - np.log(-np.log(U[:, lo:hi]))
    order = np.lexsort((np.arange(lo, hi)[None, :].repeat(len(L), 0), -g), axis=1)[:, :KG]
    gv = np.take_along_axis(g, order, axis=1)
    gi = order + lo
    own = (tree_tok >= lo) & (tree_tok < hi)
    tl = np.where(own[None, :], L[:, np.clip(tree_tok, 0, L.shape[1] - 1)], np.nan)
    return m, s, gv, gi, tl


def _merge(recs):
    m = np.stack([r[0] for r in recs])                  # [G, rows]
    s = np.stack([r[1] for r in recs])
    M = m.max(axis=0)
    lse = M + np.log((s * np.exp(m - M)).sum(axis=0))
    gv = np.concatenate([r[2] for r in recs], axis=1)
    gi = np.concatenate([r[3] for r in recs], axis=1)
    order = np.lexsort((gi, -gv), axis=1)[:, :KG]
    tl = np.nanmax(np.stack([np.where(np.isnan(r[4]), -np.inf, r[4]) for r in recs]), axis=0)
    return lse, np.take_along_axis(gv, order, 1), np.take_along_axis(gi, order, 1), tl


def _stoch_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_21224_b200.hsd import vocab_shard_bounds
    from oracle.philox import gumbel_uniforms
    V, rows, T = 1000, 6, 0.7
    rng = np.random.default_rng(11)                     # the same inputs on every rank
    L = rng.standard_normal((rows, V)) * 3.0
    tree_tok = rng.choice(V, size=9, replace=False)
    U = np.stack([gumbel_uniforms(seed=3, req=2, step=1, slot=r, vocab=V) for r in range(rows)])
    lo = vocab_shard_bounds(V, world)
    rec = _records(L, lo[rank], lo[rank + 1], T, U, tree_tok)
    allrec = [None] * world
    dist.all_gather_object(allrec, rec)                 # the records all-gather (gloo here, NCCL on GPUs)
    out[rank] = _merge(allrec)
    dist.destroy_process_group()


def test_gloo_world2_stochastic_shard_merge():
    """World-2 processes each reduce their vocab columns to R29 records, all-gather
    them and merge: the merged lse is logsumexp(l/T) of the full rows, the tree-token
    logits are the full rows' values, and the residual Gumbel-max over V minus any
    rejected set of < 16 tokens (the oracle's gumbel_argmax on the full row) is the
    best merged candidate outside it."""
    from oracle.philox import gumbel_uniforms
    from oracle.accept import gumbel_argmax
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stoch_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    V, rows, T = 1000, 6, 0.7
    rng = np.random.default_rng(11)
    L = rng.standard_normal((rows, V)) * 3.0
    tree_tok = rng.choice(V, size=9, replace=False)
    for r in range(world):
        lse, gv, gi, tl = out[r]
        ref = np.log(np.exp(L / T - (L / T).max(1, keepdims=True)).sum(1)) + (L / T).max(1)
        assert np.allclose(lse, ref, rtol=0, atol=1e-12)
        assert np.array_equal(tl, L[:, tree_tok])
        for row in range(rows):
            U = gumbel_uniforms(seed=3, req=2, step=1, slot=row, vocab=V)
            for k in (0, 4, 15):                       # rejected sets of 0 / 4 / 15 tokens
                excl = [int(x) for x in gi[row, :k]]
                want, _ = gumbel_argmax(L[row], T, U, exclude=excl)
                got = next(int(v) for v in gi[row] if int(v) not in excl)
                assert got == want
