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
