"""GPU tests of the vocab-sharded lm_head (BASELINE configs[4]).

The draft one-pass logits (S1a) and the verify head (S2) are split by
vocabulary column into G shards (include/hsd.h). Verify rows keep only a
per-shard partial argmax, merged exactly (max value, lowest token id, R8); the
draft logits rows are reassembled from the shards' column slices.

- HSD_SHARD_SIM (one GPU computes every shard and merges through the same
  kernels): in fp32-verify mode the sharded context emits exactly the unsharded
  context's tokens, which are the oracle's plain greedy decode (losslessness),
  and its draft logits / verify argmax are bit-identical (the SIMT GEMM's
  per-element k order does not depend on the column tiling).
- bf16 tcgen05 at several shard counts, including uneven 128-aligned widths:
  draft logits within the bf16 bar (2e-2 row-normwise, R21); verify argmax
  identical wherever the unsharded top-2 margin exceeds 1e-2.
- HSD_SHARD_NCCL with a one-rank communicator (the only NCCL group one GPU
  allows): the all-gather / send-recv path inside the step's CUDA graph.
"""
import numpy as np
import pytest
import torch

from synth import get_config, prompts
from oracle.model import Model
from oracle.engine import greedy_decode

pytestmark = pytest.mark.gpu

hsd = pytest.importorskip("paper_2602_21224_b200.hsd")


def _wide(vocab=1024):
    return get_config("c1").replace(hidden=256, q_heads=4, kv_heads=2, head_dim=64, ffn=512, vocab=vocab,
                                    layers=2, steps_N=4, branch_k=3, budget_B=16, prompt_len=40)


def _run(cfg, precision, steps, tcgen05=False, seed=0, **shard):
    stream = torch.cuda.Stream()
    ctx = hsd.init_model(cfg, device=0, precision=precision, seed=seed, stream=stream.cuda_stream,
                         max_ctx=cfg.prompt_len + steps * (cfg.steps_N + 1) + 16, tcgen05=tcgen05, **shard)
    ctx.prefill(prompts(cfg))
    out = []
    for _ in range(steps):
        e, n = ctx.step_host()
        out += [int(t) for t in e[0, :n[0]]]
    ctx.destroy()
    return out


@pytest.mark.parametrize("G", [2, 3, 8])
def test_sim_shards_fp32_lossless_and_identical(G):
    cfg = _wide()
    steps = 8
    base = _run(cfg, hsd.FP32_VERIFY, steps)
    got = _run(cfg, hsd.FP32_VERIFY, steps, shard_mode=hsd.SHARD_SIM, vocab_shards=G)
    assert got == base
    m = Model(cfg, seed=0, precision="fp32")
    ref, _ = greedy_decode(m, prompts(cfg)[0], len(got) + 2)
    assert got == list(ref[1:len(got) + 1]), "sharded speculative output != oracle plain greedy decode"


def _staged_pair(cfg, precision, G, tcgen05, force=False):
    """Unsharded and SIM-sharded contexts driven through the same staged step;
    returns (draft logits, tree, verify argmax, unsharded verify logits) of both.
    force: both contexts verify the UNSHARDED context's tree (hsd_force_tree) right
    after prefill, so their verify rows are always comparable (bf16: the two
    contexts' draft logits differ by rounding, which may reorder near-equal
    siblings)."""
    res, tree0 = [], None
    for shard in ({}, dict(shard_mode=hsd.SHARD_SIM, vocab_shards=G)):
        ctx = hsd.init_model(cfg, device=0, precision=precision, seed=1, max_ctx=cfg.prompt_len + 64,
                             tcgen05=tcgen05, stream=torch.cuda.Stream().cuda_stream, **shard)
        ctx.prefill(prompts(cfg))
        if not force:
            ctx.step()                           # one full step, then a staged one
        ctx.build_tree()
        L = ctx.tensor("draft_logits").clone()
        tree = [ctx.tensor(k).clone() for k in ("tree_tok", "tree_par", "tree_depth", "tree_n")]
        if force:
            if tree0 is None:
                tree0 = [t.cpu().numpy() for t in tree]
            else:
                ctx.force_tree(*tree0)
                tree = [ctx.tensor(k).clone() for k in ("tree_tok", "tree_par", "tree_depth", "tree_n")]
        v = ctx.verify_tree()
        am = ctx.tensor("verify_argmax").clone()
        logits = ctx.tensor("verify_logits").clone() if not shard else None
        assert (v.logits is None or v.logits == 0) if shard else v.logits
        ctx.accept_and_compact()
        ctx.destroy()
        res.append((L, tree, am, logits))
    return res


def test_sim_shards_fp32_bit_identical_heads():
    (L0, t0, a0, _), (L1, t1, a1, _) = _staged_pair(_wide(), hsd.FP32_VERIFY, 3, False)
    assert torch.equal(L0, L1)
    assert all(torch.equal(x, y) for x, y in zip(t0, t1))
    assert torch.equal(a0, a1)


@pytest.mark.parametrize("G,vocab", [(2, 1024), (5, 1024), (8, 2048), (3, 1000)])
def test_sim_shards_bf16_tcgen05(G, vocab):
    """bf16 tcgen05: both contexts verify the same (forced) tree right after the
    same prefill; draft logits within 2e-2 row-normwise (R21) and the sharded
    partial-argmax merge equals the unsharded argmax wherever the top-2 margin
    exceeds 1e-2 -- on every step, never skipped."""
    (L0, t0, a0, lg), (L1, t1, a1, _) = _staged_pair(_wide(vocab), hsd.BF16, G, True, force=True)
    scale = L0.abs().amax(dim=-1, keepdim=True).clamp_min(1e-6)
    assert ((L1 - L0).abs() / scale).max().item() <= 2e-2
    assert all(torch.equal(x, y) for x, y in zip(t0, t1))            # the forced tree
    top2 = lg.topk(2, dim=-1).values
    margin = (top2[..., 0] - top2[..., 1]) / lg.abs().amax(dim=-1).clamp_min(1e-6)
    decided = (a0 >= 0) & (margin > 1e-2)
    assert decided.sum() > 0
    assert torch.equal(a0[decided], a1[decided])
    assert torch.equal(a0 < 0, a1 < 0)                                # inactive slots stay -1


def test_nccl_single_rank_group_in_graph():
    """HSD_SHARD_NCCL with one rank: ncclAllGather + grouped ncclSend/ncclRecv run
    inside the step's CUDA graph; the result equals the unsharded context."""
    cfg = _wide()
    steps = 6
    base = _run(cfg, hsd.FP32_VERIFY, steps)
    nid = hsd.nccl_unique_id()
    got = _run(cfg, hsd.FP32_VERIFY, steps, shard_mode=hsd.SHARD_NCCL, vocab_shards=1, shard_rank=0, nccl_id=nid)
    assert got == base


# ------------------------------------------------------------- stochastic (R13)
def _stoch(vocab=1024):
    return _wide(vocab).replace(accept="stochastic")


@pytest.mark.parametrize("G", [2, 3, 8])
def test_sim_shards_stochastic_fp32_identical(G):
    """Stochastic acceptance over the vocab-sharded head: per-row records of each
    shard (max / sum of l/T, Gumbel top-KG, tree-token logits), merged exactly. In
    fp32-verify the sharded context emits the unsharded context's tokens: Gumbel
    scores are computed per element by the same expression on bit-identical logits,
    the lse merge differs only in summation order."""
    cfg = _stoch()
    steps = 10
    base = _run(cfg, hsd.FP32_VERIFY, steps, seed=3)
    got = _run(cfg, hsd.FP32_VERIFY, steps, seed=3, shard_mode=hsd.SHARD_SIM, vocab_shards=G)
    assert got == base


def _staged_stoch(cfg, precision, G, tcgen05, seed=4, force=False):
    """force: the sharded context verifies the unsharded context's tree
    (hsd_force_tree), so the two sets of verify rows are always comparable."""
    res, tree0 = [], None
    for shard in ({}, dict(shard_mode=hsd.SHARD_SIM, vocab_shards=G)):
        ctx = hsd.init_model(cfg, device=0, precision=precision, seed=seed, max_ctx=cfg.prompt_len + 64,
                             tcgen05=tcgen05, stream=torch.cuda.Stream().cuda_stream, **shard)
        ctx.prefill(prompts(cfg))
        ctx.build_tree()
        if force:
            if tree0 is None:
                tree0 = [ctx.tensor(k).cpu().numpy() for k in ("tree_tok", "tree_par", "tree_depth", "tree_n")]
            else:
                ctx.force_tree(*tree0)
        tree = (ctx.tensor("tree_tok").clone(), ctx.tensor("tree_par").clone(), int(ctx.tensor("tree_n").cpu()[0]))
        ctx.verify_tree()
        if shard:
            out = {k: ctx.tensor("shard_" + k).clone() for k in ("lse", "tl", "gv", "gi")}
        else:
            out = {"logits": ctx.tensor("verify_logits").clone()}
        out["tree"] = tree
        ctx.accept_and_compact()
        out["emitted"] = ctx.tensor("emitted").clone()
        ctx.destroy()
        res.append(out)
    return res


@pytest.mark.parametrize("G", [2, 5])
def test_sim_shards_stochastic_partials_match_full_rows(G):
    """The merged partials against the unsharded context's full verify-logits rows
    (same tree, fp32-verify): lse = logsumexp(l / T) to fp32 rounding, tree-token
    logits exactly, the Gumbel top-KG exactly (scores by the walk's own stream)."""
    cfg = _stoch()
    T = cfg.budget_B + cfg.resample_budget_Br + 1
    full, sh = _staged_stoch(cfg, hsd.FP32_VERIFY, G, False)
    assert all(torch.equal(x, y) for x, y in zip(full["tree"][:2], sh["tree"][:2]))
    n = full["tree"][2]
    L = full["logits"][0, :n].double()                    # [n, V]
    lse = torch.logsumexp(L / cfg.temperature, dim=-1)
    assert torch.allclose(sh["lse"][0, :n].double(), lse, rtol=0, atol=2e-5 * lse.abs().max().item())
    tok = full["tree"][0][0, :T].long()
    tl = sh["tl"][0, :n]
    for s2 in range(n):
        assert torch.equal(tl[:, s2], full["logits"][0, :n, tok[s2]])
    # Gumbel: the walk's kernel draws the same scores -> hsd_debug_gumbel gives the argmax
    assert torch.equal(sh["emitted"], full["emitted"])
    gi = sh["gi"][0, :n]
    assert (gi[:, 1:] != gi[:, :1]).all()                 # distinct candidates, sorted lists
    assert (sh["gv"][0, :n, 1:] <= sh["gv"][0, :n, :-1]).all()


def test_stochastic_shard_contract():
    """k + B_r must leave a Gumbel candidate after the largest rejected set."""
    cfg = _stoch().replace(branch_k=8, resample_budget_Br=12)
    with pytest.raises(hsd.HsdError):
        hsd.init_model(cfg, device=0, precision=hsd.FP32_VERIFY, seed=0, shard_mode=hsd.SHARD_SIM, vocab_shards=2)


@pytest.mark.parametrize("G", [2, 5])
def test_sim_shards_stochastic_bf16_tcgen05(G):
    """bf16 tcgen05 with the stochastic sharded head: both contexts verify the same
    (forced) tree after the same prefill; the merged lse within the bf16 bar of the
    unsharded rows' logsumexp; tree-token logits within it too."""
    cfg = _stoch(1024)
    full, sh = _staged_stoch(cfg, hsd.BF16, G, True, force=True)
    assert all(torch.equal(x, y) for x, y in zip(full["tree"][:2], sh["tree"][:2]))   # the forced tree
    n = full["tree"][2]
    L = full["logits"][0, :n].double()
    lse = torch.logsumexp(L / cfg.temperature, dim=-1)
    assert ((sh["lse"][0, :n].double() - lse).abs() / lse.abs().clamp_min(1)).max().item() <= 2e-2
    tok = full["tree"][0][0, :n].long()
    tl_ref = L[:, tok]                                     # [rows, tree slots]
    scale = L.abs().amax(dim=-1, keepdim=True).clamp_min(1e-6)
    assert ((sh["tl"][0, :n, :n].double() - tl_ref).abs() / scale).max().item() <= 2e-2


def test_nccl_single_rank_stochastic_in_graph():
    """The NCCL stochastic path (all-gathers of rows, tree tokens, request ids and
    records) with a one-rank group inside the step graph == the unsharded context."""
    cfg = _stoch()
    steps = 6
    base = _run(cfg, hsd.FP32_VERIFY, steps, seed=5)
    got = _run(cfg, hsd.FP32_VERIFY, steps, seed=5, shard_mode=hsd.SHARD_NCCL, vocab_shards=1, shard_rank=0,
               nccl_id=hsd.nccl_unique_id())
    assert got == base
