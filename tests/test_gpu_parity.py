"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

fp32-verify mode: identical tree topology, accepted slots,
emitted tokens and compaction, flagged decisions (oracle margin < 1e-4 x row
max |logit|) excepted; bf16 mode: logits within 2e-2 row-normwise relative
error (reading R21), identical decisions where the margin exceeds 1e-2.
"""
import numpy as np
import pytest
import torch

from synth import get_config, prompts, vocab_permutation
from oracle.model import Model, layer_tid
from oracle.table import TokenInfoTable
from oracle.engine import Engine, greedy_decode
from oracle.fp8 import round_e4m3
from tests.gpu_lockstep import Lockstep

pytestmark = pytest.mark.gpu

hsd = pytest.importorskip("paper_2602_21224_b200.hsd")


def ctx_for(cfg, precision, **kw):
    return hsd.init_model(cfg, device=0, precision=precision, **kw)


@pytest.mark.parametrize("precision", [hsd.FP32_VERIFY, hsd.BF16])
def test_weights_bit_exact(precision):
    cfg = get_config("c1")
    ctx = ctx_for(cfg, precision, seed=7)
    m = Model(cfg, seed=7, precision="fp32" if precision == hsd.FP32_VERIFY else "bf16")
    emb = ctx.tensor("embed").float().cpu().numpy()
    head = ctx.tensor("head").float().cpu().numpy()
    wqkv = ctx.tensor("layer0_wqkv").float().cpu().numpy()
    assert np.array_equal(emb, m.embed) and np.array_equal(head, m.head)
    lw = m.layers[0]
    assert np.array_equal(wqkv, np.concatenate([lw.wq, lw.wk, lw.wv]))
    ctx.destroy()


@pytest.mark.parametrize("precision,hot", [(hsd.FP32_VERIFY, 0), (hsd.BF16, 0), (hsd.FP32_VERIFY, 64)])
def test_token_info_table(precision, hot):
    cfg = get_config("c1").replace(vocab=512 if hot else 256, hot_tokens=hot)
    perm = vocab_permutation(cfg.vocab, 0)
    ctx = ctx_for(cfg, precision, seed=3, vocab_perm=perm if hot else None)
    tab = ctx.tensor("table").float().cpu().numpy()
    m = Model(cfg, seed=3, precision="fp32" if precision == hsd.FP32_VERIFY else "bf16", layers=0)
    ot = TokenInfoTable(m, hot_tokens=hot, perm=perm if hot else None)
    Vh = hot or cfg.vocab
    rank_tok = perm[:Vh] if hot else np.arange(cfg.vocab)
    tol = 1e-5 if precision == hsd.FP32_VERIFY else 1e-2
    for rk in range(0, Vh, max(1, Vh // 16)):
        ref = ot.row(int(rank_tok[rk]))[rank_tok]
        np.testing.assert_allclose(tab[rk], ref, atol=tol * np.abs(ref).max())
    ctx.destroy()


def e4m3_step(q):
    """Spacing of e4m3 values around |q| (3 mantissa bits; 2^-9 in the subnormal range)."""
    a = np.abs(q)
    return np.where(a < 2.0 ** -6, 2.0 ** -9, 2.0 ** (np.floor(np.log2(np.maximum(a, 2.0 ** -6))) - 3))


@pytest.mark.parametrize("precision,hot", [(hsd.FP32_VERIFY, 0), (hsd.BF16, 0), (hsd.BF16, 128)])
def test_token_info_table_fp8(precision, hot):
    """FP8 table (R25): per-row scale = max|row| / 448 and e4m3 codes. The GPU row
    (fp32) and the oracle row (fp64) may straddle a rounding midpoint, so codes are
    compared to within one e4m3 step and must agree almost everywhere."""
    cfg = get_config("c1").replace(vocab=512 if hot else 256, hot_tokens=hot)
    perm = vocab_permutation(cfg.vocab, 0)
    ctx = ctx_for(cfg, precision, seed=3, vocab_perm=perm if hot else None,
                  flags=hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_TABLE_FP8)
    codes = ctx.tensor("table")
    assert codes.dtype == torch.uint8
    q = codes.view(torch.float8_e4m3fn).to(torch.float64).cpu().numpy()
    sc = ctx.tensor("table_scale").cpu().numpy().astype(np.float64)
    m = Model(cfg, seed=3, precision="fp32" if precision == hsd.FP32_VERIFY else "bf16", layers=0)
    o8 = TokenInfoTable(m, hot_tokens=hot, perm=perm if hot else None, fp8=True)
    Vh = hot or cfg.vocab
    rank_tok = perm[:Vh] if hot else np.arange(cfg.vocab)
    same = total = 0
    for rk in range(0, Vh, max(1, Vh // 16)):
        tok = int(rank_tok[rk])
        r64 = o8.fp64_row(tok)[rank_tok]
        s_ref = np.abs(r64).max() / 448.0
        assert sc[rk] == pytest.approx(s_ref, rel=1e-5)
        qref = round_e4m3(r64 / s_ref)                     # the oracle's codes (R25)
        assert np.allclose(o8.row(tok)[rank_tok], qref * s_ref, rtol=1e-15, atol=0)
        assert np.all(np.abs(q[rk] - qref) <= e4m3_step(np.maximum(np.abs(q[rk]), np.abs(qref))) + 1e-12)
        assert np.max(np.abs(q[rk])) == 448.0
        same += int(np.sum(q[rk] == qref)); total += qref.size
    assert same / total > 0.99, same / total
    ctx.destroy()


def test_lockstep_c1_fp8_table():
    """The whole step with the FP8 table in fp32-verify mode: the oracle's Alg. 1
    uses its own e4m3 rows; output stays the plain greedy decode (lossless)."""
    ls, accs = run_lockstep(get_config("c1"), hsd.FP32_VERIFY, steps=12, seed=1, table_fp8=True)
    assert ls.checked["tree"] == 12 and ls.checked["accept"] == 12


def run_lockstep(cfg, precision, steps, seed=0, batch=1, planted=False, accept="greedy", hot=0, tol=None,
                 flag=None, expect_no_flags=False, tcgen05=False, table_fp8=False, extra_ctx=0,
                 block_table_seed=None, zero_table=False, resample=True, first_token=True):
    perm = vocab_permutation(cfg.vocab, 0) if hot else None
    pr = prompts(cfg, batch=batch)
    m = Model(cfg, seed=seed, precision="fp32" if precision == hsd.FP32_VERIFY else "bf16")
    table = TokenInfoTable(m, hot_tokens=hot, perm=perm, fp8=table_fp8, zero=zero_table)
    plant, rates, flags = None, None, (hsd.FLAG_RESAMPLE if resample else 0) | hsd.FLAG_FUSION
    if zero_table:
        flags |= hsd.FLAG_ZERO_TABLE
    if not first_token:
        flags |= hsd.FLAG_NO_FIRST_TOKEN
    if table_fp8:
        flags |= hsd.FLAG_TABLE_FP8
    ref = [greedy_decode(m, p, steps * (cfg.steps_N + 1) + cfg.steps_N + 4)[0] for p in pr] \
        if (planted or accept == "greedy") else None
    if planted:
        plant = [np.concatenate([p, r]) for p, r in zip(pr, ref)]
        rates = [1.0, 0.9, 0.8, 0.7, 0.7, 0.7, 0.7, 0.7]
        flags |= hsd.FLAG_PLANTED
    ctx = ctx_for(cfg, precision, seed=seed, max_batch=batch, flags=flags, accept=accept, vocab_perm=perm,
                  plant_rates=rates, max_ctx=cfg.prompt_len + steps * (cfg.steps_N + 1) + 8 + extra_ctx,
                  tcgen05=tcgen05)
    if block_table_seed is not None:        # paged KV through a scrambled page map
        bt = ctx.tensor("block_table")
        n = bt.shape[0] * bt.shape[1]
        ctx.set_block_table(np.random.default_rng(block_table_seed).permutation(n).reshape(bt.shape[0], bt.shape[1]))
    ls = Lockstep(ctx, cfg, m, table, pr, seed=seed, accept=accept, plant=plant, plant_rates=rates, perm=perm,
                  resample=resample, first_token=first_token,
                  logit_tol=tol or (1e-4 if precision == hsd.FP32_VERIFY else 2e-2),
                  flag_margin=flag or (1e-4 if precision == hsd.FP32_VERIFY else 1e-2),
                  tree_flag_margin=None if precision == hsd.FP32_VERIFY else 2 * (tol or 2e-2))
    first, ofirst = ls.start()
    if planted:
        ctx.set_plant(np.stack(plant))
    if accept == "greedy" and precision == hsd.FP32_VERIFY:
        assert list(first) == list(ofirst)
    accs = []
    for _ in range(steps):
        rep = ls.step()
        accs += [a for a, _ in rep]
    ctx.sync()
    if ref is not None and precision == hsd.FP32_VERIFY:
        for r in range(batch):
            got = ls.emitted[r]
            assert got == ref[r][:len(got)], "GPU speculative output != oracle plain greedy decode"
    if expect_no_flags:
        assert ls.flags == 0
    ctx.destroy()
    return ls, accs


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_lockstep_c1_fp32_greedy(seed):
    ls, accs = run_lockstep(get_config("c1"), hsd.FP32_VERIFY, steps=16, seed=seed, expect_no_flags=True)
    assert ls.checked["tree"] == 16 and ls.checked["accept"] == 16


def test_lockstep_c1_fp32_planted_accepts():
    ls, accs = run_lockstep(get_config("c1"), hsd.FP32_VERIFY, steps=12, planted=True)
    assert max(accs) >= 2 and ls.checked["accept"] >= 10


def test_lockstep_c1_bf16():
    ls, accs = run_lockstep(get_config("c1"), hsd.BF16, steps=10)
    assert ls.max_err["verify"] <= 2e-2 and ls.max_err["L"] <= 2e-2


def test_lockstep_c1_stochastic():
    cfg = get_config("c1").replace(accept="stochastic")
    ls, accs = run_lockstep(cfg, hsd.FP32_VERIFY, steps=12, accept="stochastic")
    assert ls.checked["accept"] >= 10


def test_lockstep_stochastic_admit_fresh_request_id():
    """Continuous batching in stochastic mode: a request admitted into a used slot
    draws its first token and its acceptance uniforms from its OWN global request
    id (hsd_admit's req_id), not the slot's earlier request's noise; the oracle
    (Engine.admit) follows the same rule, so the lockstep stays exact."""
    cfg = get_config("c1").replace(accept="stochastic", batch=2)
    pr = prompts(cfg, batch=2)
    seed = 3
    m = Model(cfg, seed=seed, precision="fp32")
    table = TokenInfoTable(m)
    ctx = ctx_for(cfg, hsd.FP32_VERIFY, seed=seed, max_batch=2, accept="stochastic",
                  flags=hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION, max_ctx=cfg.prompt_len + 12 * (cfg.steps_N + 1) + 8)
    ls = Lockstep(ctx, cfg, m, table, pr, seed=seed, accept="stochastic")
    ls.start()
    for _ in range(4):
        ls.step()
    fresh = prompts(cfg.replace(prompt_len=19), batch=6)[5]
    firsts = []
    for rid in (11, 12):                       # the same prompt under two fresh ids
        g, o = ls.admit(1, fresh, rid)
        assert g == o, f"admitted first token {g} != oracle {o} (req_id {rid})"
        firsts.append(g)
        for _ in range(3):
            ls.step()
    ctx.sync()
    assert ls.checked["accept"] >= 14, ls.checked
    ctx.destroy()


def test_lockstep_hot_pruned_gqa_batch2():
    cfg = get_config("c1").replace(vocab=512, hot_tokens=64, kv_heads=2, batch=2)
    ls, accs = run_lockstep(cfg, hsd.FP32_VERIFY, steps=8, batch=2, hot=64, planted=True)
    assert ls.checked["tree"] >= 14


def test_step_graph_equals_staged_calls():
    """hsd_step (CUDA-graph replay) emits exactly what the staged calls emit."""
    cfg = get_config("c1")
    pr = prompts(cfg)
    outs = []
    for graph in (False, True):
        stream = torch.cuda.Stream()
        ctx = ctx_for(cfg, hsd.FP32_VERIFY, seed=1, max_ctx=200)
        ctx2 = hsd.init_model(cfg, device=0, precision=hsd.FP32_VERIFY, seed=1, max_ctx=200,
                              stream=stream.cuda_stream)
        c = ctx2 if graph else ctx
        c.prefill(pr)
        em = []
        for _ in range(10):
            if graph:
                e, n = c.step_host()
            else:
                c.build_tree(); c.verify_tree(); c.accept_and_compact()
                e = c.tensor("emitted").cpu().numpy(); n = c.tensor("n_emitted").cpu().numpy()
            em += list(e[0, :n[0]])
        outs.append(em)
        assert c.kernel_launches() > 0
        ctx.destroy(); ctx2.destroy()
    assert outs[0] == outs[1]


def test_contract_violations_are_host_checked():
    cfg = get_config("c1")
    ctx = ctx_for(cfg, hsd.FP32_VERIFY, seed=0)
    with pytest.raises(hsd.HsdError) as e:
        ctx.prefill(np.array([[1, 2, 999]]))          # token outside [0, V)
    assert e.value.status == hsd.HSD_EINVAL
    with pytest.raises(hsd.HsdError) as e:
        ctx.verify_tree()                             # call order
    assert e.value.status in (hsd.HSD_ESTATE,)
    ctx.destroy()


def test_lockstep_c1_bf16_tcgen05():
    ls, accs = run_lockstep(get_config("c1"), hsd.BF16, steps=10, tcgen05=True)
    assert ls.max_err["verify"] <= 2e-2 and ls.max_err["L"] <= 2e-2


@pytest.mark.parametrize("hd,q_heads,kv_heads,prompt_len", [(64, 8, 2, 32), (64, 4, 4, 100), (128, 4, 4, 150),
                                                           (128, 8, 2, 200), (128, 8, 2, 32), (64, 16, 2, 100),
                                                           (128, 16, 2, 150), (128, 32, 2, 300)])
def test_lockstep_wide_bf16_tcgen05_planted(hd, q_heads, kv_heads, prompt_len):
    """Wider models so every GEMM spans several 128-row tiles and k-blocks of the
    tcgen05 GEMM, and the tcgen05 tree attention (hd 64/128, MHA and GQA) runs
    over several 64-key pages and key splits. GQA 16/2 and 32/2 (21 verify slots x
    8 or 16 heads = 168 / 336 (row, head) pairs, 2 / 3 q-tiles) run the CTA-pair
    (cta_group::2) attention, including an all-padding follower tile."""
    cfg = get_config("c1").replace(hidden=512, q_heads=q_heads, kv_heads=kv_heads, head_dim=hd, ffn=1024,
                                   vocab=1024, layers=2, steps_N=5, branch_k=3, budget_B=16,
                                   prompt_len=prompt_len)
    ls, accs = run_lockstep(cfg, hsd.BF16, steps=6, tcgen05=True, planted=True)
    assert ls.max_err["verify"] <= 2e-2 and max(accs) >= 2


@pytest.mark.parametrize("variant", ["zero_table", "no_resample"])
def test_lockstep_ablation_variants(variant):
    """NEXT-1 ablation toggles (Table 4 / Fig. 12) in full lockstep with the
    oracle's same variant, fp32-verify, planted acceptance: token info off
    (HSD_FLAG_ZERO_TABLE: Alg. 1 on the draft logits alone, Fig. 5a) and Alg. 2
    re-sampling off. Every variant stays the oracle's plain greedy decode (lossless)."""
    kw = {"zero_table": dict(zero_table=True), "no_resample": dict(resample=False)}[variant]
    ls, accs = run_lockstep(get_config("c1"), hsd.FP32_VERIFY, steps=10, planted=True, **kw)
    assert ls.checked["tree"] >= 9 and ls.checked["accept"] >= 9 and max(accs) >= 2


def _stream_vs_oracle(flags, steps=12, check_first_draft=False, cfg=None, rates=None, **engine_kw):
    """GPU hsd_step stream vs an oracle Engine that runs the same variant through the
    whole decode (no per-step restart: variants whose draft state depends on the step
    history); planted greedy, fp32-verify. Returns (GPU tokens, oracle engine)."""
    cfg = cfg or get_config("c1")
    pr = prompts(cfg)
    m = Model(cfg, seed=0, precision="fp32")
    table = TokenInfoTable(m)
    ref = greedy_decode(m, pr[0], steps * (cfg.steps_N + 1) + 4)[0]
    plant = [np.concatenate([pr[0], ref])]
    rates = rates or [1.0, 0.9, 0.8, 0.7, 0.7, 0.7, 0.7, 0.7]
    ctx = ctx_for(cfg, hsd.FP32_VERIFY, seed=0, flags=flags | hsd.FLAG_PLANTED, plant_rates=rates,
                  max_ctx=cfg.prompt_len + (steps + 2) * (cfg.steps_N + 1) + 8)
    ctx.prefill(pr)
    ctx.set_plant(np.stack(plant))
    e = Engine(m, table, cfg, seed=0, plant=plant, plant_rates=rates, **engine_kw)
    first = e.prefill(pr)
    got = [int(ctx.tensor("root_tok").cpu()[0])]
    assert got == first
    for i in range(steps):
        if check_first_draft and i == 0:     # the variant's draft arithmetic itself (step-1 logits)
            ctx.build_tree()
            Lg = ctx.tensor("draft_logits").cpu().numpy()[0].astype(np.float64)
            ctx.verify_tree()
            ctx.accept_and_compact()
            g = [int(t) for t in ctx.tensor("emitted").cpu().numpy()[0, :int(ctx.tensor("n_emitted").cpu()[0])]]
        else:
            em, n = ctx.step_host()
            g = [int(t) for t in em[0, :n[0]]]
        o = e.step()[0]
        if check_first_draft and i == 0:
            Lo = e.trace[-1][2]["L"]
            assert np.max(np.abs(Lg - Lo)) <= 1e-4 * np.max(np.abs(Lo)), "step-1 draft logits differ"
        assert g == o, f"step {i + 1} tokens differ: gpu {g} oracle {o}"
        got += g
    ctx.sync()
    assert got == ref[:len(got)], "GPU output != plain greedy decode"
    ctx.destroy()
    return got, e


def test_no_first_token_variant():
    """"w/o first token" (Table 4; HSD_FLAG_NO_FIRST_TOKEN, R26): the root
    pair enters the draft as W_fc [H; 0]. Step-1 draft logits match the oracle's
    variant (1e-4), every step emits the oracle's tokens, output lossless."""
    got, e = _stream_vs_oracle(hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_NO_FIRST_TOKEN, check_first_draft=True,
                               first_token=False)
    # the variant changes the draft itself (not a no-op)
    cfg = get_config("c1")
    m = e.m
    e_on = Engine(m, TokenInfoTable(m), cfg, seed=0)
    e_on.prefill(prompts(cfg))
    e_on.step()
    assert np.max(np.abs(e_on.trace[-1][2]["L"] - e.trace[0][2]["L"])) > 1e-3


def test_token_ar_draft_mode():
    """NEXT-2 token-level AR draft (HSD_FLAG_TOKEN_AR, R27): per-step lm_head GEMV +
    argmax + fc feeding back the draft's own token. Step-1 draft logits match the
    oracle's token-AR chain (1e-4), every step emits the oracle's tokens, lossless."""
    _stream_vs_oracle(hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_TOKEN_AR, check_first_draft=True,
                      draft_mode="token_ar")


def test_fusion_off_dedicated_verify_pass():
    """Re-sampling WITHOUT verification fusion (HSD_FLAG_RESAMPLE alone): the
    Alg. 2 tree is verified by its own target pass inside the step. Per step the GPU
    emits exactly the oracle's tokens (Engine(fusion=False) runs the same extra pass),
    the stream is the plain greedy decode, and extra passes really emit tokens."""
    # a deeper draft and lower planted rates so that Alg. 2 (N - m - 1 > r) really fires
    cfg = get_config("c1").replace(steps_N=6, budget_B=12)
    got, e = _stream_vs_oracle(hsd.FLAG_RESAMPLE, steps=14, cfg=cfg, rates=[0.9, 0.5, 0.5, 0.5, 0.5, 0.5],
                               fusion=False)
    assert sum("acc2" in rec for _, _, rec in e.trace) > 0


def test_lockstep_permuted_block_table():
    """Paged KV with a scrambled block table (hsd_set_block_table): every K / V read
    and write -- prefill, qkv_rope_kv, the SIMT and tcgen05 tree attention, the draft
    layer, compaction -- goes through the page map. fp32-verify stays the oracle's
    plain greedy decode; bf16 tcgen05 (GQA hd 128, multi-page prompts, 2 requests)
    stays in lockstep, compacted KV rows read back through the same map."""
    ls, accs = run_lockstep(get_config("c1").replace(batch=2), hsd.FP32_VERIFY, steps=8, batch=2, planted=True,
                            block_table_seed=5)
    assert ls.checked["accept"] >= 14 and max(accs) >= 2
    cfg = get_config("c1").replace(hidden=512, q_heads=8, kv_heads=2, head_dim=128, ffn=1024, vocab=1024,
                                   layers=2, steps_N=5, branch_k=3, budget_B=16, prompt_len=200, batch=2)
    ls, accs = run_lockstep(cfg, hsd.BF16, steps=5, batch=2, tcgen05=True, planted=True, block_table_seed=9)
    assert ls.max_err["verify"] <= 2e-2 and max(accs) >= 2


def test_block_table_contract():
    cfg = get_config("c1")
    ctx = ctx_for(cfg, hsd.FP32_VERIFY, seed=0)
    bt = ctx.tensor("block_table").cpu().numpy()
    assert np.array_equal(bt.ravel(), np.arange(bt.size))          # identity by default
    bad = bt.copy()
    bad.flat[0] = bad.flat[1]                                       # not a permutation
    with pytest.raises(hsd.HsdError) as e:
        ctx.set_block_table(bad)
    assert e.value.status == hsd.HSD_EINVAL
    ctx.destroy()


def test_lockstep_attention_capacity_far_above_context():
    """Key splits are sized on the host from the context CAPACITY (max_ctx) but, in the
    latency-bound regime, divide the chunks each tile really sees on the device
    (attention_tc.cu, P.dyn): a 4k-key capacity over a ~100-key context leaves most
    capacity splits empty. MHA hd 128 and GQA hd 64, planted acceptance."""
    for hd, qh, kvh in [(128, 4, 4), (64, 8, 2)]:
        cfg = get_config("c1").replace(hidden=512, q_heads=qh, kv_heads=kvh, head_dim=hd, ffn=1024, vocab=1024,
                                       layers=2, steps_N=5, branch_k=3, budget_B=16, prompt_len=100)
        ls, accs = run_lockstep(cfg, hsd.BF16, steps=5, tcgen05=True, planted=True, extra_ctx=4096)
        assert ls.max_err["verify"] <= 2e-2 and max(accs) >= 2


def test_attention_cluster_reduction_all_widths():
    """Key splits merged inside a thread-block cluster over DSMEM (attention_tc.cu):
    by default only S = 2 takes that path, so re-run the multi-split tcgen05
    lockstep cases in a fresh process with clusters of up to 8 CTAs."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, HSD_ATTN_CLUSTER_MAX="8")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k", "tcgen05 and not cluster"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
