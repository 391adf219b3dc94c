"""Pins for oracle/accept.py and oracle/engine.py (CPU only).

- greedy losslessness: speculative output == plain greedy decode, token for
  token, over a seed x (N, k, B) x resample/fusion grid (the paper's
  implicit correctness contract at T = 0);
- compaction: committed KV == the KV a plain decode writes;
- stochastic acceptance preserves the target distribution (chi-square).
"""
import math
import numpy as np
import pytest
from scipy.stats import chi2

from synth import get_config, prompts
from oracle.model import Model
from oracle.table import TokenInfoTable
from oracle.engine import Engine, greedy_decode
from oracle import tree as T
from oracle.accept import greedy_walk, stochastic_walk, softmax_T


def tiny(**kw):
    base = dict(vocab=64, hidden=32, layers=1, q_heads=2, kv_heads=1, head_dim=16, ffn=64,
                prompt_len=8, max_new=24)
    base.update(kw)
    return get_config("c1").replace(**base)


GRID = [(1, 1, 4), (2, 2, 4), (3, 2, 6), (4, 3, 12), (5, 4, 16)]


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("N,k,B", GRID)
@pytest.mark.parametrize("resample,fusion", [(True, True), (True, False), (False, False)])
def test_greedy_lossless_grid(seed, N, k, B, resample, fusion):
    cfg = tiny(steps_N=N, branch_k=k, budget_B=B)
    m = Model(cfg, seed=seed)
    pr = prompts(cfg, batch=2, length=8, prompt_seed=77 + seed)
    ref = [greedy_decode(m, p, cfg.max_new + 2 * N + 2)[0] for p in pr]
    # planted continuation so that drafts are really accepted
    plant = [np.concatenate([p, r]) for p, r in zip(pr, ref)]
    e = Engine(m, TokenInfoTable(m), cfg, seed=seed, resample=resample, fusion=fusion,
               plant=plant, plant_rates=[0.9, 0.8, 0.7, 0.7, 0.7])
    out = e.decode(pr, cfg.max_new)
    for o, r in zip(out, ref):
        assert o == r[:cfg.max_new]
    acc = [len(rec["acc"]) for _, _, rec in e.trace]
    assert max(acc) >= min(N, 2)  # the planted path really is accepted
    extra = 0
    for _, _, rec in e.trace:
        lin = rec["lin"]
        assert lin["T"] <= B + (cfg.resample_budget_Br if fusion else 0) + 1
        n2 = len(rec["acc2"]) + 1 if "acc2" in rec else 0    # fusion off: the dedicated extra verify
        assert len(rec["emitted"]) == len(rec["acc"]) + 1 + n2
        assert len(rec["emitted"]) <= N + 1
        extra += "acc2" in rec
    if resample and not fusion and N >= 3:
        assert extra > 0            # the re-sampled tree was really verified on its own


def test_unplanted_random_weights_lossless_c1():
    cfg = get_config("c1")
    m = Model(cfg, seed=0)
    pr = prompts(cfg)
    out = Engine(m, TokenInfoTable(m), cfg).decode(pr, 32)
    assert out[0] == greedy_decode(m, pr[0], 32)[0]


def test_compaction_equals_plain_decode_kv():
    """After every step the committed target KV [0, p) equals, bit for bit, the
    KV rows a plain greedy decode of the same tokens writes."""
    cfg = tiny(steps_N=4, branch_k=2, budget_B=8)
    m = Model(cfg, seed=5)
    pr = prompts(cfg, batch=1, length=8)
    ref, _ = greedy_decode(m, pr[0], 40)
    plant = [np.concatenate([pr[0], ref])]
    e = Engine(m, TokenInfoTable(m), cfg, plant=plant, plant_rates=[1.0, 1.0, 0.8, 0.8])
    e.prefill(pr)
    for _ in range(6):
        e.step()
    q = e.reqs[0]
    p = len(q.tokens) - 1
    _, kv_ref = greedy_decode(m, pr[0], p - len(pr[0]) + 1)
    for l in range(m.n_layers):
        assert len(q.kv[l][0]) == p
        for j in range(p):
            assert np.array_equal(q.kv[l][0][j], kv_ref[l][0][j])
            assert np.array_equal(q.kv[l][1][j], kv_ref[l][1][j])
    # compaction indices = accepted slots, strictly increasing depth-major
    for _, _, rec in e.trace:
        acc = rec["acc"]
        assert all(rec["lin"]["depth"][s] == j + 1 for j, s in enumerate(acc))
        assert all(s >= j + 1 for j, s in enumerate(acc))


def test_resampled_tree_is_fused_and_rooted_at_bonus():
    cfg = tiny(steps_N=5, branch_k=2, budget_B=6)
    m = Model(cfg, seed=8)
    e = Engine(m, TokenInfoTable(m), cfg)
    pr = prompts(cfg, batch=1, length=8)
    e.prefill(pr)
    e.step()
    rec = e.trace[-1][2]
    if len(rec["acc"]) < cfg.steps_N - 1 - cfg.resample_threshold_r:
        pend = rec["pending"]
        assert pend is not None and pend[0]["tok"] == rec["bonus"]
        assert len(pend) == 1 + cfg.resample_budget_Br
        e.step()
        lin = e.trace[-1][2]["lin"]
        assert lin["tok"][0] == rec["bonus"]
        assert set(T.paths(pend)) <= set(T.paths(T.fuse(e.trace[-1][2]["fresh"], pend)))


# ---------------------------------------------------------------------------
# Acceptance walks.
# ---------------------------------------------------------------------------

def toy_tree():
    # root(0) -> children tokens 3, 5, 9 ; child tok 3 -> children 1, 2
    nodes = [T._node(7, -1, 0, 1, 0)]
    for t, lj in [(3, -0.5), (5, -1.0), (9, -2.0)]:
        nodes.append(T._node(t, 0, 1, math.exp(lj), lj))
    for t, lj in [(1, -0.7), (2, -0.9)]:
        nodes.append(T._node(t, 1, 2, math.exp(lj), lj))
    return T.linearize(nodes)


def test_greedy_walk_semantics():
    lin = toy_tree()
    V = 16
    lg = np.zeros((lin["T"], V))
    lg[0, 3] = 5            # root: argmax 3 -> accept child slot 1
    lg[1, 2] = 4            # tok-3 node: argmax 2 -> accept
    lg[lin["T"] - 1, 11] = 1  # tok-2 node (leaf): bonus 11
    acc, bonus = greedy_walk(lin, lg)
    assert [int(lin["tok"][s]) for s in acc] == [3, 2] and bonus == 11
    lg[0, 3] = 0; lg[0, 4] = 9   # argmax 4 is not a child -> stop, bonus 4
    acc, bonus = greedy_walk(lin, lg)
    assert acc == [] and bonus == 4


def test_stochastic_walk_preserves_target_distribution():
    """Every emitted token is distributed as the target's softmax (chi-square,
    alpha = 0.01), first token and second-given-first (reading R13)."""
    lin = toy_tree()
    V = 16
    rng = np.random.default_rng(0)
    lg = rng.standard_normal((lin["T"], V)) * 1.5
    lg[0, 3] += 1.0; lg[1, 1] += 1.0
    n = 40000
    first = np.zeros(V)
    second = np.zeros(V)
    for i in range(n):
        acc, bonus = stochastic_walk(lin, lg, 1.0, 0, 0, 0,
                                     uniform=lambda s, r: rng.random(),
                                     gumbel=lambda s: rng.random(V))
        toks = [int(lin["tok"][s]) for s in acc] + [bonus]
        first[toks[0]] += 1
        if acc and acc[0] == 1:     # went through the tok-3 node: 2nd token ~ its p
            second[toks[1]] += 1
    for counts, p in [(first, softmax_T(lg[0], 1.0)), (second, softmax_T(lg[1], 1.0))]:
        exp = p * counts.sum()
        stat = float(((counts - exp) ** 2 / exp).sum())
        assert stat < chi2.ppf(0.99, V - 1), stat


def test_stochastic_low_temperature_is_greedy():
    lin = toy_tree()
    rng = np.random.default_rng(3)
    lg = rng.standard_normal((lin["T"], 16)) * 3
    lg[0, 3] = 10
    g = greedy_walk(lin, lg)
    for s in range(20):
        st = stochastic_walk(lin, lg, 1e-4, s, 0, 1)
        assert st == g


def test_admit_is_lossless_and_uses_the_new_request_id():
    """Engine.admit (continuous batching around the path): the admitted
    slot decodes its new prompt losslessly while the other slot continues
    untouched, and its random streams use the NEW global request id (stochastic
    first token = the Gumbel-max sample under that id; a different id gives
    independent noise)."""
    cfg = tiny(steps_N=3, branch_k=2, budget_B=6)
    m = Model(cfg, seed=4)
    table = TokenInfoTable(m)
    pr = prompts(cfg, batch=3, length=8, prompt_seed=5)
    e = Engine(m, table, cfg)
    e.prefill(pr[:2])
    outs = [[q.tokens[-1]] for q in e.reqs]
    for _ in range(3):
        for o, new in zip(outs, e.step()):
            o.extend(new)
    t1 = e.admit(1, pr[2], req_id=9)
    assert e.req_ids == [0, 9]
    new_out = [t1]
    for _ in range(4):
        a, b = e.step()
        outs[0].extend(a)
        new_out.extend(b)
    assert outs[0] == greedy_decode(m, pr[0], len(outs[0]))[0]
    assert new_out == greedy_decode(m, pr[2], len(new_out))[0]
    # stochastic: the admitted first token is the Gumbel-max sample of ITS id
    from oracle.philox import gumbel_uniforms
    from oracle.accept import gumbel_argmax
    es = Engine(m, table, cfg.replace(accept="stochastic"), seed=1, accept="stochastic", temperature=1.0)
    es.prefill(pr[:2])
    kv = [([], []) for _ in range(m.n_layers)]          # the prompt's last-position logits, plain
    for pos, t in enumerate(pr[2]):
        _, logits, rows = m.target_one(int(t), pos, kv)
        for l, (k, v) in enumerate(rows):
            kv[l][0].append(k); kv[l][1].append(v)
    picks = {rid: es.admit(1, pr[2], req_id=rid) for rid in (5, 6, 7, 8)}
    for rid, t in picks.items():
        assert t == gumbel_argmax(logits, 1.0, gumbel_uniforms(1, rid, 0, 0, cfg.vocab))[0]


@pytest.mark.parametrize("seed", [0, 1])
def test_no_first_token_variant_lossless_and_distinct(seed):
    """R26 ("w/o first token", Table 4): the root pair enters the draft as W_fc [H; 0].
    The draft changes (different one-pass logits) but the output stays the plain
    greedy decode -- losslessness does not depend on the draft."""
    cfg = tiny(steps_N=3, branch_k=2, budget_B=6)
    m = Model(cfg, seed=seed)
    pr = prompts(cfg, batch=1, length=8, prompt_seed=40 + seed)
    ref = greedy_decode(m, pr[0], cfg.max_new + 8)[0]
    e = Engine(m, TokenInfoTable(m), cfg, first_token=False)
    out = e.decode(pr, cfg.max_new)
    assert out[0] == ref[:cfg.max_new]
    e_on = Engine(m, TokenInfoTable(m), cfg)
    e_on.prefill(pr)
    e_on.step()
    assert np.max(np.abs(e.trace[0][2]["L"] - e_on.trace[0][2]["L"])) > 1e-6
    # the input of the root pair is W_fc [H; 0]
    H = np.arange(cfg.hidden, dtype=np.float64) / cfg.hidden
    assert np.allclose(m.draft_input(H, 3, with_token=False), m.fc[:, :cfg.hidden] @ H)


def test_token_ar_draft_mode_lossless_and_distinct():
    """R27 (NEXT-2): the token-level AR draft feeds back its own top-1
    token, x_{i+1} = W_fc [h_i ; E(argmax l_i)]. A different draft (different L rows
    after the first), the same lossless output."""
    cfg = tiny(steps_N=4, branch_k=2, budget_B=8)
    m = Model(cfg, seed=3)
    pr = prompts(cfg, batch=1, length=8, prompt_seed=9)
    ref = greedy_decode(m, pr[0], cfg.max_new + 8)[0]
    e = Engine(m, TokenInfoTable(m), cfg, draft_mode="token_ar")
    assert e.decode(pr, cfg.max_new)[0] == ref[:cfg.max_new]
    e_h = Engine(m, TokenInfoTable(m), cfg)
    e_h.prefill(pr)
    e_h.step()
    L_tok, L_hid = e.trace[0][2]["L"], e_h.trace[0][2]["L"]
    assert np.allclose(L_tok[0], L_hid[0])              # h_1 is the same draft prefill output
    assert np.max(np.abs(L_tok[1:] - L_hid[1:])) > 1e-6
