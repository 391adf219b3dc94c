"""Pin of the oracle's S0 draft chain and S1a one-pass logits (CPU only).

PAPER.md:206-214 (section 4.1): the draft head fuses the target's hidden state
with the next token's embedding, h_1 = TL(h_0 (+) E(t_1)), and then runs the
same transformer layer autoregressively on its own output, h_{i+1} = TL(h_i),
with no token input; PAPER.md:237-244 (section 4.2) turns the N chain states
into logits with ONE product, L = RMSNorm_f(H_chain) W_head^T.
DESIGN.md readings: R1 ((+) = W_fc [H_{j-1}; E(t_j)] at every committed
position j, draft position j, prompt position 0 skipped), R2 (TL is one decoder
layer with its own KV over positions 1..p; chain row i sits at position p+i),
R3 (the root / last committed token t_p feeds h_1), R4 (the target's final
RMSNorm and the shared W_head).

The independent side is HuggingFace `transformers`: the target's pre-norm
hidden states H come from `LlamaForCausalLM`, and TL is a one-layer
`LlamaModel` loaded with the draft weights and run over the WHOLE causal
sequence [x_1 .. x_p, h_1 .. h_{N-1}] at positions [1 .. p, p+1 .. p+N-1],
recomputed from scratch for every chain step. The oracle instead keeps a draft
KV cache across steps, feeds the verification-pass H of the accepted path, and
extends the chain one row at a time. Any off-by-one position, a wrong draft KV
row, H_j in place of H_{j-1}, or a stale pending pair changes the rows by O(1).
Steps run with the planted continuation so that m > 0 drafts are accepted and
several tokens are committed per step (the case where those mistakes show).
"""
import numpy as np
import pytest
import torch

from synth import get_config, prompts
from oracle.model import Model, rmsnorm
from oracle.table import TokenInfoTable
from oracle.engine import Engine, greedy_decode
from tests.oracle_hf import hf_model, hf_draft_layer, hf_layer_outputs, hf_prenorm_hidden


def _cfg(gqa):
    base = dict(vocab=96, hidden=48, layers=2, q_heads=4, kv_heads=2 if gqa else 4, head_dim=12, ffn=96,
                steps_N=4, branch_k=2, budget_B=8)
    if gqa:
        base["rope_theta"] = 500000.0
    return get_config("c1").replace(**base)


@pytest.mark.parametrize("gqa", [False, True])
def test_draft_chain_matches_hf_one_layer_llama(gqa):
    cfg = _cfg(gqa)
    m = Model(cfg, seed=11 if gqa else 4)
    pr = prompts(cfg, batch=1, length=10, prompt_seed=900)
    ref, _ = greedy_decode(m, pr[0], 40)
    plant = [np.concatenate([pr[0], ref])]
    e = Engine(m, TokenInfoTable(m), cfg, plant=plant, plant_rates=[1.0, 1.0, 0.9, 0.9])
    e.prefill(pr)
    hf_t, hf_d = hf_model(m), hf_draft_layer(m)
    N = cfg.steps_N
    committed_more = 0
    for _ in range(5):
        e.step()
        rec = e.trace[-1][2]
        p = rec["p"]
        toks = e.reqs[0].tokens[:p + 1]          # t_0 .. t_p committed before this step
        H = hf_prenorm_hidden(hf_t, toks[:p])    # H_0 .. H_{p-1}
        # x_j = W_fc [H_{j-1}; E(t_j)], j = 1..p (reading R1)
        X = np.stack([m.fc @ np.concatenate([H[j - 1], m.embed[toks[j]]]) for j in range(1, p + 1)])
        seq, pos = list(X), list(range(1, p + 1))
        chain = []
        for i in range(N):
            out = hf_layer_outputs(hf_d, np.stack(seq), pos)
            chain.append(out[-1])                # h_{i+1}
            seq.append(out[-1])                  # h_{i+1} = TL(h_i), no token input
            pos.append(p + i + 1)
        chain = np.stack(chain)
        np.testing.assert_allclose(rec["chain"], chain, rtol=0, atol=1e-10 * max(1.0, np.abs(chain).max()))
        # S1a: one product of the stacked chain with the shared head after the target's final norm
        with torch.no_grad():
            L = hf_t.lm_head(hf_t.model.norm(torch.from_numpy(chain))).numpy()
        np.testing.assert_allclose(rec["L"], L, rtol=0, atol=1e-10 * max(1.0, np.abs(L).max()))
        committed_more += len(rec["acc"]) > 0
    assert committed_more >= 3, "planted steps must accept drafts (m > 0) for the pin to bite"


def test_one_pass_logits_equal_iterated_gemvs():
    """the one-pass product equals the N separate lm_head GEMVs."""
    cfg = _cfg(False)
    m = Model(cfg, seed=2)
    rng = np.random.default_rng(0)
    Hc = rng.standard_normal((cfg.steps_N, cfg.hidden))
    one_pass = rmsnorm(Hc, cfg.rms_eps) @ m.head.T
    iterated = np.stack([m.logits(h) for h in Hc])
    np.testing.assert_allclose(one_pass, iterated, rtol=0, atol=1e-12)
