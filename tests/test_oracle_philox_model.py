"""Pins for oracle/philox.py and oracle/model.py (CPU only)."""
import numpy as np
import pytest
import torch

from synth import get_config
from oracle.philox import philox4x32_10, uniform_weights, linear_scale, round_bf16, raw_stream
from oracle.model import Model, rmsnorm
from oracle.engine import greedy_decode
from tests.oracle_hf import hf_model, hf_logits_and_hidden

# Random123 kat_vectors, philox4x32 R=10: (ctr0..3, key0..1) -> out0..3
KAT = [
    ((0, 0, 0, 0, 0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 6, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344, 0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("inp,out", KAT)
def test_philox_known_answer(inp, out):
    got = tuple(int(x) for x in philox4x32_10(*inp))
    assert got == out


def test_weight_stream_layout_and_range():
    w = uniform_weights(7, 3, (5, 6), linear_scale(6))
    x = raw_stream(7, 3, 30)
    s = np.float32(np.sqrt(np.float32(3.0) / np.float32(6)))
    u = (x >> 8).astype(np.float64) * 2.0 ** -24
    # w = s*(2u-1) with a single float32 rounding of the product
    assert np.array_equal(w.reshape(-1), (np.float32(s) * (2 * u - 1).astype(np.float32)).astype(np.float32))
    assert np.all(np.abs(w) <= s)
    # statistical check (SPEC.md:76 analogue): mean of 1e5 draws near 0
    big = uniform_weights(1, 1, (100000,), np.float32(1.0))
    assert abs(big.mean()) < 3 * np.sqrt(1 / 3 / 1e5)


def test_round_bf16_matches_torch():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 10
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(round_bf16(x), ref)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("gqa", [False, True])
def test_target_forward_matches_hf_llama(precision, gqa):
    """The oracle's Llama forward == transformers' LlamaForCausalLM (an
    independent implementation) on the same weights, float64."""
    cfg = get_config("c1")
    if gqa:
        cfg = cfg.replace(kv_heads=2, rope_theta=500000.0)
    m = Model(cfg, seed=3, precision=precision, with_draft=False, with_table_factors=False)
    hf = hf_model(m)
    toks = [5, 77, 200, 13, 13, 99, 0, 255, 31, 64]
    ref_logits, ref_normed = hf_logits_and_hidden(hf, toks)
    kv = [([], []) for _ in range(m.n_layers)]
    for pos, t in enumerate(toks):
        H, logits, rows = m.target_one(t, pos, kv)
        for l, (k, v) in enumerate(rows):
            kv[l][0].append(k); kv[l][1].append(v)
        # HF runs with float64 RoPE angles and RMSNorm (tests/oracle_hf.py), so the
        # two agree to rounding; any real mistake is O(1).
        np.testing.assert_allclose(logits, ref_logits[pos], rtol=0, atol=1e-10)
        np.testing.assert_allclose(rmsnorm(H, cfg.rms_eps), ref_normed[pos], rtol=0, atol=1e-10)


def test_greedy_decode_matches_hf_generate():
    cfg = get_config("c1")
    m = Model(cfg, seed=1, with_draft=False, with_table_factors=False)
    hf = hf_model(m)
    prompt = [1, 2, 3, 4, 250]
    ours, _ = greedy_decode(m, prompt, 12)
    ids = list(prompt)
    for _ in range(12):
        lg, _ = hf_logits_and_hidden(hf, ids)
        ids.append(int(np.argmax(lg[-1])))
    assert ours == ids[len(prompt):]


def test_one_pass_logits_equal_iterated_gemv():
    """[l_1..l_k] = [h_1..h_k]^T W_head (one GEMM) equals k GEMVs."""
    cfg = get_config("c1")
    m = Model(cfg, seed=2, with_draft=False, with_table_factors=False)
    Hs = np.random.default_rng(0).standard_normal((5, cfg.hidden))
    one_pass = rmsnorm(Hs, cfg.rms_eps) @ m.head.T
    for i in range(5):
        np.testing.assert_allclose(one_pass[i], m.logits(Hs[i]), atol=1e-12)


def test_tree_verify_equals_per_path_hf_forward():
    """Tree attention pin: each tree slot's logits equal an
    independent causal forward (HF Llama) of prompt + the slot's root path."""
    from synth import prompts
    from oracle.table import TokenInfoTable
    from oracle.engine import Engine
    from oracle import tree as T
    cfg = get_config("c1").replace(kv_heads=2)
    m = Model(cfg, seed=6)
    hf = hf_model(m)
    pr = prompts(cfg, batch=1, length=12)
    e = Engine(m, TokenInfoTable(m), cfg)
    e.prefill(pr)
    q = e.reqs[0]
    rng = np.random.default_rng(1)
    L = rng.standard_normal((3, cfg.vocab))
    lin = T.linearize(T.prune(T.build_subtree(L, q.tokens[-1], 3, 3, e.table), 9))
    H, logits, _ = e.verify(q, lin)
    paths = []
    for u in range(lin["T"]):
        path, a = [], u
        while a > 0:
            path.append(int(lin["tok"][a])); a = int(lin["par"][a])
        paths.append(path[::-1])
    for u in range(lin["T"]):
        seq = list(q.tokens) + paths[u]
        ref, _ = hf_logits_and_hidden(hf, seq)
        np.testing.assert_allclose(logits[u], ref[-1], atol=1e-5)


def test_stochastic_engine_runs_and_is_reproducible():
    from synth import prompts
    from oracle.table import TokenInfoTable
    from oracle.engine import Engine
    cfg = get_config("c1").replace(accept="stochastic", max_new=12)
    m = Model(cfg, seed=0)
    pr = prompts(cfg)
    a = Engine(m, TokenInfoTable(m), cfg, seed=3).decode(pr, 12)
    b = Engine(m, TokenInfoTable(m), cfg, seed=3).decode(pr, 12)
    c = Engine(m, TokenInfoTable(m), cfg, seed=4).decode(pr, 12)
    assert a == b and a != c
    assert all(0 <= t < cfg.vocab for t in a[0])


def test_uniform_rows_equals_full_tensor_rows():
    from oracle.philox import uniform_rows
    full = uniform_weights(3, 9, (37, 23), linear_scale(23))
    rows = [0, 5, 36, 17]
    np.testing.assert_array_equal(uniform_rows(3, 9, 23, linear_scale(23), rows), full[rows].astype(np.float64))
    fb = round_bf16(full)
    np.testing.assert_array_equal(uniform_rows(3, 9, 23, linear_scale(23), rows, "bf16"), fb[rows].astype(np.float64))


def test_sampling_uniform_exact_in_fp32_and_open():
    """unit_open over all 2^23 distinct values: strictly inside (0, 1), equal to
    its float32 rounding (the GPU computes it in fp32), strictly increasing, and
    -log(-log u) finite everywhere (reading R13's Gumbel-max)."""
    from oracle.philox import unit_open
    k = np.arange(2 ** 23, dtype=np.uint32)
    u = unit_open(k << np.uint32(9))
    assert u.min() > 0.0 and u.max() < 1.0
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    assert np.all(np.diff(u) > 0)
    assert np.all(np.isfinite(-np.log(-np.log(u))))
    # the low 9 bits of the word do not matter; extremes of the 32-bit word
    assert unit_open(np.uint32(0xFFFFFFFF)) == 1.0 - 2.0 ** -24
    assert unit_open(np.uint32(0)) == 2.0 ** -24
