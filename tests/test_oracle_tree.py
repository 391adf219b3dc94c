"""Pins for oracle/tree.py (Alg. 1, prune, Alg. 2, fusion, linearisation) and
oracle/table.py. CPU only."""
import math
import itertools
import numpy as np
import pytest
from scipy.special import logsumexp as sp_logsumexp

from synth import get_config, vocab_permutation
from oracle import tree as T
from oracle.table import ExplicitTable, TokenInfoTable, table_bytes
from oracle.model import Model

MODEL, TRAINING, INFERENCE, SERVER, SPEED, OPTIMIZATION, QUANT, ACCURACY, METHOD = range(9)


def joint(nodes, tokpath):
    paths = T.paths(nodes)
    i = paths.index(tuple(tokpath))
    return math.exp(nodes[i]["lj"])


def probs_row(V, d, rest):
    p = np.full(V, rest)
    for t, v in d.items():
        p[t] = v
    assert abs(p.sum() - 1) < 1e-12
    return np.log(p)


# ---------------------------------------------------------------------------
# Fig. 5 worked example (PAPER.md:299 beam sampling; :303 token-info sampling;
# :385 re-sampling).
# ---------------------------------------------------------------------------

def test_fig5a_beam_sampling_order():
    """'training' (0.6) -> 'server' 0.6x0.7 = 0.42 -> 'inference'
    0.3 -> 'optimization' 0.6x0.7x0.7 = 0.294; beam width 2, no token info."""
    V = 6
    L = np.stack([probs_row(V, {TRAINING: 0.6, INFERENCE: 0.3}, 0.025),
                  probs_row(V, {SERVER: 0.7, SPEED: 0.15}, 0.0375),
                  probs_row(V, {OPTIMIZATION: 0.7, SPEED: 0.1}, 0.05)])
    tree = T.build_subtree(L, MODEL, 2, 3, ExplicitTable(V))
    order = []
    for B in range(1, 5):
        kept = T.prune(tree, B)
        new = set(T.paths(kept)) - set(order) - {()}
        assert len(new) == 1
        order.append(new.pop())
    assert order == [(TRAINING,), (TRAINING, SERVER), (INFERENCE,), (TRAINING, SERVER, OPTIMIZATION)]
    assert joint(tree, [TRAINING]) == pytest.approx(0.6, abs=1e-12)
    assert joint(tree, [TRAINING, SERVER]) == pytest.approx(0.42, abs=1e-12)
    assert joint(tree, [INFERENCE]) == pytest.approx(0.3, abs=1e-12)
    assert joint(tree, [TRAINING, SERVER, OPTIMIZATION]) == pytest.approx(0.294, abs=1e-12)


def fig5b_instance():
    V = 9
    tab = ExplicitTable(V, {
        MODEL: probs_row(V, {TRAINING: 0.6, INFERENCE: 0.3}, 0.1 / 7),
        TRAINING: probs_row(V, {SERVER: 0.7, SPEED: 0.1}, 0.2 / 7),
        INFERENCE: probs_row(V, {SPEED: 0.9}, 0.1 / 8),
        QUANT: probs_row(V, {ACCURACY: 0.5, METHOD: 0.4}, 0.1 / 7),
    })
    L = np.zeros((3, V))          # raw logits carry no preference: the table decides
    return V, tab, L


def test_fig5b_token_info_sampling():
    """top-2 of Logits 1' = 0.6 / 0.3; 'server' = 0.6x0.7 = 0.42;
    the frontier continues with (server, speed)."""
    V, tab, L = fig5b_instance()
    tree = T.build_subtree(L, MODEL, 2, 2, tab)
    d1 = [(n["tok"], n["prob"]) for n in tree if n["depth"] == 1]
    assert [t for t, _ in d1] == [TRAINING, INFERENCE]
    assert [p for _, p in d1] == pytest.approx([0.6, 0.3], abs=1e-12)
    assert joint(tree, [TRAINING, SERVER]) == pytest.approx(0.42, abs=1e-12)
    tree3 = T.build_subtree(L, MODEL, 2, 3, tab)
    expanded = {T.paths(tree3)[n["par"]] for n in tree3 if n["depth"] == 3}
    assert expanded == {(TRAINING, SERVER), (INFERENCE, SPEED)}


def test_fig5c_resampling_from_bonus_token():
    """both depth-1 drafts rejected, bonus 'quantization'; its
    token info on Logits 2 gives 'accuracy' and 'method'; each seeds Logits 3."""
    V, tab, L = fig5b_instance()
    rs = T.resample(L[1:], QUANT, 2, 1, tab)
    assert rs[0]["tok"] == QUANT
    assert [n["tok"] for n in rs if n["depth"] == 1] == [ACCURACY, METHOD]
    assert max(n["depth"] for n in rs) == 2
    # Alg. 2 else-branch: N_remain <= r -> single node
    single = T.resample(L[2:], QUANT, 2, 1, tab)
    assert len(single) == 1 and single[0]["tok"] == QUANT and single[0]["lj"] == 0.0


# ---------------------------------------------------------------------------
# Independent brute-force builder (no queue, path tuples, scipy logsumexp).
# ---------------------------------------------------------------------------

def brute_force_tree(L, root, k, N, table):
    """Level-synchronous enumeration of Alg. 1's semantics written without
    the oracle's data structures: returns {path: logjoint}."""
    out = {(): 0.0}
    frontier = [()]
    for i in range(N):
        cands = []
        for path in frontier:
            last = path[-1] if path else root
            v = np.asarray(L[i]) + table.row(last)
            lp = v - sp_logsumexp(v)
            best = sorted(range(len(v)), key=lambda e: (-v[e], e))[:k]
            for e in best:
                cands.append((path + (e,), out[path] + lp[e]))
        for pth, lj in cands:
            out[pth] = lj
        frontier = [pth for pth, lj in sorted(cands, key=lambda c: (-c[1], c[0][-1]))[:k]]
    return out


@pytest.mark.parametrize("seed", range(40))
def test_alg1_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(4, 9)); N = int(rng.integers(1, 4)); k = int(rng.integers(1, min(V, 4) + 1))
    L = rng.standard_normal((N, V)) * 2
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    root = int(rng.integers(V))
    tree = T.build_subtree(L, root, k, N, tab)
    bf = brute_force_tree(L, root, k, N, tab)
    got = {p: n["lj"] for p, n in zip(T.paths(tree), tree)}
    assert set(got) == set(bf)
    for p in bf:
        assert got[p] == pytest.approx(bf[p], abs=1e-10)
    # node count = 1 + k + (N-1)k^2 (SPEC.md:381 bound, attained when V >= k)
    assert len(tree) == 1 + k + (N - 1) * k * k if N >= 1 else 1
    # jointProb = product of probs along the path
    for n in tree[1:]:
        assert n["lj"] == pytest.approx(tree[n["par"]]["lj"] + math.log(n["prob"]), abs=1e-12)


def test_k1_is_greedy_chain():
    rng = np.random.default_rng(5)
    V, N = 12, 5
    L = rng.standard_normal((N, V))
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    tree = T.build_subtree(L, 3, 1, N, tab)
    assert len(tree) == N + 1
    prev = 3
    for i in range(N):
        assert tree[i + 1]["par"] == i
        assert tree[i + 1]["tok"] == int(np.argmax(L[i] + tab.row(prev)))
        prev = tree[i + 1]["tok"]


def test_zero_table_is_beam_tree():
    """with a zero table Alg. 1 is the beam-sampling tree (Fig. 5a):
    every node at step i conditions on the same softmax(l_i)."""
    rng = np.random.default_rng(9)
    V, N, k = 7, 3, 3
    L = rng.standard_normal((N, V))
    tree = T.build_subtree(L, 0, k, N, ExplicitTable(V))
    for n in tree[1:]:
        i = n["depth"] - 1
        assert n["prob"] == pytest.approx(float(np.exp(L[i][n["tok"]] - sp_logsumexp(L[i]))), abs=1e-12)
    # siblings of every expanded node are the same top-k tokens of l_i
    for u in range(len(tree)):
        kids = [n["tok"] for n in tree if n["par"] == u]
        if kids:
            i = tree[u]["depth"]
            assert kids == list(np.argsort(-L[i], kind="stable")[:k])


@pytest.mark.parametrize("seed", range(30))
def test_prune_is_sort_all_and_connected(seed):
    rng = np.random.default_rng(100 + seed)
    V, N, k = 10, 4, 3
    L = rng.standard_normal((N, V)) * 1.5
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    tree = T.build_subtree(L, 0, k, N, tab)
    for B in (1, 2, 5, 12, 40):
        kept = T.prune(tree, B)
        allp = sorted(((n["lj"], p) for p, n in zip(T.paths(tree), tree) if p), reverse=True)
        assert set(T.paths(kept)) - {()} == {p for _, p in allp[:B]}
        assert len(kept) == 1 + min(B, len(tree) - 1)
        kp = set(T.paths(kept))
        assert all(p[:-1] in kp for p in kp if p)
    with pytest.raises(ValueError):
        T.prune(tree, 0)


@pytest.mark.parametrize("seed", range(20))
def test_resample_reduces_to_alg1_on_truncated_chain(seed):
    rng = np.random.default_rng(200 + seed)
    V, N, k = 9, 5, 2
    L = rng.standard_normal((N, V))
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    for cut in range(N + 1):
        rem = L[cut:]
        rs = T.resample(rem, 4, k, 1, tab)
        if len(rem) > 1:
            ref = T.build_subtree(rem, 4, k, len(rem), tab)
            assert T.paths(rs) == T.paths(ref) and [n["lj"] for n in rs] == [n["lj"] for n in ref]
        else:
            assert len(rs) == 1


@pytest.mark.parametrize("seed", range(20))
def test_fuse_is_path_union_with_max_joint(seed):
    rng = np.random.default_rng(300 + seed)
    V, k = 6, 2
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    a = T.prune(T.build_subtree(rng.standard_normal((4, V)), 1, k, 4, tab), 8)
    b = T.prune(T.build_subtree(rng.standard_normal((3, V)), 1, k, 3, tab), 4)
    f = T.fuse(a, b)
    pa, pb, pf = T.paths(a), T.paths(b), T.paths(f)
    assert set(pf) == set(pa) | set(pb) and len(pf) == len(set(pf))
    ja = dict(zip(pa, (n["lj"] for n in a)))
    jb = dict(zip(pb, (n["lj"] for n in b)))
    for p, n in zip(pf, f):
        assert n["lj"] == max(ja.get(p, -np.inf), jb.get(p, -np.inf))
    # identity cases
    assert T.paths(T.fuse(a, [dict(a[0])])) == pa
    assert T.paths(T.fuse(a, a)) == pa
    # monotone: a fused node's joint never exceeds its parent's -> prune stays connected
    for n in f[1:]:
        assert n["lj"] <= f[n["par"]]["lj"]
    kept = T.prune(f, 9)
    kp = set(T.paths(kept))
    assert all(p[:-1] in kp for p in kp if p)


def test_linearize_ancestor_masks():
    rng = np.random.default_rng(11)
    V = 8
    tab = ExplicitTable(V, {t: rng.standard_normal(V) for t in range(V)})
    tree = T.prune(T.build_subtree(rng.standard_normal((4, V)), 2, 3, 4, tab), 10)
    lin = T.linearize(tree)
    n = lin["T"]
    assert n == 11 and lin["par"][0] == -1
    for u in range(1, n):
        assert lin["par"][u] < u and lin["depth"][u] == lin["depth"][lin["par"][u]] + 1
        assert lin["depth"][u] >= lin["depth"][u - 1]
        # visibility(node) = visibility(parent) + {node}
        expect = lin["anc"][lin["par"][u]].copy(); expect[u] = True
        assert np.array_equal(lin["anc"][u], expect)
    # siblings in (jointProb desc, token asc) order
    for u in range(n):
        kids = [c for c in range(n) if lin["par"][c] == u]
        keys = [(-lin["lj"][c], lin["tok"][c]) for c in kids]
        assert keys == sorted(keys) and kids == list(range(kids[0], kids[0] + len(kids))) if kids else True


# ---------------------------------------------------------------------------
# Token-info table (§5.1, §6.1).
# ---------------------------------------------------------------------------

def test_table_bytes_paper_numbers():
    # |V| = 128,256 in FP8 -> "15.3 GB" (GiB: 16,449,601,536 B)
    b = table_bytes(128256, 1)
    assert b == 16_449_601_536
    assert b / 2 ** 30 == pytest.approx(15.3, abs=0.05)
    # keeping 32K of 128,256 tokens prunes the matrix "to 1/16"
    # -- only a 2-D (rows and columns) prune gives that ratio (reading R5).
    assert table_bytes(32768, 1) / b == pytest.approx(1 / 16, rel=0.05)
    assert 32768 / 128256 == pytest.approx(1 / 4, rel=0.05)
    assert table_bytes(32768, 1) == 2 ** 30


def test_table_rows_collapse_norm_and_hot_prune():
    cfg = get_config("c1").replace(vocab=96, hidden=32, hot_tokens=24)
    m = Model(cfg, seed=4, layers=0, with_draft=False)
    perm = vocab_permutation(cfg.vocab, 0)
    dense = TokenInfoTable(m)
    hot = TokenInfoTable(m, hot_tokens=24, perm=perm)
    hot_set = set(perm[:24].tolist())
    d = cfg.table_rank
    for t in range(cfg.vocab):
        # brute-force triple loop for E'(t) = W_E[t] . W_1 . W_2 (paper orientation)
        e = np.zeros(cfg.vocab)
        for c in range(cfg.vocab):
            e[c] = sum(m.embed[t, i] * m.w1[j, i] * m.w2[c, j] for i in range(cfg.hidden) for j in range(d)) \
                if t < 3 else 0.0
        r = dense.row(t)
        if t < 3:
            np.testing.assert_allclose(r, e / np.sqrt(np.mean(e * e) + 1e-6), atol=1e-12)
        assert np.mean(r * r) == pytest.approx(1.0, rel=1e-3)     # RMSNorm, no gain (eps shifts ~1e-5)
        hr = hot.row(t)
        if t in hot_set:
            cols = sorted(hot_set)
            np.testing.assert_array_equal(hr[cols], r[cols])       # kept rows unchanged
            assert np.all(hr[[c for c in range(cfg.vocab) if c not in hot_set]] == 0)
        else:
            assert np.all(hr == 0)                                  # cold row -> zero bias
