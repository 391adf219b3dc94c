"""Oracle acceptance walks (S3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Greedy (T = 0): from the root slot, descend to the child whose
token equals argmax of the target logits at the current slot (ties -> lowest
id); stop when there is none; the bonus token is that argmax (PAPER.md:378,
"A bonus token is produced by the target model as a byproduct").

Stochastic (T > 0; not in the paper, required by north_star - reading R13):
multi-draft recursive rejection with deterministic drafts (q = delta). For the
children c_1..c_j of the current slot in slot order: accept c with probability
p(c) / (1 - sum_{rejected} p) using the Philox uniform u(req, step, slot, rank);
on rejection remove c. If every child is rejected, the bonus is drawn from the
residual (p restricted to V minus the rejected set) by Gumbel-max with the
Philox uniforms g(req, step, slot, v). At a leaf the bonus is drawn from p.
Marginally every emitted token is distributed as p (telescoping), which
tests/test_oracle_accept.py checks by chi-square.
"""
from __future__ import annotations

import math
import numpy as np

from .philox import accept_uniform, gumbel_uniforms


def children(tree, u):
    return [c for c in range(tree["T"]) if tree["par"][c] == u]


def argmax_lowest(v):
    return int(np.argmax(v))       # numpy returns the first (lowest-id) maximum


def top2_margin(v):
    s = np.sort(v)
    return float(s[-1] - s[-2]) if v.shape[0] > 1 else math.inf


def greedy_walk(tree, logits, margins=None):
    """Returns (accepted slots [s_1..s_m], bonus token)."""
    cur, acc = 0, []
    while True:
        a = argmax_lowest(logits[cur])
        if margins is not None:
            margins.append(("argmax", top2_margin(logits[cur])))
        nxt = [c for c in children(tree, cur) if tree["tok"][c] == a]
        if not nxt:
            return acc, a
        cur = nxt[0]
        acc.append(cur)


def softmax_T(l, T):
    z = np.asarray(l, dtype=np.float64) / T
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


def gumbel_argmax(logits_row, T, U, exclude=()):
    """argmax_v (l_v / T + G_v), G_v = -log(-log U_v), over v not excluded."""
    z = np.asarray(logits_row, dtype=np.float64) / T - np.log(-np.log(U))
    if exclude:
        z = z.copy()
        z[list(exclude)] = -np.inf
    return argmax_lowest(z), top2_margin(z[np.isfinite(z)])


def stochastic_walk(tree, logits, T, seed, req, step, margins=None, uniform=None, gumbel=None):
    """Returns (accepted slots, bonus). `uniform(slot, rank)` / `gumbel(slot)`
    override the Philox streams (used by the distribution tests)."""
    V = logits.shape[1]
    uniform = uniform or (lambda slot, rank: accept_uniform(seed, req, step, slot, rank))
    gumbel = gumbel or (lambda slot: gumbel_uniforms(seed, req, step, slot, V))
    cur, acc = 0, []
    while True:
        p = softmax_T(logits[cur], T)
        kids = children(tree, cur)
        rejected, S, took = [], 0.0, None
        for rank, c in enumerate(kids):
            t = int(tree["tok"][c])
            u = uniform(cur, rank)
            denom = 1.0 - S
            p_res = p[t] / denom if denom > 0 else 0.0
            if margins is not None:
                margins.append(("accept_u", abs(u - p_res)))
            if u < p_res:
                took = c
                break
            rejected.append(t)
            S += p[t]
        if took is not None:
            acc.append(took)
            cur = took
            continue
        bonus, mg = gumbel_argmax(logits[cur], T, gumbel(cur), exclude=rejected)
        if margins is not None:
            margins.append(("gumbel", mg))
        return acc, bonus
