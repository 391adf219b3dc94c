"""Oracle draft-tree algorithms (§5.2-§5.3, §6.2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A tree is a flat list of node dicts in creation order, node 0 = root:
  tok   token id
  par   index of the parent in the same list (-1 for the root)
  depth root = 0
  prob  p_j of Alg. 1 (root 1)
  lj    log jointProb (root 0), float64
Children are recovered from `par`. The list index is the node's creation index,
used by the tie-breaks (reading R8).
"""
from __future__ import annotations

import math
import numpy as np


def _node(tok, par, depth, prob, lj):
    return {"tok": int(tok), "par": int(par), "depth": int(depth), "prob": float(prob), "lj": float(lj)}


def logsumexp(v: np.ndarray) -> float:
    m = float(np.max(v))
    return m + math.log(float(np.sum(np.exp(v - m))))


def topk_desc(v: np.ndarray, k: int):
    """Top-k indices of v: value descending, ties by ascending token id
    (reading R8). Also returns the boundary margin
    v[k-th] - v[(k+1)-th] (inf if k == |V|)."""
    if k > v.shape[0]:
        raise ValueError("k > |V| (contract violation)")
    order = np.lexsort((np.arange(v.shape[0]), -v))   # primary -v, secondary id
    top = order[:k]
    margin = float(v[order[k - 1]] - v[order[k]]) if k < v.shape[0] else math.inf
    return [int(e) for e in top], margin


def build_subtree(L_rows, t_root: int, k: int, n_steps: int, table, margins=None):
    """BuildSubtree of Alg. 1, step by step:

      T_sub <- Node(t_root, 1, 1); Q <- [T_sub]
      for i = 1..N_steps:
        l_i <- L_{start+i-1}; Q_next <- []
        while Q not empty: node <- Q.pop()
          r_i <- getTokenInfo(node.token)
          l'_i <- SoftMax(l_i + r_i)
          p_1..p_k, e_1..e_k <- TopkValue/TopkIndex(l'_i)
          children t_j = Node(e_j, p_j, node.jointProb * p_j); push to Q_next
        Q <- TopkByJointProb(Q_next, k)

    jointProb is carried in log space (reading R9). TopkByJointProb ties: token
    id ascending, then parent creation index ascending (reading R8)."""
    if k < 1 or n_steps < 0:
        raise ValueError("contract violation: k >= 1, N >= 0")
    nodes = [_node(t_root, -1, 0, 1.0, 0.0)]
    Q = [0]
    for i in range(n_steps):
        l_i = np.asarray(L_rows[i], dtype=np.float64)
        Q_next = []
        for u in Q:                                   # Q.pop() in queue order
            v = l_i + table.row(nodes[u]["tok"])      # l_i + r_i
            lse = logsumexp(v)                        # SoftMax normaliser
            top, mg = topk_desc(v, k)
            if margins is not None:
                margins.append(("topk", mg))
            for e in top:
                lp = float(v[e]) - lse                # log p_j
                nodes.append(_node(e, u, nodes[u]["depth"] + 1, math.exp(lp), nodes[u]["lj"] + lp))
                Q_next.append(len(nodes) - 1)
        key = lambda c: (-nodes[c]["lj"], nodes[c]["tok"], nodes[c]["par"])
        Q_sorted = sorted(Q_next, key=key)
        if margins is not None and len(Q_sorted) > k:
            margins.append(("frontier", nodes[Q_sorted[k - 1]]["lj"] - nodes[Q_sorted[k]]["lj"]))
        Q = Q_sorted[:k]
    return nodes


def prune_order_key(nodes, i):
    """Prune priority (reading R8): jointProb desc, depth asc, token asc,
    parent creation index asc. Shallower-first on ties keeps the kept set
    connected."""
    n = nodes[i]
    return (-n["lj"], n["depth"], n["tok"], n["par"])


def _subset(nodes, keep):
    """Restrict to the index set `keep` (must contain 0 and be parent-closed),
    preserving creation order and re-indexing parents."""
    keep = sorted(keep)
    remap = {old: new for new, old in enumerate(keep)}
    out = []
    for old in keep:
        n = dict(nodes[old])
        n["par"] = remap[n["par"]] if n["par"] >= 0 else -1
        out.append(n)
    return out


def prune(nodes, B: int, margins=None):
    """Keep the top-B non-root nodes by cumulative probability."""
    if B < 1:
        raise ValueError("contract violation: B >= 1")
    rest = sorted(range(1, len(nodes)), key=lambda i: prune_order_key(nodes, i))
    if margins is not None and len(rest) > B:
        margins.append(("prune", nodes[rest[B - 1]]["lj"] - nodes[rest[B]]["lj"]))
    keep = [0] + rest[:B]
    for i in keep[1:]:
        assert nodes[i]["par"] in keep, "pruned tree must be connected"
    return _subset(nodes, keep)


def resample(L_remain, t_gt: int, k: int, r: int, table):
    """Alg. 2: if N_remain > r, BuildSubtree(L_remain, t_gt,
    k, N_remain); else the single node (t_gt, 1, 1)."""
    n_remain = len(L_remain)
    if n_remain > r:
        return build_subtree(L_remain, t_gt, k, n_remain, table)
    return [_node(t_gt, -1, 0, 1.0, 0.0)]


def paths(nodes):
    """token path (tuple, root excluded) of every node."""
    out = []
    for n in nodes:
        out.append(() if n["par"] < 0 else out[n["par"]] + (n["tok"],))
    return out


def fuse(fresh, resampled):
    """Verification fusion (§6.2): union at the shared bonus-token
    root; nodes with identical token paths are deduplicated keeping the larger
    jointProb, fresh winning ties (reading R11). Creation order: fresh nodes,
    then resampled-only nodes in their own order."""
    if fresh[0]["tok"] != resampled[0]["tok"]:
        raise ValueError("contract violation: fused trees must share the root token")
    out = [dict(n) for n in fresh]
    pmap = {p: i for i, p in enumerate(paths(out))}
    rpaths = paths(resampled)
    for j in range(1, len(resampled)):
        rn, rp = resampled[j], rpaths[j]
        if rp in pmap:
            i = pmap[rp]
            if rn["lj"] > out[i]["lj"]:
                out[i]["lj"], out[i]["prob"] = rn["lj"], rn["prob"]
        else:
            par = pmap[rp[:-1]]
            out.append(_node(rn["tok"], par, rn["depth"], rn["prob"], rn["lj"]))
            pmap[rp] = len(out) - 1
    return out


def linearize(nodes):
    """Depth-major linearisation (reading R8): BFS from the root, children of a
    node ordered by (jointProb desc, token asc). Returns dict of arrays:
    tok, par (slot), depth, lj, prob, anc (bool [T, T]: anc[u, a] iff a is u or
    an ancestor of u - the tree-attention visibility of PAPER.md:95)."""
    kids = {i: [] for i in range(len(nodes))}
    for i in range(1, len(nodes)):
        kids[nodes[i]["par"]].append(i)
    order, slot_of = [0], {0: 0}
    head = 0
    while head < len(order):
        u = order[head]; head += 1
        for c in sorted(kids[u], key=lambda c: (-nodes[c]["lj"], nodes[c]["tok"])):
            slot_of[c] = len(order)
            order.append(c)
    T = len(order)
    tok = np.array([nodes[i]["tok"] for i in order], dtype=np.int64)
    par = np.array([slot_of[nodes[i]["par"]] if nodes[i]["par"] >= 0 else -1 for i in order], dtype=np.int64)
    depth = np.array([nodes[i]["depth"] for i in order], dtype=np.int64)
    lj = np.array([nodes[i]["lj"] for i in order])
    prob = np.array([nodes[i]["prob"] for i in order])
    anc = np.zeros((T, T), dtype=bool)
    for u in range(T):
        a = u
        while a >= 0:
            anc[u, a] = True
            a = par[a]
    return {"tok": tok, "par": par, "depth": depth, "lj": lj, "prob": prob, "anc": anc, "T": T}
