"""Oracle speculative-decoding engine: the per-step draft-tree verify-and-reuse
loop (§3 overview :184, §4-§6), one request at a time.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

State of a request between steps:
  tokens      committed tokens t_0..t_p; t_p (the last bonus token) is the root of
              the next tree, at position p.
  kv[l]       target K/V rows for positions [0, p) (what plain decode wrote).
  pend        draft pairs (H_{j-1}, t_j, j) not yet run through the draft layer;
              always the m+1 pairs committed by the last step (R1).
  dkv         draft K/V rows by position (positions 1..p are valid).
  pending     Alg. 2 re-sampled tree rooted at t_p, or None (R10/R11).

One step (per request):
  S0  draft prefill of `pend`, then the chain h_{i+1} = TL(h_i), i = 1..N-1
      (PAPER.md:208-212); chain row i sits at position p+i (R2).
  S1a L = [l_1..l_N] = RMSNorm_f([h_1..h_N]) W_head^T, one product.
  S1b Alg. 1 from root t_p over L; prune to B.
  S1c fuse the pending re-sampled tree, prune to B+B_r; linearise.
  S2  verify: each slot = plain causal forward of its root path over the cache
      (tree attention), position p + depth (R12).
  S3  acceptance walk (greedy / stochastic).
  S4  commit m+1 tokens; KV of the accepted path; draft pairs; Alg. 2 over
      L rows m+1..N-1 (0-based) rooted at the bonus token.
"""
from __future__ import annotations

import numpy as np

from . import tree as T
from .accept import greedy_walk, stochastic_walk, argmax_lowest, gumbel_argmax
from .philox import gumbel_uniforms, philox4x32_10, unit_open, TAG_PLANT


class Request:
    def __init__(self, L):
        self.tokens = []
        self.kv = [([], []) for _ in range(L)]
        self.pend = []
        self.dkv = {}
        self.pending = None
        self.H = []          # target pre-norm hidden per committed position (for tests)


class Engine:
    def __init__(self, model, table, cfg, seed=0, accept=None, temperature=None,
                 resample=True, fusion=True, req_offset=0, plant=None, plant_rates=None, first_token=True,
                 draft_mode="hidden"):
        self.m, self.table, self.cfg = model, table, cfg
        self.seed = seed
        self.accept = accept or cfg.accept
        self.T = cfg.temperature if temperature is None else temperature
        self.resample, self.fusion = resample, fusion
        self.first_token = first_token   # False: the root pair's draft input omits E(t_p) (R26, Table 4)
        self.draft_mode = draft_mode     # "hidden" (the paper's chain) | "token_ar" (EAGLE-style, R27)
        self.req_offset = req_offset
        self.plant, self.plant_rates = plant, plant_rates
        self.reqs = []
        self.req_ids = []    # global request id per slot (random streams)
        self.step_idx = 0
        self.trace = []      # per step, per request: dict of intermediate results

    # ------------------------------------------------------------------
    def prefill(self, prompts, first_tokens=None):
        """Causal target forward over each prompt (plain decode of the prompt),
        first token = argmax (greedy) or a Gumbel sample (slot 0, step 0) unless
        `first_tokens` forces it (lockstep tests); then the draft layer over
        pairs j = 1..P0-1; pair P0 stays pending."""
        self.reqs, self.req_ids = [], []
        return [self._prefill_one(prompt, self.req_offset + r,
                                  None if first_tokens is None else first_tokens[r])
                for r, prompt in enumerate(prompts)]

    def admit(self, slot, prompt, req_id, first_token=None):
        """Continuous batching (the serving layer around the path): slot
        `slot` restarts with a new prompt under the fresh global request id
        `req_id` (its random streams); the other slots keep their state."""
        q_old, id_old = self.reqs, self.req_ids
        t1 = self._prefill_one(prompt, req_id, first_token)
        q_new = self.reqs.pop()
        self.req_ids.pop()
        q_old[slot], id_old[slot] = q_new, req_id
        return t1

    def _prefill_one(self, prompt, req_id, first_token):
        m = self.m
        if True:
            q = Request(m.n_layers)
            logits = None
            for pos, t in enumerate(prompt):
                H, logits, rows = m.target_one(int(t), pos, q.kv)
                for l, (k, v) in enumerate(rows):
                    q.kv[l][0].append(k); q.kv[l][1].append(v)
                q.H.append(H)
                q.tokens.append(int(t))
            if first_token is not None:
                t1 = int(first_token)
            elif self.accept == "greedy":
                t1 = argmax_lowest(logits)
            else:
                U = gumbel_uniforms(self.seed, req_id, 0, 0, m.cfg.vocab)
                t1 = gumbel_argmax(logits, self.T, U)[0]
            q.tokens.append(t1)
            P0 = len(prompt)
            pairs = [(q.H[j - 1], q.tokens[j], j) for j in range(1, P0 + 1)]
            self._draft_prefill(q, pairs[:-1])
            q.pend = pairs[-1:]
            self.reqs.append(q)
            self.req_ids.append(req_id)
        return t1

    def _draft_prefill(self, q, pairs):
        h = None
        p_root = len(q.tokens) - 1
        for H_prev, t, j in pairs:
            # R26 ("w/o first token", Table 4): the root pair -- the ground-truth token
            # just committed -- enters the draft without its embedding
            x = self.m.draft_input(H_prev, t, with_token=self.first_token or j != p_root)
            dk = [q.dkv[i][0] for i in range(1, j)]
            dv = [q.dkv[i][1] for i in range(1, j)]
            h, k, v = self.m.draft_one(x, j, dk, dv)
            q.dkv[j] = (k, v)
        return h

    # ------------------------------------------------------------------
    def draft_chain(self, q):
        """S0: returns [h_1..h_N]."""
        N = self.cfg.steps_N
        p = len(q.tokens) - 1
        h = self._draft_prefill(q, q.pend)
        chain = [h]
        tmp = {i: q.dkv[i] for i in range(1, p + 1)}
        for i in range(1, N):
            dk = [tmp[j][0] for j in range(1, p + i)]
            dv = [tmp[j][1] for j in range(1, p + i)]
            x = chain[-1]
            if self.draft_mode == "token_ar":   # R27: feed back the draft's own top-1 token
                x = self.m.draft_input(chain[-1], argmax_lowest(self.m.logits(chain[-1])))
            h, k, v = self.m.draft_one(x, p + i, dk, dv)
            tmp[p + i] = (k, v)
            chain.append(h)
        return chain

    def verify(self, q, lin, slots=None):
        """S2: per-slot plain forward of its root path over the cache. `slots`
        (tests at full size): only those slots and their ancestors are computed;
        the other rows of H / logits stay zero."""
        m = self.m
        p = len(q.tokens) - 1
        Tn = lin["T"]
        need = set(range(Tn))
        if slots is not None:
            need = set()
            for u in slots:
                while u >= 0 and u not in need:
                    need.add(u)
                    u = int(lin["par"][u])
        path_rows = [None] * Tn
        H = np.zeros((Tn, m.cfg.hidden))
        logits = np.zeros((Tn, m.cfg.vocab))
        for u in range(Tn):
            if u not in need:
                continue
            par = int(lin["par"][u])
            prev = path_rows[par] if par >= 0 else [([], []) for _ in range(m.n_layers)]
            ctx = [(q.kv[l][0] + prev[l][0], q.kv[l][1] + prev[l][1]) for l in range(m.n_layers)]
            H[u], logits[u], rows = m.target_one(int(lin["tok"][u]), p + int(lin["depth"][u]), ctx)
            path_rows[u] = [(prev[l][0] + [rows[l][0]], prev[l][1] + [rows[l][1]]) for l in range(m.n_layers)]
        return H, logits, path_rows

    # ------------------------------------------------------------------
    def step(self):
        self.step_idx += 1
        cfg = self.cfg
        N, k, B, Br, r = cfg.steps_N, cfg.branch_k, cfg.budget_B, cfg.resample_budget_Br, cfg.resample_threshold_r
        out = []
        for ri, q in enumerate(self.reqs):
            mg = []
            p = len(q.tokens) - 1
            chain = self.draft_chain(q)
            L = np.stack([self.m.logits(h) for h in chain])                # S1a
            fresh = T.prune(T.build_subtree(L, q.tokens[-1], k, N, self.table, mg), B, mg)
            tree = fresh
            if self.fusion and q.pending is not None and len(q.pending) > 1:
                tree = T.prune(T.fuse(fresh, q.pending), B + Br)
            lin = T.linearize(tree)
            if self.plant is not None:
                plant_path(lin, self.plant[ri], p, self.plant_rates, self.seed, self.req_ids[ri],
                           self.step_idx)
            H, logits, path_rows = self.verify(q, lin)                    # S2
            if self.accept == "greedy":                                   # S3
                acc, bonus = greedy_walk(lin, logits, mg)
            else:
                acc, bonus = stochastic_walk(lin, logits, self.T, self.seed, self.req_ids[ri],
                                             self.step_idx, mg)
            mm = len(acc)
            new_tokens = self._commit(q, lin, H, path_rows, acc, bonus, append=False)
            pending = None
            if self.resample and N - mm - 1 > r:                          # Alg. 2
                pending = T.prune(T.resample(L[mm + 1:], int(bonus), k, r, self.table), Br)
            q.pending = pending
            rec = {"L": L, "chain": np.stack(chain), "fresh": fresh, "lin": lin, "H": H,
                   "logits": logits, "acc": acc, "bonus": int(bonus), "emitted": list(new_tokens),
                   "pending": pending, "margins": mg, "p": p}
            if self.resample and not self.fusion and pending is not None and len(pending) > 1:
                # re-sampling WITHOUT verification fusion (the ablation of
                # Fig. 12): the re-sampled tree, rooted at the bonus token, is verified in a
                # dedicated extra pass of the same step (its own random-stream step index)
                lin2 = T.linearize(pending)
                H2, logits2, rows2 = self.verify(q, lin2)
                if self.accept == "greedy":
                    acc2, bonus2 = greedy_walk(lin2, logits2, mg)
                else:
                    acc2, bonus2 = stochastic_walk(lin2, logits2, self.T, self.seed, self.req_ids[ri],
                                                   self.step_idx + 1, mg)
                new_tokens = new_tokens + self._commit(q, lin2, H2, rows2, acc2, bonus2, append=True)
                q.pending = None
                rec.update({"lin2": lin2, "acc2": acc2, "bonus2": int(bonus2), "emitted": list(new_tokens)})
            self.trace.append((self.step_idx, ri, rec))
            out.append(new_tokens)
        if self.resample and not self.fusion:
            self.step_idx += 1      # the extra verify pass counts as a step of the random streams
        return out

    def _commit(self, q, lin, H, path_rows, acc, bonus, append):
        """S4: the accepted path's KV rows and hidden states, the new draft pairs
        (H_{j-1}, t_j) (appended to the step's earlier pairs when `append`), the
        committed tokens. Returns the new tokens."""
        p = len(q.tokens) - 1
        last = acc[-1] if acc else 0
        for l in range(self.m.n_layers):
            q.kv[l][0].extend(path_rows[last][l][0])
            q.kv[l][1].extend(path_rows[last][l][1])
        path_slots = [0] + acc
        new_tokens = [int(lin["tok"][s]) for s in acc] + [int(bonus)]
        pairs = [(H[s], new_tokens[j], p + 1 + j) for j, s in enumerate(path_slots)]
        q.pend = (q.pend + pairs) if append else pairs
        q.H.extend(H[s] for s in path_slots)
        q.tokens.extend(new_tokens)
        return new_tokens

    def decode(self, prompts, max_new):
        """Run prefill + steps until every request has max_new new tokens;
        surplus tokens of the last step are truncated (reading R15)."""
        first = self.prefill(prompts)
        outs = [[t] for t in first]
        while min(len(o) for o in outs) < max_new:
            for o, new in zip(outs, self.step()):
                o.extend(new)
        return [o[:max_new] for o in outs]


def plant_path(lin, plant_tokens, p, rates, seed, req, step):
    """Planted-continuation perf mode (never a paper claim):
    from the root, follow the first child in slot order (the best draft); with
    probability a_d (Philox (seed, TAG_PLANT), counter (d, step, req, 0)) make the
    depth-d node on that path carry the target's greedy continuation token
    plant_tokens[p + d] - by switching to the sibling that already carries it,
    else by overwriting the first child's token. Stops at the first failed draw
    or at a leaf. Mutates lin['tok']."""
    cur = 0
    for d in range(1, len(rates) + 1):
        kids = [c for c in range(lin["T"]) if lin["par"][c] == cur]
        if not kids or p + d >= len(plant_tokens):
            return
        w = philox4x32_10(d, step, req, 0, seed & 0xFFFFFFFF, TAG_PLANT)[0]
        if not unit_open(np.asarray(w))[()] < rates[d - 1]:
            return
        want = int(plant_tokens[p + d])
        hit = [c for c in kids if lin["tok"][c] == want]
        cur = hit[0] if hit else kids[0]
        lin["tok"][cur] = want


# ----------------------------------------------------------------------
# Plain (non-speculative) reference decodes: the losslessness oracle.
# ----------------------------------------------------------------------

def greedy_decode(model, prompt, n_new):
    """Target plain greedy decode: one forward per token."""
    kv = [([], []) for _ in range(model.n_layers)]
    toks = [int(t) for t in prompt]
    logits = None
    out = []
    for pos in range(len(toks) + n_new - 1):
        t = toks[pos] if pos < len(toks) else out[pos - len(toks)]
        _, logits, rows = model.target_one(t, pos, kv)
        for l, (k, v) in enumerate(rows):
            kv[l][0].append(k); kv[l][1].append(v)
        if pos >= len(toks) - 1:
            out.append(argmax_lowest(logits))
    return out[:n_new], kv
