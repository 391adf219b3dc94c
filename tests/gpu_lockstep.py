"""Lockstep GPU-vs-oracle comparison.

Each step the oracle is restarted from the GPU's committed state (committed
tokens + the GPU's pending re-sampled tree), runs the same step in float64, and
every intermediate of the GPU step is compared:
  L (draft logits), tree topology, verify logits, accepted slots / bonus,
  the new pending tree, and the KV rows written by compaction.
Discrete decisions whose oracle margin is below `flag_margin` (relative to the
row's max |logit|) are FLAGGED: a mismatch there is counted, not failed.
"""
import numpy as np

from oracle.model import Model
from oracle.table import TokenInfoTable
from oracle.engine import Engine
from oracle import tree as T


def gpu_tree(ctx, r):
    n = int(ctx.tensor("tree_n").cpu()[r])
    tok = ctx.tensor("tree_tok").cpu().numpy()[r, :n]
    par = ctx.tensor("tree_par").cpu().numpy()[r, :n]
    depth = ctx.tensor("tree_depth").cpu().numpy()[r, :n]
    lj = ctx.tensor("tree_lj").cpu().numpy()[r, :n]
    return n, tok, par, depth, lj


def gpu_pending(ctx, r):
    n = int(ctx.tensor("pt_n").cpu()[r])
    tok = ctx.tensor("pt_tok").cpu().numpy()[r]
    par = ctx.tensor("pt_par").cpu().numpy()[r]
    dep = ctx.tensor("pt_depth").cpu().numpy()[r]
    lj = ctx.tensor("pt_lj").cpu().numpy()[r]
    return [T._node(tok[i], par[i], dep[i], float(np.exp(lj[i])), float(lj[i])) for i in range(n)]


def lin_from_gpu(n, tok, par, depth, lj):
    anc = np.zeros((n, n), dtype=bool)
    for u in range(n):
        a = u
        while a >= 0:
            anc[u, a] = True
            a = par[a]
    return {"tok": np.array(tok, dtype=np.int64), "par": np.array(par, dtype=np.int64),
            "depth": np.array(depth, dtype=np.int64), "lj": np.array(lj, dtype=np.float64),
            "prob": np.exp(np.array(lj, dtype=np.float64)), "anc": anc, "T": n}


def kv_rows(ctx, cfg, layer, r, positions, page_size, pages_per_req):
    """GPU K and V rows [len(positions), Hkv*hd] of request r at `positions`
    (logical page -> physical page through the context's block table)."""
    kv = ctx.tensor("kv")[layer]                   # [pages, 2, Hkv*ps*hd]
    bt = ctx.tensor("block_table").cpu().numpy()   # [max_batch, pages_per_req]
    Hkv, hd = cfg.kv_heads, cfg.head_dim
    out_k, out_v = [], []
    for pos in positions:
        page = int(bt[r, pos // page_size])
        slot = pos % page_size
        blk = kv[page].float()
        out_k.append(blk[0].view(Hkv, page_size, hd)[:, slot, :].reshape(-1).cpu().numpy())
        # V blocks are stored transposed, [hd][page_size] per head (KVLayer)
        out_v.append(blk[1].view(Hkv, hd, page_size)[:, :, slot].reshape(-1).cpu().numpy())
    return np.stack(out_k), np.stack(out_v)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.max(np.abs(b), axis=-1, keepdims=True)
    return float(np.max(np.max(np.abs(a - b), axis=-1, keepdims=True) / np.maximum(den, 1e-30)))


class Lockstep:
    def __init__(self, ctx, cfg, model, table, prompts, seed=0, accept="greedy", temperature=1.0,
                 resample=True, fusion=True, plant=None, plant_rates=None, perm=None,
                 logit_tol=1e-4, flag_margin=1e-4, page_size=64, tree_flag_margin=None, first_token=True):
        self.ctx, self.cfg, self.m, self.table = ctx, cfg, model, table
        self.seed, self.accept, self.T = seed, accept, temperature
        self.resample, self.fusion = resample, fusion
        self.first_token = first_token
        self.plant, self.plant_rates = plant, plant_rates
        self.perm = perm
        self.tol, self.flag = logit_tol, flag_margin
        # draft-tree decisions (top-k / frontier / prune on the draft logits): exact
        # topology is required in fp32-verify mode (north_star); in bf16 the draft
        # logits carry up to logit_tol row-normwise error (R21) on the GPU side, so a
        # decision whose oracle margin is below 2 x logit_tol may legitimately flip
        self.tree_flag = flag_margin if tree_flag_margin is None else tree_flag_margin
        self.page_size = page_size
        self.prompts = [list(map(int, p)) for p in prompts]
        self.tokens = None
        self.flags = 0
        self.checked = {"tree": 0, "accept": 0, "pending": 0}
        self.max_err = {"L": 0.0, "verify": 0.0, "kv": 0.0}
        self.step_no = 0
        self.emitted = [[] for _ in prompts]
        self.req_ids = list(range(len(prompts)))     # global request id per slot (ctx req_offset 0)

    def start(self):
        import torch
        b = len(self.prompts)
        d_first = torch.empty(b, dtype=torch.int32, device="cuda")
        self.ctx.prefill(np.array(self.prompts), d_first=d_first.data_ptr())
        torch.cuda.synchronize()
        first = d_first.cpu().numpy()
        self.tokens = [p + [int(f)] for p, f in zip(self.prompts, first)]
        for r in range(b):
            self.emitted[r].append(int(first[r]))
        # oracle first token (plain argmax / Gumbel sample)
        e = Engine(self.m, self.table, self.cfg, seed=self.seed, accept=self.accept, temperature=self.T)
        ofirst = e.prefill(self.prompts)
        return first, ofirst

    def admit(self, slot, prompt, req_id):
        """hsd_admit a new request into `slot` under global id `req_id`; returns
        (GPU first token, oracle first token) of the admitted request."""
        import torch
        d_first = torch.zeros(len(self.prompts), dtype=torch.int32, device="cuda")
        prompt = [int(t) for t in prompt]
        self.ctx.admit(slot, prompt, req_id, d_first=d_first.data_ptr())
        first = int(d_first.cpu()[slot])
        e = Engine(self.m, self.table, self.cfg, seed=self.seed, accept=self.accept, temperature=self.T)
        e.prefill([self.prompts[0]])
        ofirst = e.admit(0, prompt, req_id)
        self.prompts[slot] = prompt
        self.tokens[slot] = prompt + [first]
        self.emitted[slot] = [first]
        self.req_ids[slot] = req_id
        return first, ofirst

    def _engine(self, r):
        return Engine(self.m, self.table, self.cfg, seed=self.seed, accept=self.accept,
                      temperature=self.T, resample=self.resample, fusion=self.fusion, req_offset=self.req_ids[r],
                      plant=None if self.plant is None else [self.plant[r]], plant_rates=self.plant_rates,
                      first_token=self.first_token)

    def _margins_ok(self, margins, kinds, scale, flag=None):
        flag = self.flag if flag is None else flag
        for kind, mg in margins:
            if kind in kinds and mg < flag * scale:
                return False
        return True

    def step(self):
        ctx, cfg = self.ctx, self.cfg
        b = len(self.prompts)
        self.step_no += 1
        pend_before = [gpu_pending(ctx, r) for r in range(b)]
        p_before = ctx.tensor("p").cpu().numpy().copy()
        ctx.build_tree()
        Lg = ctx.tensor("draft_logits").cpu().numpy().copy()
        trees = [gpu_tree(ctx, r) for r in range(b)]
        ctx.verify_tree()
        VL = ctx.tensor("verify_logits").cpu().numpy().copy()
        ctx.accept_and_compact()
        acc_n = ctx.tensor("acc_n").cpu().numpy().copy()
        acc = ctx.tensor("acc_slots").cpu().numpy().copy()
        bonus = ctx.tensor("bonus").cpu().numpy().copy()
        emitted = ctx.tensor("emitted").cpu().numpy().copy()
        pend_after = [gpu_pending(ctx, r) for r in range(b)]
        report = []
        for r in range(b):
            e = self._engine(r)
            e.prefill([self.tokens[r][:-1]], first_tokens=[self.tokens[r][-1]])
            q = e.reqs[0]
            q.pending = pend_before[r] if len(pend_before[r]) > 1 else None
            assert int(p_before[r]) == len(q.tokens) - 1, "GPU position differs from committed length"
            e.step_idx = self.step_no - 1
            e.step()
            rec = e.trace[-1][2]
            Lo = rec["L"]
            Lgr = Lg[r]
            if self.perm is not None:          # GPU L columns are in rank order
                tmp = np.empty_like(Lgr)
                tmp[:, self.perm] = Lgr
                Lgr = tmp
            self.max_err["L"] = max(self.max_err["L"], rel_err(Lgr, Lo))
            assert rel_err(Lgr, Lo) <= self.tol, f"draft logits rel err {rel_err(Lgr, Lo)}"
            scaleL = float(np.max(np.abs(Lo)))
            n, tok, par, depth, lj = trees[r]
            lin_o = rec["lin"]
            same_tree = (n == lin_o["T"] and np.array_equal(tok, lin_o["tok"]) and np.array_equal(par, lin_o["par"])
                         and np.array_equal(depth, lin_o["depth"]))
            if not same_tree:
                if self._margins_ok(rec["margins"], ("topk", "frontier", "prune"), scaleL, self.tree_flag):
                    raise AssertionError(f"step {self.step_no} req {r}: tree differs with clear margins\n"
                                         f"gpu {tok.tolist()} {par.tolist()}\noracle {lin_o['tok'].tolist()} "
                                         f"{lin_o['par'].tolist()}")
                self.flags += 1
            else:
                self.checked["tree"] += 1
                np.testing.assert_allclose(lj, lin_o["lj"], atol=max(self.tol, 1e-6) * 10 * max(1, scaleL))
            # verify logits on the GPU's tree, from the pre-step state
            lin_g = lin_from_gpu(n, tok, par, depth, lj)
            if same_tree:
                Vo = rec["logits"]
            else:
                ev = self._engine(r)
                ev.prefill([self.tokens[r][:-1]], first_tokens=[self.tokens[r][-1]])
                _, Vo, _ = ev.verify(ev.reqs[0], lin_g)
            verr = rel_err(VL[r, :n], Vo)
            self.max_err["verify"] = max(self.max_err["verify"], verr)
            assert verr <= self.tol, f"verify logits rel err {verr}"
            # acceptance
            m = int(acc_n[r])
            g_acc = [int(s) for s in acc[r, :m]]
            if same_tree:
                if g_acc == rec["acc"] and int(bonus[r]) == rec["bonus"]:
                    self.checked["accept"] += 1
                else:
                    scaleV = float(np.max(np.abs(Vo)))
                    if self._margins_ok(rec["margins"], ("argmax", "accept_u", "gumbel"), scaleV if self.accept ==
                                        "greedy" else 1.0):
                        raise AssertionError(f"step {self.step_no} req {r}: acceptance differs: gpu {g_acc} "
                                             f"{bonus[r]} oracle {rec['acc']} {rec['bonus']}")
                    self.flags += 1
                    same_tree = False
            # new pending tree (Alg. 2)
            if same_tree and g_acc == rec["acc"]:
                po = rec["pending"]
                pg = pend_after[r]
                if po is None:
                    assert len(pg) == 1 and pg[0]["tok"] == int(bonus[r])
                else:
                    if T.paths(pg) == T.paths(po):
                        self.checked["pending"] += 1
                        np.testing.assert_allclose([x["lj"] for x in pg], [x["lj"] for x in po],
                                                   atol=max(self.tol, 1e-6) * 10 * max(1, scaleL))
                    else:
                        mg = []
                        T.prune(T.resample(Lo[m + 1:], int(bonus[r]), cfg.branch_k, cfg.resample_threshold_r,
                                           self.table), cfg.resample_budget_Br, mg)
                        T.build_subtree(Lo[m + 1:], int(bonus[r]), cfg.branch_k, cfg.steps_N - m - 1, self.table, mg)
                        if self._margins_ok(mg, ("topk", "frontier", "prune"), scaleL, self.tree_flag):
                            raise AssertionError(f"pending tree differs: gpu {T.paths(pg)} oracle {T.paths(po)}")
                        self.flags += 1
            new = [int(t) for t in emitted[r, :m + 1]]
            assert new[-1] == int(bonus[r])
            self.tokens[r] += new
            self.emitted[r] += new
            # compaction: GPU KV rows at positions p..p+m == oracle plain-decode KV of the committed path
            p0 = int(p_before[r])
            pages_per_req = ctx.tensor("kv").shape[1] // ctx.cfg.max_batch
            e2 = self._engine(r)
            e2.prefill([self.tokens[r][:-1]], first_tokens=[self.tokens[r][-1]])
            for layer in range(self.m.n_layers):
                gk, gv = kv_rows(ctx, cfg, layer, r, range(p0, p0 + m + 1), self.page_size, pages_per_req)
                ok = np.stack(e2.reqs[0].kv[layer][0][p0:p0 + m + 1]).reshape(m + 1, -1)
                ov = np.stack(e2.reqs[0].kv[layer][1][p0:p0 + m + 1]).reshape(m + 1, -1)
                err = max(rel_err(gk, ok), rel_err(gv, ov))
                self.max_err["kv"] = max(self.max_err["kv"], err)
                assert err <= self.tol * 10, f"compacted KV rel err {err}"
            report.append((m, new))
        return report
