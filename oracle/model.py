"""Oracle target model (Llama decoder) and hidden-state draft head, float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Target: Llama decoder x L (the paper evaluates
LLaMA-2-7B / Vicuna-7B):
  RMSNorm -> Q,K,V -> RoPE(pos) -> softmax(QK^T/sqrt(hd)) V (GQA) -> Wo -> +res
  RMSNorm -> Wd (silu(Wg a) * Wu a) -> +res
  H = last-layer output before the final norm; logits = RMSNorm_f(H) W_head^T.
Draft head (§4.1 eq. for h_{i+1}):
  h_1 = TL(h_0 (+) E(t_1)), h_{i+1} = TL(h_i); (+) read as W_fc [h_0 ; E(t_1)]
  (reading R1), TL = one decoder layer with its own KV cache (R2).
Draft logits l_i = RMSNorm_f(h_i) W_head^T (R4).

Every per-token computation goes through ONE function, `layer_one`, so that
prefill, plain decode, per-path tree verification and the draft all share the
exact same float64 arithmetic: plain greedy decode and speculative decode are
then token-identical by construction when the method is lossless.
"""
from __future__ import annotations

import math
import os
import numpy as np

from .philox import uniform_weights, linear_scale, round_bf16

# tensor ids of the Philox weight streams
TID_EMBED, TID_HEAD, TID_W1, TID_W2, TID_FC = 1, 2, 3, 4, 5
TID_DRAFT_LAYER = 60
TID_LAYER0 = 100
LAYER_PARTS = ("wq", "wk", "wv", "wo", "wg", "wu", "wd")


def layer_tid(layer: int, part: int) -> int:
    return TID_LAYER0 + 8 * layer + part


def rmsnorm(x: np.ndarray, eps: float) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps), gain 1 (norm gains are 1)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def silu(x):
    return x / (1.0 + np.exp(-x))


def rope(x: np.ndarray, pos: int, theta: float) -> np.ndarray:
    """Rotary embedding, Llama 'rotate_half' convention, float64 angles.
    x: [heads, hd]."""
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / hd)
    ang = pos * inv
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


class LayerWeights:
    def __init__(self, d: dict):
        self.__dict__.update(d)


class Model:
    """Target + draft head weights, regenerated from Philox (seed) in the
    precision the GPU path stores them in ('fp32' values, or 'bf16' rounded)."""

    def __init__(self, cfg, seed: int = 0, precision: str = "fp32", layers: int | None = None,
                 with_draft: bool = True, with_table_factors: bool = True):
        self.cfg = cfg
        self.seed = seed
        self.precision = precision
        self.n_layers = cfg.layers if layers is None else layers
        n, V = cfg.hidden, cfg.vocab
        qd, kd = cfg.q_heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
        self.embed = self._w(TID_EMBED, (V, n), np.float32(1.0))
        self.head = self._w(TID_HEAD, (V, n), linear_scale(n))
        self.layers = [self._layer(lambda p, l=l: layer_tid(l, p)) for l in range(self.n_layers)]
        if with_draft:
            self.fc = self._w(TID_FC, (n, 2 * n), linear_scale(2 * n))
            self.draft = self._layer(lambda p: TID_DRAFT_LAYER + p)
        if with_table_factors:
            d = cfg.table_rank
            self.w1 = self._w(TID_W1, (d, n), linear_scale(n))      # paper W_1 = w1^T (n x d)
            self.w2 = self._w(TID_W2, (V, d), linear_scale(d))      # paper W_2 = w2^T (d x |V|)

    def _w(self, tid, shape, scale):
        w = uniform_weights(self.seed, tid, shape, scale).reshape(-1)
        out = np.empty(w.size, dtype=np.float64)

        def conv(e0, e1):   # elementwise: bf16 rounding (bf16 mode) then exact widening
            x = w[e0:e1]
            out[e0:e1] = round_bf16(x) if self.precision == "bf16" else x
        step = 1 << 22
        ranges = [(e0, min(w.size, e0 + step)) for e0 in range(0, w.size, step)]
        if len(ranges) <= 1:
            for r in ranges:
                conv(*r)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(max_workers=min(len(ranges), os.cpu_count() or 1)) as ex:
                list(ex.map(lambda r: conv(*r), ranges))
        return out.reshape(shape)

    def _layer(self, tid):
        c = self.cfg
        n, qd, kd, f = c.hidden, c.q_heads * c.head_dim, c.kv_heads * c.head_dim, c.ffn
        shapes = {"wq": (qd, n), "wk": (kd, n), "wv": (kd, n), "wo": (n, qd),
                  "wg": (f, n), "wu": (f, n), "wd": (n, f)}
        return LayerWeights({k: self._w(tid(i), shapes[k], linear_scale(shapes[k][1]))
                             for i, k in enumerate(LAYER_PARTS)})

    # ------------------------------------------------------------------
    # One token through one decoder layer.
    # ------------------------------------------------------------------
    def layer_one(self, lw: LayerWeights, x: np.ndarray, pos: int, ctx_k, ctx_v):
        """x: residual [n] at position `pos`. ctx_k/ctx_v: lists of [Hkv, hd]
        rows this token may attend to (its visible context, in position order,
        NOT including itself). Returns (x_out, k_row, v_row)."""
        c = self.cfg
        hd, Hq, Hkv = c.head_dim, c.q_heads, c.kv_heads
        a = rmsnorm(x, c.rms_eps)
        q = (lw.wq @ a).reshape(Hq, hd)
        k = (lw.wk @ a).reshape(Hkv, hd)
        v = (lw.wv @ a).reshape(Hkv, hd)
        q = rope(q, pos, c.rope_theta)
        k = rope(k, pos, c.rope_theta)
        K = np.stack(list(ctx_k) + [k])          # [S, Hkv, hd]
        Vv = np.stack(list(ctx_v) + [v])
        grp = Hq // Hkv
        o = np.empty((Hq, hd))
        for h in range(Hq):
            kh = K[:, h // grp, :]
            s = kh @ q[h] / math.sqrt(hd)
            s = np.exp(s - s.max())
            o[h] = (s / s.sum()) @ Vv[:, h // grp, :]
        x = x + lw.wo @ o.reshape(-1)
        a2 = rmsnorm(x, c.rms_eps)
        x = x + lw.wd @ (silu(lw.wg @ a2) * (lw.wu @ a2))
        return x, k, v

    def target_one(self, token: int, pos: int, kv_ctx):
        """Target forward of one token. kv_ctx: per layer (list_k, list_v) of its
        visible context. Returns (H [n], logits [V], new rows [(k, v)] per layer)."""
        x = self.embed[token].copy()
        rows = []
        for l, lw in enumerate(self.layers):
            x, k, v = self.layer_one(lw, x, pos, kv_ctx[l][0], kv_ctx[l][1])
            rows.append((k, v))
        return x, self.logits(x), rows

    def logits(self, H: np.ndarray) -> np.ndarray:
        """l = RMSNorm_f(H) W_head^T."""
        return self.head @ rmsnorm(H, self.cfg.rms_eps)

    # ------------------------------------------------------------------
    # Draft head.
    # ------------------------------------------------------------------
    def draft_input(self, H_prev: np.ndarray, token: int, with_token: bool = True) -> np.ndarray:
        """h_0 (+) E(t): W_fc [H_{j-1} ; E(t_j)] (reading R1); with_token=False
        drops the token half, W_fc [H_{j-1} ; 0] (the "w/o first token" ablation, R26)."""
        e = self.embed[token] if with_token else np.zeros(self.cfg.hidden)
        return self.fc @ np.concatenate([H_prev, e])

    def draft_one(self, x: np.ndarray, pos: int, dk, dv):
        """TransformerLayer(x) at draft position `pos` over draft KV rows dk/dv."""
        return self.layer_one(self.draft, x, pos, dk, dv)
