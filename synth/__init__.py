"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no model, no tree, no
sampling rule). It only produces inputs: configuration presets (public model
shapes), the seeded vocabulary permutation that defines the
hot-token set, and Zipf-distributed prompts over it (SURVEY.md §8(d.2):
"token ids ~ Zipf(s = 1.1) over a seeded vocab permutation (prompt seed 1234 +
request id)"). Both the oracle side and the CUDA side consume these values as
plain arrays; neither side imports the other.
"""
from __future__ import annotations

import dataclasses
import numpy as np

# ---------------------------------------------------------------------------
# Configuration presets (BASELINE.json configs[0..4]).
# Model shapes are the public configs of the named models; the paper itself only
# names LLaMA-2-7B / Vicuna-7B. Tree parameters per SURVEY.md §8.
# ---------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    vocab: int
    hidden: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float
    rms_eps: float
    steps_N: int          # draft steps = tree depth (Alg. 1 N)
    branch_k: int         # branch number k (Alg. 1)
    budget_B: int         # verification budget B, non-root nodes
    resample_budget_Br: int = 4   # SPEC.md:459 default
    resample_threshold_r: int = 1  # SPEC.md:390 default
    hot_tokens: int = 0   # 0 = dense table; else V_h hot tokens
    batch: int = 1
    prompt_len: int = 32
    max_new: int = 64
    accept: str = "greedy"   # "greedy" | "stochastic"
    temperature: float = 1.0

    @property
    def table_rank(self) -> int:
        # d = n/16: the paper never gives d; reading R7.
        return max(1, self.hidden // 16)

    @property
    def verify_slots(self) -> int:
        return self.budget_B + self.resample_budget_Br + 1

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    "c1": Config("c1", vocab=256, hidden=64, layers=2, q_heads=4, kv_heads=4, head_dim=16,
                 ffn=256, rope_theta=10000.0, rms_eps=1e-5, steps_N=4, branch_k=2,
                 budget_B=8, batch=1, prompt_len=32, max_new=64),
    "c2": Config("c2", vocab=32000, hidden=4096, layers=32, q_heads=32, kv_heads=32,
                 head_dim=128, ffn=11008, rope_theta=10000.0, rms_eps=1e-5, steps_N=6,
                 branch_k=4, budget_B=60, batch=1, prompt_len=1024, max_new=256),
    "c3": Config("c3", vocab=128256, hidden=4096, layers=32, q_heads=32, kv_heads=8,
                 head_dim=128, ffn=14336, rope_theta=500000.0, rms_eps=1e-5, steps_N=6,
                 branch_k=4, budget_B=60, hot_tokens=32768, batch=32, prompt_len=4096,
                 max_new=128, accept="stochastic"),
    "c4": Config("c4", vocab=32000, hidden=5120, layers=40, q_heads=40, kv_heads=40,
                 head_dim=128, ffn=13824, rope_theta=10000.0, rms_eps=1e-5, steps_N=6,
                 branch_k=6, budget_B=128, batch=64, prompt_len=1024, max_new=128),
    "c5": Config("c5", vocab=128256, hidden=8192, layers=80, q_heads=64, kv_heads=8,
                 head_dim=128, ffn=28672, rope_theta=500000.0, rms_eps=1e-5, steps_N=6,
                 branch_k=4, budget_B=60, hot_tokens=32768, batch=16, prompt_len=8192,
                 max_new=64),
}


def get_config(name: str, **overrides) -> Config:
    return CONFIGS[name].replace(**overrides)


# ---------------------------------------------------------------------------
# Vocabulary permutation and prompts.
# ---------------------------------------------------------------------------

def vocab_permutation(vocab: int, seed: int = 0) -> np.ndarray:
    """rank -> token id. Rank 0 is the most frequent token of the synthetic Zipf
    law; the first V_h ranks are the hot set (reading R5)."""
    rng = np.random.default_rng(np.uint64(0x9E3779B97F4A7C15) ^ np.uint64(seed))
    return rng.permutation(vocab).astype(np.int32)


def zipf_ranks(vocab: int, count: int, seed: int, s: float = 1.1) -> np.ndarray:
    """`count` i.i.d. ranks with P(r) proportional to (r+1)^-s, r in [0, vocab)."""
    w = np.arange(1, vocab + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rng = np.random.default_rng(seed)
    u = rng.random(count)
    return np.minimum(np.searchsorted(cdf, u, side="right"), vocab - 1).astype(np.int64)


def prompts(cfg: Config, batch: int | None = None, length: int | None = None,
            perm_seed: int = 0, prompt_seed: int = 1234) -> np.ndarray:
    """[batch, length] int32 prompt tokens: request r uses seed prompt_seed + r."""
    batch = cfg.batch if batch is None else batch
    length = cfg.prompt_len if length is None else length
    perm = vocab_permutation(cfg.vocab, perm_seed)
    out = np.empty((batch, length), dtype=np.int32)
    for r in range(batch):
        out[r] = perm[zipf_ranks(cfg.vocab, length, prompt_seed + r)]
    return out


def shard_requests(n_requests: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of requests owned by `rank`: [lo, hi)."""
    base, extra = divmod(n_requests, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi
