"""Oracle token-info table (§5.1, :290-296; §6.1, :404-406).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  E'(t) = t^T W_E W_1 W_2
  W_collapsed = W_E W_1 W_2, a lookup table
  bias r(t) = RMSNorm(E'(t)), eps=1e-6, no gain   (reading R4)
  hot-token sparsity: for |V| > 40K keep the 32K most frequent tokens
  (PAPER.md:406), applied in 2-D: rows AND columns (reading R5) - a cold row is a
  zero bias, a cold column gets +0. The norm is taken over the full |V| row
  before cutting.
"""
from __future__ import annotations

import numpy as np

from .fp8 import quantize_row
from .philox import round_bf16

TABLE_EPS = 1e-6


def table_bytes(vocab: int, bytes_per_entry: int) -> int:
    """|V|^2 entries ('stored as a matrix of size |V|^2')."""
    return vocab * vocab * bytes_per_entry


def collapse_row(model, t: int) -> np.ndarray:
    """E'(t) = W_E[t] W_1 W_2 (paper orientation; stored w1 = W_1^T, w2 = W_2^T)."""
    return model.w2 @ (model.w1 @ model.embed[t])


class TokenInfoTable:
    """Row lookup r(t) over the full vocabulary (zero for cold rows/columns).

    Rows are computed on demand from the factors (the collapsed matrix is
    W_collapsed row t); `precision='bf16'` rounds stored entries to bfloat16 as
    the GPU table stores them (SURVEY.md §8(a) init row); `fp8=True` stores
    them as e4m3 codes with one scale per row instead (R25)."""

    def __init__(self, model, hot_tokens: int = 0, perm: np.ndarray | None = None,
                 zero: bool = False, fp8: bool = False):
        self.model = model
        self.fp8 = fp8       # FP8 e4m3 rows with a per-row scale (reading R25, oracle/fp8.py)
        V = model.cfg.vocab
        self.V = V
        self.zero = zero
        self.hot = np.ones(V, dtype=bool)
        if hot_tokens:
            assert perm is not None, "hot pruning needs the vocab permutation"
            self.hot = np.zeros(V, dtype=bool)
            self.hot[perm[:hot_tokens]] = True
        self._cache = {}

    def fp64_row(self, t: int) -> np.ndarray:
        """The row before storage rounding: RMSNorm over the full row, cold columns 0."""
        if self.zero or not self.hot[t]:
            return np.zeros(self.V)
        r = collapse_row(self.model, t)
        r = r / np.sqrt(np.mean(r * r) + TABLE_EPS)            # RMSNorm over the full row
        return np.where(self.hot, r, 0.0)                      # 2-D prune: cold columns

    def row(self, t: int) -> np.ndarray:
        if self.zero or not self.hot[t]:
            return np.zeros(self.V)
        if t not in self._cache:
            r = self.fp64_row(t)
            if self.fp8:
                r, _ = quantize_row(r)                         # cold columns stay exactly 0
            elif self.model.precision == "bf16":
                r = round_bf16(r.astype(np.float32)).astype(np.float64)
            self._cache[t] = r
        return self._cache[t]


class ExplicitTable:
    """A table given as an explicit dict token -> bias row (tests, Fig. 5)."""

    def __init__(self, V: int, rows: dict | None = None):
        self.V = V
        self.rows = rows or {}

    def row(self, t: int) -> np.ndarray:
        return np.asarray(self.rows.get(t, np.zeros(self.V)), dtype=np.float64)
