"""Philox4x32-10 counter-based generator (Salmon et al., SC'11, "Random123").

Oracle side (test infrastructure, see oracle/__init__.py). The CUDA side has
its own independent implementation; both must reproduce the published
known-answer vectors (tests/test_oracle_philox.py).

Streams used by the method (DESIGN.md §"Random streams"):
  weights : key=(seed, tensor_id), counter=(e//4 lo, e//4 hi, 0, 0), word e%4;
            u = (x>>8)*2^-24, w = fp32(s) * fp32(2u-1)
  accept  : key=(seed, 0x5EED0001), counter=(slot, rank, step, req), word 0
  gumbel  : key=(seed, 0x5EED0002), counter=(v//4, slot, step, req), word v%4
  plant   : key=(seed, 0x5EED0003), counter=(depth, step, req, 0), word 0
  sampling uniforms are u = ((x>>9)+0.5)*2^-23 in (0,1): 2^23 values, each exact
  in float32 (k+0.5 < 2^23 needs 24 significant bits), so the GPU's fp32 u is
  this float64 u bit for bit; min 2^-24, max 1-2^-24.
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)

TAG_ACCEPT = 0x5EED0001
TAG_GUMBEL = 0x5EED0002
TAG_PLANT = 0x5EED0003


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32 with 10 rounds. Inputs: uint32-valued arrays or
    scalars (broadcast). Returns a tuple of four uint32 numpy arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK
    k1 = np.asarray(k1, dtype=np.uint64) & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0            # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return tuple(np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))


def raw_stream(seed: int, tensor_id: int, count: int) -> np.ndarray:
    """The first `count` 32-bit words of stream (seed, tensor_id): word e comes
    from counter e//4, output lane e%4."""
    nblk = (count + 3) // 4
    idx = np.arange(nblk, dtype=np.uint64)
    out = philox4x32_10(idx & MASK, idx >> np.uint64(32), 0, 0, seed & 0xFFFFFFFF, tensor_id)
    words = np.stack(out, axis=1).reshape(-1)
    return words[:count]


_CHUNK = 1 << 22      # elements per worker chunk (a multiple of 4: whole Philox blocks)


def _uniform_chunk(seed, tensor_id, scale, e0, e1, out):
    """Elements [e0, e1) of uniform_weights' stream into out[e0:e1] (e0 % 4 == 0)."""
    idx = np.arange(e0 // 4, (e1 + 3) // 4, dtype=np.uint64)
    words = np.stack(philox4x32_10(idx & MASK, idx >> np.uint64(32), 0, 0, seed & 0xFFFFFFFF, tensor_id),
                     axis=1).reshape(-1)[:e1 - e0]
    u = (words >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    t = np.float32(2.0) * u - np.float32(1.0)        # exact
    out[e0:e1] = (np.float32(scale) * t).astype(np.float32)


def uniform_weights(seed: int, tensor_id: int, shape, scale: np.float32) -> np.ndarray:
    """w = s*(2u-1), u=(x>>8)*2^-24, every step in float32 (exact except the one
    correctly-rounded multiply). Returned as float32. Large tensors are generated
    in independent element ranges on a thread pool (numpy releases the GIL); each
    element's value depends only on its own counter, so the result is the same."""
    count = int(np.prod(shape))
    out = np.empty(count, dtype=np.float32)
    ranges = [(e0, min(count, e0 + _CHUNK)) for e0 in range(0, count, _CHUNK)]
    if len(ranges) <= 1:
        for e0, e1 in ranges:
            _uniform_chunk(seed, tensor_id, scale, e0, e1, out)
    else:
        import os
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(ranges), os.cpu_count() or 1)) as ex:
            list(ex.map(lambda r: _uniform_chunk(seed, tensor_id, scale, r[0], r[1], out), ranges))
    return out.reshape(shape)


def linear_scale(fan_in: int) -> np.float32:
    """s = sqrt(3/fan_in) in float32 (IEEE division and sqrt, both correctly rounded)."""
    return np.sqrt(np.float32(3.0) / np.float32(fan_in)).astype(np.float32)


def unit_open(x: np.ndarray) -> np.ndarray:
    """Sampling uniform in (0,1): ((x>>9)+0.5)*2^-23, float64; every value is
    exactly representable in float32 (the GPU computes the same number)."""
    return ((x >> np.uint32(9)).astype(np.float64) + 0.5) * 2.0 ** -23


def accept_uniform(seed: int, req: int, step: int, slot: int, rank: int) -> float:
    w = philox4x32_10(slot, rank, step, req, seed & 0xFFFFFFFF, TAG_ACCEPT)[0]
    return float(unit_open(np.asarray(w))[()])


def gumbel_uniforms(seed: int, req: int, step: int, slot: int, vocab: int) -> np.ndarray:
    """U_v for v in [0, vocab): counter (v//4, slot, step, req), word v%4."""
    nblk = (vocab + 3) // 4
    blk = np.arange(nblk, dtype=np.uint64)
    out = philox4x32_10(blk, slot, step, req, seed & 0xFFFFFFFF, TAG_GUMBEL)
    words = np.stack(out, axis=1).reshape(-1)[:vocab]
    return unit_open(words)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 (round to nearest even) -> float32 values."""
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return (r & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)


def uniform_rows(seed: int, tensor_id: int, cols: int, scale: np.float32, rows, precision="fp32") -> np.ndarray:
    """Rows `rows` of the [*, cols] weight tensor (seed, tensor_id), without
    generating the rest: element (r, c) is stream word r*cols + c. Same
    arithmetic as uniform_weights (R23); float64 result."""
    out = np.empty((len(rows), cols), dtype=np.float64)
    for i, r in enumerate(rows):
        e0 = int(r) * cols
        b0, b1 = e0 // 4, (e0 + cols + 3) // 4
        idx = np.arange(b0, b1, dtype=np.uint64)
        w = np.stack(philox4x32_10(idx & MASK, idx >> np.uint64(32), 0, 0, seed & 0xFFFFFFFF, tensor_id),
                     axis=1).reshape(-1)[e0 - 4 * b0: e0 - 4 * b0 + cols]
        u = (w >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
        x = (np.float32(scale) * (np.float32(2.0) * u - np.float32(1.0))).astype(np.float32)
        if precision == "bf16":
            x = round_bf16(x)
        out[i] = x.astype(np.float64)
    return out
