"""Oracle FP8 (e4m3) quantisation of the token-info table.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper stores the |V|^2 table in FP8 ("15.3 GB FP8 at
128,256"). It does not name the FP8 format or the scaling; reading R25
(DESIGN.md): OCP E4M3 ("e4m3fn": 1 sign, 4 exponent bits with bias 7, 3
mantissa bits, no infinities, max finite 448, subnormal step 2^-9), one fp32
scale per table row s_t = max_j |r_t[j]| / 448, codes q = RNE_e4m3(r_t / s_t)
with saturation to +-448, lookup r_t ~ q * s_t.

Pins (tests/test_oracle_fp8.py): every one of the 254 finite codes decoded bit
by bit round-trips; torch's float8_e4m3fn cast (a library routine) agrees on
random in-range values; midpoints round to the even mantissa; out-of-range
values saturate; a quantised row has max |q| == 448 exactly.
"""
from __future__ import annotations

import numpy as np

E4M3_MAX = 448.0
E4M3_MIN_NORMAL = 2.0 ** -6
E4M3_SUBNORMAL_STEP = 2.0 ** -9


def round_e4m3(x) -> np.ndarray:
    """Nearest e4m3 value (ties to even mantissa), saturating to +-448."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    out = np.empty_like(a)
    sub = a < E4M3_MIN_NORMAL
    # subnormal range (and zero): uniform step 2^-9; rounding up to 2^-6 is the min normal
    out[sub] = np.round(a[sub] / E4M3_SUBNORMAL_STEP) * E4M3_SUBNORMAL_STEP   # np.round: half to even
    nrm = ~sub
    e = np.floor(np.log2(a[nrm]))
    step = 2.0 ** (e - 3)                     # 3 mantissa bits
    out[nrm] = np.round(a[nrm] / step) * step  # may carry into the next binade: still exact
    out = np.minimum(out, E4M3_MAX)            # satfinite
    return np.copysign(out, x)


def quantize_row(r: np.ndarray):
    """(dequantised row, scale) for one table row: s = amax / 448, q = e4m3(r / s)."""
    r = np.asarray(r, dtype=np.float64)
    amax = float(np.max(np.abs(r))) if r.size else 0.0
    s = amax / E4M3_MAX if amax > 0 else 1.0
    q = round_e4m3(r / s)
    return q * s, s


def decode_e4m3(code: int) -> float:
    """Value of an e4m3fn byte from its bit fields (NaN for 0x7f / 0xff)."""
    sign = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 0xF and m == 0x7:
        return float("nan")
    if e == 0:
        return sign * (m / 8.0) * 2.0 ** -6
    return sign * (1.0 + m / 8.0) * 2.0 ** (e - 7)
