"""Pins of the oracle FP8 (e4m3) table quantiser (oracle/fp8.py, reading R25)
against the format's bit-level definition and torch's float8_e4m3fn cast."""
import numpy as np
import pytest

from oracle.fp8 import E4M3_MAX, decode_e4m3, quantize_row, round_e4m3


def finite_values():
    vals = [decode_e4m3(c) for c in range(256)]
    return np.array([v for v in vals if not np.isnan(v)])


def test_all_finite_codes_round_trip():
    v = finite_values()
    assert len(v) == 254                       # 256 codes minus the two NaNs (+0 and -0 both finite)
    assert np.array_equal(round_e4m3(v), v)
    pos = np.unique(np.abs(v))
    assert pos.max() == 448.0 and pos[1] == 2.0 ** -9 and len(pos) == 127


def test_matches_torch_float8_e4m3fn_cast():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-448, 448, 20000), rng.normal(0, 1, 20000),
                        rng.normal(0, 0.01, 5000)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(round_e4m3(x.astype(np.float64)), ref)


def test_midpoints_round_to_even_mantissa():
    pos = np.unique(np.abs(finite_values()))
    for a, b in zip(pos[:-1], pos[1:]):
        mid = (a + b) / 2
        got = round_e4m3(np.array([mid]))[0]
        # the neighbour whose 3-bit mantissa (or subnormal count) is even
        even = a if int(round(a / _ulp(a))) % 2 == 0 else b
        assert got == even, (a, b, got)


def _ulp(a):
    if a < 2.0 ** -6:
        return 2.0 ** -9
    return 2.0 ** (np.floor(np.log2(a)) - 3)


def test_saturates():
    assert np.array_equal(round_e4m3(np.array([1000.0, -500.0, 464.1, 449.0])), [448.0, -448.0, 448.0, 448.0])


def test_row_scale_puts_amax_on_448():
    rng = np.random.default_rng(3)
    r = rng.normal(0, 1, 4096)
    r[17] = -9.5                                   # the row's largest magnitude
    deq, s = quantize_row(r)
    assert s == pytest.approx(9.5 / 448.0, rel=0, abs=0)
    assert deq[17] == pytest.approx(-9.5, rel=1e-15)
    # every entry within half an e4m3 ulp of its scaled value (3 mantissa bits -> 2^-4 relative)
    q = r / s
    assert np.all(np.abs(deq / s - q) <= np.maximum(np.abs(q) * 2.0 ** -4, 2.0 ** -10) + 1e-12)
    z, sz = quantize_row(np.zeros(8))
    assert sz == 1.0 and not z.any()


def test_fp8_table_rows_follow_the_fp64_rows():
    """TokenInfoTable(fp8=True): each row is the fp64 RMSNorm row quantised with its
    own scale; cold columns (2-D hot prune) stay exactly zero."""
    from oracle.model import Model
    from oracle.table import TokenInfoTable
    from synth import get_config, vocab_permutation
    cfg = get_config("c1").replace(vocab=256)
    m = Model(cfg, seed=0, precision="fp32")
    perm = vocab_permutation(cfg.vocab, 0)
    t64 = TokenInfoTable(m, hot_tokens=128, perm=perm)
    t8 = TokenInfoTable(m, hot_tokens=128, perm=perm, fp8=True)
    for tok in perm[:5]:
        r, q = t64.row(int(tok)), t8.row(int(tok))
        s = np.max(np.abs(r)) / E4M3_MAX
        assert np.max(np.abs(q)) == pytest.approx(np.max(np.abs(r)), rel=1e-15)
        assert np.all(q[r == 0] == 0)
        assert np.all(np.abs(q - r) <= np.maximum(np.abs(r) * 2.0 ** -4, s * 2.0 ** -10) + 1e-12)
