"""CPU-side checks of the C ABI boundary (no GPU needed): the library loads,
exports every symbol include/hsd.h declares, the ctypes structs match the C
layout, and host-checked contract violations return HSD_EINVAL before any
CUDA call."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from synth import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hsd():
    from paper_2602_21224_b200 import hsd as h
    if not os.path.exists(h.LIB_PATH):
        from paper_2602_21224_b200.build import build
        build()
    h.load()
    return h


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hsd.h")).read()
    return sorted(set(re.findall(r"\b(hsd_[a-z_]+)\s*\(", text)))


def test_exports_every_declared_symbol(hsd):
    lib = hsd.load()
    names = declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(hsd.EXPORTS) == set(names)


def test_struct_layout_matches_c(hsd):
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "hsd.h"
int main(){ printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(hsd_config), offsetof(hsd_config, seed),
  offsetof(hsd_config, vocab_perm), offsetof(hsd_config, plant_rates), sizeof(hsd_tensor),
  sizeof(hsd_tree_view), sizeof(hsd_verify_view), offsetof(hsd_config, vocab_shards),
  offsetof(hsd_config, nccl_id)); return 0; }
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        got = list(map(int, subprocess.check_output([exe]).split()))
    py = [ctypes.sizeof(hsd.HsdConfig), hsd.HsdConfig.seed.offset, hsd.HsdConfig.vocab_perm.offset,
          hsd.HsdConfig.plant_rates.offset, ctypes.sizeof(hsd.Tensor), ctypes.sizeof(hsd.TreeView),
          ctypes.sizeof(hsd.VerifyView), hsd.HsdConfig.vocab_shards.offset, hsd.HsdConfig.nccl_id.offset]
    assert got == py


@pytest.mark.parametrize("bad", [dict(steps_N=0), dict(budget_B=0), dict(branch_k=9),
                                 dict(vocab=1), dict(kv_heads=3), dict(hot_tokens=16),
                                 dict(shard_mode=3, vocab_shards=2),
                                 dict(shard_mode=2, vocab_shards=17),
                                 dict(shard_mode=2, vocab_shards=3),          # c1: V = 256 < 128 * 3
                                 dict(shard_mode=2, vocab_shards=2, shard_rank=1),
                                 dict(shard_mode=1, vocab_shards=2, shard_rank=2)])
def test_invalid_config_rejected_before_cuda(hsd, bad):
    cfg = get_config("c1")
    c, keep = hsd.make_config(cfg)
    for k, v in bad.items():
        setattr(c, k, v)
    h = ctypes.c_void_p()
    s = hsd.load().hsd_init_model(ctypes.byref(c), 0, None, ctypes.byref(h))
    assert s == hsd.HSD_EINVAL and not h.value


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_21224_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_sharded_stochastic_needs_room_for_a_candidate(hsd):
    """Stochastic acceptance over the vocab-sharded head merges each shard's Gumbel
    top-16 (R29): the largest rejected set (<= branch_k + B_r children) must leave
    a candidate, so branch_k + B_r >= 16 is refused with HSD_EUNSUP before any CUDA
    call (nothing allocated). The token-AR draft is not combined with sharding."""
    c, keep = hsd.make_config(get_config("c1").replace(branch_k=8, resample_budget_Br=8), accept="stochastic", temperature=1.0,
                              shard_mode=hsd.SHARD_SIM, vocab_shards=2)
    h = ctypes.c_void_p()
    s = hsd.load().hsd_init_model(ctypes.byref(c), 0, None, ctypes.byref(h))
    assert s == hsd.HSD_EUNSUP and not h.value
    c, keep = hsd.make_config(get_config("c1"), accept="greedy", shard_mode=hsd.SHARD_SIM, vocab_shards=2,
                              flags=hsd.FLAG_RESAMPLE | hsd.FLAG_FUSION | hsd.FLAG_TOKEN_AR)
    s = hsd.load().hsd_init_model(ctypes.byref(c), 0, None, ctypes.byref(h))
    assert s == hsd.HSD_EUNSUP and not h.value


def test_vocab_shard_bounds(hsd):
    """Shard column bounds (include/hsd.h): 128-aligned starts, cover [0, V) exactly,
    every shard non-empty, widths differ by at most 128 + V mod 128."""
    for V, G in [(256, 2), (32000, 8), (128256, 8), (128256, 3), (1000, 7), (128256, 16)]:
        lo = hsd.vocab_shard_bounds(V, G)
        assert lo[0] == 0 and lo[-1] == V and len(lo) == G + 1
        assert all(x % 128 == 0 for x in lo[:-1])
        w = [b - a for a, b in zip(lo, lo[1:])]
        assert min(w) >= 1 and sum(w) == V
        assert max(w) - min(w) <= 128 + V % 128


def test_nccl_unique_id_loads_nccl_at_run_time(hsd):
    """hsd_nccl_unique_id dlopens libnccl.so.2 (no link-time NCCL dependency) and
    returns 128 fresh bytes (host only, no device work)."""
    a, b = hsd.nccl_unique_id(), hsd.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
