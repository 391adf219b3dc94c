"""GPU tests of the serving-layer entry points around the path:
ragged prompt lengths in one batch and continuous batching (hsd_admit replaces the
request in one slot while the others keep decoding).

Pinned by losslessness: in fp32-verify greedy mode every slot's
emitted stream must equal the oracle's plain greedy decode of that slot's prompt,
before and after another slot is re-admitted.
"""
import numpy as np
import pytest

from synth import get_config, prompts
from oracle.model import Model
from oracle.engine import greedy_decode

pytestmark = pytest.mark.gpu

hsd = pytest.importorskip("paper_2602_21224_b200.hsd")


def _collect(ctx, steps, out):
    for _ in range(steps):
        e, n = ctx.step_host()
        for r in range(e.shape[0]):
            out[r] += [int(t) for t in e[r, :n[r]]]


@pytest.mark.parametrize("precision", [hsd.FP32_VERIFY])
def test_ragged_batch_then_admit_is_lossless(precision):
    cfg = get_config("c1").replace(batch=3)
    base = prompts(cfg, batch=3)
    lens = [20, 32, 9]                                     # ragged
    stride = max(lens)
    toks = np.zeros((3, stride), np.int32)
    for r, L in enumerate(lens):
        toks[r, :L] = base[r][:L]
    fresh = np.array(prompts(cfg.replace(prompt_len=27), batch=5)[4], np.int32)   # a new request
    steps = 6
    ctx = hsd.init_model(cfg, device=0, precision=precision, seed=2, max_batch=3,
                         max_ctx=64 + 3 * steps * (cfg.steps_N + 1))
    ctx.prefill(toks, lens)
    first = [[int(x)] for x in ctx.tensor("root_tok").cpu().numpy()]    # the first token of each slot
    got = [list(f) for f in first]
    _collect(ctx, steps, got)
    ctx.admit(1, fresh, 7)                                 # slot 1: new request, others continue
    got_admit = [int(ctx.tensor("root_tok").cpu().numpy()[1])]
    rest = [[], [], []]
    _collect(ctx, steps, rest)
    ctx.destroy()

    m = Model(cfg, seed=2, precision="fp32")
    for r in (0, 2):                                      # untouched slots: one uninterrupted decode
        stream = got[r] + rest[r]
        ref, _ = greedy_decode(m, toks[r, :lens[r]], len(stream) + 1)
        assert stream == list(ref[:len(stream)]), f"slot {r} diverged from its greedy decode"
    ref1, _ = greedy_decode(m, toks[1, :lens[1]], len(got[1]) + 1)
    assert got[1] == list(ref1[:len(got[1])])
    stream1 = got_admit + rest[1]                         # the admitted request from its first token
    refn, _ = greedy_decode(m, fresh, len(stream1) + 1)
    assert stream1 == list(refn[:len(stream1)]), "admitted request != its greedy decode"
    assert len(rest[1]) >= steps                          # it really decoded after admission


def test_admit_contract():
    cfg = get_config("c1").replace(batch=2)
    ctx = hsd.init_model(cfg, device=0, precision=hsd.FP32_VERIFY, seed=0, max_batch=2, max_ctx=96)
    with pytest.raises(hsd.HsdError) as e:
        ctx.admit(0, [1, 2, 3], 5)                         # before prefill
    assert e.value.status == hsd.HSD_ESTATE
    ctx.prefill(np.stack(prompts(cfg, batch=2)))
    for bad_slot, toks in [(2, [1, 2, 3]), (-1, [1, 2, 3]), (0, [5]), (0, [1, cfg.vocab])]:
        with pytest.raises(hsd.HsdError) as e:
            ctx.admit(bad_slot, toks, 5)
        assert e.value.status == hsd.HSD_EINVAL
    ctx.destroy()


def test_step_refuses_at_kv_capacity():
    """Capacity contract (include/hsd.h, hsd_prefill): a step writes KV rows up to
    p + T - 1, so once a slot's committed length could pass max_pos - T, hsd_step
    returns HSD_ESTATE and launches nothing -- never writing past the slot's pages
    into the next request's. The host bound is refreshed from the device's p, so
    a slot is refused only when it is really full."""
    cfg = get_config("c1").replace(batch=2)
    ctx = hsd.init_model(cfg, device=0, precision=hsd.FP32_VERIFY, seed=0, max_batch=2, max_ctx=40)
    ctx.prefill(np.stack(prompts(cfg, batch=2)))
    T = cfg.budget_B + cfg.resample_budget_Br + 1
    page = 64
    max_pos = ctx.tensor("kv").shape[1] // 2 * page
    refused = False
    for _ in range(200):
        p = ctx.tensor("p").cpu().numpy()
        try:
            ctx.step_host()
        except hsd.HsdError as e:
            assert e.status == hsd.HSD_ESTATE and "capacity" in str(e)
            assert int(p.max()) + T > max_pos            # refused only when really full
            refused = True
            break
        assert int(ctx.tensor("p").cpu().numpy().max()) <= max_pos
    assert refused
    # the refusal is sticky and harmless: a second call refuses again, state unchanged
    p_before = ctx.tensor("p").cpu().numpy().copy()
    with pytest.raises(hsd.HsdError):
        ctx.step_host()
    assert np.array_equal(ctx.tensor("p").cpu().numpy(), p_before)
    ctx.destroy()
