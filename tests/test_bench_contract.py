"""bench.py's JSON-line contract (the driver parses it): the reference arm runs on
CPU here (it times the oracle), the GPU arm on a B200 with a tiny config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "tokens/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "c1" and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0 and 0 < r["frac"] and r["unit"] in ("GB/s", "TFLOP/s")
    assert "traffic" in r
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["step_latency_ms"]["median"] > 0 and d["verify_latency_ms"]["median"] > 0


def test_plan_shard_weak_and_strong():
    """weak-scaled configs give every rank its own fixed block of
    requests (distinct prompts and global request ids, never duplicated work);
    strong-scaled configs split the fixed global batch into a partition."""
    sys.path.insert(0, ROOT)
    from bench import plan_shard
    for world in (1, 2, 4, 8):
        blocks = [plan_shard("c3", 32, world, r) for r in range(world)]
        assert all(b[2] == 32 * world and b[3] == "weak" and b[1] - b[0] == 32 for b in blocks)
        assert sorted(x for b in blocks for x in range(b[0], b[1])) == list(range(32 * world))
        reps = [plan_shard("c2", 1, world, r) for r in range(world)]
        assert [(b[0], b[1]) for b in reps] == [(r, r + 1) for r in range(world)]
        st = [plan_shard("c4", 64, world, r) for r in range(world)]
        assert all(b[2] == 64 and b[3] == "strong" for b in st)
        assert sorted(x for b in st for x in range(b[0], b[1])) == list(range(64))
    assert plan_shard("c3", 32, 2, 1, batch_per_gpu=8)[:3] == (8, 16, 16)
    assert plan_shard("c3", 32, 2, 1, strong=True)[:4] == (16, 32, 32, "strong")
