"""One-line summaries of bench.py JSON lines: python scripts/bench_summary.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:
        print(f, "unreadable", ex)
        continue
    r = d.get("roofline") or {}
    oe = r.get("other_kernels_eager", {}).get("attn_verify", {})
    ag = r.get("attn_verify_in_graph", {})
    prof = d.get("profile_ms_per_step", {})
    print(f"{f}: {d['config']['workload']} {d['value']} tok/s {d['ms_per_step']} ms/step launches {d.get('gpu_launches')} "
          f"| {r.get('kernel')} frac {r.get('frac')} | attn eager {oe.get('frac')} ({oe.get('us_per_launch')} us) "
          f"in-graph {ag.get('frac')} ({ag.get('us_per_launch')} us) | clocks {d.get('clocks', {}).get('sm_mhz')}")
    print("   ", {k: v for k, v in prof.items()})
