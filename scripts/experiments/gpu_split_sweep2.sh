#!/bin/bash
python -m paper_2602_21224_b200.build >/dev/null
for s in 0 3 4 5 6; do
  r=$(HSD_ATTN_SPLITS=$s timeout 600 python bench.py --config c2 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-planted 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['profile_ms_per_step']['attn_verify'], d['profile_ms_per_step']['attn_draft'])")
  echo "c2 S=$s $r"
done
for cfg in "c3" "c5 --batch 2"; do
  r=$(timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-planted 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['profile_ms_per_step']['attn_verify'])")
  echo "$cfg auto $r"
done
