#!/bin/bash
# sweep the attention key-split count (HSD_ATTN_SPLITS) on c3 and c5 (batch 2)
python -m paper_2602_21224_b200.build >/dev/null
for cfg in "c3" "c5 --batch 2"; do
  for s in 0 1 2 3 4 6 8 12; do
    r=$(HSD_ATTN_SPLITS=$s timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-planted 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['profile_ms_per_step']['attn_verify'])")
    echo "$cfg S=$s $r"
  done
done
