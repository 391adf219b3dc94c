# A/B: softmax warps per TMEM lane quarter in tree attention (HSD_ATTN_SW 2 / 4)
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted --steps 20"
for cfg in c3 c2; do for w in 2 4; do
  HSD_ATTN_SW=$w timeout 900 $B --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg SW=$w', d['ms_per_step'], 'attn_verify', d['profile_ms_per_step'].get('attn_verify'), 'attn_draft', d['profile_ms_per_step'].get('attn_draft'))"
done; done
HSD_ATTN_SW=4 python scripts/attn_trace.py c2 1 | head -12
HSD_ATTN_SW=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" 2>&1 | tail -2
HSD_ATTN_SW=4 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
