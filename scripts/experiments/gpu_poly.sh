# A/B of the FMA-pipe exp2 share in tree attention (HSD_ATTN_POLY 0/1/2): step time c2/c3, trace, parity
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted --steps 20"
for cfg in c3 c2; do for p in 0 1 2; do
  HSD_ATTN_POLY=$p timeout 900 $B --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg poly=$p', d['ms_per_step'], 'attn_verify', d['profile_ms_per_step'].get('attn_verify'))"
done; done
HSD_ATTN_POLY=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" 2>&1 | tail -2
HSD_ATTN_POLY=2 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
