# qkv_rope_kv: loads hoisted ahead of stores -- step time c2/c3/c4 + parity
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted"
for cfg in "c2 --steps 30" "c3 --steps 20" "c4 --steps 6"; do
  timeout 900 $B --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['roofline']['frac'], 'rowwise', d['profile_ms_per_step'].get('rowwise'))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
