# A/B: device-side even key splits over the visible chunks + one-wave cap (HSD_ATTN_DYNSPLIT)
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted"
for cfg in "c2 --steps 30" "c5 --batch 2 --steps 10" "c3 --steps 20"; do for d in 0 1; do
  HSD_ATTN_DYNSPLIT=$d timeout 900 $B --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg dyn=$d', d['ms_per_step'], 'attn_verify', d['profile_ms_per_step'].get('attn_verify'))"
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
