# A/B: CTA-pair data-parallel GEMMs for c3's QKV / O / down (HSD_GEMM_DP_WAVE)
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted --steps 20"
for cfg in c3 c2 "c5 --batch 2"; do for w in 0 1; do
  HSD_GEMM_DP_WAVE=$w timeout 900 $B --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg wave=$w', d['ms_per_step'], d['roofline']['frac'], 'gemm_verify', d['profile_ms_per_step'].get('gemm_verify'))"
done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
