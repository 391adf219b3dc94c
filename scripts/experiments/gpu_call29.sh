cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
: > $O/c29.txt
for v in "X=0" "HSD_L2PF_MB=0" "HSD_L2PF_MB=48" "HSD_L2PF_MB=160" "HSD_GEMM_MIN_STAGES=4" "HSD_ATTN_CLUSTER_MAX=4" "X=1"; do
  env $v timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-planted --no-profile > $O/c29_tmp.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$O/c29_tmp.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'])" >> $O/c29.txt
done
cat $O/c29.txt
