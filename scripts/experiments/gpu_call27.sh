cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
: > $O/c27.txt
for v in "X=0" "HSD_ATTN_SPLITS=2" "HSD_ATTN_SPLITS=3" "HSD_ATTN_SW=4" "HSD_GEMM_RING_KB=90" "HSD_GEMM_CTAS_PER_SM=1" "X=1"; do
  env $v timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-planted --no-profile > $O/c27_tmp.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$O/c27_tmp.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'])" >> $O/c27.txt
done
cat $O/c27.txt
