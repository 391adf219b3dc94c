cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
: > $O/c30.txt
for v in "X=0" "HSD_ATTN_SW=2" "HSD_L2PF_MB=0" "HSD_GEMM_TMA_OUT=1" "HSD_ATTN_DYNSPLIT=0" "X=1"; do
  env $v timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c30_tmp.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$O/c30_tmp.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])" >> $O/c30.txt
done
cat $O/c30.txt
