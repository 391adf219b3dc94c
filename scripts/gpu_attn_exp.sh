# attention timing experiments on c3 (bench line per variant) + ncu of the current kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out; T=${TAG:-x}
B="python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline --no-planted --no-e2e"
timeout 300 $B > $O/${T}_base.json 2>&1
HSD_ATTN_EXP=1 timeout 300 $B > $O/${T}_notile3.json 2>&1
NF="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 900 $NF -k regex:attention_tc_kernel -c 1 -o $O/${T}_attn_c3 python scripts/profile_step.py c3 > $O/${T}_ncu.log 2>&1
