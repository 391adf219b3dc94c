# ncu evidence for profiles/ (one GPU; never a multi-rank command). Round-1 refresh.
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
mkdir -p gpurun_out
O=gpurun_out
# c2: launch list of bench.py's step (launch_summary.py slices one step), then
# ncu --set full of verify layer 0's 4 GEMMs + attention, and the 2 K-TREE launches
B="python bench.py --steps 2 --warmup 1 --no-profile --no-cpu-baseline --no-e2e --no-planted"
[ -n "$SKIP_C2_LAUNCHES" ] || timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/r01_launches_c2.csv $B > $O/ncu_launch_c2.log 2>&1
NF="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 600 $NF -k regex:gemm_tc_kernel -c 4 -o $O/r01_gemm_c2 python scripts/profile_step.py c2 > $O/ncu_gemm_c2.log 2>&1
timeout 600 $NF -k regex:attention_tc_kernel -c 1 -o $O/r01_attn_c2 python scripts/profile_step.py c2 > $O/ncu_attn_c2.log 2>&1
timeout 600 $NF -k regex:tree_kernel -c 2 -o $O/r01_tree_c2 python scripts/profile_step.py c2 --stage step > $O/ncu_tree_c2.log 2>&1
# c3 (batch 32): launch list of one profiled step, verify layer-0 GEMMs + attention
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/r01_launches_c3.csv python scripts/profile_step.py c3 --stage step > $O/ncu_launch_c3.log 2>&1
timeout 900 $NF -k regex:gemm_tc -c 4 -o $O/r01_gemm_c3 python scripts/profile_step.py c3 > $O/ncu_gemm_c3.log 2>&1
timeout 900 $NF -k regex:attention_tc_kernel -c 1 -o $O/r01_attn_c3 python scripts/profile_step.py c3 > $O/ncu_attn_c3.log 2>&1
ls -la $O | tail -12
