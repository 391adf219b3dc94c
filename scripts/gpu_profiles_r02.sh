# ncu evidence for profiles/ (one GPU; never a multi-rank command). Round 2.
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
mkdir -p gpurun_out
O=gpurun_out
M="--metrics sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum"
NF="ncu --set full --clock-control none --import-source on --profile-from-start off $M"
# c3 (the bench default): launch list of one profiled step, verify layer-0 GEMMs + attention, K-TREE
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/r02_launches_c3.csv python scripts/profile_step.py c3 --stage step > $O/ncu_launch_c3.log 2>&1
timeout 900 $NF -k regex:gemm_tc -c 4 -o $O/r02_gemm_c3 python scripts/profile_step.py c3 > $O/ncu_gemm_c3.log 2>&1
timeout 900 $NF -k regex:attention_tc_kernel -c 1 -o $O/r02_attn_c3 python scripts/profile_step.py c3 > $O/ncu_attn_c3.log 2>&1
timeout 900 $NF -k regex:tree_kernel -c 2 -o $O/r02_tree_c3 python scripts/profile_step.py c3 --stage step > $O/ncu_tree_c3.log 2>&1
# c2: launch list of one profiled step + the verify layer-0 GEMMs and attention
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/r02_launches_c2.csv python scripts/profile_step.py c2 --stage step > $O/ncu_launch_c2.log 2>&1
timeout 900 $NF -k regex:gemm_tc -c 4 -o $O/r02_gemm_c2 python scripts/profile_step.py c2 > $O/ncu_gemm_c2.log 2>&1
timeout 900 $NF -k regex:attention_tc_kernel -c 1 -o $O/r02_attn_c2 python scripts/profile_step.py c2 > $O/ncu_attn_c2.log 2>&1
ls -la $O | grep r02
