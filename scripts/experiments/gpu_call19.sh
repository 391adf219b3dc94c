cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
M="--metrics sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum"
HSD_ATTN_DUAL=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off $M -k regex:attention_dual -c 1 -o $O/c19_dual python scripts/profile_step.py c3 > $O/c19.log 2>&1
tail -2 $O/c19.log
