cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "fullsize_logits or production_k or serving or parity" 2>&1 | tail -15 > $O/r2c_tests.txt
NF="ncu --set full --clock-control none --import-source on --profile-from-start off --metrics sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum"
timeout 900 $NF -k regex:gemm_tc -c 4 -o $O/r02_gemm_c3 python scripts/profile_step.py c3 > $O/ncu_gemm_c3.log 2>&1
timeout 900 $NF -k regex:attention_tc_kernel -c 1 -o $O/r02_attn_c3 python scripts/profile_step.py c3 > $O/ncu_attn_c3.log 2>&1
tail -3 $O/r2c_tests.txt
