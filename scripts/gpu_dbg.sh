cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
NF="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 900 $NF -k regex:attention_tc2_kernel -c 1 -o gpurun_out/tc2_attn_c3 python scripts/profile_step.py c3 > gpurun_out/tc2_ncu.log 2>&1
HSD_EXTRA_NVCC=-DHSD_ATTN_TRACE_ON python -m paper_2602_21224_b200.build > /dev/null
TC2_TRACE=1 timeout 600 python scripts/attn_trace.py c3 32 > gpurun_out/tc2_trace.txt 2>&1
