cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HSD_EXTRA_NVCC=-DHSD_ATTN_TRACE_ON python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 600 python scripts/attn_trace.py c3 32 > $O/t4_default.txt 2>&1
timeout 600 python scripts/attn_trace.py c3 4 > $O/t4_b4.txt 2>&1
