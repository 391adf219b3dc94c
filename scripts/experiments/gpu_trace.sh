# attention phase trace (HSD_ATTN_TRACE_ON build): CTA (0,0,0) of the last verify attention launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HSD_EXTRA_NVCC=-DHSD_ATTN_TRACE_ON python -m paper_2602_21224_b200.build > /dev/null
timeout 600 python scripts/attn_trace.py ${1:-c3} ${2:-32} > gpurun_out/${TAG:-t}_trace.txt 2>&1
