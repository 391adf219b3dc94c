cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
HSD_ATTN_PAIR=0 timeout 900 python -m pytest tests -m gpu -q -x -k "wide_bf16 or capacity_far or lockstep_c1_bf16" 2>&1 | tail -3 > gpurun_out/dbg.txt
HSD_ATTN_PAIR=0 timeout 300 python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline --no-planted --no-e2e > gpurun_out/dbg_c3.json 2>&1
HSD_ATTN_PAIR=0 timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-e2e > gpurun_out/dbg_c2.json 2>&1
HSD_EXTRA_NVCC=-DHSD_ATTN_TRACE_ON python -m paper_2602_21224_b200.build > /dev/null
HSD_ATTN_PAIR=0 timeout 600 python scripts/attn_trace.py c3 32 > gpurun_out/dbg_trace.txt 2>&1
