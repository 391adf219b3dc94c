cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out; T=${TAG:-m}
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "wide_bf16 or capacity_far or fullsize_logits or c3_stochastic or c5" 2>&1 | tail -5 > $O/${T}_tests.txt
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err
HSD_EXTRA_NVCC=-DHSD_ATTN_TRACE_ON python -m paper_2602_21224_b200.build > /dev/null
timeout 600 python scripts/attn_trace.py c3 32 > $O/${T}_trace.txt 2>&1
