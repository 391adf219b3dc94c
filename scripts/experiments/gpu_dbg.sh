cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or c4 or fullsize_logits" 2>&1 | tail -2 > gpurun_out/dbg.txt
for i in 1 2; do timeout 300 python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline --no-planted --no-e2e > gpurun_out/dbg_c3.json 2>&1; python scripts/bench_summary.py gpurun_out/dbg_c3.json >> gpurun_out/dbg.txt; done
NF="ncu --set full --clock-control none --profile-from-start off"
timeout 900 $NF -k regex:gemm_tc -c 4 -o gpurun_out/dbg_gemm_c3 python scripts/profile_step.py c3 > /dev/null 2>&1
