cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
HSD_TREE_CL=4 timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_c1 or hot_pruned or c3_stochastic or c4" 2>&1 | tail -2 > gpurun_out/dbg.txt
B="python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline --no-planted --no-e2e"
for cl in 8 4; do HSD_TREE_CL=$cl timeout 300 $B > gpurun_out/dbg_cl$cl.json 2>&1; python scripts/bench_summary.py gpurun_out/dbg_cl$cl.json >> gpurun_out/dbg.txt; done
