cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep or fullsize_logits or c3_stochastic" 2>&1 | tail -2 > gpurun_out/dbg.txt
for c in c3 c2; do timeout 300 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-planted --no-e2e > gpurun_out/dbg_$c.json 2>&1; python scripts/bench_summary.py gpurun_out/dbg_$c.json >> gpurun_out/dbg.txt; done
