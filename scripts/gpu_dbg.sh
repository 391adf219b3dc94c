cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6 > gpurun_out/dbg.txt
timeout 300 python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline --no-planted --no-e2e > gpurun_out/dbg_c3.json 2>&1
