cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_bench_short.sh "$@" 2>&1 | tail -3
