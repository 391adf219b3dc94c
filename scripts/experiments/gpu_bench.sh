cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
timeout 900 python bench.py "$@" 2>&1 | tail -20
