cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40
