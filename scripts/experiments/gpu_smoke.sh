set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2602_21224_b200.build
timeout 300 python __graft_entry__.py 2>&1 | tail -30
