cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -25
