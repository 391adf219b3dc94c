cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf -k "fusion_off or first_token" 2>&1 | tail -8 > gpurun_out/dbg.txt
