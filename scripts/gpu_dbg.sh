cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_vocab_shard.py -q -rf 2>&1 | tail -12 > gpurun_out/dbg.txt
