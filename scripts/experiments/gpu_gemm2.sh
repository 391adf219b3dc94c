cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
python scripts/gemm_bench.py | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'], d['profile_ms_per_step'])"
