cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_vocab_shard.py -q -rs 2>&1 | tail -4 > $O/c11_vs.txt
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c11_bench_c3.json 2> $O/c11_bench_c3.err
timeout 600 python bench.py --config c5 --batch-per-gpu 2 --steps 5 --warmup 3 --no-cpu-baseline --no-planted > $O/c11_bench_c5.json 2> $O/c11_bench_c5.err
bash scripts/gpu_profiles_r02.sh > /dev/null 2>&1
N=30 bash scripts/gpu_repeat_c3.sh
cat $O/c11_vs.txt
