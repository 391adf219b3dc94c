cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -8 > $O/c10_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/c10_smoke.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c10_bench_c3.json 2> $O/c10_bench_c3.err
HSD_GEMM_TMA_OUT=2 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c10_bench_c3_t2.json 2> $O/c10_bench_c3_t2.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c10_bench_c2.json 2> $O/c10_bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-planted > $O/c10_bench_c4.json 2> $O/c10_bench_c4.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-planted > $O/c10_bench_c5.json 2> $O/c10_bench_c5.err
cat $O/c10_tests.txt; tail -1 $O/c10_smoke.txt
