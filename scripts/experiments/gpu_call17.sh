cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -5 > $O/c17_tests.txt
for i in 1 2; do
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c17_bench_c3_$i.json 2> /dev/null
HSD_GEMM_PRE=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c17_bench_c3_pre0_$i.json 2> /dev/null
done
cat $O/c17_tests.txt
