cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c7_bench_c3.json 2> $O/c7_bench_c3.err
HSD_GEMM_QKV_EPI=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c7_bench_c3_noqkv.json 2> $O/c7_bench_c3_noqkv.err
timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "fullsize or tcgen05 or bf16 or gemm" 2>&1 | tail -5 > $O/c7_tests.txt
cat $O/c7_tests.txt
