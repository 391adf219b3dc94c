cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2 > $O/c13_gemmtests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c13_c3.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c13_bench_c3.json 2> $O/c13_bench_c3.err
HSD_GEMM_NT_WT1=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c13_bench_c3_nt0.json 2> $O/c13_bench_c3_nt0.err
HSD_GEMM_PRE=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c13_bench_c3_pre0.json 2> $O/c13_bench_c3_pre0.err
timeout 1500 python -m pytest tests -m gpu -q -x -k "fullsize or tcgen05 or bf16 or serving" 2>&1 | tail -3 > $O/c13_tests.txt
cat $O/c13_gemmtests.txt $O/c13_c3.txt $O/c13_tests.txt
