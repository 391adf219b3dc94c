cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -rf -x 2>&1 | tail -5 > $O/c4_gemmtests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c4_cublas_c3.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c4_bench_c3.json 2> $O/c4_bench_c3.err
HSD_GEMM_QKV_EPI=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c4_bench_c3_noqkv.json 2> $O/c4_bench_c3_noqkv.err
timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "fullsize or tcgen05 or bf16" 2>&1 | tail -5 > $O/c4_tests.txt
timeout 300 ncu --metrics gpu__time_duration.sum --csv python scripts/experiments/cublas_names.py > $O/c4_cublas_names.csv 2>&1
cat $O/c4_gemmtests.txt $O/c4_tests.txt
