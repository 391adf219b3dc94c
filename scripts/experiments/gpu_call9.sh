cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3 > $O/c9_gemmtests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c9_c3.txt 2>&1
HSD_GEMM_TMA_OUT=0 timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c9_c3_notma.txt 2>&1
timeout 300 python scripts/gemm_vs_cublas.py c4 > $O/c9_c4.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c9_bench_c3.json 2> $O/c9_bench_c3.err
cat $O/c9_gemmtests.txt $O/c9_c3.txt $O/c9_c3_notma.txt $O/c9_c4.txt
