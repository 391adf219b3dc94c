cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -rf -x 2>&1 | tail -5 > $O/c3_gemmtests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c3_cublas_c3.txt 2>&1
timeout 300 python scripts/gemm_vs_cublas.py c4 > $O/c3_cublas_c4.txt 2>&1
HSD_GEMM_WT=2 timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c3_cublas_c3_wt2.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c3_bench_c3.json 2> $O/c3_bench_c3.err
HSD_ATTN_ORDER=1 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c3_bench_c3_order.json 2> $O/c3_bench_c3_order.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c3_bench_c2.json 2> $O/c3_bench_c2.err
timeout 1200 python -m pytest tests -m gpu -q -rf -x -k "tcgen05 or fullsize_logits or bf16" 2>&1 | tail -5 > $O/c3_tests.txt
cat $O/c3_gemmtests.txt $O/c3_tests.txt
