cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2 > $O/c14_gemmtests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c14_c3.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c14_bench_c3_$i.json 2> $O/c14_bench_c3.err
HSD_GEMM_NT_ALT=0 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c14_bench_c3_alt0_$i.json 2> $O/c14_bench_c3_alt0.err
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "fullsize or tcgen05 or bf16 or serving" 2>&1 | tail -3 > $O/c14_tests.txt
cat $O/c14_gemmtests.txt $O/c14_c3.txt $O/c14_tests.txt
for sd in 2 4; do HSD_ATTN_SPLITS_DRAFT=$sd timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c14_bench_c3_sd$sd.json 2> /dev/null; done
