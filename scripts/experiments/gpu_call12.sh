cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2 > $O/c12_gemmtests.txt
for v in "HSD_GEMM_PRE=0" "HSD_GEMM_PRE=1" "HSD_GEMM_PF_AHEAD=4" "HSD_GEMM_PF_AHEAD=8" "HSD_GEMM_PF_AHEAD=16" "HSD_GEMM_MAX_NT=176" "HSD_GEMM_MAX_NT=208"; do
  echo "== $v" >> $O/c12_sweep.txt
  env $v timeout 300 python scripts/gemm_vs_cublas.py c3 --head >> $O/c12_sweep.txt 2>&1
done
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c12_bench_c3.json 2> $O/c12_bench_c3.err
cat $O/c12_gemmtests.txt $O/c12_sweep.txt
