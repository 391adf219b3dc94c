cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2 > $O/c26_gemm.txt
cat $O/c26_gemm.txt
for i in 1 2; do
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-planted --no-profile > $O/c26_c2_$i.json 2>/dev/null
HSD_GEMM_TMA_SK=0 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-planted --no-profile > $O/c26_c2_sk0_$i.json 2>/dev/null
done
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c26_c3.json 2>/dev/null
HSD_GEMM_TMA_SK=0 timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c26_c3_sk0.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > $O/c26_tests.txt
cat $O/c26_tests.txt
