cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
for i in 1 2 3; do
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c20_def_$i.json 2> /dev/null
HSD_GEMM_NT_ALT=176 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c20_alt_$i.json 2> /dev/null
done
HSD_GEMM_NT_ALT=176 timeout 900 python -m pytest tests -m gpu -q -x -k "fullsize_logits or test_gpu_gemm" > $O/c20_tests.txt 2>&1
tail -2 $O/c20_tests.txt
