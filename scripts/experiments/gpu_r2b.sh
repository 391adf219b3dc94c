cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build
timeout 600 python -m pytest tests -m gpu -q -rf -k "admit or capacity or bench or sampling" 2>&1 | tail -15 > gpurun_out/r2b_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench_c3.json 2> gpurun_out/r2b_bench_c3.err
ncu --query-metrics 2>/dev/null | grep -i -E "tensor|utc|umma|tmem|pipe_tc|mma" > gpurun_out/r2b_metrics.txt
ncu --query-metrics-mode suffix --metrics sm__pipe_tensor_op_hmma_cycles_active 2>/dev/null | head -20 >> gpurun_out/r2b_metrics.txt
tail -3 gpurun_out/r2b_tests.txt
