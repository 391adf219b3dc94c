cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -x -k "parity or fullsize" 2>&1 | tail -8 > $O/c2_tests.txt
timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/cublas_c3.txt 2>&1
timeout 300 python scripts/gemm_vs_cublas.py c4 > $O/cublas_c4.txt 2>&1
bash scripts/gpu_profiles_r02.sh
tail -3 $O/c2_tests.txt
