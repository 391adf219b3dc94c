cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2 > $O/c6_gemmtests.txt
for e in 0 8 1; do HSD_GEMM_EXP=$e timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c6_cublas_c3_exp$e.txt 2>&1; done
cat $O/c6_gemmtests.txt $O/c6_cublas_c3_exp*.txt
