cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
for e in 0 1 4; do HSD_GEMM_EXP=$e timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c5_cublas_c3_exp$e.txt 2>&1; done
HSD_GEMM_WT=2 HSD_GEMM_EXP=4 timeout 300 python scripts/gemm_vs_cublas.py c3 > $O/c5_cublas_c3_wt2_exp4.txt 2>&1
cat $O/c5_cublas_c3_exp*.txt
