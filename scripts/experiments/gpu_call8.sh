cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
for w in 0 1 2; do HSD_GEMM_WT=$w timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c8_wt$w.txt 2>&1; done
HSD_GEMM_EXP=1 timeout 300 python scripts/gemm_vs_cublas.py c3 --head > $O/c8_exp1.txt 2>&1
cat $O/c8_*.txt
