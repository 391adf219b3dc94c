# pair-GEMM super-tile width check: c3 / c4 verify shapes vs cuBLAS at WT = auto / 1 / 2
cd $GRAFT_REPO_ROOT; python -m paper_2602_21224_b200.build >/dev/null
O=gpurun_out/gwt.txt; : > $O
for wt in 0 1 2; do echo "WT=$wt" >> $O; HSD_GEMM_WT=$wt python scripts/gemm_vs_cublas.py c3 >> $O 2>&1; done
echo "c4 auto" >> $O; python scripts/gemm_vs_cublas.py c4 >> $O 2>&1
