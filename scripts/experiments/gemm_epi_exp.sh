cd $GRAFT_REPO_ROOT; python -m paper_2602_21224_b200.build >/dev/null
O=gpurun_out/gexp.txt; : > $O
for wt in 1 2; do for ex in 0 1 2; do echo "WT=$wt EXP=$ex" >> $O; HSD_GEMM_WT=$wt HSD_GEMM_EXP=$ex python scripts/gemm_vs_cublas.py c3 >> $O 2>&1; done; done
