# same-box A/B: committed gemm_tc.cu (scripts/experiments/gemm_tc_head.cu.txt) vs the working copy
cd $GRAFT_REPO_ROOT; O=gpurun_out/gon.txt; : > $O
D=paper_2602_21224_b200/csrc
cp $D/gemm_tc.cu /tmp/gemm_new.cu
for v in old new old new; do
  if [ $v = old ]; then cp scripts/experiments/gemm_tc_head.cu.txt $D/gemm_tc.cu; else cp /tmp/gemm_new.cu $D/gemm_tc.cu; fi
  python -m paper_2602_21224_b200.build >/dev/null 2>&1
  echo "== $v" >> $O; python scripts/gemm_vs_cublas.py c3 >> $O 2>&1
done
cp /tmp/gemm_new.cu $D/gemm_tc.cu
