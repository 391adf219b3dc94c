cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
: > $O/c16.txt
for v in "X=0" "HSD_PREFILL_CHUNK=1024" "HSD_GEMM_QKV_EPI=0" "HSD_GEMM_PRE=0" "HSD_GEMM_TMA_OUT=0" "HSD_GEMM_NT_ALT=176"; do
  echo "== $v" >> $O/c16.txt
  env $v timeout 600 python -m pytest tests/test_gpu_fullsize_logits.py -q -x -k "c3" 2>&1 | grep -E "AssertionError: \{|passed|failed" >> $O/c16.txt
done
cat $O/c16.txt
