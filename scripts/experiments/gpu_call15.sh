cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize_logits.py -q -x -k "c3" > $O/c15_default.txt 2>&1
HSD_GEMM_NT_ALT=176 timeout 900 python -m pytest tests/test_gpu_fullsize_logits.py -q -x -k "c3" > $O/c15_alt176.txt 2>&1
tail -3 $O/c15_default.txt $O/c15_alt176.txt
