cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 300 python scripts/prefill_time.py c3 > $O/c22_pt.txt 2>&1
HSD_GEMM_QKV_WT2=1 timeout 300 python scripts/prefill_time.py c3 >> $O/c22_pt.txt 2>&1
timeout 300 python scripts/prefill_time.py c2 >> $O/c22_pt.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c22_def_$i.json 2> /dev/null
done
timeout 900 python -m pytest tests -m gpu -q -x -k "fullsize_logits or serving" > $O/c22_tests.txt 2>&1
cat $O/c22_pt.txt; tail -2 $O/c22_tests.txt
