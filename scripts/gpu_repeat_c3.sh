# VERDICT r1 "done" criterion for the sampling fix: the c3 full-size stochastic
# test (margin 1e-5) green in N consecutive runs, each a fresh process (new
# weights init, new prefill, new graph). Log: profiles/r02_c3_stochastic_repeat.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out/c3_repeat.txt
: > $O
N=${N:-30}
pass=0
for i in $(seq 1 $N); do
  if timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_stochastic" -p no:cacheprovider > gpurun_out/rep_$i.log 2>&1; then
    pass=$((pass+1)); echo "run $i: pass" >> $O
  else
    echo "run $i: FAIL" >> $O; tail -30 gpurun_out/rep_$i.log >> $O
  fi
  rm -f gpurun_out/rep_$i.log
done
echo "$pass / $N consecutive runs green" >> $O
tail -1 $O
