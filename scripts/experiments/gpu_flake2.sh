# hunt the rare full-size c3 parity failure: 10 runs of the c3 full-size tests, with a c3 bench between
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
for i in 1 2 3 4 5 6 7 8 9 10; do
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x --tb=long -k c3 > gpurun_out/flake_$i.log 2>&1
  echo "run $i: $(tail -1 gpurun_out/flake_$i.log)"
  grep -E "^E " gpurun_out/flake_$i.log | head -8
  if [ $((i % 3)) -eq 0 ]; then timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-planted --steps 10 > /dev/null 2>&1; fi
done
