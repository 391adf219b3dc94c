# hunt the rare full-size c3 parity failure: bench first (as in the round-end order), then the suite x6
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-planted --steps 20 2>&1 | tail -1 | cut -c1-150
for i in 1 2 3 4 5 6; do
  timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --tb=long 2>&1 | grep -E "^E |passed|failed|test_gpu_fullsize.py:[0-9]+:" | head -20
done
