# Round-end evidence: GPU suite, smoke, default bench (c2) + c3/c4/c5 lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_gpu.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 3500 gpurun_out/bench_c2.json
for extra in "--config c3" "--config c4 --steps 8" "--config c5 --batch 2 --steps 10"; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-planted $extra 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$extra', d['ms_per_step'], d['value'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['kernel'], d['step_latency_ms']['median'], d['verify_latency_ms']['median'], d['profile_ms_per_step'])"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-600
