cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
(time timeout 900 python bench.py) > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
tail -4 gpurun_out/bench_c2_full.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c2_full.json').read().strip().splitlines()[-1]); print(json.dumps({k: d[k] for k in ['value','ms_per_step','tau','planted','tau_curve','cpu_baseline','e2e','roofline','gpu_launches','clocks']}, indent=None)[:3000])"
