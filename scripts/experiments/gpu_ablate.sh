cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
for a in none attn rms rope swiglu tree gemm "attn,rms,rope,swiglu,tree" "attn,rms,rope,swiglu,tree,gemm"; do
  HSD_ABLATE=$a timeout 600 python bench.py --steps 30 --warmup 5 --config ${CFG:-c2} --no-cpu-baseline --no-profile --no-e2e --no-planted 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['ms_per_step'])"
done
