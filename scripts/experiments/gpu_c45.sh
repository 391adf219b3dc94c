cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-planted > /tmp/b_$c.json 2>/tmp/b_$c.err
  tail -2 /tmp/b_$c.err | cut -c1-300
  python -c "import json; d=json.loads(open('/tmp/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['bound'], d['roofline']['frac'], d['init_s'], d['profile_ms_per_step'])" 2>&1 | tail -1
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
